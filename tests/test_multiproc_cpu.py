"""world_size-2 host-side tests of the N > 1 path on CPU (gloo backend):
placement, the per-rank engine-replay plans with their epoch waits, and the
peer-blob / NCCL-id exchange protocol of the binding."""
import os

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import synth

WORLD = 2


def _worker(rank, port, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=WORLD)
        import paper_1710_06952_b200 as P
        n = 8 * WORLD
        e, _ = synth.ring(n)
        out = {}
        for placement in (0, 1):
            wr, wl = P.plan_placement(n, WORLD, placement)
            ev, _ = synth.schedule_iid(n, e, K=300, seed=5, no_grad=True)
            plan, ep = P.plan_replay(wr, rank, ev, k0=1000)
            allp = [None] * WORLD
            dist.all_gather_object(allp, (wr.tolist(), plan.tolist(), ep.tolist()))
            out[placement] = allp
        # blob exchange protocol (fake blobs; the NCCL id comes from rank 0 only)
        blobs, nid = P.exchange_peer_blobs(bytes([rank]) * 64, rank, WORLD,
                                           (lambda: b"ID" * 64) if rank == 0 else None)
        out["blobs"] = (blobs, nid)
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, out))
    except Exception as ex:  # surfaced by the parent
        q.put((rank, repr(ex)))


@pytest.fixture(scope="module")
def results():
    from paper_1710_06952_b200 import build
    build.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29600 + os.getpid() % 300
    ps = [ctx.Process(target=_worker, args=(r, port, q)) for r in range(WORLD)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(WORLD))
    for p in ps:
        p.join(timeout=60)
    for r in range(WORLD):
        assert not isinstance(res[r], str), res[r]
    return res


def test_placement_consistent_across_ranks(results):
    n = 8 * WORLD
    for placement in (0, 1):
        wr0 = results[0][placement][0][0]
        assert all(results[r][placement][r][0] == wr0 for r in range(WORLD))
        if placement == 0:
            assert wr0 == [w * WORLD // n for w in range(n)]           # contiguous ring segments
        else:
            assert wr0 == [w % WORLD for w in range(n)]


def test_replay_plans_partition_schedule_and_epochs_are_exact(results):
    n = 8 * WORLD
    e, _ = synth.ring(n)
    ev, _ = synth.schedule_iid(n, e, K=300, seed=5, no_grad=True)
    for placement in (0, 1):
        allp = results[0][placement]
        wr = allp[0][0]
        rows = [tuple(x) for r in range(WORLD) for x in allp[r][1]]
        assert sorted(x[0] for x in rows) == list(range(1000, 1300))   # every event exactly once
        for r in range(WORLD):
            assert all(wr[x[1]] == r for x in allp[r][1])            # owned by the updating worker's rank
            assert allp[r][2] == allp[0][2]                            # identical epoch mirrors
        # brute force: e_i, e_j = number of earlier events touching i, j
        for (k, i, j, fl, ei, ej, kind, grow) in rows:
            assert kind == 0 and grow == -1
            prev = ev[:k - 1000]
            assert ei == int(((prev[:, 0] == i) | (prev[:, 1] == i)).sum())
            if j >= 0:
                assert ej == int(((prev[:, 0] == j) | (prev[:, 1] == j)).sum())
        touches = np.zeros(n, np.int64)
        for i, j, _, _ in ev:
            touches[i] += 1
            touches[j] += 1
        assert allp[0][2] == touches.tolist()


def test_peer_blob_exchange(results):
    for r in range(WORLD):
        blobs, nid = results[r]["blobs"]
        assert blobs == [bytes([q]) * 64 for q in range(WORLD)]
        assert nid == b"ID" * 64


def test_replay_plan_stale_reads_are_placed_at_their_read_points():
    """Engine replay with tau > 0 (X_hat_k = X_{k - tau}): each stale
    gradient event f of worker i gets a read op in i's op sequence after every
    event < f - tau touching i and before every event >= f - tau touching i, in
    read row m mod (T + 1) for i's m-th such event; e_i / e_j of every op equal
    its position in the worker's sequence (brute force over the schedule)."""
    import paper_1710_06952_b200 as P
    n, T, K = 8, 3, 400
    e, _ = synth.ring(n)
    ev, _ = synth.schedule_iid(n, e, K=K, T=T, seed=17, local_prob=0.25)
    ev[::7, 3] = 1                                   # some pure averages (no read)
    wr = np.array([w % 2 for w in range(n)], np.int32)
    rows = np.concatenate([P.plan_replay(wr, r, ev, k0=50, T=T, stale_reads=True)[0] for r in range(2)])
    events = rows[rows[:, 6] == 0]
    reads = rows[rows[:, 6] == 2]
    assert sorted(events[:, 0].tolist()) == list(range(50, 50 + K))
    stale = [f for f in range(K) if ev[f, 2] > 0 and not (ev[f, 3] & 1)]
    assert len(reads) == len(stale)
    # reconstruct every worker's op sequence in global order and check positions
    seq = {w: [] for w in range(n)}
    for f in range(K):
        for g in [g for g in stale if g - ev[g, 2] == f]:
            seq[ev[g, 0]].append(("r", g))
        seq[ev[f, 0]].append(("e", f))
        if ev[f, 1] >= 0:
            seq[ev[f, 1]].append(("e", f))
    pos = {w: {op: p for p, op in enumerate(s)} for w, s in seq.items()}
    m = np.zeros(n, np.int64)
    row_of = {}
    for f in range(K):                               # rows in order of the reads (= m-th stale event)
        for g in [g for g in stale if g - ev[g, 2] == f]:
            i = ev[g, 0]
            row_of[g] = m[i] % (T + 1)
            m[i] += 1
    for (k, i, j, fl, ei, ej, kind, grow) in events:
        f = k - 50
        assert ei == pos[i][("e", f)]
        if j >= 0:
            assert ej == pos[j][("e", f)]
        assert grow == (row_of[f] if f in row_of else -1)
    by_row = {}
    for (k, i, j, fl, ei, ej, kind, grow) in reads:
        assert j == -1
        cand = [g for g in stale if ev[g, 0] == i and pos[i][("r", g)] == ei]
        assert len(cand) == 1
        g = cand[0]
        assert grow == row_of[g] and k == 50 + g   # Alg. 1 events: the key is the event's k


def test_replay_plan_fits_the_preallocated_op_list():
    """The engine replay sizes its device op list before the collective that lets a peer's
    engine start (runtime.cu replay_engine: 3 K + n_local + 1 entries), so the plan of any rank
    must fit that bound -- events, stale reads and pure averages alike, at world 1, 2 and 4."""
    import paper_1710_06952_b200 as P
    n, T, K = 16, 4, 600
    e, _ = synth.ring(n)
    ev, _ = synth.schedule_iid(n, e, K=K, T=T, seed=23, local_prob=0.3)
    ev[::5, 3] = 1
    for world in (1, 2, 4):
        wr = np.array([w % world for w in range(n)], np.int32)
        for r in range(world):
            rows, _ = P.plan_replay(wr, r, ev, k0=7, T=T, stale_reads=True)
            n_local = int((wr == r).sum())
            assert len(rows) <= 3 * K + n_local + 1, (world, r, len(rows))
