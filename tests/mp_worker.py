"""Multi-rank parity worker.  Two launchers run the same body:
  * one process per GPU (tests/test_multigpu.py::test_nvlink_parity through
    torch.distributed.run; CUDA IPC peers + NCCL);
  * in-process ranks on host threads (tests/test_multigpu.py::
    test_virtual_ranks_parity; comm_local contexts, which may all share ONE GPU:
    the same cross-rank engine protocol -- remote try-locks, cooperative
    mailboxes, commit flags, tickets -- with local pointers, and fixed-order
    in-process collectives instead of NCCL).
Rank 0 compares against the oracle; any mismatch is returned / exits non-zero.

Checks:
  1. engine replay of a pure-gossip schedule whose ring edges cross GPUs
     (interleave placement: every edge is an NVLink edge) -- bitwise;
  2. engine replay with the quadratic (block placement) -- bitwise;
  3. free-running engine, quadratic: the device event log replayed through the
     oracle reproduces every rank's models bitwise;
  4. consensus mean (NCCL fp64 all-reduce) within 1 ulp;
  5. AllReduce-SGD baseline (NCCL fp32) within 1e-5 relative;
  6. D-PSGD baseline (NCCL halo exchange) bitwise;
  7. App. A wait-free engine loop across GPUs: log replay bitwise.
  8. host-driven adpsgd_step across GPUs (ranks step concurrently): log replay
     bitwise; a collective run afterwards starts from the agreed device ticket;
  9. the bench workload at full size (d = 25.6M, 8 workers/GPU, block placement,
     10x straggler, cooperative cross events on their grid/4 CTA footprint):
     free-running log replay bitwise, compared through per-row SHA-1 digests.
"""
import hashlib
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch
import torch.distributed as dist

import synth
import paper_1710_06952_b200 as P


class DistGroup:
    """torch.distributed (one process per rank)."""

    def __init__(self, rank, world):
        self.rank, self.world = rank, world

    def barrier(self):
        dist.barrier()

    def all_gather(self, obj):
        out = [None] * self.world
        dist.all_gather_object(out, obj)
        return out

    def ctx_kw(self):
        return {}


class ThreadRanks:
    """In-process ranks (P.ThreadGroup): same interface."""

    def __init__(self, tg, rank):
        self.tg, self.rank, self.world = tg, rank, tg.world

    def barrier(self):
        self.tg.barrier()

    def all_gather(self, obj):
        out = [None] * self.world
        self.tg.all_gather_object(out, obj, self.rank)
        return out

    def ctx_kw(self):
        return {"group": self.tg}


def gather_models(ctx, G):
    mine = {w: ctx.read_model(w) for w in ctx.local_workers()}
    allm = G.all_gather(mine)
    X = np.zeros((ctx.n, ctx.d), np.float32)
    for m in allm:
        for w, x in m.items():
            X[w] = x
    return X


_T0 = time.time()


def progress(rank, what):
    print(f"[rank {rank} {time.time() - _T0:7.1f}s] {what}", file=sys.stderr, flush=True)


def body(rank, world, local, G, full_size=True):
    """The checks; G is a DistGroup or ThreadRanks.  Returns rank 0's failures."""
    kw = G.ctx_kw()
    fails = []
    if rank == 0:
        from oracle import oracle as O
    n = 8 * world
    e, r = synth.ring(n)
    dk, nk = synth.quad_keys(3)
    s = float(np.float32(0.1 * math.sqrt(96)))
    prob_q = None
    if rank == 0:
        prob_q = O.OracleProblem(O.MODEL_QUADRATIC, M=32, gamma=0.01, data_key=dk, noise_key=nk, noise_s=s)

    # 1. pure gossip replay over NVLink (interleave: every edge crosses GPUs),
    #    one-sided (cooperative events off) and with the auto policy
    d = 1 << 20
    X0 = synth.x0_uniform(n, d, seed=21)
    ev, _ = synth.schedule_iid(n, e, K=1500, seed=4, no_grad=True)
    if rank == 0:
        Xo, _ = O.replay(O.OracleProblem(), X0, e, r, ev)
    for variant in (-1, 0):          # cooperative events off (one-sided) / auto
        ctx = P.Context(e, n, d, role=r, rank=rank, world_size=world, device=local, **kw, placement=1,
                        x0_per_worker=X0, engine_coop=False if variant == -1 else None)
        ctx.replay(ev, flags=P.REPLAY_ENGINE)
        ctx.sync()
        G.barrier()
        st = ctx.stats()
        X = gather_models(ctx, G)
        cross = G.all_gather(st["local_cross_events"])
        hbm = G.all_gather(st["local_bytes"])
        if rank == 0:
            # every pair reads + writes two rows: 16d bytes system-wide, 8d on each GPU's HBM
            if abs(sum(hbm) - 1500 * 16.0 * d) > 1e-6 * 1500 * 16.0 * d or min(hbm) <= 0:
                fails.append(f"HBM byte accounting {hbm} != {1500 * 16 * d} (variant {variant})")
            if not np.array_equal(X.view(np.uint32), Xo.view(np.uint32)):
                fails.append(f"pure-gossip engine replay over NVLink not bit-exact (variant {variant})")
            if sum(cross) != 1500:
                fails.append(f"expected every event to cross GPUs, got {sum(cross)}")
        if variant == -1:
            ctx.destroy()
            G.barrier()
    progress(rank, "1 pure-gossip replay done")
    # 4. consensus mean (NCCL fp64)
    out = torch.empty(d, dtype=torch.float32, device=f"cuda:{local}")
    mk = ctx.consensus_mean(out.data_ptr())
    if rank == 0:
        xo, mko = O.consensus_mean(Xo)
        ulp = np.abs(out.cpu().numpy().view(np.int32).astype(np.int64) - xo.view(np.int32).astype(np.int64))
        if ulp.max() > 1:
            fails.append(f"consensus mean {ulp.max()} ulp")
        if abs(mk - mko) > 1e-9 * mko:
            fails.append(f"M_k {mk} vs {mko}")
    ctx.destroy()
    G.barrier()

    progress(rank, "4 consensus done")
    # 2./3. quadratic: engine replay then free-running, block placement
    d = 1 << 20
    ev, _ = synth.schedule_iid(n, e, K=400, seed=8, local_prob=0.3)
    ctx = P.Context(e, n, d, role=r, rank=rank, world_size=world, device=local, **kw, placement=0,
                    model=P.MODEL_QUADRATIC, gamma=0.01, batch_M=32, quad_keys=(dk, nk), quad_noise_s=s,
                    straggler=synth.stragglers(n), compute_ns=20_000, seed=9)
    ctx.replay(ev, flags=P.REPLAY_ENGINE)
    ctx.sync()
    G.barrier()
    X = gather_models(ctx, G)
    if rank == 0:
        Xo, _ = O.replay(prob_q, np.zeros((n, d), np.float32), e, r, ev)
        if not np.array_equal(X.view(np.uint32), Xo.view(np.uint32)):
            fails.append("quadratic engine replay (block placement) not bit-exact")
    ctx.run(3000)
    ctx.sync()
    G.barrier()
    X2 = gather_models(ctx, G)
    if rank == 0:
        log = ctx.read_log(400)
        evs = np.stack([log["i"], log["j"], log["tau"], log["flags"].astype(np.int32)], 1)
        if len(log) != 3000:
            fails.append(f"log has {len(log)} entries")
        Xo2, _ = O.replay(prob_q, Xo, e, r, evs, k0=400)
        if not np.array_equal(X2.view(np.uint32), Xo2.view(np.uint32)):
            bad = np.where((X2 != Xo2).any(1))[0]
            fails.append(f"free-running multi-GPU log replay not bit-exact (workers {bad.tolist()})")
    progress(rank, "2/3 quadratic replay + free-running done")
    # 2b. engine replay with stale reads tau ~ U{0..3} across ranks: each
    #     stale gradient is a read op at X_{k - tau} of the worker's sequence
    T = 3
    ev_s, _ = synth.schedule_iid(n, e, K=300, T=T, seed=12, local_prob=0.25)
    X0s = synth.x0_uniform(n, d, seed=29)
    cs = P.Context(e, n, d, role=r, rank=rank, world_size=world, device=local, **kw, placement=0, T=T,
                   model=P.MODEL_QUADRATIC, gamma=0.01, batch_M=32, quad_keys=(dk, nk), quad_noise_s=s,
                   x0_per_worker=X0s, seed=9)
    cs.replay(ev_s, flags=P.REPLAY_ENGINE)
    cs.sync()
    G.barrier()
    Xs_ = gather_models(cs, G)
    if rank == 0:
        Xso, _ = O.replay(prob_q, X0s, e, r, ev_s, T=T)
        if not np.array_equal(Xs_.view(np.uint32), Xso.view(np.uint32)):
            fails.append("multi-rank engine replay with stale reads not bit-exact")
    cs.destroy()
    G.barrier()
    progress(rank, "2b stale-read engine replay done")
    # 6. D-PSGD baseline: halo exchange of neighbour rows by NCCL send/recv
    X0d = synth.x0_uniform(n, d, seed=23)
    ctx.dpsgd_reset(X0d)
    ctx.dpsgd(4)
    mine = {w: ctx.dpsgd_read_model(w) for w in ctx.local_workers()}
    allm = G.all_gather(mine)
    if rank == 0:
        Xd = np.zeros((n, d), np.float32)
        for m in allm:
            for w, x in m.items():
                Xd[w] = x
        Xdo = X0d
        for rr in range(4):
            Xdo = O.dpsgd_round(prob_q, Xdo, e, k_base=rr * n)
        if not np.array_equal(Xd.view(np.uint32), Xdo.view(np.uint32)):
            fails.append("D-PSGD multi-GPU not bit-exact")
    # 5. AllReduce-SGD baseline over NCCL
    ctx.allreduce_reset()
    ctx.allreduce_sgd(5)
    xa = ctx.allreduce_read_model()
    if rank == 0:
        x = np.zeros(d, np.float32)
        for rr in range(5):
            Gm = np.stack([O.gradient(prob_q, x, k=rr * n + w) for w in range(n)])
            x = O.allreduce_update(x, Gm, 0.01)
        if not np.allclose(xa, x, rtol=1e-5, atol=1e-6):
            fails.append(f"allreduce baseline max err {np.abs(xa - x).max()}")
    ctx.destroy()
    G.barrier()

    progress(rank, "5/6 baselines done")
    # 8. host-driven adpsgd_step across GPUs (device try-lock + ticket, fused pass over
    #    NVLink, commit): ranks step their own workers concurrently; the log replays bitwise
    d = (1 << 14) + 20
    X0s = synth.x0_uniform(n, d, seed=27)
    ctx = P.Context(e, n, d, role=r, rank=rank, world_size=world, device=local, **kw, placement=1,
                    model=P.MODEL_QUADRATIC, gamma=0.01, batch_M=32, quad_keys=(dk, nk), quad_noise_s=s,
                    x0_per_worker=X0s, seed=13)
    for _ in range(25):
        for w in ctx.local_workers():
            ctx.step(w)
    ctx.sync()
    G.barrier()
    Xs = gather_models(ctx, G)
    if rank == 0:
        log = ctx.read_log(0)
        evs = np.stack([log["i"], log["j"], log["tau"], log["flags"].astype(np.int32)], 1)
        if len(log) != 25 * n or not np.array_equal(np.sort(log["k"]), np.arange(25 * n)):
            fails.append(f"multi-GPU step log: {len(log)} entries")
        else:
            order = np.argsort(log["k"])
            Xso, _ = O.replay(prob_q, X0s, e, r, evs[order])
            if not np.array_equal(Xs.view(np.uint32), Xso.view(np.uint32)):
                fails.append("multi-GPU adpsgd_step log replay not bit-exact")
    progress(rank, "8 steps done")
    ctx.run(200)                                  # the device ticket is settled before the collective run
    ctx.sync()
    G.barrier()
    if rank == 0 and ctx.ticket() != 25 * n + 200:
        fails.append(f"ticket after steps + run: {ctx.ticket()}")
    ctx.destroy()
    G.barrier()

    progress(rank, "8 run after steps done")
    # 7. App. A wait-free engine loop (reading R20), interleave placement: pulls,
    #    buffered-gradient flushes and continuous averages across NVLink; the log
    #    (tau = k - t_read, FLUSH_FIRST | COMPENSATE) replays bitwise
    d = (1 << 14) + 20
    X0w = synth.x0_uniform(n, d, seed=25)
    ctx = P.Context(e, n, d, role=r, rank=rank, world_size=world, device=local, **kw, placement=1,
                    model=P.MODEL_QUADRATIC, gamma=0.01, batch_M=32, quad_keys=(dk, nk), quad_noise_s=s,
                    x0_per_worker=X0w, straggler=synth.stragglers(n, slow=3.0), compute_ns=30_000, seed=11,
                    wait_free=2)
    ctx.run(2000)
    ctx.sync()
    G.barrier()
    Xw = gather_models(ctx, G)
    if rank == 0:
        log = ctx.read_log(0)
        evs = np.stack([log["i"], log["j"], log["tau"], log["flags"].astype(np.int32)], 1)
        grad = (evs[:, 3] & 1) == 0
        if len(log) != 2000 or grad.sum() == 0 or not (evs[grad, 3] & 4).any():
            fails.append(f"wait-free log: {len(log)} entries, {int(grad.sum())} flushes")
        else:
            Xwo, _ = O.replay(prob_q, X0w, e, r, evs, T=int(evs[:, 2].max()))
            if not np.array_equal(Xw.view(np.uint32), Xwo.view(np.uint32)):
                fails.append("wait-free multi-GPU log replay not bit-exact")
    ctx.destroy()
    G.barrier()

    progress(rank, "7 wait-free done")
    if not full_size:
        return fails
    # 9. full-size bench workload across GPUs: digests of every row vs the oracle's replay
    d, U = 25_600_000, 32 * world
    ctx = P.Context(e, n, d, role=r, rank=rank, world_size=world, device=local, **kw, placement=0,
                    model=P.MODEL_QUADRATIC, gamma=0.01, batch_M=32, quad_keys=(dk, nk), quad_noise_s=s,
                    straggler=synth.stragglers(n), compute_ns=50_000, seed=17)
    ctx.run(U)
    ctx.sync()
    G.barrier()
    mine = {w: hashlib.sha1(ctx.read_model(w).tobytes()).hexdigest() for w in ctx.local_workers()}
    cross = ctx.stats()["local_cross_events"]
    alld = G.all_gather(mine)
    allc = G.all_gather(cross)
    if rank == 0:
        dig = {w: h for m in alld for w, h in m.items()}
        log = ctx.read_log(0)
        evs = np.stack([log["i"], log["j"], log["tau"], log["flags"].astype(np.int32)], 1)
        if len(log) != U:
            fails.append(f"full-size log has {len(log)} entries")
        else:
            Xf, _ = O.replay(prob_q, np.zeros((n, d), np.float32), e, r, evs)
            bad = [w for w in range(n) if hashlib.sha1(Xf[w].tobytes()).hexdigest() != dig[w]]
            if bad:
                fails.append(f"full-size multi-GPU log replay not bit-exact (workers {bad})")
            del Xf
        if sum(allc) == 0:
            fails.append("full-size run had no cross-GPU event")
        progress(rank, f"9 full size: {sum(allc)} cross events of {U}")
    ctx.destroy()
    G.barrier()
    return fails


def main():
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    fails = body(rank, world, local, DistGroup(rank, world))
    if rank == 0:
        print("MULTIGPU", "FAIL" if fails else "OK", fails, flush=True)
    dist.destroy_process_group()
    sys.exit(1 if (rank == 0 and fails) else 0)


if __name__ == "__main__":
    main()
