"""GPU parity of the App. A wait-free runtime (DESIGN.md reading
R20): flush-then-average events, read-point-keyed gradients, local-update
compensation -- host replay, engine replay and the free-running engine loop
(wait_free = 1 / 2) against the oracle, through the C-ABI."""
import math

import numpy as np
import pytest

import synth
from oracle import oracle as O

pytestmark = pytest.mark.gpu

FF, COMP = O.EV_FLUSH_FIRST, O.EV_COMPENSATE


@pytest.fixture(scope="module")
def P():
    from paper_1710_06952_b200 import build
    build.build()
    import paper_1710_06952_b200 as P
    return P


def read_all(ctx):
    return np.stack([ctx.read_model(w) for w in range(ctx.n)])


def log_events(log):
    return np.stack([log["i"], log["j"], log["tau"], log["flags"].astype(np.int32)], 1)


def quad_setup(seed):
    dk, nk = synth.quad_keys(seed)
    s = float(np.float32(0.1 * math.sqrt(3 * 32)))
    prob = O.OracleProblem(O.MODEL_QUADRATIC, M=32, gamma=0.01, data_key=dk, noise_key=nk, noise_s=s)
    return dict(model=2, gamma=0.01, batch_M=32, quad_keys=(dk, nk), quad_noise_s=s), prob


@pytest.mark.parametrize("compensate", [True, False])
@pytest.mark.parametrize("d", [3 * 4096 + 37, 1 << 18])
def test_appa_host_replay_quadratic_bitwise(P, compensate, d):
    """Valid App. A schedules (stale reads, buffered gradient compensation,
    no-gradient averages) replayed by the host executor: bitwise."""
    n, K, T = 8, 400, 12
    e, r = synth.ring(n)
    kw, prob = quad_setup(21)
    ev = synth.schedule_appa(n, e, r, K, T, seed=5, compensate=compensate)
    assert (ev[:, 2] > 0).any() and (ev[:, 3] == 1).any()
    X0 = synth.x0_uniform(n, d, seed=3)
    ctx = P.Context(e, n, d, role=r, T=T, x0_per_worker=X0, **kw)
    ctx.replay(ev, flags=P.REPLAY_HOST)
    ctx.sync()
    Xo, _ = O.replay(prob, X0, e, r, ev, T=T)
    assert np.array_equal(read_all(ctx).view(np.uint32), Xo.view(np.uint32))
    ctx.destroy()


def test_appa_host_replay_lsq_within_1e4(P):
    """Config-1 shapes (least squares, d = 1024, M = 32) under an App. A
    schedule with compensation: within reading c11's 1e-4."""
    n, d, K, T, S, M = 4, 1024, 1500, 6, 8192, 32
    e, r = synth.ring(n)
    A, b = synth.lsq_data(S=S, d=d, seed=1)
    ev = synth.schedule_appa(n, e, r, K, T, seed=42)
    bi = np.random.default_rng(8).integers(0, S, size=(K, M)).astype(np.int32)
    ctx = P.Context(e, n, d, role=r, T=T, model=P.MODEL_LSQ, gamma=0.5, batch_M=M, data_A=A, data_b=b)
    ctx.replay(ev, batch_idx=bi, flags=P.REPLAY_HOST)
    ctx.sync()
    prob = O.OracleProblem(O.MODEL_LSQ, M=M, gamma=0.5, A=A, b=b)
    Xo, _ = O.replay(prob, np.zeros((n, d), np.float32), e, r, ev, bi, T=T)
    Xg = read_all(ctx)
    rms = np.sqrt(np.mean(Xo.astype(np.float64) ** 2, axis=1, keepdims=True))
    assert (np.abs(Xg.astype(np.float64) - Xo) <= 1e-4 * np.maximum(np.abs(Xo), rms)).all()
    ctx.destroy()


def test_appa_compensation_causality_rejected(P):
    n, d = 1, 64
    kw, _ = quad_setup(2)
    ctx = P.Context(np.zeros((0, 2), np.int32), n, d, T=2, **kw)
    with pytest.raises(P.AdpsgdError) as ei:
        ctx.replay([[0, -1, 0, 0], [0, -1, 0, COMP], [0, -1, 2, FF | COMP]], flags=P.REPLAY_HOST)
    assert ei.value.code == 5
    ctx.destroy()


@pytest.mark.parametrize("d", [100003, 1 << 20])
def test_appa_engine_replay_flush_first_bitwise(P, d):
    """tau = 0 flush-first events through the persistent engine (inline
    gradient, App. A order and keys): bitwise."""
    n, K = 8, 300
    e, r = synth.ring(n)
    kw, prob = quad_setup(9)
    ev, _ = synth.schedule_iid(n, e, K=K, seed=4, local_prob=0.2)
    ev[:, 3] = np.where(np.arange(K) % 3 == 0, 1, FF | COMP)
    X0 = synth.x0_uniform(n, d, seed=6)
    ctx = P.Context(e, n, d, role=r, x0_per_worker=X0, **kw)
    ctx.replay(ev, flags=P.REPLAY_ENGINE)
    ctx.sync()
    Xo, _ = O.replay(prob, X0, e, r, ev)
    assert np.array_equal(read_all(ctx).view(np.uint32), Xo.view(np.uint32))
    ctx.destroy()


@pytest.mark.parametrize("wait_free", [1, 2])
def test_wait_free_free_running_log_replays_bitwise(P, wait_free):
    """The wait-free engine loop (pull -> compute s_w t_c -> buffer -> flush,
    continuous averaging by actives): its event log -- flush events carry
    tau = k - t_read and FLUSH_FIRST | COMPENSATE -- replayed through the
    oracle reproduces every model bitwise, across two run() calls."""
    n, d, U = 8, (1 << 14) + 20, 1500
    e, r = synth.ring(n)
    kw, prob = quad_setup(13)
    X0 = synth.x0_uniform(n, d, seed=14)
    st = synth.stragglers(n, slow_worker=0, slow=4.0)
    ctx = P.Context(e, n, d, role=r, x0_per_worker=X0, seed=5, wait_free=wait_free, straggler=st,
                    compute_ns=30_000, **kw)
    ctx.run(U)
    ctx.run(U)
    ctx.sync()
    assert ctx.ticket() == 2 * U
    log = ctx.read_log(0)
    assert len(log) == 2 * U and np.array_equal(log["k"], np.arange(2 * U))
    ev = log_events(log)
    grad = (ev[:, 3] & 1) == 0
    assert grad.sum() > 50 and (~grad).sum() > 50                # flushes and pure averages
    assert ((ev[grad, 3] & FF) != 0).all()
    # COMPENSATE marks the gradients pulled while the previous one was buffered
    assert ((ev[grad, 3] & COMP) != 0).any() == (wait_free == 2)
    assert (ev[grad, 2] > 0).any()                               # reads are stale by the gossip in between
    cnt = ctx.update_counts()
    assert sum(cnt.values()) == int(grad.sum())
    T = int(ev[:, 2].max())
    Xo, _ = O.replay(prob, X0, e, r, ev, T=T)
    assert np.array_equal(read_all(ctx).view(np.uint32), Xo.view(np.uint32))
    ctx.destroy()


def test_wait_free_configuration_errors(P):
    n, d = 4, 256
    e, r = synth.ring(n)
    with pytest.raises(P.AdpsgdError) as ei:
        P.Context(e, n, d, role=r, wait_free=1)                  # needs the quadratic model
    assert ei.value.code == 12
    kw, _ = quad_setup(1)
    with pytest.raises(P.AdpsgdError) as ei:
        P.Context(e, n, d, role=r, wait_free=1, engine_variant=1, **kw)
    assert ei.value.code == 12
    with pytest.raises(P.AdpsgdError) as ei:
        P.Context(e, n, d, role=r, wait_free=3, **kw)
    assert ei.value.code == 1
