"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the
same seeded inputs (-m gpu).  Bars:
  * pure-gossip replay and the synthetic quadratic (no reductions): bit-exact;
  * lsq / logreg replay: |x_gpu - x_orc| <= 1e-4 * max(|x_orc|, rms(x_orc)) (reading c11);
  * consensus mean: <= 1 ulp; M_k: 1e-9 relative;
  * free-running engine: its event log replayed through the oracle reproduces
    the GPU models bitwise; column sum within the c10 tolerances.
"""
import math
import os
import sys

import numpy as np
import pytest

import synth
from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    from paper_1710_06952_b200 import build
    build.build()
    import paper_1710_06952_b200 as P
    return P


def torch_out(d):
    import torch
    return torch.empty(d, dtype=torch.float32, device="cuda")


def read_all(ctx):
    return np.stack([ctx.read_model(w) for w in range(ctx.n)])


def c11_ok(x_gpu, x_orc, tol=1e-4):
    rms = np.sqrt(np.mean(x_orc.astype(np.float64) ** 2, axis=1, keepdims=True))
    bound = tol * np.maximum(np.abs(x_orc), rms)
    return np.abs(x_gpu.astype(np.float64) - x_orc) <= bound


def log_events(log):
    return np.stack([log["i"], log["j"], log["tau"], log["flags"].astype(np.int32)], 1)


# ------------------------------------------------------------ pure gossip ---
@pytest.mark.parametrize("d", [1 << 20, 1000, 4099, 1])
@pytest.mark.parametrize("path", [1, 2])
def test_pure_gossip_replay_bit_exact(P, d, path):
    """Config 2 (n=16 bipartite ring), pure averaging, bit-exact vs the oracle;
    ragged d (not a multiple of 4 / 64) and d=1 as edge cases; HOST and ENGINE."""
    n = 16
    e, r = synth.ring(n)
    K = 4000 if d == 1 << 20 else 600
    for seed in ([0, 1] if d == 1 << 20 else [3]):
        X0 = synth.x0_uniform(n, d, seed=100 + seed)
        ev, _ = synth.schedule_iid(n, e, K=K, seed=seed, no_grad=True)
        ctx = P.Context(e, n, d, role=r, x0_per_worker=X0)
        ctx.replay(ev, flags=path)
        ctx.sync()
        Xg = read_all(ctx)
        Xo, _ = O.replay(O.OracleProblem(), X0, e, r, ev)
        assert np.array_equal(Xg.view(np.uint32), Xo.view(np.uint32)), (seed, path)
        ctx.destroy()


def test_empty_and_partnerless_events(P):
    n, d = 4, 300
    e, r = synth.ring(n)
    X0 = synth.x0_uniform(n, d, seed=5)
    ctx = P.Context(e, n, d, role=r, x0_per_worker=X0)
    ctx.replay(np.zeros((0, 4), np.int32))                       # empty schedule
    ctx.replay([[2, -1, 0, P.EV_NO_GRAD]])                          # W = I, no gradient
    ctx.sync()
    assert np.array_equal(read_all(ctx), X0)
    assert ctx.ticket() == 1                                     # k still advances
    ctx.destroy()


def test_replay_errors(P):
    n, d = 4, 64
    e, r = synth.ring(n)
    ctx = P.Context(e, n, d, role=r, T=1, model=P.MODEL_QUADRATIC, gamma=0.1, quad_keys=(1, 2))
    with pytest.raises(P.AdpsgdError) as ei:
        ctx.replay([[0, 2, 0, 0]])
    assert ei.value.code == 4
    with pytest.raises(P.AdpsgdError) as ei:
        ctx.replay([[0, 1, 0, 0], [1, 0, 2, 0]])
    assert ei.value.code == 5
    with pytest.raises(P.AdpsgdError) as ei:
        ctx.replay([[0, 1, 1, 0]])                              # tau > k
    assert ei.value.code == 5
    ctx.destroy()


# ------------------------------------------------------ synthetic quadratic --
@pytest.mark.parametrize("d,n,K,T", [(100003, 8, 300, 3), (4096, 4, 2000, 4)])
def test_quadratic_replay_bit_exact_with_staleness(P, d, n, K, T):
    """Quadratic gradients (elementwise, no reductions) with stale reads
    tau ~ U{0..T}: bit-exact vs the oracle's Alg. 1."""
    e, r = synth.ring(n)
    dk, nk = synth.quad_keys(4)
    s = float(np.float32(0.1 * math.sqrt(3 * 32)))
    ev, _ = synth.schedule_iid(n, e, K=K, T=T, seed=7, local_prob=0.2)
    ctx = P.Context(e, n, d, role=r, T=T, model=P.MODEL_QUADRATIC, gamma=0.01, batch_M=32,
                    quad_keys=(dk, nk), quad_noise_s=s)
    ctx.replay(ev)
    ctx.sync()
    prob = O.OracleProblem(O.MODEL_QUADRATIC, M=32, gamma=0.01, data_key=dk, noise_key=nk, noise_s=s)
    Xo, _ = O.replay(prob, np.zeros((n, d), np.float32), e, r, ev, T=T)
    assert np.array_equal(read_all(ctx).view(np.uint32), Xo.view(np.uint32))
    ctx.destroy()


@pytest.mark.parametrize("d,n,K,T,ff", [(100003, 8, 400, 3, False), (1 << 20, 16, 600, 4, False),
                                        (4099, 4, 300, 2, True)])
def test_engine_replay_with_stale_reads_bit_exact(P, d, n, K, T, ff):
    """The persistent engine replays tau ~ U{0..T} (X_hat = X_{k - tau}):
    each stale gradient is a read op of the worker's op sequence at X_{k - tau}
    (adpsgd_plan_replay) -- bit-exact vs the oracle's Alg. 1 (and App. A
    flush-first events when ff, reading R20)."""
    e, r = synth.ring(n)
    dk, nk = synth.quad_keys(6)
    s = float(np.float32(0.1 * math.sqrt(3 * 32)))
    ev, _ = synth.schedule_iid(n, e, K=K, T=T, seed=19, local_prob=0.2)
    ev[::9, 3] = 1                                        # some pure averages in between
    if ff:
        ev[(ev[:, 3] & 1) == 0, 3] |= P.EV_FLUSH_FIRST
    X0 = synth.x0_uniform(n, d, seed=5)
    ctx = P.Context(e, n, d, role=r, T=T, model=P.MODEL_QUADRATIC, gamma=0.01, batch_M=32,
                    quad_keys=(dk, nk), quad_noise_s=s, x0_per_worker=X0)
    ctx.replay(ev, flags=P.REPLAY_ENGINE)
    ctx.sync()
    prob = O.OracleProblem(O.MODEL_QUADRATIC, M=32, gamma=0.01, data_key=dk, noise_key=nk, noise_s=s)
    Xo, _ = O.replay(prob, X0, e, r, ev, T=T)
    assert np.array_equal(read_all(ctx).view(np.uint32), Xo.view(np.uint32))
    assert ctx.ticket() == K
    ctx.destroy()


def test_quadratic_engine_replay_full_size(P):
    """BASELINE size d = 25.6M, n = 8, tau = 0, through the persistent engine
    (the launch configuration bench.py times): bit-exact vs the oracle."""
    n, d, K = 8, 25_600_000, 24
    e, r = synth.ring(n)
    dk, nk = synth.quad_keys(5)
    s = float(np.float32(0.1 * math.sqrt(3 * 32)))
    ev, _ = synth.schedule_iid(n, e, K=K, seed=11, local_prob=0.3)
    ctx = P.Context(e, n, d, role=r, model=P.MODEL_QUADRATIC, gamma=0.01, batch_M=32,
                    quad_keys=(dk, nk), quad_noise_s=s)
    ctx.replay(ev, flags=P.REPLAY_ENGINE)
    ctx.sync()
    prob = O.OracleProblem(O.MODEL_QUADRATIC, M=32, gamma=0.01, data_key=dk, noise_key=nk, noise_s=s)
    Xo, _ = O.replay(prob, np.zeros((n, d), np.float32), e, r, ev)
    for w in range(n):
        assert np.array_equal(ctx.read_model(w).view(np.uint32), Xo[w].view(np.uint32)), w
    ctx.destroy()


# -------------------------------------------------------- lsq / logreg -------
@pytest.mark.parametrize("kind", ["lsq", "logreg"])
def test_config1_replay_within_1e4(P, kind):
    """Config 1: n=4 ring, d=1024, M=32, T=4, 2000 steps, explicit batches:
    max relative error <= 1e-4 per parameter (reading c11)."""
    n, d, M, K, T = 4, 1024, 32, 2000, 4
    e, r = synth.ring(n)
    if kind == "lsq":
        A, b = synth.lsq_data(S=8192, d=d, seed=1)
        model, okind, gamma = P.MODEL_LSQ, O.MODEL_LSQ, 0.5
    else:
        A, b = synth.logreg_data(S=8192, d=d, seed=2)
        model, okind, gamma = P.MODEL_LOGREG, O.MODEL_LOGREG, 0.5
    ev, bi = synth.schedule_iid(n, e, K=K, T=T, M=M, S=8192, seed=42)
    ctx = P.Context(e, n, d, role=r, T=T, model=model, gamma=gamma, batch_M=M, data_A=A, data_b=b)
    ctx.replay(ev, batch_idx=bi)
    ctx.sync()
    Xg = read_all(ctx)
    prob = O.OracleProblem(okind, M=M, gamma=gamma, A=A, b=b)
    Xo, _ = O.replay(prob, np.zeros((n, d), np.float32), e, r, ev, bi, T=T)
    ok = c11_ok(Xg, Xo)
    assert ok.all(), (np.abs(Xg - Xo).max(), (~ok).sum(), O.full_loss(prob, Xg.mean(0)),
                      O.full_loss(prob, Xo.mean(0)))
    # progress sanity (not parity -- that is the c11 check above): least squares
    # starts at f(0) = mean(b^2)/2 ~ 1/2 and its optimum is ~1e-4 of that (SURVEY
    # config 1); the logistic loss starts at ln 2 and decreases far
    # more slowly (label noise in synth.logreg_data, a flat loss far from the
    # margin) -- so the bar is 1/10 of f(0) for lsq and 1/2 for logreg
    frac = 0.1 if kind == "lsq" else 0.5
    assert O.full_loss(prob, Xo.mean(0)) < O.full_loss(prob, np.zeros(d, np.float32)) * frac
    ctx.destroy()


def test_device_batch_sampling_matches_oracle_philox(P):
    """batch_idx = NULL: both sides draw idx = (Philox(seed; k, m, BATCH).x * S) >> 32."""
    n, d, M, K = 4, 256, 8, 200
    e, r = synth.ring(n)
    A, b = synth.lsq_data(S=512, d=d, seed=3)
    seed = 0x1234_5678_9ABC
    ev, _ = synth.schedule_iid(n, e, K=K, seed=1)
    ctx = P.Context(e, n, d, role=r, model=P.MODEL_LSQ, gamma=0.1, batch_M=M, data_A=A, data_b=b, seed=seed)
    ctx.replay(ev)
    ctx.sync()
    prob = O.OracleProblem(O.MODEL_LSQ, M=M, gamma=0.1, A=A, b=b,
                           batch_key=(seed & 0xFFFFFFFF, seed >> 32))
    Xo, _ = O.replay(prob, np.zeros((n, d), np.float32), e, r, ev)
    assert c11_ok(read_all(ctx), Xo).all()
    ctx.destroy()


# -------------------------------------------------------- consensus output ---
@pytest.mark.parametrize("n,d", [(16, 1 << 20), (8, 1 << 20), (6, 4100), (4, 1001), (2, 4)])
def test_consensus_mean_within_one_ulp(P, n, d):
    """n > 8 or d % 4 != 0: scalar kernel; otherwise the float4 register form."""
    e, r = synth.ring(n)
    X0 = synth.x0_uniform(n, d, seed=9) * np.float32(1000.0)
    ctx = P.Context(e, n, d, role=r, x0_per_worker=X0)
    out = torch_out(d)
    mk = ctx.consensus_mean(out.data_ptr())
    xg = out.cpu().numpy()
    xo, mko = O.consensus_mean(X0)
    ulp = np.abs(xg.view(np.int32).astype(np.int64) - xo.view(np.int32).astype(np.int64))
    assert ulp.max() <= 1
    assert abs(mk - mko) <= 1e-9 * mko
    ctx.destroy()


# ------------------------------------------------------ free-running engine --
@pytest.mark.parametrize("model", ["none", "quadratic"])
def test_free_running_log_replays_bitwise(P, model):
    """Free-running engine (device try-locks, tickets): its event log, replayed
    through the oracle, reproduces every GPU model bitwise."""
    n, d, U = 8, 1 << 18, 3000
    e, r = synth.ring(n)
    dk, nk = synth.quad_keys(6)
    s = float(np.float32(0.1 * math.sqrt(3 * 32)))
    X0 = synth.x0_uniform(n, d, seed=12)
    kw = dict(model=P.MODEL_QUADRATIC, gamma=0.01, batch_M=32, quad_keys=(dk, nk), quad_noise_s=s) \
        if model == "quadratic" else {}
    ctx = P.Context(e, n, d, role=r, x0_per_worker=X0, seed=77, **kw)
    ctx.run(U)
    ctx.sync()
    assert ctx.ticket() == U
    log = ctx.read_log(0)
    assert len(log) == U and np.array_equal(log["k"], np.arange(U))
    Xg = read_all(ctx)
    prob = O.OracleProblem(O.MODEL_QUADRATIC, M=32, gamma=0.01, data_key=dk, noise_key=nk, noise_s=s) \
        if model == "quadratic" else O.OracleProblem()
    Xo, _ = O.replay(prob, X0, e, r, log_events(log))
    assert np.array_equal(Xg.view(np.uint32), Xo.view(np.uint32))
    if model == "none":
        S0 = X0.astype(np.float64).sum(0)
        S1 = Xg.astype(np.float64).sum(0)
        assert np.linalg.norm(S1 - S0) / np.linalg.norm(S0) <= 1e-5
        assert np.max(np.abs(S1 - S0) / np.abs(X0.astype(np.float64)).sum(0)) <= 1e-5
    else:
        cnt = ctx.update_counts()
        assert sum(cnt.values()) == U
    ctx.destroy()


def test_free_running_straggler_locality(P):
    """One worker 10x slower: it makes ~10x fewer updates while
    the others keep their pace."""
    n, d = 8, 1 << 16
    e, r = synth.ring(n)
    st = synth.stragglers(n, slow_worker=0, slow=10.0)
    ctx = P.Context(e, n, d, role=r, model=P.MODEL_QUADRATIC, gamma=0.01, batch_M=32, quad_keys=(1, 2),
                    straggler=st, compute_ns=200_000)
    ctx.run(4000)
    ctx.sync()
    c = ctx.update_counts()
    others = np.mean([c[w] for w in range(1, n)])
    assert c[0] < others / 5
    assert sum(c.values()) == 4000
    ctx.destroy()


def test_full_size_free_running_parity(P):
    """BASELINE workload (d = 25.6M, n = 8 on one GPU, 10x straggler), the
    configuration bench.py times: log replay through the oracle is bitwise."""
    n, d, U = 8, 25_600_000, 32
    e, r = synth.ring(n)
    dk, nk = synth.quad_keys(7)
    s = float(np.float32(0.1 * math.sqrt(3 * 32)))
    ctx = P.Context(e, n, d, role=r, model=P.MODEL_QUADRATIC, gamma=0.01, batch_M=32, quad_keys=(dk, nk),
                    quad_noise_s=s, straggler=synth.stragglers(n), compute_ns=50_000)
    ctx.run(U)
    ctx.sync()
    log = ctx.read_log(0)
    prob = O.OracleProblem(O.MODEL_QUADRATIC, M=32, gamma=0.01, data_key=dk, noise_key=nk, noise_s=s)
    Xo, _ = O.replay(prob, np.zeros((n, d), np.float32), e, r, log_events(log))
    for w in range(n):
        assert np.array_equal(ctx.read_model(w).view(np.uint32), Xo[w].view(np.uint32)), w
    ctx.destroy()


# --------------------------------------------------------- step / gossip ----
def test_step_and_gossip_match_oracle(P):
    n, d = 4, 5000
    e, r = synth.ring(n)
    dk, nk = synth.quad_keys(8)
    X0 = synth.x0_uniform(n, d, seed=3)
    ctx = P.Context(e, n, d, role=r, x0_per_worker=X0, model=P.MODEL_QUADRATIC, gamma=0.05, batch_M=4,
                    quad_keys=(dk, nk), quad_noise_s=0.2, seed=5)
    for t in range(40):
        ctx.step(t % n)
    ctx.sync()
    log = ctx.read_log(0)
    assert len(log) == 40
    prob = O.OracleProblem(O.MODEL_QUADRATIC, M=4, gamma=0.05, data_key=dk, noise_key=nk, noise_s=0.2)
    Xo, _ = O.replay(prob, X0, e, r, log_events(log))
    assert np.array_equal(read_all(ctx).view(np.uint32), Xo.view(np.uint32))
    ctx.gossip(0, 1)
    ctx.gossip(3, 0)                    # passive named first: the same pair average
    ctx.sync()
    Xo2, _ = O.replay(O.OracleProblem(), Xo, e, r, [[0, 1, 0, 1], [3, 0, 0, 1]])
    assert np.array_equal(read_all(ctx).view(np.uint32), Xo2.view(np.uint32))
    # reading R23: pure averages take tickets 40, 41 and are logged with NO_GRAD
    log2 = ctx.read_log(0)
    assert ctx.ticket() == 42 and len(log2) == 42
    assert log_events(log2)[40:].tolist() == [[0, 1, 0, 1], [3, 0, 0, 1]]
    Xo3, _ = O.replay(prob, X0, e, r, log_events(log2))
    assert np.array_equal(read_all(ctx).view(np.uint32), Xo3.view(np.uint32))
    ctx.destroy()


# ---------------------------------------------------- AllReduce baseline ----
def test_allreduce_sgd_matches_oracle(P):
    n, d, R = 8, 10007, 20
    e, r = synth.ring(n)
    dk, nk = synth.quad_keys(9)
    ctx = P.Context(e, n, d, role=r, model=P.MODEL_QUADRATIC, gamma=0.01, batch_M=32, quad_keys=(dk, nk),
                    quad_noise_s=0.5)
    ctx.allreduce_reset()
    ctx.allreduce_sgd(R)
    xg = ctx.allreduce_read_model()
    prob = O.OracleProblem(O.MODEL_QUADRATIC, M=32, gamma=0.01, data_key=dk, noise_key=nk, noise_s=0.5)
    x = np.zeros(d, np.float32)
    for rr in range(R):
        G = np.stack([O.gradient(prob, x, k=rr * n + w) for w in range(n)])
        x = O.allreduce_update(x, G, 0.01)
    np.testing.assert_allclose(xg, x, rtol=1e-5, atol=1e-6)
    ctx.destroy()


# ------------------------------------------------------------- MLP (tcgen05) --
@pytest.mark.parametrize("dims,K,T", [((256, 128, 10), 2000, 2), ((3072, 512, 10), 6, 1)])
def test_mlp_replay_within_1e4(P, dims, K, T):
    """Config 3 MLP gradients (3xTF32 tcgen05 GEMMs) with stale reads: after K
    replayed events every parameter within reading R11 of the fp64 oracle."""
    I, H, Ocl = dims
    n, M = 4, 128
    e, r = synth.ring(n)
    X, y = synth.mlp_data(S=2048 if I == 256 else 4096, n_in=I, n_out=Ocl, s=0.02 if I == 3072 else 0.3, seed=3)
    x0 = synth.mlp_init(I, H, Ocl, seed=4)
    d = x0.size
    gamma = 0.002 if I == 3072 else 0.01
    ev, bi = synth.schedule_iid(n, e, K=K, T=T, M=M, S=X.shape[0], seed=21)
    ctx = P.Context(e, n, d, role=r, T=T, model=P.MODEL_MLP, gamma=gamma, batch_M=M, data_A=X, data_y=y,
                    mlp_dims=dims, x0=x0)
    ctx.replay(ev, batch_idx=bi)
    ctx.sync()
    Xg = read_all(ctx)
    prob = O.OracleProblem(O.MODEL_MLP, M=M, gamma=gamma, A=X, y=y, dims=dims)
    Xo, _ = O.replay(prob, np.tile(x0, (n, 1)), e, r, ev, bi, T=T)
    ok = c11_ok(Xg, Xo)
    assert ok.all(), (np.abs(Xg - Xo).max(), (~ok).sum())
    if K >= 1000:
        assert O.full_loss(prob, Xo.mean(0)) < 0.7 * O.full_loss(prob, x0)
    ctx.destroy()


def test_mlp_batch_256_multi_tile_within_1e4(P):
    """MLP gradients at batch M = 256: two M tiles in GEMM1 (each drawing and publishing its own
    batch rows), GEMM1's split-K left as two cluster-reduced planes that the per-sample kernel
    sums, and GEMM2's K = 256 contraction refilling its gathered stages -- replayed with stale
    reads against the fp64 oracle under reading R11."""
    I, H, Ocl = 256, 128, 10
    n, M, T, K = 4, 256, 2, 40
    e, r = synth.ring(n)
    X, y = synth.mlp_data(S=2048, n_in=I, n_out=Ocl, s=0.3, seed=5)
    x0 = synth.mlp_init(I, H, Ocl, seed=6)
    ev, bi = synth.schedule_iid(n, e, K=K, T=T, M=M, S=X.shape[0], seed=33)
    ctx = P.Context(e, n, x0.size, role=r, T=T, model=P.MODEL_MLP, gamma=0.005, batch_M=M, data_A=X, data_y=y,
                    mlp_dims=(I, H, Ocl), x0=x0)
    ctx.replay(ev, batch_idx=bi)
    ctx.sync()
    Xg = read_all(ctx)
    prob = O.OracleProblem(O.MODEL_MLP, M=M, gamma=0.005, A=X, y=y, dims=(I, H, Ocl))
    Xo, _ = O.replay(prob, np.tile(x0, (n, 1)), e, r, ev, bi, T=T)
    ok = c11_ok(Xg, Xo)
    assert ok.all(), (np.abs(Xg - Xo).max(), (~ok).sum())
    ctx.destroy()


# ------------------------------------------------- spectral-gap contraction --
def test_pure_gossip_contracts_at_the_spectral_rate(P):
    """Config 2 property (north star): on the n = 16 bipartite ring, the seed-mean
    consensus error E||Y_k||^2/||Y_0||^2 of GPU pure-gossip replays equals the
    exact second moment tr(T^k(G0))/tr(G0) (reading R9) within 4 SE, stays below
    the lemma's rho^k + 4 SE, and its fitted per-event log-rate
    matches log r_T."""
    from oracle import theory as TH
    n, d, K, R = 16, 2048, 1600, 48
    e, r = synth.ring(n)
    rho = TH.rho(TH.expected_gram(n, e))
    checkpoints = [100, 400, 800, 1200, 1600]
    ratios = np.zeros((R, len(checkpoints)))
    want = np.zeros((R, len(checkpoints)))
    for s in range(R):
        X0 = synth.x0_uniform(n, d, seed=500 + s)
        ev, _ = synth.schedule_iid(n, e, K=K, seed=900 + s, no_grad=True)
        ctx = P.Context(e, n, d, role=r, x0_per_worker=X0)
        Y0 = X0.astype(np.float64) - X0.astype(np.float64).mean(0)
        tr = TH.second_moment_trace(n, e, X0, K)
        done = 0
        for c, kc in enumerate(checkpoints):
            ctx.replay(ev[done:kc], flags=P.REPLAY_HOST)
            done = kc
            X = read_all(ctx).astype(np.float64)
            Y = X - X.mean(0)
            ratios[s, c] = (Y ** 2).sum() / (Y0 ** 2).sum()
            want[s, c] = tr[kc] / tr[0]
        ctx.destroy()
    m, se = ratios.mean(0), ratios.std(0) / np.sqrt(R)
    assert np.all(np.abs(m - want.mean(0)) < 4 * se + 1e-12), (m, want.mean(0), se)
    assert np.all(m <= rho ** np.array(checkpoints) + 4 * se)
    slope = np.polyfit(checkpoints[1:], np.log(want.mean(0)[1:]), 1)[0]
    fit = np.polyfit(checkpoints[1:], np.log(m[1:]), 1)[0]
    assert abs(fit - slope) < 5e-4, (fit, slope)


@pytest.mark.parametrize("topo", ["ring", "skip"])
def test_dpsgd_baseline_bit_exact(P, topo):
    """D-PSGD baseline (reading R19): synchronous rounds bit-exact
    against the oracle (fixed fp32 op order, elementwise gradient)."""
    n, d, R = 16, 10007, 12
    e, r = synth.ring(n) if topo == "ring" else synth.skip_ring(n)
    dk, nk = synth.quad_keys(13)
    X0 = synth.x0_uniform(n, d, seed=41)
    ctx = P.Context(e, n, d, role=r, model=P.MODEL_QUADRATIC, gamma=0.02, batch_M=8, quad_keys=(dk, nk),
                    quad_noise_s=0.3)
    ctx.dpsgd_reset(X0)
    ctx.dpsgd(R)
    Xg = np.stack([ctx.dpsgd_read_model(w) for w in range(n)])
    prob = O.OracleProblem(O.MODEL_QUADRATIC, M=8, gamma=0.02, data_key=dk, noise_key=nk, noise_s=0.3)
    Xo = X0
    for rr in range(R):
        Xo = O.dpsgd_round(prob, Xo, e, k_base=rr * n)
    assert np.array_equal(Xg.view(np.uint32), Xo.view(np.uint32))
    ctx.destroy()


def test_skip_ring_free_running_log_replay(P):
    """the skip ring (odd offsets 2^i+1 keep the
    bipartite split) runs through the same engine; log replay is bitwise and
    its rho is below the plain ring's (faster mixing)."""
    from oracle import theory as TH
    n, d, U = 16, 1 << 16, 2000
    e, r = synth.skip_ring(n)
    assert TH.rho(TH.expected_gram(n, e)) < TH.rho(TH.expected_gram(n, synth.ring(n)[0])) - 0.03
    X0 = synth.x0_uniform(n, d, seed=31)
    dk, nk = synth.quad_keys(12)
    ctx = P.Context(e, n, d, role=r, x0_per_worker=X0, model=P.MODEL_QUADRATIC, gamma=0.01, batch_M=32,
                    quad_keys=(dk, nk), quad_noise_s=0.3, seed=3)
    ctx.run(U)
    ctx.sync()
    log = ctx.read_log(0)
    prob = O.OracleProblem(O.MODEL_QUADRATIC, M=32, gamma=0.01, data_key=dk, noise_key=nk, noise_s=0.3)
    Xo, _ = O.replay(prob, X0, e, r, log_events(log))
    assert np.array_equal(read_all(ctx).view(np.uint32), Xo.view(np.uint32))
    ctx.destroy()


def test_slow_link_locality_and_log_replay(P):
    """Heterogeneous communication (reading R21): worker 1's link
    is 10x slower.  Only the averages touching it wait; actives away from it
    keep their pace; the event log still replays bitwise through the oracle."""
    n, d, U = 8, (1 << 16) + 12, 3000
    e, r = synth.ring(n)
    dk, nk = synth.quad_keys(17)
    s = float(np.float32(0.1 * math.sqrt(3 * 32)))
    X0 = synth.x0_uniform(n, d, seed=18)
    link = np.ones(n, np.float32)
    link[1] = 10.0
    ctx = P.Context(e, n, d, role=r, x0_per_worker=X0, model=P.MODEL_QUADRATIC, gamma=0.01, batch_M=32,
                    quad_keys=(dk, nk), quad_noise_s=s, compute_ns=20_000, link_slow=link, link_ns=100_000,
                    seed=3)
    ctx.run(U)
    ctx.sync()
    log = ctx.read_log(0)
    ev = log_events(log)
    prob = O.OracleProblem(O.MODEL_QUADRATIC, M=32, gamma=0.01, data_key=dk, noise_key=nk, noise_s=s)
    Xo, _ = O.replay(prob, X0, e, r, ev)
    assert np.array_equal(read_all(ctx).view(np.uint32), Xo.view(np.uint32))
    served = {w: int((ev[:, 1] == w).sum()) for w in range(1, n, 2)}
    assert served[1] < 0.5 * np.mean([served[w] for w in (3, 5, 7)])
    cnt = ctx.update_counts()
    assert min(cnt[4], cnt[6]) > max(cnt[0], cnt[2])            # actives not adjacent to worker 1
    ctx.destroy()


def test_fused_passive_steps_replay_bitwise(P):
    """Engine fusion: a due passive's local step run inside the pair pass that
    holds its lock (events k-1 = (j, -1) and k = (i, j), one pass).  A long
    passive wait makes fusion frequent; the log must still replay bitwise and
    every fused step must sit right before its pair, sharing its start time."""
    n, d, U = 8, (1 << 18) + 44, 3000
    e, r = synth.ring(n)
    dk, nk = synth.quad_keys(19)
    s = float(np.float32(0.1 * math.sqrt(3 * 32)))
    X0 = synth.x0_uniform(n, d, seed=20)
    ctx = P.Context(e, n, d, role=r, x0_per_worker=X0, model=P.MODEL_QUADRATIC, gamma=0.01, batch_M=32,
                    quad_keys=(dk, nk), quad_noise_s=s, compute_ns=20_000, seed=4,
                    engine_fuse_wait_ns=200_000)
    ctx.run(U)
    ctx.sync()
    log = ctx.read_log(0)
    loc = log["j"] < 0
    fused = loc[:-1] & (log["j"][1:] == log["i"][:-1]) & (log["t0"][1:] == log["t0"][:-1])
    assert fused.sum() > 20
    prob = O.OracleProblem(O.MODEL_QUADRATIC, M=32, gamma=0.01, data_key=dk, noise_key=nk, noise_s=s)
    Xo, _ = O.replay(prob, X0, e, r, log_events(log))
    assert np.array_equal(read_all(ctx).view(np.uint32), Xo.view(np.uint32))
    assert sum(ctx.update_counts().values()) == U
    ctx.destroy()


def test_max_local_workers_free_running(P):
    """The engine's limit of 128 workers on one GPU (config 5 at one GPU): a
    free-running quadratic run at n = 128 replays bitwise; n = 129 is refused."""
    n, d, U = 128, 4096 + 8, 2000
    e, r = synth.ring(n)
    dk, nk = synth.quad_keys(23)
    s = float(np.float32(0.1 * math.sqrt(3 * 32)))
    X0 = synth.x0_uniform(n, d, seed=24)
    ctx = P.Context(e, n, d, role=r, x0_per_worker=X0, model=P.MODEL_QUADRATIC, gamma=0.01, batch_M=32,
                    quad_keys=(dk, nk), quad_noise_s=s, compute_ns=5_000,
                    straggler=synth.stragglers(n, hetero=True), seed=6)
    ctx.run(U)
    ctx.sync()
    log = ctx.read_log(0)
    prob = O.OracleProblem(O.MODEL_QUADRATIC, M=32, gamma=0.01, data_key=dk, noise_key=nk, noise_s=s)
    Xo, _ = O.replay(prob, X0, e, r, log_events(log))
    assert np.array_equal(read_all(ctx).view(np.uint32), Xo.view(np.uint32))
    assert len({int(w) for w in log["i"]}) > 100                  # most workers made progress
    ctx.destroy()
    e2, r2 = synth.ring(130)
    with pytest.raises(P.AdpsgdError) as ei:
        P.Context(e2, 130, 64, role=r2)
    assert ei.value.code == 12


def test_divergence_is_reported(P):
    """a diverging run (gamma * M * h_max far above 2) is reported as
    ADPSGD_E_DIVERGED by the consensus output and the next sync -- as the oracle
    reports it for the same schedule."""
    n, d = 4, 1000
    e, r = synth.ring(n)
    ctx = P.Context(e, n, d, role=r, model=P.MODEL_QUADRATIC, gamma=50.0, batch_M=32, quad_keys=(1, 2),
                    quad_noise_s=1.0, compute_ns=0)
    ctx.run(400)
    out = torch_out(d)
    with pytest.raises(P.AdpsgdError) as ei:
        ctx.consensus_mean(out.data_ptr(), with_mk=True)
    assert ei.value.code == 6
    with pytest.raises(P.AdpsgdError) as ei:
        ctx.sync()
    assert ei.value.code == 6
    ctx.sync()                                                   # the latch is cleared once reported
    ctx.destroy()
    ev, _ = synth.schedule_iid(n, e, K=400, seed=1)
    prob = O.OracleProblem(O.MODEL_QUADRATIC, M=32, gamma=50.0, data_key=1, noise_key=2, noise_s=1.0)
    with pytest.raises(O.OracleError) as eo:
        O.replay(prob, np.zeros((n, d), np.float32), e, r, ev)
    assert eo.value.code == 6


def test_config3_full_size_2000_steps_vs_oracle_fixture(P):
    """Config 3 at its own size (BASELINE configs[2]): 3072 -> 512 -> 10
    tanh MLP, n = 8 ring, M = 128, tau ~ U{0..4}, 2000 events, tcgen05 3xTF32
    gradients, against the ORACLE's result stored by tools/make_config3_reference.py
    (tests/golden/config3_mlp_2000_oracle.json: seeded coordinate subset + row rms).
    Acceptance: reading R11 (|x_gpu - x_orc| <= 1e-4 max(|x_orc|, rms)) on every
    stored coordinate of every worker."""
    import json
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
    import make_config3_reference as R
    with open(R.OUT_PATH) as f:
        ref = json.load(f)
    X, y, x0, e, r, ev, bi = R.inputs()
    assert ref["digest_inputs"] == {"data": R.digest(X, y), "x0": R.digest(x0), "schedule": R.digest(ev, bi)}
    ctx = P.Context(e, R.N, x0.size, role=r, T=R.T, model=P.MODEL_MLP, gamma=R.GAMMA, batch_M=R.M, data_A=X,
                    data_y=y, mlp_dims=(R.I, R.H, R.OUT), x0=x0)
    ctx.replay(ev, batch_idx=bi)
    ctx.sync()
    idx = np.array(ref["idx"], np.int64)
    worst = 0.0
    for w in range(R.N):
        xg = ctx.read_model(w)[idx].astype(np.float64)
        xo = np.array(ref["values"][w], np.float64)
        err = np.abs(xg - xo) / np.maximum(np.abs(xo), ref["rms"][w])
        worst = max(worst, float(err.max()))
    assert worst <= 1e-4, worst
    assert ref["loss_xbar"] < 0.9 * ref["loss_x0"]          # the run made progress (oracle's own)
    ctx.destroy()


def test_free_running_reaches_oracle_loss_threshold(P):
    """Reading c20 (north star: free-running 'reaches the oracle's loss
    threshold'; P:861-863 'w.r.t. epochs ... converge similar'): L* = f(x_bar)
    after K_ref updates of a seeded i.i.d. Algorithm-1 schedule replayed by the
    oracle; the free-running engine (worker 0 slowed 10x) must reach
    f(x_bar) <= L* within 1.5 K_ref committed updates.  Config-4 quadratic at
    d = 2^20, n = 16."""
    n, d, K_ref = 16, 1 << 20, 3000
    e, r = synth.ring(n)
    dk, nk = synth.quad_keys(12)
    s = float(np.float32(0.1 * math.sqrt(3 * 32)))
    prob = O.OracleProblem(O.MODEL_QUADRATIC, M=32, gamma=0.01, data_key=dk, noise_key=nk, noise_s=s)
    ev = synth.schedule_alg1(n, e, r, K_ref, seed=31)
    Xo, _ = O.replay(prob, np.zeros((n, d), np.float32), e, r, ev)
    L_star = O.full_loss(prob, Xo.astype(np.float64).mean(0).astype(np.float32))
    L0 = O.full_loss(prob, np.zeros(d, np.float32))
    assert L_star < 0.9 * L0
    ctx = P.Context(e, n, d, role=r, model=P.MODEL_QUADRATIC, gamma=0.01, batch_M=32, quad_keys=(dk, nk),
                    quad_noise_s=s, straggler=synth.stragglers(n), compute_ns=20_000, seed=5)
    ctx.run(int(1.5 * K_ref))
    ctx.sync()
    xbar = read_all(ctx).astype(np.float64).mean(0).astype(np.float32)
    L_gpu = O.full_loss(prob, xbar)
    assert L_gpu <= L_star, (L_gpu, L_star, L0)
    ctx.destroy()
