"""Pins for the CPU oracle (-m "not gpu").  Each test checks the oracle against
something other than itself: a value printed in the paper / SPEC / SURVEY
(cited), a closed form, an invariant, a special case that reduces to a
textbook routine, or brute force on tiny inputs."""
import itertools
import math

import numpy as np
import pytest

import synth
from oracle import oracle as O
from oracle import theory as TH


def f32bits(x):
    return int(np.asarray(x, np.float32).view(np.uint32))


def bits2f(b):
    return np.array([b], np.uint32).view(np.float32)[0]


def quad(h, xstar, gamma, M=1, s=0.0):
    return O.OracleProblem(O.MODEL_QUADRATIC, M=M, gamma=gamma, noise_s=s, h=h, xstar=xstar)


# ------------------------------------------------------------------ RNG ----
def test_philox_known_answers():
    """Philox4x32-10 KATs (Random123 kat_vectors; SURVEY 8(c) 'RNG' row)."""
    assert [hex(v) for v in O.philox([0, 0, 0, 0], [0, 0])] == \
        ["0x6627e8d5", "0xe169c58d", "0xbc57ac4c", "0x9b00dbd8"]
    f = 0xFFFFFFFF
    assert [hex(v) for v in O.philox([f, f, f, f], [f, f])] == \
        ["0x408f276d", "0x41c83b0e", "0xa20bc7c6", "0x6d5451fd"]
    assert [hex(v) for v in O.philox([0x243f6a88, 0x85a308d3, 0x13198a2e, 0x03707344],
                                     [0xa4093822, 0x299f31d0])] == \
        ["0xd16cfe09", "0x94fdcceb", "0x5001e420", "0x24126ea1"]


# lowbias32's published inverse ("lowbias32_r", C. Wellons, hash-prospector):
#   x ^= x >> 16; x *= 0x43021123; x ^= x >> 15 ^ x >> 30; x *= 0x1d69e2a5; x ^= x >> 16
# 0x43021123 and 0x1d69e2a5 are the inverses mod 2^32 of 0x846ca68b and
# 0x7feb352d, and x ^ x>>15 ^ x>>30 undoes the xorshift by 15.  The inverse only
# round-trips if every constant and shift of the forward hash is the published one.
_M = 0xFFFFFFFF


def _xs15_inv(x):
    return x ^ (x >> 15) ^ (x >> 30)


def test_lowbias32_known_inverse():
    rng = np.random.default_rng(5)
    for x in [0, 1, 2, 0xFFFFFFFF, 0x80000000] + rng.integers(0, 2**32, 2000).tolist():
        y = O.lowbias32(int(x))
        y ^= y >> 16
        y = (y * 0x43021123) & _M
        y = _xs15_inv(y)
        y = (y * 0x1d69e2a5) & _M
        y ^= y >> 16
        assert y == x


def test_quad_noise_mix_known_inverse_and_grid():
    """The quadratic's noise mix (DESIGN.md definition v3: u = ((x A) ^ (x A) >> 15) B
    with lowbias32's multipliers A = 0x7feb352d, B = 0x846ca68b) inverts with the
    published inverse multipliers; and the noise v = (u >> 9) 2^-22 - 1 it feeds is
    the 23-bit uniform grid on [-1, 1): mean 0, variance 1/3 (so s v has the
    variance M sigma^2 of a batch sum when s = sigma sqrt(3M), reading R2)."""
    rng = np.random.default_rng(6)
    for x in [0, 1, 0xFFFFFFFF] + rng.integers(0, 2**32, 2000).tolist():
        y = (O.quad_noise_mix(int(x)) * 0x43021123) & _M
        y = (_xs15_inv(y) * 0x1d69e2a5) & _M
        assert y == x
    d = 1 << 18
    p = O.OracleProblem(O.MODEL_QUADRATIC, M=1, noise_key=0x5EED, noise_s=1.0,
                        h=np.ones(d, np.float32), xstar=np.zeros(d, np.float32))
    v = O.gradient(p, np.zeros(d, np.float32), k=3).astype(np.float64)   # det part 0: g = 1 * v
    assert v.min() >= -1.0 and v.max() < 1.0
    grid = (v + 1.0) * 2.0 ** 22
    assert np.array_equal(grid, np.round(grid))
    se = math.sqrt(1 / 3 / d)
    assert abs(v.mean()) < 5 * se
    assert abs(v.var() - 1 / 3) < 5 * math.sqrt(4 / 45 / d)


def test_lowbias32_is_a_bijection_sample():
    """lowbias32 is a composition of invertible steps: no collisions on a block,
    and 0 is its fixed point (every step maps 0 to 0)."""
    vals = {O.lowbias32(x) for x in range(20000)}
    assert len(vals) == 20000
    assert O.lowbias32(0) == 0


# --------------------------------------------------------------- graphs ----
def test_ring_roles_and_errors():
    e, r = synth.ring(4)
    st, roles = O.check_graph(4, e)
    assert st == 0 and list(roles) == [0, 1, 0, 1]
    e5, _ = synth.ring(5)
    assert O.check_graph(5, e5)[0] == 2                      # odd cycle
    assert O.check_graph(4, [[0, 1], [2, 3]])[0] == 3        # disconnected
    assert O.check_graph(3, [[1, 1]])[0] == 1                # self loop
    assert O.check_graph(4, e, role=[0, 0, 1, 1])[0] == 2    # edge joins same roles


def test_bipartite_verdict_matches_brute_force_all_graphs_n5():
    """verdicts equal brute-force 2-colourings on every graph (n <= 5)."""
    for n in range(2, 6):
        pairs = [(a, b) for a in range(n) for b in range(a + 1, n)]
        for mask in range(1 << len(pairs)):
            E = [pairs[t] for t in range(len(pairs)) if mask >> t & 1]
            st, _ = O.check_graph(n, np.array(E, np.int32).reshape(-1, 2))
            # brute force connectivity
            adj = {v: set() for v in range(n)}
            for a, b in E:
                adj[a].add(b); adj[b].add(a)
            seen, stack = {0}, [0]
            while stack:
                u = stack.pop()
                for w in adj[u] - seen:
                    seen.add(w); stack.append(w)
            if len(seen) != n:
                assert st == 3
                continue
            bip = any(all(c[a] != c[b] for a, b in E) for c in itertools.product([0, 1], repeat=n))
            assert st == (0 if bip else 2), (n, E)


# ---------------------------------------------------- update-rule goldens ---
def test_average_golden_vectors():
    """SURVEY 8(c)/App. A.3: (a+b)*0.5 in RN-even fp32, no FTZ.
    avg(1.0f, 3*2^-24): the sum 1 + 3*2^-24 is a tie between 1+2^-23 (odd
    mantissa) and 1+2^-22 (even) -> 0x3f800002, avg 0x3f000002.  (App. A.3
    prints the operand as 0x33c00000, which is 3*2^-25, not 3*2^-24 =
    0x34400000; 0x33c00000 is kept as a non-tie case: 1+3*2^-25 rounds to
    1+2^-23 -> avg 0x3f000001.)"""
    for a, b, want in [(0x00000001, 0x00000001, 0x00000001),
                       (0x3f800000, 0x34400000, 0x3f000002),
                       (0x3f800000, 0x33c00000, 0x3f000001)]:
        X = np.array([[bits2f(a)], [bits2f(b)]], np.float32)
        e, r = synth.ring(2)
        Xo, _ = O.replay(O.OracleProblem(), X, e, r, [[0, 1, 0, synth.EV_NO_GRAD]])
        assert f32bits(Xo[0, 0]) == want and f32bits(Xo[1, 0]) == want


@pytest.mark.parametrize("m,g,want", [(0x3f001907, 0x404b5f9b, 0x3e3afe56),
                                      (0x3efa391b, 0x407a58fc, 0x3dc7c7ac)])
def test_update_golden_vectors_no_fma(m, g, want):
    """x <- fl(m - fl(gamma*g)), gamma = 0x3dcccccd (FMA gives +-1 ulp)."""
    mf, gf = bits2f(m), bits2f(g)
    xstar = np.float32(mf - gf)
    assert np.float32(mf - xstar) == gf          # the quadratic then yields exactly g
    X = np.array([[mf]], np.float32)
    prob = quad([1.0], [xstar], gamma=float(bits2f(0x3dcccccd)))
    Xo, _ = O.replay(prob, X, np.zeros((0, 2), np.int32), None, [[0, -1, 0, 0]])
    assert f32bits(Xo[0, 0]) == want


def test_spec_worked_examples():
    """n=1, x=1, f=x^2/2, gamma=0.1 -> 0.9.  S:255: n=2, (1,3), pair (0,1),
    i_k=0, tau=0 -> (1.9, 2.0) = (0x3ff33333, 0x40000000)."""
    p = quad([1.0], [0.0], gamma=0.1)
    X1, _ = O.replay(p, [[1.0]], np.zeros((0, 2), np.int32), None, [[0, -1, 0, 0]])
    assert X1[0, 0] == np.float32(0.9) or abs(X1[0, 0] - 0.9) < 1e-7
    e, r = synth.ring(2)
    X2, _ = O.replay(p, [[1.0], [3.0]], e, r, [[0, 1, 0, 0]])
    assert f32bits(X2[0, 0]) == 0x3ff33333 and f32bits(X2[1, 0]) == 0x40000000


def test_stale_read_hand_trace():
    """X_hat_k = X_{k - tau}: hand trace, n=2, f = x^2/2, gamma = 0.5.
    k=0 (0,1,tau=0): xhat=1, m=2 -> (1.5, 2).  k=1 (1,0,tau=1): xhat = x_1 of X_0
    = 3, m = 1.75 -> x_1 = 1.75 - 1.5 = 0.25.  (tau = 0 would give 0.75.)"""
    p = quad([1.0], [0.0], gamma=0.5)
    e, r = synth.ring(2)
    X, _ = O.replay(p, [[1.0], [3.0]], e, r, [[0, 1, 0, 0], [1, 0, 1, 0]], T=1)
    assert X[0, 0] == 1.75 and X[1, 0] == 0.25
    X0, _ = O.replay(p, [[1.0], [3.0]], e, r, [[0, 1, 0, 0], [1, 0, 0, 0]], T=1)
    assert X0[1, 0] == 0.75
    with pytest.raises(O.OracleError) as ei:                  # tau > T
        O.replay(p, [[1.0], [3.0]], e, r, [[0, 1, 0, 0], [1, 0, 1, 0]], T=0)
    assert ei.value.code == 5
    with pytest.raises(O.OracleError) as ei:                  # tau > k
        O.replay(p, [[1.0], [3.0]], e, r, [[0, 1, 1, 0]], T=1)
    assert ei.value.code == 5


def test_replay_validation():
    e, r = synth.ring(4)
    p = O.OracleProblem()
    X = np.zeros((4, 2), np.float32)
    with pytest.raises(O.OracleError) as ei:
        O.replay(p, X, e, r, [[0, 2, 0, 1]])                  # (0,2) not an edge
    assert ei.value.code == 4
    with pytest.raises(O.OracleError) as ei:
        O.replay(p, X, e, r, [[1, 1, 0, 1]])                  # i == j
    assert ei.value.code == 1


# ------------------------------------------------- reductions / closed forms
def test_n1_reduces_to_gd_closed_form():
    """P:699-705 (n=1, T=0 is SGD) and S:291: gamma=0.5, f=x^2/2, x0=1 -> 0.5^k exactly."""
    p = quad([1.0], [0.0], gamma=0.5)
    K = 60
    X, _ = O.replay(p, [[1.0]], np.zeros((0, 2), np.int32), None, [[0, -1, 0, 0]] * K)
    assert X[0, 0] == np.float32(2.0 ** -K)


def test_n1_lsq_equals_serial_sgd():
    """n=1, T=0 replay == a serial minibatch-SGD loop written with
    numpy's BLAS (fp64) -- equal to fp32 rounding."""
    A, b = synth.lsq_data(S=256, d=64, seed=5)
    ev, bi = synth.schedule_iid(1, np.zeros((0, 2), np.int32), K=200, M=8, S=256, seed=3)
    p = O.OracleProblem(O.MODEL_LSQ, M=8, gamma=0.05, A=A, b=b)
    X, _ = O.replay(p, np.zeros((1, 64), np.float32), np.zeros((0, 2), np.int32), None, ev, bi)
    x = np.zeros(64, np.float32)
    for k in range(200):
        Ab = A[bi[k]].astype(np.float64)
        g = (Ab.T @ (Ab @ x.astype(np.float64) - b[bi[k]])).astype(np.float32)
        x = (x - np.float32(0.05) * g).astype(np.float32)
    np.testing.assert_allclose(X[0], x, rtol=1e-5, atol=1e-6)


FF, COMP = O.EV_FLUSH_FIRST, O.EV_COMPENSATE


def test_appa_flush_first_hand_example():
    """App. A, Alg. 2: flush g, then average -- both endpoints get
    (x_i - gamma g + x_j)/2.  Alg. 1: average, then x_i -= gamma g.
    f = x^2/2 (g = x), gamma = 0.5, x = (1, 3): App. A -> (1.75, 1.75);
    Alg. 1 -> (1.5, 2).  All values are exact in fp32."""
    p = quad([1.0], [0.0], gamma=0.5)
    e = np.array([[0, 1]], np.int32)
    X, _ = O.replay(p, [[1.0], [3.0]], e, [0, 1], [[0, 1, 0, FF]])
    assert X[:, 0].tolist() == [1.75, 1.75]
    X, _ = O.replay(p, [[1.0], [3.0]], e, [0, 1], [[0, 1, 0, 0]])
    assert X[:, 0].tolist() == [1.5, 2.0]
    # the passive flushes its own gradient with no partner (Alg. 3)
    X, _ = O.replay(p, [[1.0], [3.0]], e, [0, 1], [[1, -1, 0, FF]])
    assert X[:, 0].tolist() == [1.0, 1.5]


def test_appa_compensation_reduces_to_gd_and_delayed_gd():
    """Footnote at P:1265-1268: the computation thread pulls x while g is still
    in the buffer and applies x -= gamma g locally.  n = 1, f = x^2/2, gamma =
    0.5, x0 = 1, every read one event stale (tau = 1): with compensation the
    pulled model equals the current one, so x_k = 0.5^k (plain GD);
    without it, delayed GD x_{k+1} = x_k - 0.5 x_{k-1} (exact rationals)."""
    from fractions import Fraction
    p = quad([1.0], [0.0], gamma=0.5)
    K = 40
    none = np.zeros((0, 2), np.int32)
    ev = [[0, -1, 0, FF | COMP]] + [[0, -1, 1, FF | COMP]] * (K - 1)
    X, _ = O.replay(p, [[1.0]], none, None, ev, T=1)
    assert X[0, 0] == np.float32(2.0 ** -K)
    ev = [[0, -1, 0, FF]] + [[0, -1, 1, FF]] * (K - 1)
    X, _ = O.replay(p, [[1.0]], none, None, ev, T=1)
    xs = [Fraction(1), Fraction(1, 2)]
    for _ in range(K - 1):
        xs.append(xs[-1] - Fraction(1, 2) * xs[-2])
    assert X[0, 0] == np.float32(float(xs[-1]))


def test_appa_compensation_causality_and_lsq_serial_equivalence():
    """(a) A worker computes one gradient at a time (Alg. 1 blocks until g = 0):
    a compensated read older than the previous gradient's read is rejected.
    (b) n = 1 least squares, every read one event stale with compensation ==
    the serial minibatch-SGD loop, numpy fp64 BLAS, to fp32 rounding."""
    p = quad([1.0], [0.0], gamma=0.5)
    none = np.zeros((0, 2), np.int32)
    with pytest.raises(O.OracleError) as ex:
        O.replay(p, [[1.0]], none, None, [[0, -1, 0, 0], [0, -1, 0, COMP], [0, -1, 2, FF | COMP]], T=2)
    assert ex.value.code == 5
    A, b = synth.lsq_data(S=256, d=64, seed=5)
    ev, bi = synth.schedule_iid(1, none, K=200, M=8, S=256, seed=3)
    ev[:, 3] = FF | COMP
    ev[1:, 2] = 1
    pl = O.OracleProblem(O.MODEL_LSQ, M=8, gamma=0.05, A=A, b=b)
    X, _ = O.replay(pl, np.zeros((1, 64), np.float32), none, None, ev, bi, T=1)
    x = np.zeros(64, np.float32)
    for k in range(200):
        Ab = A[bi[k]].astype(np.float64)
        g = (Ab.T @ (Ab @ x.astype(np.float64) - b[bi[k]])).astype(np.float32)
        x = (x - np.float32(0.05) * g).astype(np.float32)
    np.testing.assert_allclose(X[0], x, rtol=1e-5, atol=1e-6)


def test_appa_pair_endpoints_equal_and_sum_moves_by_gradient():
    """Invariants of a flush-first pair event (Alg. 2/3): both endpoints hold
    the same bits afterwards, and the pair sum (hence sum_i x_i) moves by
    -gamma g (S:297 analogue, fp64-tracked, tolerance of reading c10)."""
    n, d = 8, 512
    e, r = synth.ring(n)
    dk, nk = synth.quad_keys(2)
    p = O.OracleProblem(O.MODEL_QUADRATIC, M=8, gamma=0.01, data_key=dk, noise_key=nk, noise_s=0.3)
    X = synth.x0_uniform(n, d, seed=6)
    ev, _ = synth.schedule_iid(n, e, K=40, seed=7, local_prob=0.0)
    ev[:, 3] = FF
    for k in range(40):
        i, j = int(ev[k, 0]), int(ev[k, 1])
        Xn, _ = O.replay(p, X, e, r, ev[k:k + 1], k0=k)
        assert np.array_equal(Xn[i].view(np.uint32), Xn[j].view(np.uint32))
        g = O.gradient(p, X[i], k=O.read_key(k, i))        # tau = 0: read at X_k
        pair0 = X[i].astype(np.float64) + X[j].astype(np.float64)
        pair1 = 2.0 * Xn[i].astype(np.float64)
        np.testing.assert_allclose(pair1 - pair0, -0.01 * g.astype(np.float64), atol=4e-7)
        X = Xn


def test_noiseless_quadratic_converges_to_closed_form_minimiser():
    """Shared noiseless quadratic f = 1/2 sum h (x - x*)^2 with gamma*M*h_max < 1:
    every worker converges to the closed-form minimiser x* (a fixed point of
    both the averaging and the gradient step)."""
    n, d = 8, 256
    e, r = synth.ring(n)
    rng = np.random.default_rng(0)
    h = rng.uniform(0.5, 1.0, d).astype(np.float32)
    xstar = rng.uniform(-1, 1, d).astype(np.float32)
    p = O.OracleProblem(O.MODEL_QUADRATIC, M=4, gamma=0.2, h=h, xstar=xstar)
    ev, _ = synth.schedule_iid(n, e, K=4000, seed=9)
    X, _ = O.replay(p, np.zeros((n, d), np.float32), e, r, ev)
    assert np.abs(X - xstar[None]).max() < 1e-6


def test_column_sum_invariant_pure_gossip():
    """W_k doubly stochastic => sum_i x_i preserved;
    tolerances of reading c10; and x_i == x_j bitwise after an average."""
    n, d = 16, 4096
    e, r = synth.ring(n)
    X0 = synth.x0_uniform(n, d, seed=1)
    ev, _ = synth.schedule_iid(n, e, K=2000, seed=2, no_grad=True)
    X, _ = O.replay(O.OracleProblem(), X0, e, r, ev)
    S0 = X0.astype(np.float64).sum(0)
    S1 = X.astype(np.float64).sum(0)
    assert np.linalg.norm(S1 - S0) / np.linalg.norm(S0) <= 1e-5
    assert np.max(np.abs(S1 - S0) / np.abs(X0.astype(np.float64)).sum(0)) <= 1e-5
    X1, _ = O.replay(O.OracleProblem(), X0, e, r, ev[:1])
    i, j = ev[0, 0], ev[0, 1]
    assert np.array_equal(X1[i].view(np.uint32), X1[j].view(np.uint32))


def test_mean_moves_by_minus_gamma_g():
    """per event, sum_i x_i changes by exactly -gamma*g (fp64-tracked)."""
    n, d = 4, 512
    e, r = synth.ring(n)
    dk, nk = synth.quad_keys(1)
    p = O.OracleProblem(O.MODEL_QUADRATIC, M=8, gamma=0.01, data_key=dk, noise_key=nk, noise_s=0.3)
    X = synth.x0_uniform(n, d, seed=4)
    ev, _ = synth.schedule_iid(n, e, K=50, seed=5)
    for k in range(50):
        i = ev[k, 0]
        g = O.gradient(p, X[i], k=k)
        Xn, _ = O.replay(p, X, e, r, ev[k:k + 1], k0=k)
        dS = Xn.astype(np.float64).sum(0) - X.astype(np.float64).sum(0)
        np.testing.assert_allclose(dS, -0.01 * g.astype(np.float64), atol=4e-7)
        X = Xn


# -------------------------------------------------------------- brute force
def test_bruteforce_enumeration_matches_linear_recursion():
    """ring n=4, d=1, X0=(1,2,3,4), gamma=0.1, h=1, x*=0.5, tau=1
    (clipped at k<tau), 5 events: the probability-weighted mean over all 8^5
    schedules equals the fp64 recursion and SURVEY's printed values."""
    n, K = 4, 5
    e, r = synth.ring(n)
    p = quad([1.0], [0.5], gamma=0.1)
    X0 = np.array([[1.0], [2.0], [3.0], [4.0]], np.float32)
    mean = np.zeros(n)
    tot = 0.0
    for prob, evs in TH.enumerate_schedules(n, e, K):
        ev = [[i, j, min(1, k), 0] for k, (i, j) in enumerate(evs)]
        X, _ = O.replay(p, X0, e, r, ev, T=1)
        mean += prob * X[:, 0].astype(np.float64)
        tot += prob
    assert abs(tot - 1.0) < 1e-12
    rec = TH.mean_recursion_quadratic(n, e, X0, [1.0], [0.5], 0.1, 1, 1, K)[:, 0]
    np.testing.assert_allclose(mean, rec, atol=1e-6)
    np.testing.assert_allclose(rec, [2.05852734, 2.07710547, 2.43783203, 2.45641016], atol=1e-8)


# ------------------------------------------------------- spectral / lemma --
def test_expected_gram_spec_examples():
    """ring n=3 gram diag 2/3 off 1/6, rho=0.5; n=2 rho=0."""
    G3 = TH.expected_gram(3, [[0, 1], [1, 2], [2, 0]])
    assert np.allclose(np.diag(G3), 2 / 3) and np.allclose(G3[0, 1], 1 / 6)
    assert abs(TH.rho(G3) - 0.5) < 1e-12
    assert abs(TH.rho(TH.expected_gram(2, [[0, 1]]))) < 1e-12
    assert abs(TH.rho(np.eye(4)) - 1.0) < 1e-12


@pytest.mark.parametrize("n", [4, 8, 16])
def test_ring_rho_closed_form(n):
    """Reading c8: on a ring under law c4, rho = 1 - (1 - cos(2 pi/n))/n, and
    E[W^T W] = E[W] (pair averages are symmetric idempotent)."""
    e, _ = synth.ring(n)
    G = TH.expected_gram(n, e)
    assert np.abs(G - TH.expected_W(n, e)).max() < 1e-15
    assert abs(TH.rho(G) - (1 - (1 - math.cos(2 * math.pi / n)) / n)) < 1e-12


def test_consensus_lemma_monte_carlo_with_oracle_replay():
    """E||1/n - prod W_k e_i||^2 <= ((n-1)/n) rho^K, with the W
    products produced by the oracle's own averaging (X0 = I: row i of X_K is
    column i of prod W)."""
    n = 6
    e, r = synth.ring(n)
    rho = TH.rho(TH.expected_gram(n, e))
    trials = 3000
    for K in (1, 5, 10, 25):
        vals = np.zeros((trials, n))
        for t in range(trials):
            ev, _ = synth.schedule_iid(n, e, K=K, seed=1000 * K + t, no_grad=True)
            X, _ = O.replay(O.OracleProblem(), np.eye(n, dtype=np.float32), e, r, ev)
            vals[t] = ((X.astype(np.float64) - 1.0 / n) ** 2).sum(1)
        m = vals.mean(0)
        se = vals.std(0) / math.sqrt(trials)
        assert np.all(m <= TH.lemma_bound(n, rho, K) + 3 * se + 1e-12), (K, m)


def test_pure_gossip_second_moment_matches_T_operator():
    """Reading c9: E||Y_k||^2 = tr(T^k(G0)) exactly; Monte-Carlo within 4 SE."""
    n, d = 8, 16
    e, r = synth.ring(n)
    X0 = synth.x0_uniform(n, d, seed=3)
    K, R = 40, 1500
    want = TH.second_moment_trace(n, e, X0, K)
    got = np.zeros((R, K + 1))
    for s in range(R):
        ev, _ = synth.schedule_iid(n, e, K=K, seed=s, no_grad=True)
        for k in (10, 20, 40):
            X, _ = O.replay(O.OracleProblem(), X0, e, r, ev[:k])
            Y = X.astype(np.float64) - X.astype(np.float64).mean(0)
            got[s, k] = (Y ** 2).sum()
    for k in (10, 20, 40):
        se = got[:, k].std() / math.sqrt(R)
        assert abs(got[:, k].mean() - want[k]) < 4 * se + 1e-9, (k, got[:, k].mean(), want[k])


# ------------------------------------------------------------- gradients --
def _fd(loss, x, h):
    g = np.zeros(x.size)
    for c in range(x.size):
        xp = x.copy(); xm = x.copy()
        xp[c] += h; xm[c] -= h
        g[c] = (loss(xp) - loss(xm)) / (float(xp[c]) - float(xm[c]))
    return g


def test_lsq_logreg_gradients_match_finite_differences():
    """analytic batch gradient == central FD of the loss (within 1e-4)."""
    for kind, (A, b) in [(O.MODEL_LSQ, synth.lsq_data(S=32, d=12, seed=7)),
                         (O.MODEL_LOGREG, synth.logreg_data(S=32, d=12, seed=8))]:
        p = O.OracleProblem(kind, M=32, gamma=0.1, A=A, b=b)
        x = np.random.default_rng(0).standard_normal(12).astype(np.float32)
        g = O.gradient(p, x, idx=np.arange(32))
        fd = _fd(lambda z: O.full_loss(p, z) * 32, x, 2.0 ** -9)
        np.testing.assert_allclose(g, fd, rtol=1e-4, atol=1e-4)


def test_logistic_spec_values():
    """single sample x=[1], y=+1 at w=0: gradient -0.5, loss ln 2."""
    p = O.OracleProblem(O.MODEL_LOGREG, M=1, A=np.array([[1.0]], np.float32),
                        b=np.array([1.0], np.float32))
    assert O.gradient(p, [0.0], idx=[0])[0] == np.float32(-0.5)
    assert abs(O.full_loss(p, [0.0]) - math.log(2)) < 1e-15


def test_mlp_gradient_matches_finite_differences():
    I, H, Ocl = 5, 4, 3
    X, y = synth.mlp_data(S=6, n_in=I, n_out=Ocl, s=1.0, seed=1)
    p = O.OracleProblem(O.MODEL_MLP, M=6, A=X, y=y, dims=(I, H, Ocl))
    w = synth.mlp_init(I, H, Ocl, seed=2)
    w[H * I:H * I + H] = 0.3                    # hidden pre-activations in tanh's curved range (reading R18)
    assert w.size == O.mlp_dim(I, H, Ocl)
    g = O.gradient(p, w, idx=np.arange(6))
    fd = _fd(lambda z: O.full_loss(p, z) * 6, w, 2.0 ** -12)
    np.testing.assert_allclose(g, fd, rtol=2e-3, atol=2e-4)


def test_mlp_dim_config3():
    """Config 3: 3072 -> 512 -> 10 has 1,578,506 parameters."""
    assert O.mlp_dim(3072, 512, 10) == 1578506


def test_quadratic_gradient_properties():
    """Quadratic at the optimum has zero deterministic gradient; the
    gradient equals the FD of f times M; noise has mean 0 and variance M sigma^2
    (s = sigma sqrt(3M)) within 4 SE; fp32 result within 1 ulp-ish of fp64."""
    d = 200000
    dk, nk = synth.quad_keys(2)
    M, sigma = 32, 0.1
    s = np.float32(sigma * math.sqrt(3 * M))
    p0 = O.OracleProblem(O.MODEL_QUADRATIC, M=M, data_key=dk, noise_key=nk, noise_s=0.0)
    ps = O.OracleProblem(O.MODEL_QUADRATIC, M=M, data_key=dk, noise_key=nk, noise_s=float(s))
    x = np.random.default_rng(1).uniform(-1, 1, d).astype(np.float32)
    g0 = O.gradient(p0, x, k=3)
    # FD on a small slice via the loss (M * grad f)
    p1 = O.OracleProblem(O.MODEL_QUADRATIC, M=1, data_key=dk, noise_key=nk, noise_s=0.0)
    xs = x[:50].copy()
    fd = _fd(lambda z: O.full_loss(p1, z), xs, 2.0 ** -10)
    np.testing.assert_allclose(O.gradient(p1, xs, k=0), fd, rtol=1e-4, atol=1e-5)
    gs = O.gradient(ps, x, k=3)
    nz = (gs.astype(np.float64) - g0.astype(np.float64))
    assert abs(nz.mean()) < 4 * nz.std() / math.sqrt(d)
    assert abs(nz.var() - M * sigma ** 2) < 4 * M * sigma ** 2 * math.sqrt(2.0 / d) * 1.5
    # different events draw different noise, same event reproduces bit-exactly
    assert not np.array_equal(gs, O.gradient(ps, x, k=4))
    assert np.array_equal(gs, O.gradient(ps, x, k=3))


def test_quadratic_zero_at_minimiser():
    d = 1000
    dk, nk = synth.quad_keys(3)
    p = O.OracleProblem(O.MODEL_QUADRATIC, M=8, data_key=dk, noise_key=nk, noise_s=0.0)
    # recover x* by one exact gradient step from 0 with h known: g(0) = M h (0 - x*)
    # use the loss: f(x) minimal at x*; evaluate g at x = x* obtained from two probes
    g0 = O.gradient(p, np.zeros(d, np.float32)).astype(np.float64)
    g1 = O.gradient(p, np.ones(d, np.float32)).astype(np.float64)
    Mh = g1 - g0                         # = M h (affine), exact enough in fp64
    xstar = (-g0 / Mh).astype(np.float32)
    assert np.all((Mh / 8 >= 0.0099) & (Mh / 8 <= 1.0))   # h in [0.01, 1)
    assert np.all(np.abs(xstar) <= 1.0)
    assert np.abs(O.gradient(p, xstar)).max() < 1e-5
    assert O.full_loss(p, xstar) < 1e-12


def test_batch_sampling_unbiased():
    """Assumption 1.4 / S:211: E[g]/M over device-mode (Philox) batches equals the
    full gradient within 4 SE."""
    A, b = synth.lsq_data(S=16, d=4, seed=9)
    M = 4
    p = O.OracleProblem(O.MODEL_LSQ, M=M, A=A, b=b, batch_key=(123, 456))
    x = np.array([0.3, -0.2, 0.5, 0.1], np.float32)
    R = 20000
    gs = np.array([O.gradient(p, x, k=k) for k in range(R)], np.float64) / M
    full = O.gradient(O.OracleProblem(O.MODEL_LSQ, M=16, A=A, b=b), x, idx=np.arange(16)) / 16
    se = gs.std(0) / math.sqrt(R)
    assert np.all(np.abs(gs.mean(0) - full) < 4 * se)


# ------------------------------------------------- consensus & allreduce --
def test_consensus_mean_and_Mk():
    """n=2, p=(1/2,1/2), models (0,2): mean 1, M_k = 1; all equal -> 0."""
    out, mk = O.consensus_mean([[0.0], [2.0]], p=[0.5, 0.5])
    assert out[0] == 1.0 and mk == 1.0
    out, mk = O.consensus_mean(np.ones((5, 3), np.float32))
    assert mk == 0.0 and np.all(out == 1.0)
    # fp64 sum: mean of values that cancel in fp32
    X = np.array([[1e8], [1.0], [-1e8]], np.float32)
    out, _ = O.consensus_mean(X)
    assert out[0] == np.float32(1.0 / 3)


def test_allreduce_spec_example():
    """n=2, f=x^2/2, both at 2, gamma=0.1 -> 1.8 on both (mean gradient, c12)."""
    x = O.allreduce_update([2.0], [[2.0], [2.0]], 0.1)
    assert x[0] == np.float32(2.0) - np.float32(np.float32(0.1) * np.float32(2.0))
    assert abs(x[0] - 1.8) < 1e-6


def test_replay_deterministic():
    n, d = 8, 300
    e, r = synth.ring(n)
    A, b = synth.lsq_data(S=64, d=d, seed=1)
    p = O.OracleProblem(O.MODEL_LSQ, M=4, gamma=0.1, A=A, b=b)
    ev, bi = synth.schedule_iid(n, e, K=100, T=3, M=4, S=64, seed=5)
    X1, m1 = O.replay(p, np.zeros((n, d), np.float32), e, r, ev, bi, T=3, mk_trace=True)
    X2, m2 = O.replay(p, np.zeros((n, d), np.float32), e, r, ev, bi, T=3, mk_trace=True)
    assert X1.tobytes() == X2.tobytes() and m1.tobytes() == m2.tobytes()


def test_skip_ring_rho_matches_survey_table():
    """SURVEY App. A.5 (odd-offset skip ring, law c4): n=8 0.963388, n=16 0.956747,
    n=32 0.985724; the plain ring's closed form for the same n."""
    for n, want in [(8, 0.963388), (16, 0.956747), (32, 0.985724)]:
        e, r = synth.skip_ring(n)
        st, _ = O.check_graph(n, e, role=r)
        assert st == 0                                   # bipartite with parity roles
        assert abs(TH.rho(TH.expected_gram(n, e)) - want) < 5e-7


def test_dpsgd_spec_example_and_invariants():
    """n=2, models (1,3), f=x^2/2, gamma=0.1, W = pair average -> (1.9, 1.7);
    W = I - L/(deg_max+1) is doubly stochastic: with no gradient the column sum is
    preserved and a ring contracts to consensus."""
    p = quad([1.0], [0.0], gamma=0.1)
    X = O.dpsgd_round(p, [[1.0], [3.0]], [[0, 1]])
    assert X[0, 0] == np.float32(2.0) - np.float32(0.1) and X[1, 0] == np.float32(2.0) - np.float32(np.float32(0.1) * 3)
    assert abs(X[0, 0] - 1.9) < 1e-6 and abs(X[1, 0] - 1.7) < 1e-6
    n, d = 8, 64
    e, _ = synth.ring(n)
    X0 = synth.x0_uniform(n, d, seed=2)
    X = X0
    for _ in range(200):
        X = O.dpsgd_round(O.OracleProblem(), X, e)
    assert np.abs(X.astype(np.float64).sum(0) - X0.astype(np.float64).sum(0)).max() < 1e-4
    assert np.abs(X - X.mean(0)).max() < 1e-4 * np.abs(X0).max()


# ------------------------------------------------------------ super-learner --
def test_super_gradient_noiseless_is_R_times_the_learner_gradient():
    """Reading R22: a super-learner's gradient is the all-reduce SUM of
    its R learners' minibatch gradients.  With no noise every learner computes
    M h (x - x*), so the sum is exactly R times it (R a power of two)."""
    d = 300
    rng = np.random.default_rng(3)
    h = rng.uniform(0.1, 1.0, d).astype(np.float32)
    xs = rng.uniform(-1, 1, d).astype(np.float32)
    x = rng.uniform(-2, 2, d).astype(np.float32)
    p = O.OracleProblem(O.MODEL_QUADRATIC, M=8, gamma=0.01, h=h, xstar=xs)
    g1 = O.gradient(p, x, k=5)
    for R in (1, 2, 4):
        assert np.array_equal(O.super_gradient(p, x, s=3, c=7, R=R), (np.float32(R) * g1).astype(np.float32))


def test_super_gradient_noise_statistics():
    """The R learners draw independent noise s*v, v ~ U[-1, 1) (23-bit grid): the
    summed noise has mean 0 and variance R s^2 / 3."""
    d, R, s = 200_000, 4, 0.5
    p = O.OracleProblem(O.MODEL_QUADRATIC, M=1, gamma=0.0, noise_s=s, h=np.zeros(d, np.float32),
                        xstar=np.zeros(d, np.float32))
    g = O.super_gradient(p, np.zeros(d, np.float32), s=1, c=0, R=R).astype(np.float64)
    assert abs(g.mean()) < 5 * math.sqrt(R * s * s / 3 / d)
    assert abs(g.var() / (R * s * s / 3) - 1) < 0.02


def test_super_replay_noiseless_equals_plain_replay_with_R_gamma():
    """Noiseless super-learner replay with R learners == Alg. 1 replay of the same
    events with learning rate R*gamma (R = 2: fl(2 gamma g) = fl(gamma fl(2 g))),
    bitwise -- the super-learner is an AD-PSGD worker with batch R*M."""
    S, d, K = 8, 257, 300
    e, r = synth.ring(S)
    rng = np.random.default_rng(4)
    h = rng.uniform(0.5, 1.0, d).astype(np.float32)
    xs = rng.uniform(-1, 1, d).astype(np.float32)
    X0 = synth.x0_uniform(S, d, seed=9)
    ev, _ = synth.schedule_iid(S, e, K=K, seed=10, local_prob=0.3)
    Xs = O.super_replay(O.OracleProblem(O.MODEL_QUADRATIC, M=4, gamma=0.05, h=h, xstar=xs), X0, e, r, ev, R=2)
    Xp, _ = O.replay(O.OracleProblem(O.MODEL_QUADRATIC, M=4, gamma=0.1, h=h, xstar=xs), X0, e, r, ev)
    assert np.array_equal(Xs.view(np.uint32), Xp.view(np.uint32))


def test_super_gradient_any_model_and_distinct_batches():
    """Super-learner gradients for a sampled model (lsq, device Philox batches):
    (a) with every sample identical, each learner's minibatch gradient is the
    same closed form, so the sum over R learners is exactly R times it;
    (b) with distinct samples, two super-learners at the same count draw
    different minibatches (the key's high word enters the Philox counter)."""
    d, S, M = 64, 512, 8
    a = np.random.default_rng(1).standard_normal(d).astype(np.float32) / 8
    A = np.tile(a, (S, 1))
    b = np.full(S, 0.25, np.float32)
    p = O.OracleProblem(O.MODEL_LSQ, M=M, gamma=0.1, A=A, b=b, batch_key=(3, 4))
    x = np.random.default_rng(2).standard_normal(d).astype(np.float32) / 4
    g1 = O.gradient(p, x, k=0)
    for R in (1, 2, 4):
        assert np.array_equal(O.super_gradient(p, x, s=1, c=5, R=R), (np.float32(R) * g1).astype(np.float32))
    A2, b2 = synth.lsq_data(S=S, d=d, seed=3)
    p2 = O.OracleProblem(O.MODEL_LSQ, M=M, gamma=0.1, A=A2, b=b2, batch_key=(3, 4))
    assert not np.array_equal(O.super_gradient(p2, x, s=0, c=7, R=1), O.super_gradient(p2, x, s=1, c=7, R=1))


def test_openmp_build_is_bit_identical():
    """The all-cores CPU baseline (liboracle_omp.so) runs the
    same per-coordinate loops in parallel: identical results to the serial oracle."""
    n, d = 4, 100_003
    e, r = synth.ring(n)
    dk, nk = synth.quad_keys(3)
    p = O.OracleProblem(O.MODEL_QUADRATIC, M=32, gamma=0.01, data_key=dk, noise_key=nk, noise_s=0.5)
    ev, _ = synth.schedule_iid(n, e, K=40, T=2, seed=9, local_prob=0.3)
    X0 = synth.x0_uniform(n, d, seed=4)
    Xs, _ = O.replay(p, X0, e, r, ev, T=2)
    Xp, _ = O.replay(p, X0, e, r, ev, T=2, omp=True)
    assert np.array_equal(Xs.view(np.uint32), Xp.view(np.uint32))
