"""Seeded synthetic INPUT generators shared by the oracle tests, the GPU parity
tests and bench.py.

This module holds none of the method's arithmetic: it only draws graphs,
event schedules, datasets and initial models from numpy's seeded generators.
The oracle (oracle/) and the CUDA path (paper_1710_06952_b200/) both consume
what it returns; neither side's computation lives here.  Recipes are stated in
DESIGN.md section "Input recipes" and follow the paper's workload shapes
(ring of workers P:485-487, batch 32/128 P:853, ~1 MB / ~100 MB models
P:781-783, Strategy-1 data P:386-388).
"""
from __future__ import annotations

import numpy as np

EV_NO_GRAD = 1  # event flag: pure averaging (W_k only), no gradient


def ring(n: int):
    """Ring topology: edges (j, j+1 mod n); parity roles (0 active,
    1 passive), bipartite iff n is even."""
    if n < 1:
        raise ValueError("n must be >= 1")
    if n == 1:
        return np.zeros((0, 2), np.int32), np.zeros(1, np.int8)
    if n == 2:
        return np.array([[0, 1]], np.int32), np.array([0, 1], np.int8)
    e = np.array([[j, (j + 1) % n] for j in range(n)], np.int32)
    role = (np.arange(n) % 2).astype(np.int8)
    return e, role


def skip_ring(n: int, odd_only: bool = True):
    """Skip ring: sender j talks to j + 2^i + 1 (mod n) for
    i = 0..floor(log2(n-1)) (reading c13).  odd_only keeps the offsets that
    preserve the parity bipartition."""
    if n < 3:
        return ring(n)
    offs = [2 ** i + 1 for i in range(int(np.floor(np.log2(n - 1))) + 1)]
    offs = sorted({o % n for o in offs if o % n != 0})
    if odd_only:
        offs = [o for o in offs if o % 2 == 1]
    E = set()
    for j in range(n):
        for o in offs:
            a, b = j, (j + o) % n
            if a != b:
                E.add((min(a, b), max(a, b)))
    e = np.array(sorted(E), np.int32).reshape(-1, 2)
    role = (np.arange(n) % 2).astype(np.int8)
    return e, role


def neighbours(n: int, edges: np.ndarray):
    nb = [[] for _ in range(n)]
    for a, b in np.asarray(edges).reshape(-1, 2):
        nb[int(a)].append(int(b))
        nb[int(b)].append(int(a))
    return [sorted(x) for x in nb]


def schedule_iid(n, edges, K, T=0, seed=0, M=0, S=0, no_grad=False, tau=None,
                 local_prob=0.0):
    """Event schedule under law c4: i_k ~ U{0..n-1}, j_k ~ U(N(i_k)),
    tau_k ~ U{0..min(k,T)} (or the fixed `tau`, clipped to k).  With
    local_prob > 0 an event is a partner-less local update (j = -1) with that
    probability.  Returns (events[K,4] int32 = (i, j, tau, flags),
    batch_idx[K,M] int32 or None)."""
    rng = np.random.default_rng(seed)
    nb = neighbours(n, edges)
    ev = np.zeros((K, 4), np.int32)
    for k in range(K):
        i = int(rng.integers(n))
        if nb[i] and not (local_prob > 0 and rng.random() < local_prob):
            j = nb[i][int(rng.integers(len(nb[i])))]
        else:
            j = -1
        if tau is None:
            t = int(rng.integers(min(k, T) + 1))
        else:
            t = min(int(tau), k)
        ev[k] = (i, j, t, EV_NO_GRAD if no_grad else 0)
    bidx = None
    if M > 0 and S > 0:
        bidx = rng.integers(0, S, size=(K, M), dtype=np.int64).astype(np.int32)
    return ev, bidx


def super_ring(S: int, R: int):
    """Super-learner layout (reading R22): learner (s, r) = s*R + r on rank s*R + r;
    the learner graph is R copies of ring(S) (learner (s, r) -- (s', r)) and a
    learner takes its super-learner's role.  Returns (edges, roles, worker_rank,
    super_edges, super_roles)."""
    se, sr = ring(S)
    e = np.array([[a * R + r, b * R + r] for a, b in se for r in range(R)], np.int32).reshape(-1, 2)
    role = np.repeat(sr, R).astype(np.int8)
    return e, role, np.arange(S * R, dtype=np.int32), se, sr


def placement_xor(n: int, G: int) -> np.ndarray:
    """Worker -> GPU for a ring where EVERY edge crosses GPUs and the actives
    (even workers) are spread over all GPUs: GPU(w) = (w mod G) xor ((w div G)
    mod 2).  Needs G a power of two >= 4 and n a multiple of 2G.  (With G = 2
    no such placement exists: a connected bipartite graph has one 2-colouring,
    so 'every edge crosses' forces GPU = role, i.e. all actives on one GPU.)"""
    if G < 4 or G & (G - 1) or n % (2 * G):
        raise ValueError("placement_xor needs G = 4, 8, ... and n % 2G == 0")
    w = np.arange(n)
    return ((w % G) ^ ((w // G) % 2)).astype(np.int32)


EV_FLUSH_FIRST, EV_COMPENSATE = 2, 4


def schedule_appa(n, edges, role, K, T, seed=0, compensate=True, p_gossip=0.3):
    """A valid App. A (wait-free runtime) schedule, reading R20: actives either
    average with no gradient (probability p_gossip) or flush a buffered
    gradient and average; passives flush with no partner.  A gradient's read
    point t (tau = k - t) is drawn so that each worker reads in order and has
    at most one gradient in the buffer when it pulls:
    t in [max(k - T, previous read, flush before the previous + 1), k]."""
    rng = np.random.default_rng(seed)
    nb = neighbours(n, edges)
    last_k = [-1] * n
    last_r = [0] * n
    prev_k = [-1] * n
    flags = EV_FLUSH_FIRST | (EV_COMPENSATE if compensate else 0)
    ev = np.zeros((K, 4), np.int32)
    for k in range(K):
        i = int(rng.integers(n))
        active = role[i] == 0 and len(nb[i]) > 0
        j = nb[i][int(rng.integers(len(nb[i])))] if active else -1
        if active and rng.random() < p_gossip:
            ev[k] = (i, j, 0, EV_NO_GRAD)
            continue
        lo = max(0, k - T, last_r[i], prev_k[i] + 1)
        t = int(rng.integers(lo, k + 1))
        ev[k] = (i, j, k - t, flags)
        prev_k[i], last_k[i], last_r[i] = last_k[i], k, t
    return ev


def x0_uniform(n: int, d: int, seed: int = 7) -> np.ndarray:
    """Per-worker initial models, values 2u-1 with u = m * 2^-24 exact in fp32
    (pure-gossip tests only, reading c7)."""
    rng = np.random.default_rng(seed)
    m = rng.integers(0, 1 << 24, size=(n, d), dtype=np.int64)
    return (m.astype(np.float64) * 2.0 ** -23 - 1.0).astype(np.float32)


def schedule_alg1(n, edges, role, K, seed=0):
    """Algorithm 1 iterations as an i.i.d. schedule (law c4): i_k ~ U{0..n-1};
    an active worker averages with j_k ~ U(N(i_k)), a passive one updates alone
    (j = -1, W_k = I) -- the event mix of the free-running engine's Alg. 1 loop.
    Returns events[K,4] int32 (i, j, 0, 0)."""
    rng = np.random.default_rng(seed)
    nb = neighbours(n, edges)
    ev = np.zeros((K, 4), np.int32)
    for k in range(K):
        i = int(rng.integers(n))
        j = nb[i][int(rng.integers(len(nb[i])))] if (role[i] == 0 and nb[i]) else -1
        ev[k] = (i, j, 0, 0)
    return ev


def lsq_data(S: int = 8192, d: int = 1024, seed: int = 1, noise: float = 0.01):
    """Config 1: A ~ N(0, 1/d) fp32, x_true ~ N(0,1), b = A x_true + noise*N(0,1)."""
    rng = np.random.default_rng(seed)
    A = (rng.standard_normal((S, d)) / np.sqrt(d)).astype(np.float32)
    xt = rng.standard_normal(d)
    b = (A.astype(np.float64) @ xt + noise * rng.standard_normal(S)).astype(np.float32)
    return A, b


def logreg_data(S: int = 8192, d: int = 1024, seed: int = 2):
    """Labels y = sign(a.w_true + 0.1 N(0,1)) in {-1,+1}, a ~ N(0, 1/d)."""
    rng = np.random.default_rng(seed)
    A = (rng.standard_normal((S, d)) / np.sqrt(d)).astype(np.float32)
    w = rng.standard_normal(d)
    z = A.astype(np.float64) @ w + 0.1 * rng.standard_normal(S)
    y = np.where(z >= 0, 1.0, -1.0).astype(np.float32)
    return A, y


def mlp_data(S: int = 50000, n_in: int = 3072, n_out: int = 10, s: float = 0.02, seed: int = 3):
    """Config 3: CIFAR-shaped synthetic data x = mu_y + N(0, I), mu_c ~ N(0, s^2 I)."""
    rng = np.random.default_rng(seed)
    mu = rng.standard_normal((n_out, n_in)) * s
    y = rng.integers(0, n_out, size=S).astype(np.int32)
    X = (mu[y] + rng.standard_normal((S, n_in))).astype(np.float32)
    return X, y


def mlp_init(n_in: int = 3072, n_hid: int = 512, n_out: int = 10, seed: int = 4) -> np.ndarray:
    """He-uniform init, flat layout [W1 (hid x in) | b1 | W2 (out x hid) | b2]
    (reading c18), identical for all workers."""
    rng = np.random.default_rng(seed)
    l1 = np.sqrt(6.0 / n_in)
    l2 = np.sqrt(6.0 / n_hid)
    W1 = rng.uniform(-l1, l1, (n_hid, n_in))
    W2 = rng.uniform(-l2, l2, (n_out, n_hid))
    return np.concatenate([W1.ravel(), np.zeros(n_hid), W2.ravel(), np.zeros(n_out)]).astype(np.float32)


def quad_keys(seed: int = 11):
    """Two u32 keys for the synthetic quadratic (data landscape, noise)."""
    rng = np.random.default_rng(seed)
    k = rng.integers(0, 1 << 32, size=2, dtype=np.uint64)
    return int(k[0]), int(k[1])


def stragglers(n: int, seed: int = 99, slow_worker: int | None = 0, slow: float = 10.0,
               hetero: bool = False) -> np.ndarray:
    """Per-worker slowdown factors s_w >= 1 (config 4: one worker 10x, P:1078-1081;
    config 5: s_w = 10^u log-uniform in [1,10] plus worker 0 at 10x)."""
    f = np.ones(n, np.float32)
    if hetero:
        f = (10.0 ** np.random.default_rng(seed).random(n)).astype(np.float32)
    if slow_worker is not None and n > 0:
        f[slow_worker] = slow
    return f
