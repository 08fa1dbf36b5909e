"""Theory-side oracle helpers (numpy, fp64) -- TEST INFRASTRUCTURE ONLY.

Each function writes out a definition from the paper:
  * pair averaging matrix W
  * E[W^T W] and rho = max(|lambda_2|, |lambda_n|) (Assumption 1.3)
  * the consensus-decay lemma bound ((n-1)/n) rho^K
  * the exact second-moment operator T(G) = sum_e q_e W_e G W_e (reading c9)
  * the fp64 linear recursion for E[X_k] under an affine gradient
"""
from __future__ import annotations

import itertools

import numpy as np


def pair_matrix(i: int, j: int, n: int) -> np.ndarray:
    """W: identity except W_ii = W_jj = W_ij = W_ji = 1/2."""
    if i == j or not (0 <= i < n and 0 <= j < n):
        raise ValueError("invalid pair")
    W = np.eye(n)
    W[i, i] = W[j, j] = W[i, j] = W[j, i] = 0.5
    return W


def event_law(n: int, edges, p=None):
    """Law c4: P(i) = p_i (default 1/n), j uniform over N(i).  Returns list of
    (prob, i, j) over ordered pairs."""
    nb = [[] for _ in range(n)]
    for a, b in np.asarray(edges).reshape(-1, 2):
        nb[int(a)].append(int(b))
        nb[int(b)].append(int(a))
    p = np.full(n, 1.0 / n) if p is None else np.asarray(p, float)
    law = []
    for i in range(n):
        for j in nb[i]:
            law.append((p[i] / len(nb[i]), i, j))
    return law


def expected_W(n, edges, p=None):
    return sum(q * pair_matrix(i, j, n) for q, i, j in event_law(n, edges, p))


def expected_gram(n, edges, p=None):
    """E[W^T W] (Assumption 1.3) by enumerating every (i, j)."""
    return sum(q * pair_matrix(i, j, n).T @ pair_matrix(i, j, n) for q, i, j in event_law(n, edges, p))


def rho(gram) -> float:
    """rho = max{|lambda_2|, |lambda_n|} with eigenvalues sorted descending."""
    ev = np.sort(np.linalg.eigvalsh(np.asarray(gram, float)))[::-1]
    if ev.size < 2:
        return 0.0
    return float(max(abs(ev[1]), abs(ev[-1])))


def lemma_bound(n: int, r: float, K: int) -> float:
    """E||1/n - prod_k W_k e_i||^2 <= ((n-1)/n) rho^K."""
    return (n - 1) / n * r ** K


def T_op(n, edges, G, p=None):
    """Second-moment operator of pure gossip, T(G) = E[W G W] (W symmetric)."""
    return sum(q * pair_matrix(i, j, n) @ G @ pair_matrix(i, j, n) for q, i, j in event_law(n, edges, p))


def second_moment_trace(n, edges, X0, K):
    """tr(T^k(G0)) for k = 0..K with G0 = Y0^T Y0, Y0 = X0 minus its worker mean
    (X0 is n x d worker-major; Y^T Y in the paper's N x n orientation is n x n)."""
    X0 = np.asarray(X0, float)
    Y = X0 - X0.mean(axis=0, keepdims=True)
    G = Y @ Y.T
    out = [np.trace(G)]
    for _ in range(K):
        G = T_op(n, edges, G)
        out.append(np.trace(G))
    return np.array(out)


def mean_recursion_quadratic(n, edges, X0, h, xstar, gamma, M, tau, K):
    """fp64 recursion for E[X_k] under law c4, deterministic affine gradient
    g = M h (x - x*) and fixed staleness tau clipped to k:
      E[X_{k+1}] = E[X_k] E[W] - (gamma/n) [M h (E[X_{k-tau_k}] e_i - x*)]_i
    (worker-major rows; from X_{k+1} = X_k W_k - gamma dg, with i_k, W_k
    independent of X_k and P(i_k = i) = 1/n)."""
    EW = expected_W(n, edges)
    hist = [np.asarray(X0, float)]
    h = np.asarray(h, float)
    xs = np.asarray(xstar, float)
    for k in range(K):
        t = min(tau, k)
        Xs = hist[k - t]
        G = M * h[None, :] * (Xs - xs[None, :])
        hist.append(EW.T @ hist[k] - (gamma / n) * G)   # rows: (X W) in worker-major = W^T X
    return hist[-1]


def enumerate_schedules(n, edges, K):
    """All (i, j) sequences of length K under law c4, with their probabilities."""
    law = event_law(n, edges)
    for combo in itertools.product(range(len(law)), repeat=K):
        prob = 1.0
        evs = []
        for c in combo:
            q, i, j = law[c]
            prob *= q
            evs.append((i, j))
        yield prob, evs
