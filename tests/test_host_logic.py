"""Host-side logic without a GPU: synthetic placements and schedules."""
import numpy as np
import pytest

import synth


@pytest.mark.parametrize("G", [4, 8, 16])
def test_placement_xor_every_edge_crosses_and_balances_roles(G):
    n = 8 * G
    p = synth.placement_xor(n, G)
    e, r = synth.ring(n)
    assert all(p[a] != p[b] for a, b in e)
    for g in range(G):
        assert (p == g).sum() == n // G
        assert ((p == g) & (r == 0)).sum() == n // (2 * G)        # actives spread evenly


def test_placement_xor_rejects_two_gpus():
    # a connected bipartite ring has one 2-colouring: all-cross at G = 2 forces GPU = role
    with pytest.raises(ValueError):
        synth.placement_xor(16, 2)


def test_schedule_appa_is_causal():
    n, K, T = 8, 500, 9
    e, r = synth.ring(n)
    ev = synth.schedule_appa(n, e, r, K, T, seed=1)
    last_k, last_r, prev_k = [-1] * n, [0] * n, [-1] * n
    for k, (i, j, tau, fl) in enumerate(ev):
        if fl & 1:
            assert r[i] == 0 and j >= 0 and tau == 0
            continue
        t = k - tau
        assert 0 <= tau <= min(k, T) and t >= last_r[i] and t > prev_k[i]
        assert (j >= 0) == (r[i] == 0)
        prev_k[i], last_k[i], last_r[i] = last_k[i], k, t


@pytest.mark.parametrize("S,R", [(2, 2), (4, 2), (1, 4), (8, 1)])
def test_super_ring_layout(S, R):
    e, role, wr, se, sr = synth.super_ring(S, R)
    assert e.shape[0] == se.shape[0] * R
    for a, b in e:
        assert a % R == b % R and role[a] != role[b]            # (s, r) -- (s', r), bipartite
    assert np.array_equal(wr, np.arange(S * R))
    assert all(role[s * R + r] == sr[s] for s in range(S) for r in range(R))
