"""Writes tests/golden/config3_mlp_2000_oracle.json: the ORACLE's result of the
config-3 parity replay (BASELINE configs[2]):
2-layer tanh MLP 3072 -> 512 -> 10 (reading R18), n = 8 workers on the
bipartite ring, M = 128, gamma = 0.002, T = 4 with tau ~ U{0..4}, 2000 events of
Algorithm 1 (gradient a batch SUM), explicit
batch indices, CIFAR-shaped synthetic data S = 50,000 (synth.mlp_data).

It calls only oracle/ (and synth/ for the seeded inputs).  The whole model is
1.58M parameters per worker, so the fixture keeps, per worker, 512 coordinates
drawn with a fixed seed (plus every bias of both layers) and the rms of the
worker's full row -- what reading R11's guard max(|x|, rms(row)) needs --
together with f(x_bar) before / after and SHA-1 digests of the generated inputs
so the test can tell that synth regenerated the same arrays.
Run time: ~20 min on one core (0.57 s per fp64 gradient)."""
import hashlib
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np

import synth
from oracle import oracle as O

I, H, OUT = 3072, 512, 10
N, M, GAMMA, T, K, S = 8, 128, 0.002, 4, 2000, 50_000
SEED_DATA, SEED_INIT, SEED_SCHED, SEED_PICK = 3, 4, 21, 77
OUT_PATH = os.path.join(ROOT, "tests", "golden", "config3_mlp_2000_oracle.json")


def inputs():
    X, y = synth.mlp_data(S=S, n_in=I, n_out=OUT, s=0.02, seed=SEED_DATA)
    x0 = synth.mlp_init(I, H, OUT, seed=SEED_INIT)
    e, r = synth.ring(N)
    ev, bi = synth.schedule_iid(N, e, K=K, T=T, M=M, S=S, seed=SEED_SCHED)
    return X, y, x0, e, r, ev, bi


def digest(*arrs):
    h = hashlib.sha1()
    for a in arrs:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def picks(d):
    """Coordinates kept per worker: 512 seeded draws + b1 + b2 (W2 is drawn from too)."""
    rng = np.random.default_rng(SEED_PICK)
    sel = set(rng.choice(d, 512, replace=False).tolist())
    sel.update(range(H * I, H * I + H))                    # b1
    sel.update(range(d - OUT, d))                          # b2
    return np.array(sorted(sel), np.int64)


def main():
    X, y, x0, e, r, ev, bi = inputs()
    d = x0.size
    prob = O.OracleProblem(O.MODEL_MLP, M=M, gamma=GAMMA, A=X, y=y, dims=(I, H, OUT))
    t = time.time()
    Xo, _ = O.replay(prob, np.tile(x0, (N, 1)), e, r, ev, bi, T=T)
    took = time.time() - t
    idx = picks(d)
    rms = np.sqrt(np.mean(Xo.astype(np.float64) ** 2, axis=1))
    xbar = Xo.astype(np.float64).mean(0).astype(np.float32)
    out = {
        "what": "oracle result of the config-3 MLP replay (tools/make_config3_reference.py)",
        "cite": "PAPER.md P:498-535 (Alg. 1), P:402-406 / P:515-519 (batch-sum gradient), P:561 (stale read); "
                "DESIGN.md readings R2, R3, R11, R18",
        "recipe": {"n_in": I, "n_hid": H, "n_out": OUT, "n": N, "M": M, "gamma": GAMMA, "T": T, "K": K, "S": S,
                   "seed_data": SEED_DATA, "seed_init": SEED_INIT, "seed_sched": SEED_SCHED, "seed_pick": SEED_PICK},
        "digest_inputs": {"data": digest(X, y), "x0": digest(x0), "schedule": digest(ev, bi)},
        "oracle_seconds": took,
        "loss_x0": O.full_loss(prob, x0),
        "loss_xbar": O.full_loss(prob, xbar),
        "idx": idx.tolist(),
        "rms": rms.tolist(),
        "values": [[float(v) for v in Xo[w, idx]] for w in range(N)],
    }
    with open(OUT_PATH, "w") as f:
        json.dump(out, f)
    print(f"wrote {OUT_PATH}: oracle {took:.0f} s, f(x0) {out['loss_x0']:.4f} -> f(xbar) {out['loss_xbar']:.4f}")


if __name__ == "__main__":
    main()
