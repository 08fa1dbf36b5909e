"""Small driver for ncu captures of the hot kernels (one GPU).

  python tools/prof_engine.py --what engine  --d 25600000 --n 8 --updates 64 --runs 2
  python tools/prof_engine.py --what event   (standalone k_event pair pass)
"""
import argparse
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import synth
import paper_1710_06952_b200 as P

ap = argparse.ArgumentParser()
ap.add_argument("--what", default="engine")
ap.add_argument("--d", type=int, default=25_600_000)
ap.add_argument("--n", type=int, default=8)
ap.add_argument("--updates", type=int, default=64)
ap.add_argument("--runs", type=int, default=2)
ap.add_argument("--compute-us", type=float, default=50.0)
a = ap.parse_args()

e, r = synth.ring(a.n)
dk, nk = synth.quad_keys(5)
s = float(np.float32(0.1 * math.sqrt(96)))
ctx = P.Context(e, a.n, a.d, role=r, model=P.MODEL_QUADRATIC, gamma=0.01, batch_M=32, quad_keys=(dk, nk),
                quad_noise_s=s, straggler=synth.stragglers(a.n), compute_ns=int(a.compute_us * 1000))
if a.what == "engine":
    for it in range(a.runs):
        s0 = ctx.stats()
        ctx.run(a.updates)
        ctx.sync()
        s1 = ctx.stats()
        print(f"run {it}: events {s1['local_events'] - s0['local_events']}, "
              f"pair {s1['local_pair_events'] - s0['local_pair_events']}, "
              f"algorithmic_bytes {s1['local_bytes'] - s0['local_bytes']:.6e}", flush=True)
elif a.what == "event":
    ev, _ = synth.schedule_iid(a.n, e, K=a.updates, seed=1)
    for _ in range(a.runs):
        ctx.replay(ev, flags=P.REPLAY_HOST)
        ctx.sync()
st = ctx.stats()
print({k: v for k, v in st.items()})
ctx.destroy()
