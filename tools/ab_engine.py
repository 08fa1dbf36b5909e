"""A/B of engine variants on a FIXED event mix (engine replay of one schedule),
so that GB/s differences are not confounded by the free-running pair/local mix.

  python tools/ab_engine.py --variants 0,1,2 --n 8 --events 512 --local 0.5
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import synth
import paper_1710_06952_b200 as P

ap = argparse.ArgumentParser()
ap.add_argument("--d", type=int, default=25_600_000)
ap.add_argument("--n", type=int, default=8)
ap.add_argument("--events", type=int, default=512)
ap.add_argument("--local", type=float, default=0.5)
ap.add_argument("--variants", default="0,1,2")
ap.add_argument("--model", default="quad")
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()

e, r = synth.ring(a.n)
ev, _ = synth.schedule_iid(a.n, e, K=a.events, seed=3, local_prob=a.local,
                           no_grad=(a.model == "none"))
if a.model == "none":
    ev = ev[ev[:, 1] >= 0]
pairs = int((ev[:, 1] >= 0).sum())
locs = len(ev) - pairs
alg = (16.0 * pairs + 8.0 * locs) * a.d
for v in [int(x) for x in a.variants.split(",")]:
    ctx = P.Context(e, a.n, a.d, role=r, model=P.MODEL_QUADRATIC if a.model == "quad" else P.MODEL_NONE,
                    gamma=0.01, batch_M=32, quad_keys=(1, 2), quad_noise_s=0.5, engine_variant=v)
    ctx.replay(ev, flags=P.REPLAY_ENGINE)
    ctx.sync()
    s = torch.cuda.Stream()
    best = 1e30
    for _ in range(a.reps):
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record(s)
        ctx.replay(ev, flags=P.REPLAY_ENGINE, stream=s)
        t1.record(s)
        torch.cuda.synchronize()
        best = min(best, t0.elapsed_time(t1))
    print(f"variant {v}: {len(ev)} events ({pairs} pair, {locs} local), {best:.2f} ms, "
          f"{alg / (best / 1e3) / 1e9:.0f} GB/s", flush=True)
    ctx.destroy()
