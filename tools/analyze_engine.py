"""Engine occupancy analysis from the device event log (t0/t1 per event).

Prints, per configuration: engine time (CUDA events), algorithmic GB/s,
fraction of the launch with >= 1 event in flight, mean events in flight,
mean pass duration of pair / local events.
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
ap.add_argument("--d", type=int, default=25_600_000)
ap.add_argument("--configs", default="8:50:0,8:0:0,16:50:0")   # n:compute_us:0[:none]
ap.add_argument("--updates", type=int, default=512)
a = ap.parse_args()

for cfgs in a.configs.split(","):
    parts = cfgs.split(":")
    n, cus, var = int(parts[0]), float(parts[1]), int(parts[2])
    model = P.MODEL_NONE if len(parts) > 3 and parts[3] == "none" else P.MODEL_QUADRATIC
    e, r = synth.ring(n)
    dk, nk = synth.quad_keys(5)
    ctx = P.Context(e, n, a.d, role=r, model=model, gamma=0.01, batch_M=32, quad_keys=(dk, nk),
                    quad_noise_s=0.5, straggler=synth.stragglers(n), compute_ns=int(cus * 1000),
                    log_capacity=1 << 16)
    ctx.run(64)
    ctx.sync()
    k0 = ctx.ticket()
    st0 = ctx.stats()
    s = torch.cuda.Stream()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(s)
    ctx.run(a.updates, s)
    t1.record(s)
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1)
    st1 = ctx.stats()
    log = ctx.read_log(k0)
    ts = log["t0"].astype(np.int64)
    te = log["t1"].astype(np.int64)
    T0, T1 = ts.min(), te.max()
    pts = np.concatenate([np.stack([ts, np.ones_like(ts)], 1), np.stack([te, -np.ones_like(te)], 1)])
    pts = pts[np.lexsort((pts[:, 1], pts[:, 0]))]
    cur, last, cover, area = 0, T0, 0, 0
    for t, dlt in pts:
        if cur > 0:
            cover += t - last
        area += cur * (t - last)
        cur += dlt
        last = t
    pair = log["j"] >= 0
    gb = (st1["local_bytes"] - st0["local_bytes"]) / 1e9
    print(f"n={n} t_c={cus}us variant={var}: launch {ms:.2f} ms, span {(T1 - T0) / 1e6:.2f} ms, "
          f"{gb / (ms / 1e3):.0f} GB/s alg, busy-cover {cover / (T1 - T0):.3f}, mean in-flight "
          f"{area / (T1 - T0):.2f}, pair pass {np.mean((te - ts)[pair]) / 1e3:.0f} us ({pair.sum()}), "
          f"local pass {np.mean((te - ts)[~pair]) / 1e3 if (~pair).any() else 0:.0f} us ({(~pair).sum()})",
          flush=True)
    ctx.destroy()

# standalone stream-ordered pass (host executor), for comparison
n = 8
e, r = synth.ring(n)
for flags, name in ((P.EV_NO_GRAD, "pair avg only"), (0, "pair avg + quad grad")):
    ctx = P.Context(e, n, a.d, role=r, model=P.MODEL_QUADRATIC, gamma=0.01, batch_M=32, quad_keys=(1, 2),
                    quad_noise_s=0.5)
    ev = np.array([[0, 1, 0, flags]] * 64, np.int32)
    ctx.replay(ev, flags=P.REPLAY_HOST)
    ctx.sync()
    s = torch.cuda.Stream()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(s)
    ctx.replay(ev, flags=P.REPLAY_HOST, stream=s)
    t1.record(s)
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / 64
    print(f"k_event {name}: {ms * 1e3:.1f} us/event, {16 * a.d / (ms / 1e3) / 1e9:.0f} GB/s", flush=True)
    ctx.destroy()
