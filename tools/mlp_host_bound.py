"""Is the config-3 replay host-bound?  Host enqueue time of ctx.replay() vs the device time."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import synth
import paper_1710_06952_b200 as P

I, H, O, M, n, T = 3072, 512, 10, 128, 8, 4
X, y = synth.mlp_data(S=8192, n_in=I, n_out=O, s=0.02, seed=3)
x0 = synth.mlp_init(I, H, O, seed=4)
e, r = synth.ring(n)
ctx = P.Context(e, n, x0.size, role=r, T=T, model=P.MODEL_MLP, gamma=0.002, batch_M=M, data_A=X, data_y=y,
                mlp_dims=(I, H, O), x0=x0)
for events in (64, 256):
    ev, bi = synth.schedule_iid(n, e, K=events, T=T, M=M, S=8192, seed=7)
    ctx.replay(ev[:8], batch_idx=bi[:8])
    ctx.sync()
    s = torch.cuda.Stream()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(s)
    h0 = time.perf_counter()
    ctx.replay(ev, batch_idx=bi, stream=s)
    h1 = time.perf_counter()
    t1.record(s)
    torch.cuda.synchronize()
    h2 = time.perf_counter()
    print(f"{events} events: host enqueue {1e6 * (h1 - h0) / events:.1f} us/event, device "
          f"{1e3 * t0.elapsed_time(t1) / events:.1f} us/event, wall {1e6 * (h2 - h0) / events:.1f} us/event")
ctx.destroy()
