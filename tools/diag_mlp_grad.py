"""One MLP gradient on the GPU against the oracle, error by parameter group (diagnostic)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import synth
import paper_1710_06952_b200 as P
from oracle import oracle as O

for (I, H, Ocl) in ((256, 128, 10), (3072, 512, 10)):
    n, M = 4, 128
    e, r = synth.ring(n)
    X, y = synth.mlp_data(S=2048, n_in=I, n_out=Ocl, s=0.3 if I == 256 else 0.02, seed=3)
    x0 = synth.mlp_init(I, H, Ocl, seed=4)
    d = x0.size
    groups = {"W1": (0, H * I), "b1": (H * I, H * I + H), "W2": (H * I + H, H * I + H + Ocl * H),
              "b2": (d - Ocl, d)}
    prob = O.OracleProblem(O.MODEL_MLP, M=M, gamma=1.0, A=X, y=y, dims=(I, H, Ocl))
    ev, bi = synth.schedule_iid(n, e, K=4, T=0, M=M, S=X.shape[0], seed=21)
    g_or = O.gradient(prob, x0, idx=bi[0])
    ctx = P.Context(e, n, d, role=r, T=0, model=P.MODEL_MLP, gamma=1.0, batch_M=M, data_A=X, data_y=y,
                    mlp_dims=(I, H, Ocl), x0=x0)
    ctx.replay([[int(ev[0, 0]), -1, 0, 0]], batch_idx=bi[:1])
    ctx.sync()
    g_gpu = x0 - ctx.read_model(int(ev[0, 0]))
    for name, (a, b) in groups.items():
        err = np.abs(g_gpu[a:b] - g_or[a:b])
        print(f"{I}x{H}: {name}: max|g| {np.abs(g_or[a:b]).max():.3e} max err {err.max():.3e} "
              f"argmax {err.argmax()} gpu {g_gpu[a:b].ravel()[:4]} ref {g_or[a:b].ravel()[:4]}", flush=True)
    ctx.destroy()
