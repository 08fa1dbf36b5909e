"""MLP GPU-vs-oracle error growth by parameter group (diagnostic)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import synth
import paper_1710_06952_b200 as P
from oracle import oracle as O

I, H, Ocl = 256, 128, 10
n, M, T = 4, 128, 2
e, r = synth.ring(n)
X, y = synth.mlp_data(S=2048, n_in=I, n_out=Ocl, s=0.3, seed=3)
x0 = synth.mlp_init(I, H, Ocl, seed=4)
d = x0.size
groups = {"W1": (0, H * I), "b1": (H * I, H * I + H), "W2": (H * I + H, H * I + H + Ocl * H), "b2": (d - Ocl, d)}
prob = O.OracleProblem(O.MODEL_MLP, M=M, gamma=0.01, A=X, y=y, dims=(I, H, Ocl))
# single gradient accuracy
xg = x0.copy()
ev, bi = synth.schedule_iid(n, e, K=2000, T=T, M=M, S=X.shape[0], seed=21)
g_or = O.gradient(prob, xg, idx=bi[0])
ctx = P.Context(e, n, d, role=r, T=T, model=P.MODEL_MLP, gamma=1.0, batch_M=M, data_A=X, data_y=y,
                mlp_dims=(I, H, Ocl), x0=x0)
ctx.replay([[int(ev[0, 0]), -1, 0, 0]], batch_idx=bi[:1])
ctx.sync()
g_gpu = x0 - ctx.read_model(int(ev[0, 0]))          # gamma = 1: x - g  (fl rounding of x - g)
for name, (a, b) in groups.items():
    err = np.abs(g_gpu[a:b] - g_or[a:b]).max()
    print(f"one gradient {name}: max|g| {np.abs(g_or[a:b]).max():.3e} max err {err:.3e}")
ctx.destroy()
for K in (100, 300, 1000, 2000):
    ctx = P.Context(e, n, d, role=r, T=T, model=P.MODEL_MLP, gamma=0.01, batch_M=M, data_A=X, data_y=y,
                    mlp_dims=(I, H, Ocl), x0=x0)
    ctx.replay(ev[:K], batch_idx=bi[:K])
    ctx.sync()
    Xg = np.stack([ctx.read_model(w) for w in range(n)])
    Xo, _ = O.replay(prob, np.tile(x0, (n, 1)), e, r, ev[:K], bi[:K], T=T)
    rms = np.sqrt((Xo.astype(np.float64) ** 2).mean(1, keepdims=True))
    rel = np.abs(Xg - Xo) / np.maximum(np.abs(Xo), rms)
    s = ", ".join(f"{nm} {rel[:, a:b].max():.2e}" for nm, (a, b) in groups.items())
    print(f"K={K}: c11 max rel by group: {s}", flush=True)
    ctx.destroy()
