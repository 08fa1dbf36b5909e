"""Find the first event where the GPU lsq replay departs from the oracle (diagnostic)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import synth
import paper_1710_06952_b200 as P
from oracle import oracle as O

n, d, M, K, T = 4, 1024, 32, 2000, 4
e, r = synth.ring(n)
A, b = synth.lsq_data(S=8192, d=d, seed=1)
ev, bi = synth.schedule_iid(n, e, K=K, T=T, M=M, S=8192, seed=42)
prob = O.OracleProblem(O.MODEL_LSQ, M=M, gamma=0.5, A=A, b=b)
for rep in range(3):
    ctx = P.Context(e, n, d, role=r, T=T, model=P.MODEL_LSQ, gamma=0.5, batch_M=M, data_A=A, data_b=b)
    ctx.replay(ev, batch_idx=bi)
    ctx.sync()
    Xg = np.stack([ctx.read_model(w) for w in range(n)])
    ctx.destroy()
    Xo, _ = O.replay(prob, np.zeros((n, d), np.float32), e, r, ev, bi, T=T)
    print("rep", rep, "max abs diff", np.abs(Xg - Xo).max(), "loss gpu", O.full_loss(prob, Xg.mean(0)),
          "loss orc", O.full_loss(prob, Xo.mean(0)), flush=True)
# chunked
for chunk in (1, 10, 100):
    ctx = P.Context(e, n, d, role=r, T=T, model=P.MODEL_LSQ, gamma=0.5, batch_M=M, data_A=A, data_b=b)
    ctx.replay(ev[:chunk], batch_idx=bi[:chunk])
    ctx.sync()
    Xg = np.stack([ctx.read_model(w) for w in range(n)])
    Xo, _ = O.replay(prob, np.zeros((n, d), np.float32), e, r, ev[:chunk], bi[:chunk], T=T)
    print("first", chunk, "events: max abs diff", np.abs(Xg - Xo).max(), flush=True)
    ctx.destroy()
