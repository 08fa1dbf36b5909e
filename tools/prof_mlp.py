"""Driver for ncu captures of the MLP gradient (tcgen05 GEMMs), config 3 shapes."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
import paper_1710_06952_b200 as P

I, H, O, M, n = 3072, 512, 10, 128, 4
X, y = synth.mlp_data(S=4096, n_in=I, n_out=O, s=0.02, seed=3)
x0 = synth.mlp_init(I, H, O, seed=4)
e, r = synth.ring(n)
ev, bi = synth.schedule_iid(n, e, K=6, M=M, S=4096, seed=7)
ctx = P.Context(e, n, x0.size, role=r, model=P.MODEL_MLP, gamma=0.002, batch_M=M, data_A=X, data_y=y,
                mlp_dims=(I, H, O), x0=x0)
ctx.replay(ev, batch_idx=bi)
ctx.sync()
print("ok", ctx.launch_count())
ctx.destroy()
