"""Config 3 free-running on ONE GPU: n in-process ranks (host threads, comm_local),
one MLP worker each, running the host-driven AD-PSGD loop (super-learners with R = 1):
gradient at the worker's own model (tcgen05 3xTF32, device Philox minibatch), passive
lock + ticket on the device, pair average + update, commit.  Prints updates/s."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import synth
import paper_1710_06952_b200 as P


def run(n=8, steps=40, warm=5, S=8192):
    I, H, O, M = 3072, 512, 10, 128
    X, y = synth.mlp_data(S=S, n_in=I, n_out=O, s=0.02, seed=3)
    w0 = synth.mlp_init(I, H, O, seed=4)
    e, r, wr, _, _ = synth.super_ring(n, 1)
    tg = P.ThreadGroup(n)
    out = {}

    def body(rank):
        ctx = P.Context(e, n, w0.size, role=r, rank=rank, world_size=n, device=0, placement=2, worker_rank=wr,
                        model=P.MODEL_MLP, gamma=0.002, batch_M=M, data_A=X, data_y=y, mlp_dims=(I, H, O), x0=w0,
                        seed=99, super_R=1, log_capacity=1 << 14, group=tg)
        ctx.super_run(warm)
        ctx.sync()
        tg.barrier()
        t0 = time.perf_counter()
        ctx.super_run(steps)
        ctx.sync()
        tg.barrier()
        t1 = time.perf_counter()
        if rank == 0:
            out["updates_per_s"] = n * steps / (t1 - t0)
        tg.barrier()
        ctx.destroy()
    P.run_ranks(n, body, group=tg)
    return {"workload": f"config3: MLP {I}->{H}->{O}, M={M}, n={n} workers free-running on ONE GPU "
                        "(in-process ranks, host-driven loop, device Philox batches)",
            "updates_per_s": out["updates_per_s"], "samples_per_s": out["updates_per_s"] * M}


if __name__ == "__main__":
    print(json.dumps(run(int(sys.argv[1]) if len(sys.argv) > 1 else 8)))
