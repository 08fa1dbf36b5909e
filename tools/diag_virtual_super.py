import os, sys, time, math
print("CUDA_DEVICE_MAX_CONNECTIONS", os.environ.get("CUDA_DEVICE_MAX_CONNECTIONS"), flush=True)
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np
import synth, paper_1710_06952_b200 as P
world = int(sys.argv[1]); R = int(sys.argv[2]); steps = int(sys.argv[3])
S = world // R
d = (1 << 16) + 36
dk, nk = synth.quad_keys(8)
sn = float(np.float32(0.1 * math.sqrt(96)))
e, role, wr, se, sr = synth.super_ring(S, R)
print("edges", e.tolist() if hasattr(e, "tolist") else e, "role", list(role), "wr", list(wr), flush=True)
Xs0 = synth.x0_uniform(S, d, seed=30 + R); X0 = np.repeat(Xs0, R, axis=0)
tg = P.ThreadGroup(world)
def body(rank):
    ctx = P.Context(e, world, d, role=role, rank=rank, world_size=world, device=0, placement=2, worker_rank=wr,
                    x0_per_worker=X0, model=P.MODEL_QUADRATIC, gamma=0.01, batch_M=32, quad_keys=(dk, nk),
                    quad_noise_s=sn, seed=3 + R, super_R=R, group=tg)
    t = time.time()
    for s in range(steps):
        ctx.super_run(1)
        print(f"rank {rank} step {s} enqueued {time.time()-t:.3f}", flush=True)
    ctx.sync()
    print(f"rank {rank} synced {time.time()-t:.3f}", flush=True)
    tg.barrier()
    if rank == 0: print("log", ctx.read_log(0)[["k","i","j"]].tolist(), flush=True)
    tg.barrier()
    ctx.destroy()
P.run_ranks(world, body, group=tg)
print("DONE", flush=True)
