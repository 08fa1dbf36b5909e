import math, os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch, torch.distributed as dist
import synth, paper_1710_06952_b200 as P
rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
n = 8 * world
e, r = synth.ring(n)
d = (1 << 14) + 20
ctx = P.Context(e, n, d, role=r, rank=rank, world_size=world, device=local, placement=1,
                model=P.MODEL_QUADRATIC, gamma=0.01, batch_M=32, quad_keys=(1, 2), quad_noise_s=0.5,
                x0_per_worker=synth.x0_uniform(n, d, seed=27), seed=13)
print(f"rank {rank} ctx ok, local {ctx.local_workers()}", flush=True)
for it in range(25):
    for w in ctx.local_workers():
        try:
            k = ctx.step(w)
        except Exception as ex:
            print(f"rank {rank} step {it} w {w} FAILED {ex}", flush=True)
            raise
    print(f"rank {rank} round {it} done", flush=True)
ctx.sync()
print(f"rank {rank} steps done", flush=True)
dist.barrier()
print(f"rank {rank} ticket {ctx.ticket()}", flush=True)
import time
if rank == 0:
    time.sleep(3)
ctx.run(200)
print(f"rank {rank} run launched", flush=True)
ctx.sync()
print(f"rank {rank} run done, ticket {ctx.ticket()}", flush=True)
ctx.destroy()
dist.destroy_process_group()
