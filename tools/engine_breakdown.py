"""Per-rank engine time breakdown on the bench workload (config 4), local vs cross-GPU events.

  python tools/engine_breakdown.py                       (1 GPU)
  python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 tools/engine_breakdown.py
Prints, per rank: committed events / pairs / cross pairs, the engine's CUDA-event time per
launch, algorithmic HBM GB/s, and the mean start-to-commit duration of local and cross events
(engine counters engine_busy_ns / engine_busy_cross_ns).
"""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import synth
import paper_1710_06952_b200 as P

rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
local = int(os.environ.get("LOCAL_RANK", 0))
torch.cuda.set_device(local)
dist = None
if world > 1:
    import torch.distributed as dist
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
n, d, steps = 8 * world, 25_600_000, 10
U = 32 * n
e, r = synth.ring(n)
dk, nk = synth.quad_keys(5)
s = float(np.float32(0.1 * math.sqrt(3 * 32)))
ctx = P.Context(e, n, d, role=r, rank=rank, world_size=world, device=local, placement=0,
                model=P.MODEL_QUADRATIC, gamma=0.01, batch_M=32, quad_keys=(dk, nk), quad_noise_s=s,
                straggler=synth.stragglers(n, slow_worker=0, slow=10.0), compute_ns=50_000, seed=1234,
                log_capacity=1 << 16)
stream = torch.cuda.Stream()
for _ in range(3):
    ctx.run(U, stream)
torch.cuda.synchronize()
ctx.sync()
if dist:
    dist.barrier()
s0 = ctx.stats()
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
for a, b in ev:
    a.record(stream)
    ctx.run(U, stream)
    b.record(stream)
torch.cuda.synchronize()
ctx.sync()
s1 = ctx.stats()
ms = sum(a.elapsed_time(b) for a, b in ev) / steps
D = {k: s1[k] - s0[k] for k in ("local_events", "local_pair_events", "local_cross_events", "local_bytes",
                                 "engine_busy_ns", "engine_busy_cross_ns")}
nl = D["local_events"] - D["local_cross_events"]
line = (f"rank {rank}/{world}: per launch {D['local_events'] / steps:.1f} events, {D['local_pair_events'] / steps:.1f} "
        f"pairs, {D['local_cross_events'] / steps:.1f} cross; engine {ms:.3f} ms, "
        f"{D['local_bytes'] / steps / (ms / 1e3) / 1e9:.0f} GB/s; mean duration local "
        f"{(D['engine_busy_ns'] - D['engine_busy_cross_ns']) / max(nl, 1) / 1e3:.1f} us, cross "
        f"{D['engine_busy_cross_ns'] / max(D['local_cross_events'], 1) / 1e3:.1f} us")
if dist:
    lines = [None] * world
    dist.all_gather_object(lines, line)
    if rank == 0:
        print("\n".join(lines), flush=True)
else:
    print(line, flush=True)
ctx.destroy()
if dist:
    dist.barrier()
    dist.destroy_process_group()
