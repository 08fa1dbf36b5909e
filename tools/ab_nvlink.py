"""NVLink throughput of the engine on an all-NVLink schedule (torchrun, N GPUs); set
ADPSGD_LIB to an A/B build from tools/ab_build.py to compare engine constants.

  python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 tools/ab_nvlink.py
Interleave placement on a ring: every edge joins two GPUs.  Pure gossip (W_k
only) replayed through the engine; NVLink algorithmic bytes per event = 8d
(4d of x_j one way, 4d of the average back).
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import torch.distributed as dist

import synth
import paper_1710_06952_b200 as P

ap = argparse.ArgumentParser()
ap.add_argument("--d", type=int, default=25_600_000)
ap.add_argument("--events", type=int, default=128)
ap.add_argument("--libs", default="", help="comma-separated ADPSGD_LIB builds to compare (tools/ab_build.py); "
                                           "empty = the in-tree library")
ap.add_argument("--model", default="none")
ap.add_argument("--mode", default="replay", choices=["replay", "run"])
ap.add_argument("--wpg", type=int, default=8, help="workers per GPU")
ap.add_argument("--placement", default="interleave", choices=["interleave", "xor"])
ap.add_argument("--coop", type=int, default=0, help="cooperative cross-GPU events: 0 auto, 1 on, -1 off")
a = ap.parse_args()
rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
n = a.wpg * world
e, r = synth.ring(n)
quad = a.model == "quad"
ev, _ = synth.schedule_iid(n, e, K=a.events, seed=2, no_grad=not quad)
for v in [0]:
    xor = a.placement == "xor"
    ctx = P.Context(e, n, a.d, role=r, rank=rank, world_size=world, device=local, placement=2 if xor else 1,
                    worker_rank=synth.placement_xor(n, world) if xor else None, engine_coop=None if a.coop == 0 else a.coop > 0,
                    model=P.MODEL_QUADRATIC if quad else P.MODEL_NONE, gamma=0.01, batch_M=32,
                    quad_keys=(1, 2), quad_noise_s=0.5)
    s = torch.cuda.Stream()
    go = (lambda: ctx.replay(ev, flags=P.REPLAY_ENGINE, stream=s)) if a.mode == "replay" else \
        (lambda: ctx.run(len(ev), stream=s))
    go()
    torch.cuda.synchronize()
    ctx.sync()
    dist.barrier()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(s)
    go()
    t1.record(s)
    torch.cuda.synchronize()
    ms = torch.tensor([t0.elapsed_time(t1)], device="cuda")
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms = float(ms.item())
    cross = len(ev)
    nvl = cross * 8.0 * a.d / world / (ms / 1e3) / 1e9
    if rank == 0:
        print(f"{a.mode} {a.placement} wpg={a.wpg} coop={a.coop} variant {v}: {len(ev)} cross events in {ms:.2f} ms -> {len(ev) / (ms / 1e3):.0f} events/s, "
              f"NVLink {nvl:.0f} GB/s per GPU per direction", flush=True)
    ctx.destroy()
    dist.barrier()
dist.destroy_process_group()
