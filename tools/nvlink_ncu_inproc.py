"""NVLink counter capture (ncu) of the fused engine kernel with every pair event
crossing GPUs, ONE process driving G GPUs (in-process ranks, comm_local).

ncu serialises the kernels of the process it profiles and replays a kernel once
per metric pass, so the captured engine must not depend on another GPU's
concurrently running engine: cooperative events are off (engine_coop = -1) and
every active worker lives on GPU 0 (G = 2: interleave placement, which the
bipartite ring forces to GPU = role; G > 2: passives spread over GPUs 1..G-1),
so GPU 0's engine performs all reads of x_j and writes of m over NVLink while
the other GPUs' engines only hold passives (they exit at once).  Free-running
pure gossip (NO_GRAD averages): each pass takes and releases the
remote try-locks itself, so kernel replay sees the same protocol state.
Run:  ncu --devices 0 -k regex:k_engine ... python tools/nvlink_ncu_inproc.py G
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import synth
import paper_1710_06952_b200 as P


def main():
    G = int(sys.argv[1]) if len(sys.argv) > 1 else torch.cuda.device_count()
    d = int(sys.argv[2]) if len(sys.argv) > 2 else 25_600_000
    per = 16
    n = 2 * per * (G - 1) if G > 2 else 2 * per
    e, r = synth.ring(n)
    wr = np.array([0 if w % 2 == 0 else 1 + (w // 2) % (G - 1) for w in range(n)], np.int32)
    tg = P.ThreadGroup(G)
    sms = torch.cuda.get_device_properties(0).multi_processor_count

    def body(rank):
        ctx = P.Context(e, n, d, role=r, rank=rank, world_size=G, device=rank, placement=2, worker_rank=wr,
                        engine_coop=False, group=tg, engine_grid=2 * sms, log_capacity=1 << 16)
        for it in range(2):
            tg.barrier()
            s0 = ctx.stats()
            ctx.run(8 * n)
            ctx.sync()
            s1 = ctx.stats()
            tg.barrier()
            print(f"[rank {rank}] launch {it}: pairs {s1['local_pair_events'] - s0['local_pair_events']}, cross "
                  f"{s1['local_cross_events'] - s0['local_cross_events']}, algorithmic NVLink bytes "
                  f"{s1['local_nvlink_bytes'] - s0['local_nvlink_bytes']:.6g}", flush=True)
        tg.barrier()
        ctx.destroy()

    P.run_ranks(G, body, group=tg)


if __name__ == "__main__":
    main()
