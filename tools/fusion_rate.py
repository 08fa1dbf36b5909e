"""How often the engine fuses a passive's due local step into the pair pass that
holds its lock (bench workload, config 4).  A fused step is logged as event
k-1 = (j, -1) with the same start time as the pair event k = (i, j)."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np

import synth
import paper_1710_06952_b200 as P


def main():
    n, d, U = 8, 25_600_000, 4096
    e, r = synth.ring(n)
    dk, nk = synth.quad_keys(5)
    s = float(np.float32(0.1 * math.sqrt(96)))
    waits = [int(x) for x in sys.argv[1:]] or [0]
    for fuse, wait in [(False, 0)] + [(True, w) for w in waits]:
        ctx = P.Context(e, n, d, role=r, model=P.MODEL_QUADRATIC, gamma=0.01, batch_M=32, quad_keys=(dk, nk),
                        quad_noise_s=s, straggler=synth.stragglers(n, slow_worker=0, slow=10.0), compute_ns=50_000,
                        seed=1234, engine_fuse=fuse, engine_fuse_wait_ns=wait * 1000)
        ctx.run(U)   # warm-up run
        ctx.sync()
        k0 = ctx.ticket()
        ctx.run(U)
        ctx.sync()
        log = ctx.read_log(k0)
        loc = log["j"] < 0
        fused = loc[:-1] & (log["j"][1:] == log["i"][:-1]) & (log["t0"][1:] == log["t0"][:-1])
        t = (log["t1"].max() - log["t0"].min()) / 1e9
        print(f"fuse={fuse} wait={wait}us: events {len(log)}, pair {int((~loc).sum())}, local {int(loc.sum())}, "
              f"fused local {int(fused.sum())} ({fused.sum() / max(1, loc.sum()):.1%} of local), "
              f"{len(log) / t:.0f} events/s, {(~loc).sum() / t:.0f} gossip-steps/s")
        ctx.destroy()


if __name__ == "__main__":
    main()
