"""Small, ragged instances of every device path in one process (host and engine
replay, free-running, wait-free + slow link, step/gossip, consensus, both
synchronous baselines, lsq/logreg, the tcgen05 MLP) -- a quick all-paths smoke,
sized to run under compute-sanitizer (memcheck / racecheck / synccheck) -- which
this GPU pool refuses ("closed ... runs under it have left GPUs needing a reset",
profiles/r02_sanitizer_refused.log); the driver-side parity suite is the check.

    python tools/sanitize_smoke.py
"""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import synth
import paper_1710_06952_b200 as P


def main():
    n, d = 8, 4099
    e, r = synth.ring(n)
    dk, nk = synth.quad_keys(3)
    s = float(np.float32(0.1 * math.sqrt(96)))
    q = dict(model=P.MODEL_QUADRATIC, gamma=0.01, batch_M=32, quad_keys=(dk, nk), quad_noise_s=s)
    X0 = synth.x0_uniform(n, d, seed=1)
    # pure gossip, host and engine replay
    ev, _ = synth.schedule_iid(n, e, K=60, seed=1, no_grad=True)
    for path in (P.REPLAY_HOST, P.REPLAY_ENGINE):
        c = P.Context(e, n, d, role=r, x0_per_worker=X0)
        c.replay(ev, flags=path)
        c.sync()
        c.destroy()
    # quadratic with staleness (host), engine replay, free-running, step/gossip, consensus
    c = P.Context(e, n, d, role=r, T=3, x0_per_worker=X0, compute_ns=5_000, log_capacity=4096, **q)
    ev, _ = synth.schedule_iid(n, e, K=60, T=3, seed=2, local_prob=0.3)
    c.replay(ev, flags=P.REPLAY_HOST)
    ev0, _ = synth.schedule_iid(n, e, K=40, seed=3, local_prob=0.3)
    c.replay(ev0, flags=P.REPLAY_ENGINE)
    ev1, _ = synth.schedule_iid(n, e, K=40, T=3, seed=7, local_prob=0.3)     # engine stale-read ops
    c.replay(ev1, flags=P.REPLAY_ENGINE)
    c.run(200)
    c.step(0)
    c.gossip(2, 3)
    out = torch.empty(d, dtype=torch.float32, device="cuda")
    c.consensus_mean(out.data_ptr(), with_mk=True)
    c.read_log(0)
    c.allreduce_reset()
    c.allreduce_sgd(2)
    c.dpsgd_reset(X0)
    c.dpsgd(2)
    c.sync()
    c.destroy()
    # App. A: host replay with compensation, wait-free engine loop, slow link
    ev = synth.schedule_appa(n, e, r, 80, 6, seed=4)
    c = P.Context(e, n, d, role=r, T=6, x0_per_worker=X0, **q)
    c.replay(ev, flags=P.REPLAY_HOST)
    c.sync()
    c.destroy()
    link = np.ones(n, np.float32)
    link[1] = 4.0
    c = P.Context(e, n, d, role=r, x0_per_worker=X0, wait_free=2, compute_ns=5_000, link_slow=link,
                  link_ns=5_000, **q)
    c.run(200)
    c.sync()
    c.destroy()
    # least squares / logistic (1-CTA gradient kernels), device Philox batches
    A, b = synth.lsq_data(S=512, d=1000, seed=1)
    for kind in (P.MODEL_LSQ, P.MODEL_LOGREG):
        bb = b if kind == P.MODEL_LSQ else np.where(b > 0, 1.0, -1.0).astype(np.float32)
        c = P.Context(np.array([[0, 1], [1, 2], [2, 3], [3, 0]], np.int32), 4, 1000, T=2, model=kind,
                      gamma=0.1, batch_M=16, data_A=A, data_b=bb)
        ev, _ = synth.schedule_iid(4, np.array([[0, 1], [1, 2], [2, 3], [3, 0]]), K=40, T=2, seed=5)
        c.replay(ev)
        c.sync()
        c.destroy()
    # MLP on tcgen05 (3xTF32 GEMMs, TMA tensor maps, TMEM)
    I, H, O, M = 256, 128, 10, 128
    Xd, y = synth.mlp_data(S=1024, n_in=I, n_out=O, s=0.02, seed=3)
    dm = (H * I + H + O * H + O)
    x0 = synth.mlp_init(I, H, O, seed=4)
    c = P.Context(np.array([[0, 1], [1, 2], [2, 3], [3, 0]], np.int32), 4, dm, T=2, model=P.MODEL_MLP,
                  gamma=0.002, batch_M=M, data_A=Xd, data_y=y, mlp_dims=(I, H, O), x0=x0)
    ev, _ = synth.schedule_iid(4, np.array([[0, 1], [1, 2], [2, 3], [3, 0]]), K=12, T=2, seed=6)
    c.replay(ev)
    c.sync()
    c.destroy()
    # two in-process ranks on this GPU: cooperative cross-rank events, remote locks, mailboxes
    tg = P.ThreadGroup(2)

    def rank_body(rk):
        cc = P.Context(e, n, d, role=r, rank=rk, world_size=2, device=0, placement=1, x0_per_worker=X0,
                       compute_ns=5_000, group=tg, **q)
        cc.run(100)
        cc.sync()
        tg.barrier()
        cc.destroy()
    P.run_ranks(2, rank_body, group=tg)
    torch.cuda.synchronize()
    print("SANITIZE_SMOKE OK")


if __name__ == "__main__":
    main()
