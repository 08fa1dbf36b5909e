"""Super-learner parity worker (reading R22), run one process per GPU
(tests/test_multigpu.py through torch.distributed.run) or as in-process ranks on
host threads sharing one GPU (comm_local; tests/test_multigpu.py::
test_virtual_super_learner) -- the same body.  For every factorisation
world = S * R: R learners per super-learner (NCCL all-reduce of their
gradients), S super-learners gossiping on a bipartite ring over NVLink.  Checks
that every super-learner's R replicas are bitwise equal and that the event log,
replayed through the oracle's super-learner replay, reproduces them -- bitwise
for R <= 2, within reading c11's 1e-4 for R > 2 (NCCL's own summation order)."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

import numpy as np
import torch
import torch.distributed as dist

import synth
import paper_1710_06952_b200 as P


def body(rank, world, local, G):
    """G: mp_worker.DistGroup or ThreadRanks.  Returns rank 0's failures."""
    ckw = G.ctx_kw()
    if rank == 0:
        from oracle import oracle as O
    fails = []
    d, steps = (1 << 16) + 36, 60
    dk, nk = synth.quad_keys(8)
    s_noise = float(np.float32(0.1 * math.sqrt(96)))
    for R in [r for r in range(1, world + 1) if world % r == 0]:
        S = world // R
        e, role, wr, se, sr = synth.super_ring(S, R)
        Xs0 = synth.x0_uniform(S, d, seed=30 + R)                   # one model per super-learner
        X0 = np.repeat(Xs0, R, axis=0)                               # identical replicas
        ctx = P.Context(e, world, d, role=role, rank=rank, world_size=world, device=local, **ckw, placement=2,
                        worker_rank=wr, x0_per_worker=X0, model=P.MODEL_QUADRATIC, gamma=0.01, batch_M=32,
                        quad_keys=(dk, nk), quad_noise_s=s_noise, seed=3 + R, super_R=R)
        ctx.super_run(steps)
        ctx.sync()
        G.barrier()
        allm = G.all_gather({w: ctx.read_model(w) for w in ctx.local_workers()})
        if rank == 0:
            X = np.zeros((world, d), np.float32)
            for m in allm:
                for w, x in m.items():
                    X[w] = x
            for s in range(S):
                for r in range(1, R):
                    if not np.array_equal(X[s * R].view(np.uint32), X[s * R + r].view(np.uint32)):
                        fails.append(f"S={S} R={R}: replicas of super-learner {s} differ")
            log = ctx.read_log(0)
            if len(log) != S * steps or not np.array_equal(np.sort(log["k"]), np.arange(S * steps)):
                fails.append(f"S={S} R={R}: log has {len(log)} entries")
            else:
                ev = np.stack([log["i"], log["j"], log["tau"], log["flags"].astype(np.int32)], 1)
                prob = O.OracleProblem(O.MODEL_QUADRATIC, M=32, gamma=0.01, data_key=dk, noise_key=nk,
                                       noise_s=s_noise)
                Xo = O.super_replay(prob, Xs0, se, sr, ev, R)
                if R <= 2:      # an all-reduce of two fp32 values is one correctly rounded add
                    if not np.array_equal(X[::R].view(np.uint32), Xo.view(np.uint32)):
                        fails.append(f"S={S} R={R}: log replay not bit-exact")
                else:           # NCCL's summation order is its own: reading c11's 1e-4
                    rms = np.sqrt(np.mean(Xo.astype(np.float64) ** 2, axis=1, keepdims=True))
                    err = np.abs(X[::R].astype(np.float64) - Xo) / np.maximum(np.abs(Xo), rms)
                    if err.max() > 1e-4:
                        fails.append(f"S={S} R={R}: log replay error {err.max():.2e} > 1e-4")
                if S > 1 and not (ev[:, 1] >= 0).any():
                    fails.append(f"S={S} R={R}: no averaging events")
        ctx.destroy()
        G.barrier()
    # sampled models (device Philox minibatches keyed by the super-learner key):
    # the tcgen05 MLP (config 3 with one worker per GPU when R = 1) and lsq
    I, H, O_, M, S = 256, 128, 10, 128, 2048
    Xd, yd = synth.mlp_data(S=S, n_in=I, n_out=O_, s=0.02, seed=3)
    w0 = synth.mlp_init(I, H, O_, seed=4)
    A, b = synth.lsq_data(S=S, d=1024, seed=1)
    seed = 0x5EED_0000_1234
    for kind in ("mlp", "lsq"):
        for R in [r for r in range(1, world + 1) if world % r == 0]:
            S_ = world // R
            e, role, wr, se, sr = synth.super_ring(S_, R)
            if kind == "mlp":
                dm, x0 = w0.size, w0
                kw = dict(model=P.MODEL_MLP, gamma=0.002, batch_M=M, data_A=Xd, data_y=yd, mlp_dims=(I, H, O_))
            else:
                dm, x0 = 1024, np.zeros(1024, np.float32)
                kw = dict(model=P.MODEL_LSQ, gamma=0.02, batch_M=32, data_A=A, data_b=b)
            ctx = P.Context(e, world, dm, role=role, rank=rank, world_size=world, device=local, **ckw, placement=2,
                            worker_rank=wr, x0=x0, seed=seed, super_R=R, **kw)
            ctx.super_run(20)
            ctx.sync()
            G.barrier()
            allm = G.all_gather({w: ctx.read_model(w) for w in ctx.local_workers()})
            if rank == 0:
                X = np.zeros((world, dm), np.float32)
                for m in allm:
                    for w, x in m.items():
                        X[w] = x
                for s_ in range(S_):
                    for r_ in range(1, R):
                        if not np.array_equal(X[s_ * R].view(np.uint32), X[s_ * R + r_].view(np.uint32)):
                            fails.append(f"{kind} S={S_} R={R}: replicas differ")
                log = ctx.read_log(0)
                ev = np.stack([log["i"], log["j"], log["tau"], log["flags"].astype(np.int32)], 1)
                bk = (seed & 0xFFFFFFFF, seed >> 32)
                prob = O.OracleProblem(O.MODEL_MLP, M=M, gamma=0.002, A=Xd, y=yd, dims=(I, H, O_), batch_key=bk) \
                    if kind == "mlp" else O.OracleProblem(O.MODEL_LSQ, M=32, gamma=0.02, A=A, b=b, batch_key=bk)
                Xo = O.super_replay(prob, np.tile(x0, (S_, 1)), se, sr, ev, R)
                rms = np.sqrt(np.mean(Xo.astype(np.float64) ** 2, axis=1, keepdims=True))
                err = np.abs(X[::R].astype(np.float64) - Xo) / np.maximum(np.abs(Xo), rms)
                if len(log) != S_ * 20 or err.max() > 1e-4:
                    fails.append(f"{kind} S={S_} R={R}: {len(log)} events, log replay error {err.max():.2e}")
            ctx.destroy()
            G.barrier()
    return fails


def main():
    from mp_worker import DistGroup
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    fails = body(rank, world, local, DistGroup(rank, world))
    if rank == 0:
        print("SUPER", "FAIL" if fails else "OK", fails, flush=True)
    dist.destroy_process_group()
    sys.exit(1 if (rank == 0 and fails) else 0)


if __name__ == "__main__":
    main()
