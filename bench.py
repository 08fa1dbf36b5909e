#!/usr/bin/env python
"""bench.py -- AD-PSGD hot path on B200: gossip-steps/s at 25.6M parameters.

Workload (BASELINE.json configs[3], "config 4"): a ResNet-50-sized flat model,
d = 25,600,000 fp32, synthetic quadratic gradients (M = 32, sigma = 0.1,
gamma = 0.01), n = 8 workers per GPU on one bipartite ring (block placement),
worker 0 slowed 10x, emulated per-gradient compute t_c.
One STEP = the system commits U gradient updates through the free-running
persistent engine (stale-free fused gradient, pair average over HBM/NVLink,
device try-locks, tickets) followed by the consensus output x_bar.

Contract: python bench.py --gpus N --steps K --warmup W [--impl reference]
prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
# the config-3 free-running leg drives 8 in-process ranks: one hardware queue per stream
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

D_FULL = 25_600_000
M_BATCH = 32
SIGMA = 0.1
GAMMA = 0.01


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--d", type=int, default=D_FULL)
    ap.add_argument("--workers-per-gpu", type=int, default=8)
    ap.add_argument("--updates-per-step", type=int, default=0, help="0 = 32 per worker")
    ap.add_argument("--compute-us", type=float, default=50.0, help="emulated t_c of a 1x worker")
    ap.add_argument("--straggler", type=float, default=10.0)
    ap.add_argument("--placement", type=int, default=0)
    ap.add_argument("--no-extras", action="store_true", help="skip baseline/no-straggler/cpu legs")
    ap.add_argument("--cpu-events", type=int, default=12)
    ap.add_argument("--ctas-per-sm", type=int, default=0)
    ap.add_argument("--topology", default="ring", choices=["ring", "skip"])
    ap.add_argument("--no-fuse", action="store_true", help="never fuse a due passive step into a pair pass")
    ap.add_argument("--coop", type=int, default=0, help="cooperative cross-GPU events: 0 auto, 1 on, -1 off")
    return ap.parse_args()


# ------------------------------------------------------------------ clocks --
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled DURING the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, dev):
        self.dev, self.rows, self.proc = dev, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-i", str(self.dev), "-lms", "50"], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            p = [x.strip() for x in line.split(",")]
            if len(p) == 6:
                self.rows.append([time.perf_counter()] + p)

    def window(self, t0, t1):
        """keep only samples taken inside the timed region [t0, t1] (host clock)"""
        inside = [r for r in self.rows if t0 <= r[0] <= t1]
        self.rows = [r[1:] for r in (inside or self.rows[-1:])]

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


class NvlCounters:
    """NVML NVLink byte counters of this rank's GPU (hardware counters, not the
    engine's algorithmic accounting), read before and after a timed region.
    Scheme "throughput": fields 138 / 139 (data TX / RX) and 140 / 141 (raw TX /
    RX incl. protocol), cumulative KiB over all links; scheme "per_link": fields
    202 / 204 (XMIT / RCV bytes) summed over every link.  The first scheme the
    driver supports is used; None when NVML has neither."""

    FIELDS = {"data_tx": 138, "data_rx": 139, "raw_tx": 140, "raw_rx": 141}
    LINK_FIELDS = {"data_tx": 202, "data_rx": 204}
    MAX_LINKS = 18

    def __init__(self, dev):
        self.h, self.scheme, self.err = None, None, None
        try:
            import pynvml as N
            import torch
            N.nvmlInit()
            self.N = N
            try:
                uuid = str(torch.cuda.get_device_properties(dev).uuid)
                self.h = N.nvmlDeviceGetHandleByUUID(uuid if uuid.startswith("GPU-") else "GPU-" + uuid)
            except Exception:
                self.h = N.nvmlDeviceGetHandleByIndex(dev)
            for scheme in ("throughput", "per_link"):
                self.scheme = scheme
                if self.read() is not None:
                    break
                self.scheme = None
        except Exception as ex:
            self.h, self.err = None, repr(ex)

    def _fields(self):
        if self.scheme == "throughput":
            return [(k, (f, 0)) for k, f in self.FIELDS.items()]
        return [(k, (f, l)) for k, f in self.LINK_FIELDS.items() for l in range(self.MAX_LINKS)]

    def read(self):
        if self.h is None or self.scheme is None:
            return None
        try:
            fl = self._fields()
            vals = self.N.nvmlDeviceGetFieldValues(self.h, [f for _, f in fl])
            out = {}
            for (k, _), v in zip(fl, vals):
                if v.nvmlReturn != 0:
                    if self.scheme == "per_link":
                        continue                       # a link that is absent
                    self.err = f"field {k}: nvmlReturn {v.nvmlReturn}"
                    return None
                out[k] = out.get(k, 0.0) + float(v.value.ullVal) * (1024.0 if self.scheme == "throughput" else 1.0)
            return out if out else None
        except Exception as ex:
            self.err = repr(ex)
            return None

    @staticmethod
    def delta(a, b):
        return None if (a is None or b is None) else {k: b[k] - a[k] for k in a}


def traffic_per_launch(alg_bytes):
    """DRAM bytes per engine launch: the dram/algorithmic ratio of the committed
    ncu --set full capture (profiles/engine_traffic.json) times this launch's
    algorithmic bytes, and the capture it came from; (None, None) if no capture
    is committed."""
    try:
        t = json.load(open(os.path.join(ROOT, "profiles", "engine_traffic.json")))
        return alg_bytes * t["dram_bytes_per_algorithmic_byte"], t["source"]
    except Exception:
        return None, None


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


# --------------------------------------------------------- CPU oracle legs --
def oracle_sample(n, d, events, seed=5, omp=False):
    """Time the oracle (as it stands) on `events` events of the same workload:
    the replay core only -- a call's fixed cost (copying the n x d state in and
    out, allocating its history) is timed with an empty schedule and subtracted."""
    import numpy as np
    import synth
    from oracle import oracle as O
    e, r = synth.ring(n)
    dk, nk = synth.quad_keys(seed)
    s = float(np.float32(SIGMA * math.sqrt(3 * M_BATCH)))
    prob = O.OracleProblem(O.MODEL_QUADRATIC, M=M_BATCH, gamma=GAMMA, data_key=dk, noise_key=nk, noise_s=s)
    ev, _ = synth.schedule_iid(n, e, K=events, seed=seed, local_prob=0.0)
    X = np.zeros((n, d), np.float32)
    O.replay(prob, X, e, r, ev[:1], omp=omp)        # page in the library / first-touch the state
    t0 = time.perf_counter()
    O.replay(prob, X, e, r, ev[:0], omp=omp)
    t1 = time.perf_counter()
    O.replay(prob, X, e, r, ev, omp=omp)
    t2 = time.perf_counter()
    dt = max((t2 - t1) - (t1 - t0), 1e-9)
    pairs = int((ev[:, 1] >= 0).sum())
    return pairs, dt


def host_info():
    """nproc and the CPU model (lscpu) of the box the CPU legs ran on."""
    model = None
    try:
        for line in subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout.splitlines():
            if line.startswith("Model name:"):
                model = line.split(":", 1)[1].strip()
    except Exception:
        pass
    return {"nproc": os.cpu_count(), "cpu_model": model}


def run_reference(a):
    """--impl reference: the CPU oracle (this tier's reference arm), rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    n = a.workers_per_gpu * a.gpus
    # an event's work (2 rows of d) does not depend on n; the oracle copies the whole
    # n x d state per call, so the sample uses a ring of min(n, 8) workers to keep
    # every step bounded (n = 64 at 8 GPUs would be 6.5 GB per copy)
    n_s = min(n, 8)
    per_step = 4
    for _ in range(a.warmup):
        oracle_sample(n_s, a.d, per_step)
    tot_pairs, tot_t = 0, 0.0
    for _ in range(a.steps):
        p, t = oracle_sample(n_s, a.d, per_step)
        tot_pairs += p
        tot_t += t
    v = tot_pairs / tot_t
    line = {"impl": "reference", "metric": "gossip-steps/s", "value": v, "unit": "gossip-steps/s",
            "n_gpus": a.gpus, "steps": a.steps, "warmup": a.warmup, "ms_per_step": 1e3 * tot_t / a.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": {"workload": f"config4: quadratic d={a.d}, n={n} ring, M={M_BATCH}, oracle sample",
                       "parallelism": "none (1 CPU core)"},
            "cpu_baseline": {"value": v, "unit": "gossip-steps/s", "cores": 1, "kind": "oracle",
                             "sample": f"{per_step} pair events per step on a ring of {n_s} workers (the "
                                       f"workload has n={n}), d={a.d}; replay core (fixed per-call copy "
                                       f"cost subtracted)", "host": host_info()},
            "e2e": {"value": v, "unit": "gossip-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def mlp_leg(P, synth, torch, events=64):
    """Config 3 (BASELINE configs[2]): 2-layer MLP 3072 -> 512 -> 10, M = 128,
    n = 8 workers co-located on this GPU, stale reads tau ~ U{0..4}; gradients
    on tcgen05 (3xTF32).  Replay of a fixed schedule through the HOST executor."""
    I, H, O, M, n, T = 3072, 512, 10, 128, 8, 4
    X, y = synth.mlp_data(S=8192, n_in=I, n_out=O, s=0.02, seed=3)
    x0 = synth.mlp_init(I, H, O, seed=4)
    e, r = synth.ring(n)
    warm, bw = synth.schedule_iid(n, e, K=8, T=T, M=M, S=8192, seed=6)
    ev, bi = synth.schedule_iid(n, e, K=events, T=T, M=M, S=8192, seed=7)
    ctx = P.Context(e, n, x0.size, role=r, T=T, model=P.MODEL_MLP, gamma=0.002, batch_M=M, data_A=X,
                    data_y=y, mlp_dims=(I, H, O), x0=x0)
    ctx.replay(warm, batch_idx=bw)
    ctx.sync()
    s = torch.cuda.Stream()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = ctx.launch_count()
    t0.record(s)
    ctx.replay(ev, batch_idx=bi, stream=s)
    t1.record(s)
    torch.cuda.synchronize()
    sec = t0.elapsed_time(t1) / 1e3
    flops = 2.0 * 2 * M * I * H + 2.0 * 3 * M * H * O      # the two big GEMMs + the N=10 layer
    launches = ctx.launch_count() - l0
    ctx.destroy()
    return {"workload": f"config3: MLP {I}->{H}->{O}, M={M}, n={n} ring on 1 GPU, tau~U{{0..{T}}}, "
                        f"{events} replayed events", "updates_per_s": events / sec,
            "samples_per_s": events * M / sec, "ms_per_update": 1e3 * sec / events,
            "algorithmic_tflops": flops * events / sec / 1e12, "kernel_launches": launches}


def config1_leg(P, synth, torch, K=2000):
    """Config 1 (BASELINE configs[0]): least squares, n = 4 ring, d = 1024, M = 32,
    T = 4, a seeded 2000-event replay with explicit batches.  Latency-bound
    (4 KB rows): us/event of the HOST executor, which runs the whole lsq schedule
    in ONE launch (k_lin_replay: per event its stale-read gradients, then the
    event), next to the same schedule as pure averaging issued one kernel per
    event (the floor of any one-launch-per-event executor)."""
    n, d, M, T, S = 4, 1024, 32, 4, 8192
    e, r = synth.ring(n)
    A, b = synth.lsq_data(S=S, d=d, seed=1)
    ev, bi = synth.schedule_iid(n, e, K=K, T=T, M=M, S=S, seed=42)
    evg = ev.copy()
    evg[:, 2], evg[:, 3] = 0, 1
    out = {}
    for name, sched, kw in (("lsq", ev, dict(model=P.MODEL_LSQ, data_A=A, data_b=b)), ("averaging_only", evg, {})):
        ctx = P.Context(e, n, d, role=r, T=T, gamma=0.5, batch_M=M, **kw)
        ctx.replay(sched[:100], batch_idx=bi[:100] if name == "lsq" else None)
        ctx.sync()
        s = torch.cuda.Stream()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        l0 = ctx.launch_count()
        t0.record(s)
        ctx.replay(sched, batch_idx=bi if name == "lsq" else None, stream=s)
        t1.record(s)
        torch.cuda.synchronize()
        sec = t0.elapsed_time(t1) / 1e3
        out[name] = {"us_per_event": 1e6 * sec / K, "events_per_s": K / sec,
                     "kernel_launches_per_event": (ctx.launch_count() - l0) / K}
        ctx.destroy()
    out["workload"] = (f"config1: lsq n={n} ring, d={d}, M={M}, T={T}, {K}-event seeded replay (HOST executor: "
                       f"lsq in one launch; averaging_only one launch per event)")
    return out


def config2_leg(P, synth, torch, K=4000):
    """Config 2 (BASELINE configs[1]): pure gossip, n = 16 bipartite ring, d = 2^20,
    a 4000-event iid schedule: the persistent engine's replay (one launch; the
    64 MiB working set is L2-resident, so bytes/s can exceed HBM), the HOST
    executor's replay, and free-running gossip (actives initiate)."""
    n, d = 16, 1 << 20
    e, r = synth.ring(n)
    X0 = synth.x0_uniform(n, d, seed=100)
    ev, _ = synth.schedule_iid(n, e, K=K, seed=0, no_grad=True)
    out = {}
    for name in ("engine_replay", "host_replay", "free_running"):
        ctx = P.Context(e, n, d, role=r, x0_per_worker=X0, log_capacity=1 << 14)
        go = (lambda st: ctx.replay(ev, flags=P.REPLAY_ENGINE, stream=st)) if name == "engine_replay" else \
            (lambda st: ctx.replay(ev, flags=P.REPLAY_HOST, stream=st)) if name == "host_replay" else \
            (lambda st: ctx.run(K, stream=st))
        s = torch.cuda.Stream()
        go(s)
        torch.cuda.synchronize()
        ctx.sync()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record(s)
        go(s)
        t1.record(s)
        torch.cuda.synchronize()
        ctx.sync()
        sec = t0.elapsed_time(t1) / 1e3
        out[name] = {"gossip_steps_per_s": K / sec, "us_per_event": 1e6 * sec / K,
                     "algorithmic_gbs": K * 16.0 * d / sec / 1e9}
        ctx.destroy()
    out["workload"] = f"config2: pure gossip n={n} ring, d={d}, {K} iid events (64 MiB working set, L2-resident)"
    return out


# ---------------------------------------------------------------- our arm --
def main():
    a = parse()
    if a.impl == "reference":
        return run_reference(a)
    import numpy as np
    import torch
    import synth

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_1710_06952_b200 import build as B
    if rank == 0:
        B.build()
    if dist:
        dist.barrier()
    import paper_1710_06952_b200 as P

    n = a.workers_per_gpu * world
    d = a.d
    U = a.updates_per_step or 32 * n
    e, r = synth.skip_ring(n) if a.topology == "skip" else synth.ring(n)
    dk, nk = synth.quad_keys(5)
    s = float(np.float32(SIGMA * math.sqrt(3 * M_BATCH)))
    strag = synth.stragglers(n, slow_worker=0, slow=a.straggler)
    cns = int(a.compute_us * 1000)

    def make_ctx(st, nn=None, ee=None, rr=None, wait_free=0, compute_ns=None):
        nn = n if nn is None else nn
        ee = e if ee is None else ee
        rr = r if rr is None else rr
        return P.Context(ee, nn, d, role=rr, rank=rank, world_size=world, device=local, placement=a.placement,
                         model=P.MODEL_QUADRATIC, gamma=GAMMA, batch_M=M_BATCH, quad_keys=(dk, nk),
                         quad_noise_s=s, straggler=st, compute_ns=cns if compute_ns is None else compute_ns,
                         seed=1234, log_capacity=1 << 16,
                         engine_ctas_per_sm=a.ctas_per_sm, wait_free=wait_free,
                         engine_fuse=not a.no_fuse, engine_coop=None if a.coop == 0 else a.coop > 0)

    stream = torch.cuda.Stream()
    out = torch.empty(d, dtype=torch.float32, device="cuda")
    out_host = torch.empty(d, dtype=torch.float32, pin_memory=True)   # e2e: x_bar back to the host
    nvl = NvlCounters(local)

    def barrier():
        if dist:
            dist.barrier()

    def maxr(x):
        if not dist:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sumr(x):
        if not dist:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t)
        return float(t.item())

    def nvl_report(delta, sec):
        """counter-based NVLink GB/s of this GPU (data payload and raw incl. protocol), mean and
        max over ranks; collective"""
        ok = -maxr(-(0.0 if delta is None else 1.0)) > 0          # available on every rank
        rep = {"source": f"NVML NVLink byte counters ({nvl.scheme} scheme, see NvlCounters) read around the "
                         "timed region on every rank"}
        if delta is None or not ok:
            rep["available"] = False
            rep["error"] = nvl.err
            return rep
        vals = {k: v / sec / 1e9 for k, v in delta.items()}
        for k, v in vals.items():
            rep[f"{k}_gbs_mean"] = sumr(v) / max(world, 1)
            rep[f"{k}_gbs_max"] = maxr(v)
        rep["data_per_direction_frac_of_900"] = max(rep["data_tx_gbs_mean"], rep["data_rx_gbs_mean"]) / 900.0
        return rep

    def step(ctx, eng=None):
        if eng:
            eng[0].record(stream)
        ctx.run(U, stream)
        if eng:
            eng[1].record(stream)
        ctx.consensus_mean(out.data_ptr(), with_mk=False, stream=stream)

    def timed(ctx, K, W, engine_events=False):
        with ClockSampler(local) as clk:
            time.sleep(0.3)                     # let nvidia-smi start sampling
            for _ in range(W):
                step(ctx)
            torch.cuda.synchronize()
            ctx.sync()
            barrier()
            st0 = ctx.stats()
            l0 = ctx.launch_count()
            engs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                    for _ in range(K)] if engine_events else [None] * K
            t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            barrier()
            nv0 = nvl.read()
            h0 = time.perf_counter()
            t0.record(stream)
            for k in range(K):
                step(ctx, engs[k])
            t1.record(stream)
            torch.cuda.synchronize()
            h1 = time.perf_counter()
            nv1 = nvl.read()
        clk.window(h0, h1)
        timed.nvl = NvlCounters.delta(nv0, nv1)
        ctx.sync()
        barrier()
        ms = maxr(t0.elapsed_time(t1))
        st1 = ctx.stats()
        eng_ms = sum(x[0].elapsed_time(x[1]) for x in engs) / K if engine_events else None
        return ms, st0, st1, ctx.launch_count() - l0, clk.summary(), eng_ms

    # ------------------------------------------------ main leg: straggler --
    ctx = make_ctx(strag)
    ms, st0, st1, launches, clocks, eng_ms = timed(ctx, a.steps, a.warmup, engine_events=True)
    nvl_main = timed.nvl
    pairs = sumr(st1["local_pair_events"] - st0["local_pair_events"])
    events = sumr(st1["local_events"] - st0["local_events"])
    loc_bytes = st1["local_bytes"] - st0["local_bytes"]
    nvl_bytes = sumr(st1["local_nvlink_bytes"] - st0["local_nvlink_bytes"])
    sec = ms / 1e3
    gossip_s = pairs / sec
    upd_s = events / sec
    # roofline of the dominant kernel (k_engine): algorithmic bytes / launch duration
    pk = peaks()
    hbm_peak = pk.get("hbm_gbs", 6650.0)
    eng_s = eng_ms / 1e3
    achieved = loc_bytes / a.steps / eng_s / 1e9
    # e2e: public API with host timing.  (1) synchronous: M_k read back and x_bar copied to the host
    # before the next step starts; (2) pipelined (the reported e2e): step k's x_bar goes to pinned
    # host memory on a copy stream while step k + 1 runs (double-buffered), all copies inside the
    # timed region
    for _ in range(2):
        ctx.run(U)
        ctx.consensus_mean(out.data_ptr(), with_mk=True)
    barrier()
    st_e = ctx.stats()
    te0 = time.perf_counter()
    for _ in range(a.steps):
        ctx.run(U)
        mk = ctx.consensus_mean(out.data_ptr(), with_mk=True)
        out_host.copy_(out)                     # the step's result x_bar, device -> pinned host
    te_sync = maxr(time.perf_counter() - te0)
    pairs_sync = sumr(ctx.stats()["local_pair_events"] - st_e["local_pair_events"])
    outs = [out, torch.empty_like(out)]
    hosts = [out_host, torch.empty(d, dtype=torch.float32, pin_memory=True)]
    copy_stream = torch.cuda.Stream()
    copied = [torch.cuda.Event(), torch.cuda.Event()]
    ready = torch.cuda.Event()
    torch.cuda.synchronize()
    barrier()
    st_e = ctx.stats()
    te0 = time.perf_counter()
    for k in range(a.steps):
        b_ = k % 2
        ctx.run(U, stream)
        if k >= 2 and rank == 0:
            stream.wait_event(copied[b_])       # buffer b_'s copy from step k - 2 is done
        ctx.consensus_mean(outs[b_].data_ptr(), with_mk=False, stream=stream)
        if rank == 0:                           # x_bar is the same on every rank: rank 0 returns it
            ready.record(stream)
            copy_stream.wait_event(ready)
            with torch.cuda.stream(copy_stream):
                hosts[b_].copy_(outs[b_], non_blocking=True)
            copied[b_].record(copy_stream)
    torch.cuda.synchronize()
    te = maxr(time.perf_counter() - te0)
    pairs_e = sumr(ctx.stats()["local_pair_events"] - st_e["local_pair_events"])
    n_local = len(ctx.local_workers())
    cnts = ctx.update_counts()
    ctx.destroy()

    extras = {}
    if not a.no_extras:
        # same workload without the straggler
        c2 = make_ctx(None)
        ms2, s20, s21, _, _, _ = timed(c2, max(3, a.steps // 2), 2)
        extras["no_straggler"] = {
            "gossip_steps_per_s": sumr(s21["local_pair_events"] - s20["local_pair_events"]) / (ms2 / 1e3),
            "updates_per_s": sumr(s21["local_events"] - s20["local_events"]) / (ms2 / 1e3)}
        # synchronous baselines (Table 4): AllReduce-SGD (NCCL all-reduce) and
        # D-PSGD (neighbour averaging, NCCL halo exchange), with and without the straggler
        ar, dp = {}, {}
        for tag, stv in (("straggler", strag), ("no_straggler", None)):
            c3 = make_ctx(stv)
            R = max(4, U // n)
            for kind, out in (("ar", ar), ("dp", dp)):
                run = c3.allreduce_sgd if kind == "ar" else c3.dpsgd
                if kind == "ar":
                    c3.allreduce_reset()
                else:
                    c3.dpsgd_reset()
                run(2, stream)
                torch.cuda.synchronize()
                barrier()
                ta, tb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                ta.record(stream)
                run(R, stream)
                tb.record(stream)
                torch.cuda.synchronize()
                msa = maxr(ta.elapsed_time(tb))
                out[tag] = {"updates_per_s": R * n / (msa / 1e3), "samples_per_s": R * n * M_BATCH / (msa / 1e3),
                            "rounds_per_s": R / (msa / 1e3)}
                barrier()
            c3.destroy()
            barrier()
        extras["allreduce_sgd_baseline"] = ar
        extras["dpsgd_baseline"] = dp
        extras["adpsgd_vs_allreduce_updates_ratio_straggler"] = upd_s / ar["straggler"]["updates_per_s"]
        extras["adpsgd_vs_dpsgd_updates_ratio_straggler"] = upd_s / dp["straggler"]["updates_per_s"]
        # config 5 (BASELINE configs[4]): 16 workers per GPU, heterogeneous stragglers
        # s_w = 10^U[0,1] plus worker 0 at 10x, AD-PSGD vs the NCCL AllReduce-SGD baseline
        n5 = 128 if 128 // world <= 128 and 128 % world == 0 else 16 * world   # BASELINE configs[4]: n = 128
        e5, r5 = synth.ring(n5)
        st5 = synth.stragglers(n5, seed=99, slow_worker=0, slow=10.0, hetero=True)

        def config5(tc_ns, U5, R5):
            """AD-PSGD vs AllReduce-SGD updates/s at n5 workers, heterogeneous stragglers"""
            c5 = make_ctx(st5, n5, e5, r5, compute_ns=tc_ns)
            c5.run(U5, stream)
            torch.cuda.synchronize()
            c5.sync()
            barrier()
            s50 = c5.stats()
            ta, tb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ta.record(stream)
            for _ in range(3):
                c5.run(U5, stream)
            tb.record(stream)
            torch.cuda.synchronize()
            c5.sync()
            barrier()
            sec5 = maxr(ta.elapsed_time(tb)) / 1e3
            s51 = c5.stats()
            c5.allreduce_reset()
            c5.allreduce_sgd(2, stream)
            torch.cuda.synchronize()
            barrier()
            ta.record(stream)
            c5.allreduce_sgd(R5, stream)
            tb.record(stream)
            torch.cuda.synchronize()
            sec5ar = maxr(ta.elapsed_time(tb)) / 1e3
            c5.destroy()
            barrier()
            up5 = sumr(s51["local_events"] - s50["local_events"]) / sec5
            return {"adpsgd_updates_per_s": up5,
                    "adpsgd_gossip_steps_per_s": sumr(s51["local_pair_events"] - s50["local_pair_events"]) / sec5,
                    "allreduce_updates_per_s": R5 * n5 / sec5ar,
                    "adpsgd_vs_allreduce_updates_ratio": up5 / (R5 * n5 / sec5ar)}

        extras["config5"] = dict(config5(cns, 8 * n5, 8), workload=(
            f"n={n5} ({n5 // world}/GPU) ring, d={d}, s_w = 10^U[0,1] + worker 0 x10, t_c={a.compute_us}us"))
        # the same at t_c = 1 ms: the workers' compute (not HBM) sets the pace, as in the paper's
        # GPU clusters -- AllReduce-SGD then waits for the slowest worker every round
        extras["config5_tc_1ms"] = dict(config5(1_000_000, 2 * n5, 2), workload=(
            f"n={n5} ({n5 // world}/GPU) ring, d={d}, s_w = 10^U[0,1] + worker 0 x10, t_c=1ms"))
        def three_way(c4, Rb):
            """updates/s of AD-PSGD (free-running), AllReduce-SGD and D-PSGD on one context"""
            c4.run(U, stream)
            torch.cuda.synchronize()
            c4.sync()
            barrier()
            s0 = c4.stats()
            ta, tb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ta.record(stream)
            for _ in range(3):
                c4.run(U, stream)
            tb.record(stream)
            torch.cuda.synchronize()
            c4.sync()
            barrier()
            sec = maxr(ta.elapsed_time(tb)) / 1e3
            row = {"adpsgd": sumr(c4.stats()["local_events"] - s0["local_events"]) / sec}
            for kind in ("allreduce", "dpsgd"):
                run = c4.allreduce_sgd if kind == "allreduce" else c4.dpsgd
                (c4.allreduce_reset if kind == "allreduce" else c4.dpsgd_reset)()
                run(1, stream)
                torch.cuda.synchronize()
                barrier()
                ta.record(stream)
                run(Rb, stream)
                tb.record(stream)
                torch.cuda.synchronize()
                row[kind] = Rb * n / (maxr(ta.elapsed_time(tb)) / 1e3)
                barrier()
            c4.destroy()
            barrier()
            return row

        # Table 4's shape: one worker slowed 1x / 2x / 10x / 100x; updates/s of
        # AD-PSGD vs the two synchronous baselines (same emulated compute t_c per gradient)
        t4 = {}
        for slow in (1.0, 2.0, 10.0, 100.0):
            t4[f"x{slow:g}"] = three_way(make_ctx(synth.stragglers(n, slow_worker=0, slow=slow)),
                                         4 if slow < 50 else 2)
        extras["table4_updates_per_s"] = t4
        # emulated t_c sweep: 0.1 / 1 / 10 ms per gradient spans the paper's
        # communication-intensive and computation-intensive regimes, worker 0 slowed 10x
        tcs = {}
        for tc_us, rb in ((100.0, 4), (1000.0, 3), (10000.0, 2)):
            tcs[f"t_c_{tc_us / 1000:g}ms"] = three_way(make_ctx(strag, compute_ns=int(tc_us * 1000)), rb)
        tcs["workload"] = "config 4 workload, worker 0 x10; updates/s of AD-PSGD / AllReduce-SGD / D-PSGD"
        extras["tc_sweep_updates_per_s"] = tcs
        # heterogeneous communication (Fig. loss-link; reading R21): worker 1's
        # link 10x slower, nominal model transfer 4d / 900 GB/s; no compute straggler
        link_ns = int(4 * d / 900e9 * 1e9)
        lk = {}
        for L in (1.0, 10.0):
            lv = np.ones(n, np.float32)
            lv[1 % n] = L
            cl = P.Context(e, n, d, role=r, rank=rank, world_size=world, device=local, placement=a.placement,
                           model=P.MODEL_QUADRATIC, gamma=GAMMA, batch_M=M_BATCH, quad_keys=(dk, nk),
                           quad_noise_s=s, straggler=synth.stragglers(n, slow_worker=None), compute_ns=cns,
                           seed=1234, log_capacity=1 << 16,
                           engine_ctas_per_sm=a.ctas_per_sm, link_slow=lv, link_ns=link_ns)
            lk[f"link_x{L:g}"] = three_way(cl, 4)
        lk["workload"] = f"config 4, no compute straggler, worker 1 link slowed, link_ns = {link_ns}"
        extras["slow_link_updates_per_s"] = lk
        # App. A wait-free runtime (reading R20) on the bench workload:
        # gradients computed into a buffer, flushed before averaging; actives
        # average continuously in between (no-gradient events)
        wf = {}
        for mode in (1, 2):
            cw = make_ctx(strag, wait_free=mode)
            cw.run(U, stream)
            torch.cuda.synchronize()
            cw.sync()
            barrier()
            s0, u0 = cw.stats(), sum(cw.update_counts().values())
            ta, tb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ta.record(stream)
            for _ in range(3):
                cw.run(U, stream)
            tb.record(stream)
            torch.cuda.synchronize()
            cw.sync()
            barrier()
            secw = maxr(ta.elapsed_time(tb)) / 1e3
            s1, u1 = cw.stats(), sum(cw.update_counts().values())
            wf["compensated" if mode == 2 else "plain"] = {
                "updates_per_s": sumr(u1 - u0) / secw,
                "gossip_steps_per_s": sumr(s1["local_pair_events"] - s0["local_pair_events"]) / secw,
                "events_per_s": sumr(s1["local_events"] - s0["local_events"]) / secw}
            if rank == 0:
                # staleness of the flushed gradients, tau = k - t_read, from the event log
                lg = cw.read_log(max(0, cw.ticket() - (1 << 15)))
                flushed = lg["tau"][(lg["flags"] & 1) == 0]
                if len(flushed):
                    hist = np.bincount(flushed)
                    wf["compensated" if mode == 2 else "plain"]["staleness_histogram"] = {
                        "tau_counts": hist.tolist()[:64], "mean_tau": float(flushed.mean()),
                        "max_tau": int(flushed.max()), "events": int(len(flushed))}
            cw.destroy()
            barrier()
        wf["workload"] = "config 4 workload and straggler, adpsgd_run with wait_free = 1 / 2"
        extras["wait_free_appA"] = wf
        if world > 1:
            # NVLink stress: pure gossip, every pair event crosses GPUs.  World >= 4: the xor
            # placement also spreads the actives (the GPUs that compute events) evenly; at
            # world 2 no all-cross placement can (interleave: all actives on GPU 0)
            # 32 workers per GPU (config 5's count at 4 GPUs) keep enough disjoint pairs in flight
            ns = 32 * world
            es, rs = synth.ring(ns)
            xor = world >= 4 and (world & (world - 1)) == 0
            cn = P.Context(es, ns, d, role=rs, rank=rank, world_size=world, device=local,
                           placement=2 if xor else 1, worker_rank=synth.placement_xor(ns, world) if xor else None,
                           log_capacity=1 << 16)
            cn.run(2 * ns, stream)
            torch.cuda.synchronize()
            cn.sync()
            barrier()
            s0 = cn.stats()
            ta, tb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            nvs0 = nvl.read()
            ta.record(stream)
            for _ in range(3):
                cn.run(8 * ns, stream)
            tb.record(stream)
            torch.cuda.synchronize()
            nvs1 = nvl.read()
            cn.sync()
            barrier()
            secn = maxr(ta.elapsed_time(tb)) / 1e3
            nvl_stress = nvl_report(NvlCounters.delta(nvs0, nvs1), secn)
            s1 = cn.stats()
            nvb = sumr(s1["local_nvlink_bytes"] - s0["local_nvlink_bytes"])
            npair = sumr(s1["local_pair_events"] - s0["local_pair_events"])
            cn.destroy()
            barrier()
            extras["nvlink_stress"] = {
                "workload": f"pure gossip, free-running, n={ns} ring, {'xor' if xor else 'interleave'} placement "
                            f"(every pair crosses GPUs{'' if xor else '; all actives on even GPUs'}), d={d}",
                "gossip_steps_per_s": npair / secn,
                "per_gpu_per_direction_gbs": nvb / secn / world / 1e9,
                "frac_of_900": nvb / secn / world / 900e9,
                "frac_of_measured_peer_copy_770": nvb / secn / world / 770e9,
                "nvml_counters": nvl_stress}
        if world > 1 and world % 2 == 0:
            # super-learners (reading R22): R = 2 GPUs per super-learner (NCCL all-reduce of
            # their gradients), S = world / 2 super-learners gossiping over NVLink; one learner per GPU
            R, S = 2, world // 2
            es, rs, wrs, _, _ = synth.super_ring(S, R)
            csl = P.Context(es, world, d, role=rs, rank=rank, world_size=world, device=local, placement=2,
                            worker_rank=wrs, model=P.MODEL_QUADRATIC, gamma=GAMMA, batch_M=M_BATCH,
                            quad_keys=(dk, nk), quad_noise_s=s, seed=1234, super_R=R, log_capacity=1 << 16)
            csl.super_run(4, stream)
            torch.cuda.synchronize()
            csl.sync()
            barrier()
            ta, tb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            steps_sl = 20
            ta.record(stream)
            csl.super_run(steps_sl, stream)
            tb.record(stream)
            torch.cuda.synchronize()
            csl.sync()
            barrier()
            secs = maxr(ta.elapsed_time(tb)) / 1e3
            csl.destroy()
            barrier()
            extras["super_learner"] = {
                "workload": f"S={S} super-learners x R={R} GPUs (one learner each), ring of super-learners, d={d}",
                "super_events_per_s": S * steps_sl / secs,
                "learner_gradients_per_s": S * R * steps_sl / secs,
                "samples_per_s": S * R * steps_sl * M_BATCH / secs}
        if world > 1:
            # config 3 as stated (n workers, one per B200): the tcgen05 MLP 3072 -> 512 -> 10, M = 128,
            # free-running through the host-driven per-GPU loop (super-learners with R = 1, R22)
            I, H, O_, Mm = 3072, 512, 10, 128
            Xd, yd = synth.mlp_data(S=8192, n_in=I, n_out=O_, s=0.02, seed=3)
            w0 = synth.mlp_init(I, H, O_, seed=4)
            e3, r3, wr3, _, _ = synth.super_ring(world, 1)
            c3m = P.Context(e3, world, w0.size, role=r3, rank=rank, world_size=world, device=local, placement=2,
                            worker_rank=wr3, model=P.MODEL_MLP, gamma=0.002, batch_M=Mm, data_A=Xd, data_y=yd,
                            mlp_dims=(I, H, O_), x0=w0, seed=99, super_R=1, log_capacity=1 << 16)
            c3m.super_run(5, stream)
            torch.cuda.synchronize()
            c3m.sync()
            barrier()
            ta, tb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            steps3 = 40
            ta.record(stream)
            c3m.super_run(steps3, stream)
            tb.record(stream)
            torch.cuda.synchronize()
            c3m.sync()
            barrier()
            sec3 = maxr(ta.elapsed_time(tb)) / 1e3
            c3m.destroy()
            barrier()
            extras["mlp_config3_one_per_gpu"] = {
                "workload": f"config3: MLP {I}->{H}->{O_}, M={Mm}, n={world} workers one per GPU on a ring, "
                            "free-running host-driven loop (super-learners with R=1), device Philox batches",
                "updates_per_s": world * steps3 / sec3, "samples_per_s": world * steps3 * Mm / sec3}
        if world == 1:
            sys.path.insert(0, os.path.join(ROOT, "tools"))
            extras["config1_lsq"] = config1_leg(P, synth, torch)
            extras["config2_gossip"] = config2_leg(P, synth, torch)
            extras["mlp_config3"] = mlp_leg(P, synth, torch)
            # config 3 free-running: 8 workers as in-process ranks on this GPU, each its own
            # host-driven AD-PSGD loop (the multi-rank protocol with local pointers)
            import mlp_free_running_1gpu
            extras["mlp_config3_free_running_1gpu"] = mlp_free_running_1gpu.run(8)
            import gemm_sweep
            extras["mlp_gemm_sweep"] = gemm_sweep.sweep(reps=10)

    cpu = None
    if rank == 0 and world == 1 and not a.no_extras:
        pairs_c, dt_c = oracle_sample(n, d, a.cpu_events)
        pairs_o, dt_o = oracle_sample(n, d, a.cpu_events, omp=True)
        hi = host_info()
        cpu = {"value": pairs_c / dt_c, "unit": "gossip-steps/s", "cores": 1, "kind": "oracle",
               "sample": f"{a.cpu_events} iid events (ring n={n}, d={d}) of the oracle's Alg. 1 replay; replay "
                         f"core (the fixed per-call copy of the n x d state timed with an empty schedule and "
                         f"subtracted)", "host": hi,
               "openmp_all_cores": {"value": pairs_o / dt_o, "unit": "gossip-steps/s", "cores": hi["nproc"],
                                    "kind": "oracle built with -fopenmp (per-coordinate loops; bit-identical, "
                                            "tests/test_oracle.py)"}}

    traffic_bytes, traffic_src = traffic_per_launch(loc_bytes / a.steps)
    nvl_main_rep = nvl_report(nvl_main, sec) if world > 1 else {"available": False, "note": "one GPU"}
    line = {
        "metric": "gossip-steps/s", "value": gossip_s, "unit": "gossip-steps/s", "n_gpus": world,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms / a.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"config4: quadratic d={d} fp32, n={n} workers ({a.workers_per_gpu}/GPU) on a "
                               f"bipartite ring, M={M_BATCH}, worker 0 x{a.straggler}, t_c={a.compute_us}us; "
                               f"step = {U} committed updates + consensus mean",
                   "global_batch": U * M_BATCH, "parallelism": f"gossip over {world} GPU(s), "
                   f"{'block' if a.placement == 0 else 'interleave'} placement",
                   "l2": "inputs larger than L2 (n x 102.4 MB models)"},
        "updates_per_s": upd_s, "samples_per_s": upd_s * M_BATCH,
        # every byte that crosses NVLink leaves one GPU: per-GPU egress = total / world
        "nvlink": {"algorithmic_bytes_per_s": nvl_bytes / sec, "per_gpu_per_direction_gbs":
                   nvl_bytes / sec / max(world, 1) / 1e9, "frac_of_900": nvl_bytes / sec / max(world, 1) / 900e9,
                   "frac_of_measured_peer_copy_770": nvl_bytes / sec / max(world, 1) / 770e9,
                   "note": "this workload's block placement: one ring edge per GPU boundary crosses NVLink; "
                           "the all-cross figure is under all_cross (extras.nvlink_stress)",
                   "nvml_counters": nvl_main_rep},
        "roofline": {"kernel": "k_engine", "bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                     "frac": achieved / hbm_peak, "traffic": traffic_bytes, "traffic_source": traffic_src,
                     "per_launch_algorithmic_bytes": loc_bytes / a.steps, "avg_launch_ms": eng_ms,
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs (burst copy)"},
        "clocks": clocks,
        "e2e": {"value": pairs_e / te, "unit": "gossip-steps/s",
                "h2d_bytes_per_step": 136 * n_local * world, "d2h_bytes_per_step": 4 * d,
                "note": "public API (Context.run + consensus_mean on every rank), x_bar of every step copied "
                        "by rank 0 to pinned host memory on a copy stream while the next step runs (double-"
                        "buffered; every copy inside the timed region; x_bar is identical on all ranks), host "
                        "wall clock, max over ranks",
                "synchronous": {"value": pairs_sync / te_sync, "d2h_bytes_per_step": (16 + 4 * d) * world,
                                "note": "M_k read back and x_bar copied before the next step starts"}},
        "gpu_launches": launches,
        "update_counts_rank0": cnts,
    }
    line.update(extras)
    if "wait_free_appA" in extras:
        # the App. A runtime (real gradient buffer, real staleness tau = k - t_read) beside the
        # Alg. 1 loop's tau = 0 fused figure above
        line["realistic_staleness"] = {
            "wait_free_updates_per_s": extras["wait_free_appA"]["plain"]["updates_per_s"],
            "wait_free_compensated_updates_per_s": extras["wait_free_appA"]["compensated"]["updates_per_s"],
            "alg1_fused_updates_per_s": upd_s,
            "note": "App. A loop (P:1235-1314, reading R20): gradients computed at a pulled model into a "
                    "buffer and flushed later (tau > 0 logged); the headline runs Alg. 1 with tau = 0"}
    if "nvlink_stress" in extras:           # the fused kernel's NVLink fraction when every pair crosses GPUs
        ns = extras["nvlink_stress"]
        line["nvlink"]["all_cross"] = {"per_gpu_per_direction_gbs": ns["per_gpu_per_direction_gbs"],
                                       "frac_of_900": ns["frac_of_900"], "workload": ns["workload"],
                                       "nvml_counters": ns["nvml_counters"]}
    if cpu:
        line["cpu_baseline"] = cpu
    if rank == 0:
        print(json.dumps(line))
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
