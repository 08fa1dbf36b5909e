"""B200-native AD-PSGD hot path (arXiv 1710.06952): thin Python binding of the
C ABI in include/adpsgd.h, implemented by libadpsgd.so (CUDA, sm_100a).

This module only marshals arguments.  Every step of the path runs in the
library's kernels; there is no CPU or PyTorch fallback: if libadpsgd.so is
missing or a call fails, an exception is raised.  PyTorch is used only for
process groups (peer-handle exchange) and, optionally, streams.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ADPSGD_LIB", os.path.join(_HERE, "libadpsgd.so"))   # override: A/B builds
_lib = None

OK = 0
STATUS = {0: "OK", 1: "E_INVALID", 2: "E_NOT_BIPARTITE", 3: "E_DISCONNECTED", 4: "E_NOT_NEIGHBOURS",
          5: "E_STALENESS", 6: "E_DIVERGED", 7: "E_TIMEOUT", 8: "E_CUDA", 9: "E_NCCL", 10: "E_OOM",
          11: "E_STATE", 12: "E_UNSUPPORTED"}
EV_FLUSH_FIRST, EV_COMPENSATE = 2, 4   # App. A event flags (include/adpsgd.h, reading R20)
MODEL_NONE, MODEL_EXTERNAL, MODEL_QUADRATIC, MODEL_LSQ, MODEL_LOGREG, MODEL_MLP = range(6)
EV_NO_GRAD = 1
REPLAY_HOST, REPLAY_ENGINE = 1, 2

EXPORTED = ["adpsgd_abi_version", "adpsgd_last_error", "adpsgd_init", "adpsgd_destroy",
            "adpsgd_peer_info_size", "adpsgd_export_peer_info", "adpsgd_import_peer_info",
            "adpsgd_nccl_unique_id", "adpsgd_connect", "adpsgd_gossip", "adpsgd_step", "adpsgd_replay",
            "adpsgd_run", "adpsgd_consensus_mean", "adpsgd_allreduce_sgd", "adpsgd_allreduce_read_model",
            "adpsgd_allreduce_reset", "adpsgd_sync", "adpsgd_read_model", "adpsgd_write_model",
            "adpsgd_model_device_ptr", "adpsgd_worker_rank", "adpsgd_get_ticket", "adpsgd_read_log",
            "adpsgd_read_update_counts", "adpsgd_get_stats", "adpsgd_reset_stats", "adpsgd_launch_count",
            "adpsgd_gemm_tf32x3", "adpsgd_plan_placement", "adpsgd_plan_replay", "adpsgd_dpsgd",
            "adpsgd_dpsgd_reset", "adpsgd_dpsgd_read_model", "adpsgd_gemm_tf32x3_bench", "adpsgd_super_run"]


class AdpsgdError(RuntimeError):
    def __init__(self, code, where, msg):
        super().__init__(f"{where}: {STATUS.get(code, code)}: {msg}")
        self.code = code


class Graph(C.Structure):
    _fields_ = [("n", C.c_int32), ("n_edges", C.c_int32), ("edges", C.c_void_p), ("role", C.c_void_p)]


class Config(C.Structure):
    _fields_ = [("rank", C.c_int32), ("world_size", C.c_int32), ("device", C.c_int32),
                ("placement", C.c_int32), ("worker_rank", C.c_void_p),
                ("gamma", C.c_float), ("batch_M", C.c_int32), ("staleness_cap_T", C.c_int32),
                ("seed", C.c_uint64), ("model", C.c_int32),
                ("quad_data_key", C.c_uint32), ("quad_noise_key", C.c_uint32), ("quad_noise_s", C.c_float),
                ("n_samples", C.c_int32), ("data_A", C.c_void_p), ("data_b", C.c_void_p),
                ("data_y", C.c_void_p), ("mlp_in", C.c_int32), ("mlp_hid", C.c_int32),
                ("mlp_out", C.c_int32), ("x0", C.c_void_p), ("x0_per_worker", C.c_void_p),
                ("straggler", C.c_void_p), ("compute_ns", C.c_int64), ("engine_ctas_per_sm", C.c_int32),
                ("engine_variant", C.c_int32), ("log_capacity", C.c_int64),
                ("wait_free", C.c_int32), ("reserved0", C.c_int32),
                ("link_slow", C.c_void_p), ("link_ns", C.c_int64),
                ("engine_no_fuse", C.c_int32), ("reserved1", C.c_int32), ("engine_fuse_wait_ns", C.c_int64),
                ("super_R", C.c_int32), ("engine_coop", C.c_int32),
                ("comm_local", C.c_int32), ("engine_grid", C.c_int32)]


class Event(C.Structure):
    _fields_ = [("i", C.c_int32), ("j", C.c_int32), ("tau", C.c_int32), ("flags", C.c_uint32)]


LOG_DTYPE = np.dtype([("k", np.int64), ("i", np.int32), ("j", np.int32), ("tau", np.int32),
                      ("flags", np.uint32), ("t0", np.uint64), ("t1", np.uint64)])


class Stats(C.Structure):
    _fields_ = [("ticket", C.c_int64), ("local_events", C.c_int64), ("local_pair_events", C.c_int64),
                ("local_cross_events", C.c_int64), ("local_bytes", C.c_double),
                ("local_nvlink_bytes", C.c_double), ("engine_busy_ns", C.c_double),
                ("engine_busy_cross_ns", C.c_double)]


def lib():
    """Load libadpsgd.so (raises if it was not built: no fallback path)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built: run `python paper_1710_06952_b200/build.py` "
                              "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        P, I32, I64 = C.c_void_p, C.c_int32, C.c_int64
        sig = {
            "adpsgd_abi_version": ([], I32), "adpsgd_last_error": ([], C.c_char_p),
            "adpsgd_init": ([P, I32, I64, P, P], I32), "adpsgd_destroy": ([P], I32),
            "adpsgd_peer_info_size": ([P], I32), "adpsgd_export_peer_info": ([P, P, I64, P], I32),
            "adpsgd_import_peer_info": ([P, I32, P, I64], I32), "adpsgd_nccl_unique_id": ([P], I32),
            "adpsgd_connect": ([P, P], I32), "adpsgd_gossip": ([P, I32, I32, P], I32),
            "adpsgd_step": ([P, I32, P, P, P], I32), "adpsgd_replay": ([P, P, I64, P, C.c_uint32, P], I32),
            "adpsgd_run": ([P, I64, P], I32), "adpsgd_consensus_mean": ([P, P, P, P], I32),
            "adpsgd_allreduce_sgd": ([P, I64, P], I32), "adpsgd_allreduce_read_model": ([P, P], I32),
            "adpsgd_allreduce_reset": ([P, P], I32), "adpsgd_sync": ([P], I32),
            "adpsgd_read_model": ([P, I32, P], I32), "adpsgd_write_model": ([P, I32, P], I32),
            "adpsgd_model_device_ptr": ([P, I32, P], I32), "adpsgd_worker_rank": ([P, I32, P], I32),
            "adpsgd_get_ticket": ([P, P], I32), "adpsgd_read_log": ([P, I64, P, I64, P], I32),
            "adpsgd_read_update_counts": ([P, P], I32), "adpsgd_get_stats": ([P, P], I32),
            "adpsgd_reset_stats": ([P], I32), "adpsgd_launch_count": ([P, P], I32),
            "adpsgd_gemm_tf32x3": ([P, P, P, I32, I32, I32, I32], I32),
            "adpsgd_plan_placement": ([I32, I32, I32, P, P, P], I32),
            "adpsgd_plan_replay": ([I32, P, I32, P, I64, I64, I32, I32, P, P, I64, P], I32),
            "adpsgd_dpsgd": ([P, I64, P], I32), "adpsgd_dpsgd_reset": ([P, P], I32),
            "adpsgd_dpsgd_read_model": ([P, I32, P], I32),
            "adpsgd_gemm_tf32x3_bench": ([I32, I32, I32, I32, I32, I32, P], I32),
            "adpsgd_super_run": ([P, I64, P], I32),
        }
        for name, (args, res) in sig.items():
            f = getattr(L, name)
            f.argtypes, f.restype = args, res
        _lib = L
    return _lib


def _chk(st, where):
    if st != OK:
        raise AdpsgdError(st, where, lib().adpsgd_last_error().decode(errors="replace"))


def _arr(a, dt):
    return None if a is None else np.ascontiguousarray(np.asarray(a, dt))


def _ptr(a):
    return None if a is None else a.ctypes.data


def _stream(s):
    """Accept None, an int handle or a torch.cuda.Stream."""
    if s is None:
        return None
    return C.c_void_p(int(getattr(s, "cuda_stream", s)))


def plan_placement(n, world_size, placement=0, worker_rank=None):
    """Host-only: (worker_rank[n], local_index[n]) exactly as adpsgd_init places workers."""
    wr_in = _arr(worker_rank, np.int32)
    wr, wl = np.zeros(n, np.int32), np.zeros(n, np.int32)
    _chk(lib().adpsgd_plan_placement(n, world_size, placement, _ptr(wr_in), _ptr(wr), _ptr(wl)), "plan_placement")
    return wr, wl


def plan_replay(worker_rank, rank, events, k0=0, epochs=None, T=0, stale_reads=False):
    """Host-only: this rank's engine-replay plan, rows (k, i, j, flags, e_i, e_j,
    kind, row) -- kind 2 rows are stale reads (see adpsgd.h); returns (plan,
    advanced epoch mirror)."""
    wr = _arr(worker_rank, np.int32)
    n = wr.size
    ev = _arr(np.asarray(events).reshape(-1, 4), np.int32)
    ep = np.zeros(n, np.uint32) if epochs is None else np.array(epochs, np.uint32)
    m = C.c_int64()
    _chk(lib().adpsgd_plan_replay(n, _ptr(wr), rank, _ptr(ev), ev.shape[0], k0, T, int(stale_reads), _ptr(ep), None,
                                  0, C.byref(m)), "plan_replay")
    out = np.zeros((m.value, 8), np.int64)
    ep2 = np.zeros(n, np.uint32) if epochs is None else np.array(epochs, np.uint32)
    _chk(lib().adpsgd_plan_replay(n, _ptr(wr), rank, _ptr(ev), ev.shape[0], k0, T, int(stale_reads), _ptr(ep2),
                                  _ptr(out), m.value, C.byref(m)), "plan_replay")
    return out, ep2


def exchange_peer_blobs(mine: bytes, rank: int, world: int, make_nccl_id=None, pg=None):
    """The N > 1 wiring protocol: all-gather every rank's CUDA-IPC blob and
    broadcast rank 0's NCCL id (torch.distributed, any backend)."""
    import torch.distributed as dist
    allb = [None] * world
    dist.all_gather_object(allb, mine, group=pg)
    obj = [make_nccl_id() if (rank == 0 and make_nccl_id) else None]
    dist.broadcast_object_list(obj, src=0, group=pg)
    return allb, obj[0]


class ThreadGroup:
    """In-process rank group for comm_local contexts (include/adpsgd.h): the
    ranks are host threads of this process; this object carries the wiring
    exchange (peer blobs, the group token) between them, the role
    torch.distributed plays for one-process-per-GPU ranks."""

    def __init__(self, world):
        import threading
        self.world = int(world)
        self._bar = threading.Barrier(self.world)
        self._buf = [None] * self.world

    def barrier(self, timeout=600):
        self._bar.wait(timeout)

    def abort(self):
        """Break the barrier: ranks waiting in it raise instead of hanging."""
        self._bar.abort()

    def all_gather_object(self, out, obj, rank):
        self._buf[rank] = obj
        self.barrier()
        out[:] = list(self._buf)
        self.barrier()

    def broadcast_object(self, obj, src, rank):
        if rank == src:
            self._buf[src] = obj
        self.barrier()
        v = self._buf[src]
        self.barrier()
        return v


def run_ranks(world, fn, timeout=1800, group=None):
    """Run fn(rank) on `world` host threads (one per in-process rank); re-raise
    the first exception (a failing rank aborts `group`'s barrier so the others
    do not wait for it).  ctypes releases the GIL inside every library call."""
    import threading
    res, errs = [None] * world, [None] * world

    def body(r):
        try:
            res[r] = fn(r)
        except BaseException as ex:  # surfaced below
            errs[r] = ex
            if group is not None:
                group.abort()

    ts = [threading.Thread(target=body, args=(r,), daemon=True) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout)
    import threading as _th
    for r, ex in enumerate(errs):       # the root cause first, not a broken barrier
        if ex is not None and not isinstance(ex, _th.BrokenBarrierError):
            raise RuntimeError(f"in-process rank {r} failed: {ex!r}") from ex
    for r, ex in enumerate(errs):
        if ex is not None:
            raise RuntimeError(f"in-process rank {r} failed: {ex!r}") from ex
    if any(t.is_alive() for t in ts):
        raise TimeoutError("in-process ranks did not finish")
    return res


def gemm_tf32x3(A_ptr, B_ptr, C_ptr, M, N, K, splits=1):
    """Diagnostics: C = A . B^T on tcgen05 (3xTF32), device pointers (see adpsgd.h)."""
    _chk(lib().adpsgd_gemm_tf32x3(C.c_void_p(A_ptr), C.c_void_p(B_ptr), C.c_void_p(C_ptr), M, N, K, splits),
         "gemm_tf32x3")


def gemm_tf32x3_bench(M, N, K, splits=1, bn=128, reps=20):
    """Diagnostics: mean device ms of the tcgen05 3xTF32 GEMM kernel at this shape."""
    ms = C.c_double()
    _chk(lib().adpsgd_gemm_tf32x3_bench(M, N, K, splits, bn, reps, C.byref(ms)), "gemm_tf32x3_bench")
    return ms.value


class Context:
    """One AD-PSGD context (one process, one GPU).  Method names follow the C ABI."""

    def __init__(self, edges, n, d, *, role=None, rank=0, world_size=1, device=0, placement=0,
                 worker_rank=None, gamma=0.0, batch_M=1, T=0, seed=0, model=MODEL_NONE,
                 quad_keys=(0, 0), quad_noise_s=0.0, data_A=None, data_b=None, data_y=None,
                 mlp_dims=(0, 0, 0), x0=None, x0_per_worker=None, straggler=None, compute_ns=0,
                 engine_ctas_per_sm=0, engine_variant=0, log_capacity=0, wait_free=0, link_slow=None, link_ns=0,
                 engine_fuse=True, engine_fuse_wait_ns=0, super_R=0, engine_coop=None, connect=True,
                 pg=None, group=None, engine_grid=0):
        self.n, self.d, self.rank, self.world = int(n), int(d), int(rank), int(world_size)
        e = _arr(np.asarray(edges).reshape(-1, 2), np.int32)
        r = _arr(role, np.int8)
        keep = [e, r]
        g = Graph(self.n, e.shape[0], _ptr(e), _ptr(r))
        cfg = Config()
        cfg.rank, cfg.world_size, cfg.device, cfg.placement = rank, world_size, device, placement
        wr = _arr(worker_rank, np.int32)
        keep.append(wr)
        cfg.worker_rank = _ptr(wr)
        cfg.gamma, cfg.batch_M, cfg.staleness_cap_T, cfg.seed, cfg.model = gamma, batch_M, T, seed, model
        cfg.quad_data_key, cfg.quad_noise_key = int(quad_keys[0]), int(quad_keys[1])
        cfg.quad_noise_s = quad_noise_s
        A, b, y = _arr(data_A, np.float32), _arr(data_b, np.float32), _arr(data_y, np.int32)
        keep += [A, b, y]
        cfg.n_samples = 0 if A is None else A.shape[0]
        cfg.data_A, cfg.data_b, cfg.data_y = _ptr(A), _ptr(b), _ptr(y)
        cfg.mlp_in, cfg.mlp_hid, cfg.mlp_out = mlp_dims
        x0a, x0w, st = _arr(x0, np.float32), _arr(x0_per_worker, np.float32), _arr(straggler, np.float32)
        keep += [x0a, x0w, st]
        cfg.x0, cfg.x0_per_worker, cfg.straggler = _ptr(x0a), _ptr(x0w), _ptr(st)
        cfg.compute_ns, cfg.engine_ctas_per_sm, cfg.engine_variant = int(compute_ns), engine_ctas_per_sm, engine_variant
        cfg.log_capacity = log_capacity
        cfg.wait_free = int(wait_free)
        ls = _arr(link_slow, np.float32)
        keep.append(ls)
        cfg.link_slow, cfg.link_ns = _ptr(ls), int(link_ns)
        cfg.engine_no_fuse = 0 if engine_fuse else 1
        cfg.engine_fuse_wait_ns = int(engine_fuse_wait_ns)
        cfg.super_R = int(super_R)
        cfg.engine_coop = 0 if engine_coop is None else (1 if engine_coop else -1)   # None = auto
        cfg.comm_local = 1 if group is not None else 0       # in-process ranks (ThreadGroup)
        cfg.engine_grid = int(engine_grid)
        self.group = group
        h = C.c_void_p()
        _chk(lib().adpsgd_init(C.byref(g), self.n, self.d, C.byref(cfg), C.byref(h)), "adpsgd_init")
        self._h = h
        if world_size > 1 and connect:
            if group is not None:
                self.connect_local(group)
            else:
                self.connect_distributed(pg)

    # ---------------------------------------------------------- lifecycle --
    def connect_distributed(self, pg=None):
        """Exchange CUDA IPC peer blobs and the NCCL id over torch.distributed."""
        import torch.distributed as dist
        sz = C.c_int64()
        _chk(lib().adpsgd_peer_info_size(C.byref(sz)), "peer_info_size")
        buf = (C.c_ubyte * sz.value)()
        n = C.c_int64()
        _chk(lib().adpsgd_export_peer_info(self._h, buf, sz.value, C.byref(n)), "export_peer_info")
        mine = bytes(buf[:n.value])

        def make_id():
            nid = (C.c_ubyte * 128)()
            _chk(lib().adpsgd_nccl_unique_id(nid), "nccl_unique_id")
            return bytes(nid)

        allb, nccl_id = exchange_peer_blobs(mine, self.rank, self.world, make_id, pg)
        for r, blob in enumerate(allb):
            if r != self.rank:
                _chk(lib().adpsgd_import_peer_info(self._h, r, blob, len(blob)), "import_peer_info")
        nid2 = (C.c_ubyte * 128).from_buffer_copy(nccl_id)
        _chk(lib().adpsgd_connect(self._h, nid2), "connect")
        dist.barrier(group=pg)

    def _export(self):
        sz = C.c_int64()
        _chk(lib().adpsgd_peer_info_size(C.byref(sz)), "peer_info_size")
        buf = (C.c_ubyte * sz.value)()
        n = C.c_int64()
        _chk(lib().adpsgd_export_peer_info(self._h, buf, sz.value, C.byref(n)), "export_peer_info")
        return bytes(buf[:n.value])

    def connect_local(self, group):
        """In-process ranks (comm_local): exchange raw-pointer peer blobs and a
        random group token through a ThreadGroup; call from this rank's thread."""
        allb = [None] * self.world
        group.all_gather_object(allb, self._export(), self.rank)
        for r, blob in enumerate(allb):
            if r != self.rank:
                _chk(lib().adpsgd_import_peer_info(self._h, r, blob, len(blob)), "import_peer_info")
        tok = group.broadcast_object(os.urandom(128) if self.rank == 0 else None, 0, self.rank)
        _chk(lib().adpsgd_connect(self._h, (C.c_ubyte * 128).from_buffer_copy(tok)), "connect")
        group.barrier()

    def destroy(self):
        if getattr(self, "_h", None):
            _chk(lib().adpsgd_destroy(self._h), "destroy")
            self._h = None

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass

    # ----------------------------------------------------------- hot path --
    def gossip(self, i, j, stream=None):
        _chk(lib().adpsgd_gossip(self._h, i, j, _stream(stream)), "gossip")

    def step(self, w, grad_ptr=None, stream=None):
        k = C.c_int64()
        _chk(lib().adpsgd_step(self._h, w, grad_ptr, _stream(stream), C.byref(k)), "step")
        return k.value

    def replay(self, events, batch_idx=None, flags=0, stream=None):
        ev = _arr(np.asarray(events).reshape(-1, 4), np.int32)
        bi = _arr(batch_idx, np.int32)
        _chk(lib().adpsgd_replay(self._h, _ptr(ev), ev.shape[0], _ptr(bi), flags, _stream(stream)), "replay")

    def run(self, n_updates, stream=None):
        _chk(lib().adpsgd_run(self._h, int(n_updates), _stream(stream)), "run")

    def super_run(self, n_steps, stream=None):
        """Super-learner loop (reading R22, R = super_R): collective over all ranks."""
        _chk(lib().adpsgd_super_run(self._h, int(n_steps), _stream(stream)), "super_run")

    def consensus_mean(self, out_ptr, with_mk=True, stream=None):
        mk = C.c_double()
        _chk(lib().adpsgd_consensus_mean(self._h, C.c_void_p(out_ptr), C.byref(mk) if with_mk else None,
                                         _stream(stream)), "consensus_mean")
        return mk.value if with_mk else None

    def allreduce_sgd(self, n_rounds, stream=None):
        _chk(lib().adpsgd_allreduce_sgd(self._h, int(n_rounds), _stream(stream)), "allreduce_sgd")

    def allreduce_reset(self, x=None):
        xa = _arr(x, np.float32)
        _chk(lib().adpsgd_allreduce_reset(self._h, _ptr(xa)), "allreduce_reset")

    def allreduce_read_model(self):
        out = np.zeros(self.d, np.float32)
        _chk(lib().adpsgd_allreduce_read_model(self._h, _ptr(out)), "allreduce_read_model")
        return out

    def dpsgd(self, n_rounds, stream=None):
        _chk(lib().adpsgd_dpsgd(self._h, int(n_rounds), _stream(stream)), "dpsgd")

    def dpsgd_reset(self, x0_per_worker=None):
        xa = _arr(x0_per_worker, np.float32)
        _chk(lib().adpsgd_dpsgd_reset(self._h, _ptr(xa)), "dpsgd_reset")

    def dpsgd_read_model(self, w):
        out = np.zeros(self.d, np.float32)
        _chk(lib().adpsgd_dpsgd_read_model(self._h, w, _ptr(out)), "dpsgd_read_model")
        return out

    # --------------------------------------------------------- state access --
    def sync(self):
        _chk(lib().adpsgd_sync(self._h), "sync")

    def read_model(self, w):
        out = np.zeros(self.d, np.float32)
        _chk(lib().adpsgd_read_model(self._h, w, _ptr(out)), "read_model")
        return out

    def write_model(self, w, x):
        xa = _arr(x, np.float32)
        _chk(lib().adpsgd_write_model(self._h, w, _ptr(xa)), "write_model")

    def model_ptr(self, w):
        p = C.c_void_p()
        _chk(lib().adpsgd_model_device_ptr(self._h, w, C.byref(p)), "model_device_ptr")
        return p.value

    def worker_rank(self, w):
        r = C.c_int32()
        _chk(lib().adpsgd_worker_rank(self._h, w, C.byref(r)), "worker_rank")
        return r.value

    def local_workers(self):
        return [w for w in range(self.n) if self.worker_rank(w) == self.rank]

    def ticket(self):
        k = C.c_int64()
        _chk(lib().adpsgd_get_ticket(self._h, C.byref(k)), "get_ticket")
        return k.value

    def read_log(self, k_from=0, cap=None):
        cap = self.ticket() - k_from if cap is None else cap
        out = np.zeros(max(cap, 0), LOG_DTYPE)
        n = C.c_int64()
        _chk(lib().adpsgd_read_log(self._h, k_from, _ptr(out), len(out), C.byref(n)), "read_log")
        return out[:n.value]

    def update_counts(self):
        loc = self.local_workers()
        out = np.zeros(max(1, len(loc)), np.int64)
        _chk(lib().adpsgd_read_update_counts(self._h, _ptr(out)), "read_update_counts")
        return dict(zip(loc, out[:len(loc)].tolist()))

    def stats(self):
        s = Stats()
        _chk(lib().adpsgd_get_stats(self._h, C.byref(s)), "get_stats")
        return {f: getattr(s, f) for f, _ in Stats._fields_}

    def reset_stats(self):
        _chk(lib().adpsgd_reset_stats(self._h), "reset_stats")

    def launch_count(self):
        n = C.c_int64()
        _chk(lib().adpsgd_launch_count(self._h, C.byref(n)), "launch_count")
        return n.value
