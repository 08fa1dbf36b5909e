"""ctypes wrapper of oracle/adpsgd_oracle.c -- TEST INFRASTRUCTURE ONLY.

The C library is compiled with gcc -O2 -ffp-contract=off -fno-fast-math so that
every fp32 operation is a single IEEE round-to-nearest-even op (reading R6).
Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may use it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "adpsgd_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

MODEL_NONE, MODEL_QUADRATIC, MODEL_LSQ, MODEL_LOGREG, MODEL_MLP = 0, 2, 3, 4, 5
EV_NO_GRAD, EV_FLUSH_FIRST, EV_COMPENSATE = 1, 2, 4     # App. A flags (reading R20)
STATUS = {0: "OK", 1: "INVALID", 2: "NOT_BIPARTITE", 3: "DISCONNECTED", 4: "NOT_NEIGHBOURS",
          5: "STALENESS", 6: "DIVERGED", 10: "OOM"}


class OracleError(RuntimeError):
    def __init__(self, code):
        super().__init__(f"oracle status {code} ({STATUS.get(code, '?')})")
        self.code = code


_LIB_OMP = os.path.join(_HERE, "liboracle_omp.so")


def build(force: bool = False, omp: bool = False) -> str:
    """Compile the oracle shared library (plain gcc, no GPU).  omp=True: the same
    source with -fopenmp (per-coordinate loops over all cores, bit-identical)."""
    out = _LIB_OMP if omp else _LIB
    if force or not os.path.exists(out) or os.path.getmtime(out) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math",
                               "-fPIC", "-shared", "-Wall"] + (["-fopenmp"] if omp else []) +
                              ["-o", out + ".tmp", _SRC, "-lm"])
        os.replace(out + ".tmp", out)
    return out


class Problem(C.Structure):
    _fields_ = [("kind", C.c_int32), ("M", C.c_int32), ("gamma", C.c_float),
                ("data_key", C.c_uint32), ("noise_key", C.c_uint32), ("noise_s", C.c_float),
                ("h_explicit", C.c_void_p), ("xstar_explicit", C.c_void_p),
                ("S", C.c_int32), ("A", C.c_void_p), ("b", C.c_void_p), ("y", C.c_void_p),
                ("n_in", C.c_int32), ("n_hid", C.c_int32), ("n_out", C.c_int32),
                ("batch_key", C.c_uint32 * 2)]


_lib_omp = None


def lib(omp: bool = False):
    """The serial oracle (default), or its OpenMP build (bench.py's all-cores CPU leg)."""
    global _lib, _lib_omp
    with _lock:
        if (_lib_omp if omp else _lib) is None:
            L = C.CDLL(build(omp=omp))
            P = C.c_void_p
            L.oracle_philox4x32_10.argtypes = [P, P, P]
            L.oracle_philox4x32_10.restype = None
            L.oracle_lowbias32.argtypes = [C.c_uint32]
            L.oracle_lowbias32.restype = C.c_uint32
            L.oracle_quad_noise_mix.argtypes = [C.c_uint32]
            L.oracle_quad_noise_mix.restype = C.c_uint32
            L.oracle_quad_event_key.argtypes = [C.c_uint32, C.c_uint64]
            L.oracle_quad_event_key.restype = C.c_uint32
            L.oracle_check_graph.argtypes = [C.c_int32, C.c_int32, P, P, P]
            L.oracle_gradient.argtypes = [C.POINTER(Problem), C.c_int64, P, C.c_uint64, P, P, P]
            L.oracle_full_loss.argtypes = [C.POINTER(Problem), C.c_int64, P]
            L.oracle_full_loss.restype = C.c_double
            L.oracle_replay.argtypes = [C.POINTER(Problem), C.c_int32, C.c_int64, P, C.c_int32, P, P,
                                        P, C.c_int64, P, C.c_int32, C.c_int32, C.c_uint64, P]
            L.oracle_consensus_mean.argtypes = [C.c_int32, C.c_int64, P, P, P, P]
            L.oracle_allreduce_update.argtypes = [C.c_int32, C.c_int64, C.c_float, P, P]
            L.oracle_mlp_dim.argtypes = [C.c_int32, C.c_int32, C.c_int32]
            L.oracle_mlp_dim.restype = C.c_int64
            L.oracle_read_key.argtypes = [C.c_uint64, C.c_int32]
            L.oracle_read_key.restype = C.c_uint64
            L.oracle_super_key.argtypes = [C.c_int32, C.c_int64, C.c_int32]
            L.oracle_super_key.restype = C.c_uint64
            L.oracle_super_gradient.argtypes = [C.POINTER(Problem), C.c_int64, P, C.c_int32, C.c_int64, C.c_int32, P]
            L.oracle_super_replay.argtypes = [C.POINTER(Problem), C.c_int32, C.c_int64, P, C.c_int32, P, P, P,
                                              C.c_int64, C.c_int32]
            if omp:
                _lib_omp = L
            else:
                _lib = L
    return _lib_omp if omp else _lib


def _p(a):
    return None if a is None else a.ctypes.data


def _check(st):
    if st != 0:
        raise OracleError(st)


# ----------------------------------------------------------------- helpers --
def philox(ctr, key):
    c = np.asarray(ctr, np.uint32).copy()
    k = np.asarray(key, np.uint32).copy()
    out = np.zeros(4, np.uint32)
    lib().oracle_philox4x32_10(_p(c), _p(k), _p(out))
    return out


def read_key(t_read: int, i: int) -> int:
    """Random-draw key of an App. A gradient read at X_{t_read} by worker i (R20)."""
    return int(lib().oracle_read_key(t_read, i))


def lowbias32(x: int) -> int:
    return int(lib().oracle_lowbias32(x & 0xFFFFFFFF))


def quad_noise_mix(x: int) -> int:
    """The synthetic quadratic's noise word u = mix(c ^ K_k) (DESIGN.md definition v3)."""
    return int(lib().oracle_quad_noise_mix(x & 0xFFFFFFFF))


def check_graph(n, edges, role=None):
    e = np.ascontiguousarray(np.asarray(edges, np.int32).reshape(-1, 2))
    r = None if role is None else np.ascontiguousarray(np.asarray(role, np.int8))
    out = np.zeros(max(n, 1), np.int8)
    st = lib().oracle_check_graph(n, e.shape[0], _p(e), _p(r), _p(out))
    return st, out


class OracleProblem:
    """Keeps the numpy arrays referenced by the C struct alive."""

    def __init__(self, kind=MODEL_NONE, M=1, gamma=0.0, data_key=0, noise_key=0, noise_s=0.0,
                 h=None, xstar=None, A=None, b=None, y=None, dims=(0, 0, 0), batch_key=(0, 0)):
        self._keep = []

        def keep(a, dt):
            if a is None:
                return None
            a = np.ascontiguousarray(np.asarray(a, dt))
            self._keep.append(a)
            return a.ctypes.data

        self.s = Problem()
        self.s.kind, self.s.M, self.s.gamma = kind, M, gamma
        self.s.data_key, self.s.noise_key, self.s.noise_s = data_key, noise_key, noise_s
        self.s.h_explicit = keep(h, np.float32)
        self.s.xstar_explicit = keep(xstar, np.float32)
        self.s.A = keep(A, np.float32)
        self.s.b = keep(b, np.float32)
        self.s.y = keep(y, np.int32)
        self.s.S = 0 if A is None else int(np.asarray(A).shape[0])
        self.s.n_in, self.s.n_hid, self.s.n_out = dims
        self.s.batch_key[0], self.s.batch_key[1] = batch_key

    @property
    def ref(self):
        return C.byref(self.s)


def gradient(prob: OracleProblem, xhat, k=0, idx=None):
    x = np.ascontiguousarray(np.asarray(xhat, np.float32))
    g = np.zeros_like(x)
    loss = C.c_double(0.0)
    ix = None if idx is None else np.ascontiguousarray(np.asarray(idx, np.int32))
    _check(lib().oracle_gradient(prob.ref, x.size, _p(x), k, _p(ix), _p(g), C.byref(loss)))
    return g


def full_loss(prob: OracleProblem, x) -> float:
    x = np.ascontiguousarray(np.asarray(x, np.float32))
    return float(lib().oracle_full_loss(prob.ref, x.size, _p(x)))


def replay(prob: OracleProblem, X, edges, role, events, batch_idx=None, T=0, clamp_tau=False,
           k0=0, mk_trace=False, omp=False):
    """Run Alg. 1 over an explicit event schedule; returns (X_K, mk or None).
    omp=True runs the OpenMP build (bit-identical; bench.py's all-cores leg)."""
    X = np.ascontiguousarray(np.array(X, np.float32, copy=True))
    n, d = X.shape
    e = np.ascontiguousarray(np.asarray(edges, np.int32).reshape(-1, 2))
    r = None if role is None else np.ascontiguousarray(np.asarray(role, np.int8))
    ev = np.ascontiguousarray(np.asarray(events, np.int32).reshape(-1, 4))
    bi = None if batch_idx is None else np.ascontiguousarray(np.asarray(batch_idx, np.int32))
    mk = np.zeros(ev.shape[0] + 1, np.float64) if mk_trace else None
    _check(lib(omp).oracle_replay(prob.ref, n, d, _p(X), e.shape[0], _p(e), _p(r), _p(ev), ev.shape[0],
                               _p(bi), T, int(clamp_tau), k0, _p(mk)))
    return X, mk


def consensus_mean(X, p=None):
    X = np.ascontiguousarray(np.asarray(X, np.float32))
    n, d = X.shape
    out = np.zeros(d, np.float32)
    mk = C.c_double(0.0)
    pp = None if p is None else np.ascontiguousarray(np.asarray(p, np.float64))
    _check(lib().oracle_consensus_mean(n, d, _p(X), _p(pp), _p(out), C.byref(mk)))
    return out, mk.value


def allreduce_update(x, grads, gamma):
    x = np.ascontiguousarray(np.array(x, np.float32, copy=True))
    G = np.ascontiguousarray(np.asarray(grads, np.float32))
    _check(lib().oracle_allreduce_update(G.shape[0], x.size, gamma, _p(G), _p(x)))
    return x


def mlp_dim(n_in, n_hid, n_out) -> int:
    return int(lib().oracle_mlp_dim(n_in, n_hid, n_out))


def dpsgd_round(prob: OracleProblem, X, edges, k_base=0):
    """One synchronous D-PSGD round (reading R19); returns the new X."""
    X = np.ascontiguousarray(np.array(X, np.float32, copy=True))
    e = np.ascontiguousarray(np.asarray(edges, np.int32).reshape(-1, 2))
    L = lib()
    L.oracle_dpsgd_round.argtypes = [C.POINTER(Problem), C.c_int32, C.c_int64, C.c_void_p, C.c_int32,
                                     C.c_void_p, C.c_uint64]
    _check(L.oracle_dpsgd_round(prob.ref, X.shape[0], X.shape[1], _p(X), e.shape[0], _p(e), k_base))
    return X


def super_gradient(prob: OracleProblem, x, s, c, R):
    """Super-learner gradient (reading R22): fp64 sum of R learners' quadratic gradients."""
    x = np.ascontiguousarray(np.asarray(x, np.float32))
    g = np.zeros_like(x)
    _check(lib().oracle_super_gradient(prob.ref, x.size, _p(x), s, c, R, _p(g)))
    return g


def super_replay(prob: OracleProblem, X, edges, role, events, R):
    """Replay super-learner events (i, j, 0, flags) over S = X.shape[0] super-learners."""
    X = np.ascontiguousarray(np.array(X, np.float32, copy=True))
    S, d = X.shape
    e = np.ascontiguousarray(np.asarray(edges, np.int32).reshape(-1, 2))
    r = None if role is None else np.ascontiguousarray(np.asarray(role, np.int8))
    ev = np.ascontiguousarray(np.asarray(events, np.int32).reshape(-1, 4))
    _check(lib().oracle_super_replay(prob.ref, S, d, _p(X), e.shape[0], _p(e), _p(r), _p(ev), ev.shape[0], R))
    return X


def super_key(s, c, r) -> int:
    return int(lib().oracle_super_key(s, c, r))
