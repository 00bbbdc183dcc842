"""ctypes wrapper around the serial C++ oracle (oracle/mf_oracle.cpp).

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this package.  The product
path (paper_1610_05838_b200/) must never import it.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SO_F16C = os.path.join(_HERE, "liboracle_f16c.so")
_SRC = os.path.join(_HERE, "mf_oracle.cpp")
_lib = None
# ORACLE_F16C=1 (golden-writing scripts only): the same source built with -mf16c, so the host
# compiler's _Float16 casts become the F16C instructions vcvtps2ph / vcvtph2ps (IEEE binary16
# round-to-nearest-even under the default MXCSR, as the software routines are) -- ~4x faster fp16
# epochs.  tests/test_oracle.py checks the two builds bit for bit (all 65,536 halves, sampled
# fp32 patterns, and fp16 / bf16 epochs).  The default build, and every timing of the oracle,
# stays the plain one.
_USE_F16C = os.environ.get("ORACLE_F16C", "0") == "1"

F32, F16, BF16, F64 = 0, 1, 2, 3
STORAGE_DTYPE = {F32: np.float32, F16: np.uint16, BF16: np.uint16, F64: np.float64}
STORAGE_NAME = {"f32": F32, "fp32": F32, "f16": F16, "fp16": F16, "bf16": BF16, "f64": F64}


def build(force: bool = False, f16c: bool = False) -> str:
    so = _SO_F16C if f16c else _SO
    if force or not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(_SRC):
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-ffp-contract=off", "-fno-fast-math"]
                              + (["-mf16c"] if f16c else []) + ["-fPIC", "-shared", "-o", so, _SRC])
    return so


def host_has_f16c() -> bool:
    try:
        with open("/proc/cpuinfo") as f:
            return " f16c" in f.read()
    except OSError:
        return False


def lib():
    global _lib
    if _lib is None:
        _lib = load(_USE_F16C and host_has_f16c())
    return _lib


def load(f16c: bool = False):
    """Load one build of the oracle (a fresh ctypes handle; f16c=True is the golden-writing build)."""
    L = ctypes.CDLL(build(f16c=f16c))
    c = ctypes
    L.orc_lr.argtypes = [c.c_double, c.c_double, c.c_int32]; L.orc_lr.restype = c.c_double
    L.orc_eta.argtypes = [c.c_double, c.c_double, c.c_int32]; L.orc_eta.restype = c.c_float
    L.orc_f32_to_f16.argtypes = [c.c_float]; L.orc_f32_to_f16.restype = c.c_uint16
    L.orc_f16_to_f32.argtypes = [c.c_uint16]; L.orc_f16_to_f32.restype = c.c_float
    L.orc_f32_to_bf16.argtypes = [c.c_float]; L.orc_f32_to_bf16.restype = c.c_uint16
    L.orc_bf16_to_f32.argtypes = [c.c_uint16]; L.orc_bf16_to_f32.restype = c.c_float
    L.orc_splitmix64.argtypes = [c.c_uint64]; L.orc_splitmix64.restype = c.c_uint64
    L.orc_init.argtypes = [c.c_uint64, c.c_int64, c.c_int32, c.c_uint32, c.c_int32, c.c_void_p]
    L.orc_init.restype = None
    L.orc_shuffle_perm.argtypes = [c.c_uint64, c.c_int64, c.c_void_p]; L.orc_shuffle_perm.restype = None
    L.orc_epoch.argtypes = [c.c_int32, c.c_int32, c.c_void_p, c.c_void_p, c.c_void_p, c.c_void_p,
                            c.c_void_p, c.c_void_p, c.c_int64, c.c_float, c.c_float]
    L.orc_epoch.restype = c.c_int
    L.orc_epoch_f64.argtypes = [c.c_int32, c.c_void_p, c.c_void_p, c.c_void_p, c.c_void_p,
                                c.c_void_p, c.c_void_p, c.c_int64, c.c_double, c.c_double]
    L.orc_epoch_f64.restype = c.c_int
    L.orc_rmse.argtypes = [c.c_int32, c.c_int32, c.c_void_p, c.c_void_p, c.c_void_p, c.c_void_p,
                           c.c_void_p, c.c_int64]
    L.orc_rmse.restype = c.c_double
    L.orc_loss.argtypes = [c.c_int32, c.c_int32, c.c_void_p, c.c_void_p, c.c_void_p, c.c_void_p,
                           c.c_void_p, c.c_int64, c.c_double]
    L.orc_loss.restype = c.c_double
    L.orc_waves.argtypes = [c.c_int64, c.c_int64, c.c_void_p, c.c_void_p, c.c_void_p, c.c_int64, c.c_void_p]
    L.orc_waves.restype = c.c_int64
    return L


def _p(a):
    return None if a is None else a.ctypes.data


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


def lr(alpha, beta, t):
    return lib().orc_lr(alpha, beta, t)


def eta(alpha, beta, t):
    return lib().orc_eta(alpha, beta, t)


def init(seed, rows, k, tag, storage):
    out = np.empty((rows, k), STORAGE_DTYPE[storage])
    lib().orc_init(seed, rows, k, tag, storage, _p(out))
    return out


def shuffle_perm(seed, N):
    perm = np.empty(N, np.int64)
    lib().orc_shuffle_perm(seed, N, _p(perm))
    return perm


class Model:
    """P (m x k) and Q (n x k, row per item, reading A-4) in storage precision."""

    def __init__(self, m, n, k, storage=F32, seed=None, P=None, Q=None):
        self.m, self.n, self.k, self.storage = m, n, k, storage
        dt = STORAGE_DTYPE[storage]
        if P is not None:
            self.P, self.Q = _c(P, dt).reshape(m, k).copy(), _c(Q, dt).reshape(n, k).copy()
        else:
            self.P = init(seed, m, k, 0, storage)
            self.Q = init(seed, n, k, 1, storage)

    def epoch(self, u, v, r, eta_t, lam, order=None):
        u, v, r = _c(u, np.int32), _c(v, np.int32), _c(r, np.float32)
        o = None if order is None else _c(order, np.int64)
        N = len(u) if o is None else len(o)
        if self.storage == F64:
            return lib().orc_epoch_f64(self.k, _p(self.P), _p(self.Q), _p(u), _p(v), _p(r), _p(o), N,
                                       float(eta_t), float(lam))
        return lib().orc_epoch(self.k, self.storage, _p(self.P), _p(self.Q), _p(u), _p(v), _p(r), _p(o), N,
                               eta_t, lam)

    def rmse(self, u, v, r):
        u, v, r = _c(u, np.int32), _c(v, np.int32), _c(r, np.float32)
        return lib().orc_rmse(self.k, self.storage, _p(self.P), _p(self.Q), _p(u), _p(v), _p(r), len(u))

    def loss(self, u, v, r, lam):
        u, v, r = _c(u, np.int32), _c(v, np.int32), _c(r, np.float32)
        return lib().orc_loss(self.k, self.storage, _p(self.P), _p(self.Q), _p(u), _p(v), _p(r), len(u), lam)

    def factors_f32(self):
        return widen(self.P, self.storage), widen(self.Q, self.storage)


def widen(a, storage):
    if storage in (F32, F64):
        return a.astype(np.float32 if storage == F32 else np.float64)
    if storage == F16:
        return a.view(np.float16).astype(np.float32)
    return (a.astype(np.uint32) << 16).view(np.float32)


def waves(m, n, u, v, order=None):
    u, v = _c(u, np.int32), _c(v, np.int32)
    o = None if order is None else _c(order, np.int64)
    N = len(u) if o is None else len(o)
    w = np.empty(N, np.int32)
    nw = lib().orc_waves(m, n, _p(u), _p(v), _p(o), N, _p(w))
    return w, nw


def train(cfg_m, cfg_n, k, storage, seed_init, u, v, r, alpha, beta, lam, epochs, order=None,
          test=None, P=None, Q=None):
    """Serial SGD for `epochs` epochs over `order`; returns (model, list of test RMSE per epoch)."""
    mdl = Model(cfg_m, cfg_n, k, storage, seed=seed_init, P=P, Q=Q)
    trace = []
    for t in range(epochs):
        rc = mdl.epoch(u, v, r, eta(alpha, beta, t), lam, order)
        if rc != 0:
            raise FloatingPointError(f"oracle diverged in epoch {t}")
        if test is not None:
            trace.append(mdl.rmse(*test))
    return mdl, trace
