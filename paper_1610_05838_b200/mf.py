"""Thin ctypes binding of the C ABI in include/mf.h (argument marshalling only).

Every step of the hot path runs in libmf.so's CUDA kernels; this module only
converts Python / numpy / torch arguments to pointers and status codes to
exceptions.  There is no CPU fallback: if libmf.so is missing the import
fails loudly, and without a CUDA device every compute call raises MFError.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libmf.so")
if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`")

_lib = ctypes.CDLL(LIB_PATH)
c = ctypes

MF_OK, MF_EINVAL, MF_ENOMEM, MF_ECUDA, MF_ESTATE, MF_EDIVERGED, MF_ENCCL = 0, -1, -2, -3, -4, -5, -6
MF_SCHED_HOGWILD, MF_SCHED_WAVEFRONT, MF_SCHED_DETERMINISTIC, MF_SCHED_PARTITIONED = 0, 1, 2, 3
SCHEDULES = {"hogwild": 0, "wavefront": 1, "deterministic": 2, "partitioned": 3}
(MF_OPT_STORAGE, MF_OPT_BETA, MF_OPT_WORKERS, MF_OPT_BATCH_F, MF_OPT_WAVE_ROWS, MF_OPT_WAVE_COLS, MF_OPT_DEVICE,
 MF_OPT_STREAM, MF_OPT_SHUFFLE, MF_OPT_COUNT_UPDATES, MF_OPT_WAVE_PERM, MF_OPT_EPOCH, MF_OPT_PARTITIONS,
 MF_OPT_SEED_SHUFFLE, MF_OPT_VARIANT, MF_OPT_TRACE, MF_OPT_SUBEPOCHS, MF_OPT_WAVE_CTA,
 MF_OPT_STREAM_CHUNK, MF_OPT_PART_SPLIT, MF_OPT_R_STAGING, MF_OPT_WAVE_PASSES, MF_OPT_P_HOST,
 MF_OPT_Q_UPDATE, MF_OPT_DET_FLOW, MF_OPT_Q_KAPPA) = range(26)
STORAGE = {"f32": 0, "fp32": 0, "f16": 1, "fp16": 1, "bf16": 2}


class mf_epoch_stats(c.Structure):
    _fields_ = [("updates", c.c_int64), ("seconds", c.c_double), ("kernel_seconds", c.c_double),
                ("lr", c.c_float), ("epoch", c.c_int32), ("workers", c.c_int32), ("launches", c.c_int32)]


_P = c.c_void_p
_sig = {
    "mf_create": ([c.c_int64, c.c_int64, c.c_int32, c.c_float, c.c_float, c.c_uint64, c.POINTER(_P)], c.c_int),
    "mf_set_option": ([_P, c.c_int, c.c_double], c.c_int),
    "mf_get_option": ([_P, c.c_int, c.POINTER(c.c_double)], c.c_int),
    "mf_load_coo": ([_P, _P, _P, _P, c.c_int64], c.c_int),
    "mf_epoch": ([_P, c.c_int, c.POINTER(mf_epoch_stats)], c.c_int),
    "mf_epoch_host": ([_P, c.c_int, _P, _P, _P, c.c_int64, c.POINTER(mf_epoch_stats)], c.c_int),
    "mf_rmse": ([_P, _P, _P, _P, c.c_int64, c.POINTER(c.c_double)], c.c_int),
    "mf_get_factors": ([_P, _P, _P], c.c_int),
    "mf_set_factors": ([_P, _P, _P], c.c_int),
    "mf_get_order": ([_P, _P], c.c_int),
    "mf_wave_count": ([_P, c.POINTER(c.c_int64)], c.c_int),
    "mf_nccl_unique_id": ([_P], c.c_int),
    "mf_attach_nccl": ([_P, _P, c.c_int, c.c_int], c.c_int),
    "mf_segment": ([c.c_int64, c.c_int32, c.c_int32, c.POINTER(c.c_int64), c.POINTER(c.c_int64)], c.c_int),
    "mf_round_segment": ([c.c_uint64, c.c_int32, c.c_int32, c.c_int32, c.c_int32, c.POINTER(c.c_int32)], c.c_int),
    "mf_round_peers": ([c.c_uint64, c.c_int32, c.c_int32, c.c_int32, c.c_int32, c.POINTER(c.c_int32),
                        c.POINTER(c.c_int32)], c.c_int),
    "mf_round_unit": ([c.c_uint64, c.c_int32, c.c_int32, c.c_int32, c.c_int32, c.c_int32, c.POINTER(c.c_int32)],
                      c.c_int),
    "mf_unit_peers": ([c.c_uint64, c.c_int32, c.c_int32, c.c_int32, c.c_int32, c.c_int32, c.POINTER(c.c_int32),
                       c.POINTER(c.c_int32)], c.c_int),
    "mf_wavefront_trace": ([_P, _P, c.c_int64, c.POINTER(c.c_int64)], c.c_int),
    "mf_init_rows_host": ([_P, c.c_int32, c.c_int64, c.c_int64, _P], c.c_int),
    "mf_epoch_host_blocks": ([_P, _P, _P, _P, c.c_int64, _P, c.c_int32, _P, c.POINTER(mf_epoch_stats)], c.c_int),
    "mf_rmse_host_blocks": ([_P, _P, _P, _P, c.c_int64, _P, c.c_int32, _P, c.POINTER(c.c_double)], c.c_int),
    "mf_feasibility": ([c.c_int64, c.c_int64, c.c_int32, c.c_int32, c.c_int64, c.c_int32, c.POINTER(c.c_int64)],
                       c.c_int),
    "mf_destroy": ([_P], None),
    "mf_last_error": ([_P], c.c_char_p),
    "mf_status_string": ([c.c_int], c.c_char_p),
}
for _name, (_args, _res) in _sig.items():
    _f = getattr(_lib, _name)
    _f.argtypes = _args
    _f.restype = _res
EXPORTS = tuple(_sig)


class MFError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{_lib.mf_status_string(status).decode()}: {msg}")
        self.status = status


def _check(ctx, rc):
    if rc != MF_OK:
        msg = _lib.mf_last_error(ctx).decode() if ctx else ""
        raise MFError(rc, msg)
    return rc


def _ptr(x, dtype=None):
    """Pointer of a numpy array (converted to `dtype`, contiguous) or a torch tensor (host or device)."""
    if x is None:
        return None, None
    if hasattr(x, "data_ptr"):  # torch tensor: pass through, caller guarantees dtype / contiguity
        if not x.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return x.data_ptr(), x
    a = np.ascontiguousarray(x, dtype=dtype)
    return a.ctypes.data, a


# ------------------------------------------------------------------ C names --
def mf_create(m, n, k, lr, lam, seed):
    h = _P()
    _check(None, _lib.mf_create(m, n, k, lr, lam, seed, c.byref(h)))
    return h


def mf_set_option(ctx, key, value):
    return _check(ctx, _lib.mf_set_option(ctx, key, float(value)))


def mf_get_option(ctx, key):
    out = c.c_double()
    _check(ctx, _lib.mf_get_option(ctx, key, c.byref(out)))
    return out.value


def mf_load_coo(ctx, u, v, r):
    pu, au = _ptr(u, np.int32)
    pv, av = _ptr(v, np.int32)
    pr, ar = _ptr(r, np.float32)
    n = len(au) if not hasattr(au, "numel") else au.numel()
    return _check(ctx, _lib.mf_load_coo(ctx, pu, pv, pr, n))


def mf_epoch(ctx, schedule=MF_SCHED_HOGWILD, raise_on_error=True):
    st = mf_epoch_stats()
    rc = _lib.mf_epoch(ctx, SCHEDULES.get(schedule, schedule), c.byref(st))
    if raise_on_error:
        _check(ctx, rc)
    return st if raise_on_error else (rc, st)


def mf_epoch_host(ctx, u, v, r, schedule=MF_SCHED_HOGWILD):
    pu, au = _ptr(u, np.int32)
    pv, av = _ptr(v, np.int32)
    pr, ar = _ptr(r, np.float32)
    n = len(au) if not hasattr(au, "numel") else au.numel()
    st = mf_epoch_stats()
    _check(ctx, _lib.mf_epoch_host(ctx, SCHEDULES.get(schedule, schedule), pu, pv, pr, n, c.byref(st)))
    return st


def mf_rmse(ctx, u, v, r):
    pu, au = _ptr(u, np.int32)
    pv, av = _ptr(v, np.int32)
    pr, ar = _ptr(r, np.float32)
    n = len(au) if not hasattr(au, "numel") else au.numel()
    out = c.c_double()
    _check(ctx, _lib.mf_rmse(ctx, pu, pv, pr, n, c.byref(out)))
    return out.value


def mf_init_rows_host(ctx, tag, row0, rows, out):
    """A-7 initial values of rows [row0, row0 + rows) of P (tag 0) or Q (tag 1), in storage precision, into
    `out` (numpy array of the storage dtype: float32, or uint16 bit patterns for fp16 / bf16)."""
    _check(ctx, _lib.mf_init_rows_host(ctx, tag, row0, rows, out.ctypes.data))


def _blocks(block_off):
    bo = np.ascontiguousarray(block_off, dtype=np.int64)
    return bo, len(bo) - 1


def mf_epoch_host_blocks(ctx, u, v, r, block_off, P_host):
    pu, au = _ptr(u, np.int32)
    pv, av = _ptr(v, np.int32)
    pr, ar = _ptr(r, np.float32)
    n = len(au) if not hasattr(au, "numel") else au.numel()
    bo, nb = _blocks(block_off)
    pp, ap = _ptr(P_host)
    st = mf_epoch_stats()
    _check(ctx, _lib.mf_epoch_host_blocks(ctx, pu, pv, pr, n, bo.ctypes.data, nb, pp, c.byref(st)))
    return st


def mf_rmse_host_blocks(ctx, u, v, r, block_off, P_host):
    pu, au = _ptr(u, np.int32)
    pv, av = _ptr(v, np.int32)
    pr, ar = _ptr(r, np.float32)
    n = len(au) if not hasattr(au, "numel") else au.numel()
    bo, nb = _blocks(block_off)
    pp, ap = _ptr(P_host)
    out = c.c_double()
    _check(ctx, _lib.mf_rmse_host_blocks(ctx, pu, pv, pr, n, bo.ctypes.data, nb, pp, c.byref(out)))
    return out.value


def mf_get_factors(ctx, P=None, Q=None):
    _check(ctx, _lib.mf_get_factors(ctx, None if P is None else _ptr(P)[0], None if Q is None else _ptr(Q)[0]))


def mf_set_factors(ctx, P=None, Q=None):
    pp, ap = _ptr(P, np.float32)
    pq, aq = _ptr(Q, np.float32)
    _check(ctx, _lib.mf_set_factors(ctx, pp, pq))


def mf_get_order(ctx, n):
    out = np.empty(n, np.int64)
    _check(ctx, _lib.mf_get_order(ctx, out.ctypes.data))
    return out


def mf_wave_count(ctx):
    out = c.c_int64()
    _check(ctx, _lib.mf_wave_count(ctx, c.byref(out)))
    return out.value


def mf_nccl_unique_id():
    buf = (c.c_char * 128)()
    _check(None, _lib.mf_nccl_unique_id(buf))
    return bytes(buf)


def mf_attach_nccl(ctx, uid: bytes, rank, world):
    buf = (c.c_char * 128).from_buffer_copy(uid)
    return _check(ctx, _lib.mf_attach_nccl(ctx, buf, rank, world))


def mf_segment(extent, parts, index):
    b, e = c.c_int64(), c.c_int64()
    _check(None, _lib.mf_segment(extent, parts, index, c.byref(b), c.byref(e)))
    return b.value, e.value


def mf_round_segment(seed, epoch, G, rnd, rank):
    out = c.c_int32()
    _check(None, _lib.mf_round_segment(seed, epoch, G, rnd, rank, c.byref(out)))
    return out.value


def mf_round_peers(seed, epoch, G, rnd, rank):
    s, r = c.c_int32(), c.c_int32()
    _check(None, _lib.mf_round_peers(seed, epoch, G, rnd, rank, c.byref(s), c.byref(r)))
    return s.value, r.value


def mf_round_unit(seed, pas, G, rnd, rank, half):
    out = c.c_int32()
    _check(None, _lib.mf_round_unit(seed, pas, G, rnd, rank, half, c.byref(out)))
    return out.value


def mf_unit_peers(seed, pas, G, rnd, rank, half):
    s, r = c.c_int32(), c.c_int32()
    _check(None, _lib.mf_unit_peers(seed, pas, G, rnd, rank, half, c.byref(s), c.byref(r)))
    return s.value, r.value


def mf_wavefront_trace(ctx, cap):
    out = np.empty((cap, 4), np.int64)
    cnt = c.c_int64()
    _check(ctx, _lib.mf_wavefront_trace(ctx, out.ctypes.data, cap, c.byref(cnt)))
    return out[:cnt.value]


def mf_feasibility(m, n, i, j, s, safety=20):
    """(passes, bound) of the paper's rule s < min(m // i, n // j) / safety."""
    b = c.c_int64()
    rc = _lib.mf_feasibility(m, n, i, j, s, safety, c.byref(b))
    if rc < 0:
        raise MFError(rc, "mf_feasibility: arguments must be positive")
    return bool(rc), b.value


def mf_destroy(ctx):
    _lib.mf_destroy(ctx)


# ------------------------------------------------------------ convenience --
class MF:
    """Owning wrapper: MF(m, n, k, lr, lam, seed, storage='f32', beta=0.0, **options)."""

    def __init__(self, m, n, k, lr, lam, seed, storage="f32", beta=0.0, **opts):
        self.m, self.n, self.k = m, n, k
        self.h = mf_create(m, n, k, lr, lam, seed)
        self.set(MF_OPT_STORAGE, STORAGE.get(storage, storage))
        if beta:
            self.set(MF_OPT_BETA, beta)
        for key, val in opts.items():
            self.set(globals()["MF_OPT_" + key.upper()], val)

    def set(self, key, value):
        mf_set_option(self.h, key, value)

    def get(self, key):
        return mf_get_option(self.h, key)

    def load(self, u, v, r):
        mf_load_coo(self.h, u, v, r)
        self.N = len(u) if not hasattr(u, "numel") else u.numel()

    def epoch(self, schedule="hogwild"):
        return mf_epoch(self.h, schedule)

    def epoch_host(self, u, v, r):
        """Streamed batch-Hogwild! epoch over caller ratings (not kept resident)."""
        return mf_epoch_host(self.h, u, v, r)

    def rmse(self, u, v, r):
        return mf_rmse(self.h, u, v, r)

    def factors(self, rows=None):
        P = np.empty((self.m if rows is None else rows, self.k), np.float32)
        Q = np.empty((self.n, self.k), np.float32)
        mf_get_factors(self.h, P, Q)
        return P, Q

    def set_factors(self, P=None, Q=None):
        mf_set_factors(self.h, P, Q)

    def order(self):
        return mf_get_order(self.h, self.N)

    def close(self):
        if self.h:
            mf_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()
