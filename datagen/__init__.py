"""Seeded synthetic input generator shared by the oracle tests and the CUDA path.

Test data only: this module contains none of the SGD method's arithmetic
(see gen.c's header).  The recipe is SURVEY.md §8(d) "Synthetic inputs",
restated in DESIGN.md §3.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

from .configs import CONFIGS, Config  # noqa: F401

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libmfgen.so")
_lib = None


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "gen.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-o", _SO, src, "-lm"])
    return _SO


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_SO)
        lib.mfgen_planted_coo.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int,
                                          ctypes.c_double, ctypes.c_int64, ctypes.c_int,
                                          ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        lib.mfgen_planted_coo.restype = ctypes.c_int
        lib.mfgen_planted_factors.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int,
                                              ctypes.c_void_p, ctypes.c_void_p]
        lib.mfgen_planted_factors.restype = ctypes.c_int
        lib.mfgen_zipf_coo.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int, ctypes.c_double,
                                       ctypes.c_int64, ctypes.c_double, ctypes.c_double,
                                       ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        lib.mfgen_zipf_coo.restype = ctypes.c_int
        lib.mfgen_planted_segment.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                              ctypes.c_int64, ctypes.c_int, ctypes.c_double, ctypes.c_int64,
                                              ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        lib.mfgen_planted_segment.restype = ctypes.c_int
        _lib = lib
    return _lib


def planted_coo_into(seed, m, n, rank, sigma, total, with_replacement, u_ptr, v_ptr, r_ptr):
    """Fill caller buffers (raw host pointers: int32 u, int32 v, float32 r) with `total` samples."""
    rc = _load().mfgen_planted_coo(seed, m, n, rank, sigma, total, int(bool(with_replacement)),
                                   u_ptr, v_ptr, r_ptr)
    if rc != 0:
        raise ValueError("mfgen_planted_coo rejected its arguments")


def planted_coo(seed, m, n, rank, sigma, total, with_replacement=True):
    u = np.empty(total, np.int32)
    v = np.empty(total, np.int32)
    r = np.empty(total, np.float32)
    planted_coo_into(seed, m, n, rank, sigma, total, with_replacement,
                     u.ctypes.data, v.ctypes.data, r.ctypes.data)
    return u, v, r


def zipf_coo(seed, m, n, rank, sigma, total, s_u, s_v):
    """Skewed degrees (NEXT-4): u ~ Zipf(s_u), v ~ Zipf(s_v) over scrambled ids, same planted ratings."""
    u = np.empty(total, np.int32)
    v = np.empty(total, np.int32)
    r = np.empty(total, np.float32)
    if _load().mfgen_zipf_coo(seed, m, n, rank, sigma, total, s_u, s_v, u.ctypes.data, v.ctypes.data,
                              r.ctypes.data) != 0:
        raise ValueError("mfgen_zipf_coo rejected its arguments")
    return u, v, r


def planted_factors(seed, m, n, rank):
    P = np.empty((m, rank), np.float64)
    Q = np.empty((n, rank), np.float64)
    if _load().mfgen_planted_factors(seed, m, n, rank, P.ctypes.data, Q.ctypes.data) != 0:
        raise ValueError("bad arguments")
    return P, Q


def planted_segment(seed, m, row_lo, row_hi, n, rank, sigma, i0, total):
    """Draws i0 .. i0+total-1 of a global planted problem (m x n) restricted to rows [row_lo, row_hi)."""
    u = np.empty(total, np.int32)
    v = np.empty(total, np.int32)
    r = np.empty(total, np.float32)
    if _load().mfgen_planted_segment(seed, m, row_lo, row_hi, n, rank, sigma, i0, total, u.ctypes.data,
                                     v.ctypes.data, r.ctypes.data) != 0:
        raise ValueError("mfgen_planted_segment rejected its arguments")
    return u, v, r


TEST_STREAM = 1 << 50  # first global draw index of the test sets of segmented problems


def make_segment(cfg: "Config", m_glob, row_lo, row_hi, n_train, n_test, rank_index):
    """One rank's shard of a row-partitioned planted problem with cfg's n, rank, sigma and seed:
    train = global draws [rank_index * n_train, +n_train), test = TEST_STREAM + [rank_index * n_test, +n_test),
    rows restricted to [row_lo, row_hi)."""
    tr = planted_segment(cfg.seed_data, m_glob, row_lo, row_hi, cfg.n, cfg.rank, cfg.sigma,
                         rank_index * n_train, n_train)
    te = planted_segment(cfg.seed_data, m_glob, row_lo, row_hi, cfg.n, cfg.rank, cfg.sigma,
                         TEST_STREAM + rank_index * n_test, n_test)
    return tr, te


def split(cfg: "Config", u, v, r):
    """Train = first n_train indices, test = the next n_test (reading A-17)."""
    t = cfg.n_train
    return (u[:t], v[:t], r[:t]), (u[t:], v[t:], r[t:])


def make(cfg: "Config"):
    """Generate the config's full train+test COO; returns ((u,v,r) train, (u,v,r) test)."""
    if cfg.zipf is not None:
        u, v, r = zipf_coo(cfg.seed_data, cfg.m, cfg.n, cfg.rank, cfg.sigma, cfg.n_train + cfg.n_test, *cfg.zipf)
    else:
        u, v, r = planted_coo(cfg.seed_data, cfg.m, cfg.n, cfg.rank, cfg.sigma,
                              cfg.n_train + cfg.n_test, cfg.with_replacement)
    return split(cfg, u, v, r)
