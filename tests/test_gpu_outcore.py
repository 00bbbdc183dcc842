"""Out-of-core factors (MF_OPT_P_HOST): P in caller host memory, streamed through the GPU row block by row
block (the paper's Hugewiki path).  -m gpu.

Ratings are grouped by row block (stable, so each block keeps the given order); with one worker an epoch is
serial SGD over that grouped order, and must equal the oracle run over it (fp32 1e-5, fp16 2e-3).
"""
import numpy as np
import pytest

import datagen
import oracle

pytestmark = pytest.mark.gpu
ORC = {"f32": oracle.F32, "f16": oracle.F16}
TOL = {"f32": 1e-5, "f16": 2e-3}


@pytest.fixture(scope="module")
def mf():
    from paper_1610_05838_b200 import mf
    return mf


def _group(mf, m, u, v, r, nblocks):
    """Stable grouping of the triples by row block; returns grouped arrays and block offsets."""
    ends = np.array([mf.mf_segment(m, nblocks, b)[1] for b in range(nblocks)])
    blk = np.searchsorted(ends, u, side="right")
    o = np.argsort(blk, kind="stable")
    off = np.concatenate([[0], np.cumsum(np.bincount(blk, minlength=nblocks))]).astype(np.int64)
    return u[o], v[o], r[o], off


def _ctx(mf, cfg, storage, **kw):
    return mf.MF(cfg.m, cfg.n, cfg.k, cfg.alpha, cfg.lam, cfg.seed_init, storage=storage, beta=cfg.beta,
                 p_host=1, **kw)


@pytest.mark.parametrize("storage", ["f32", "f16"])
@pytest.mark.parametrize("nblocks", [1, 4, 7])
def test_outcore_one_worker_equals_serial_sgd(mf, storage, nblocks):
    cfg = datagen.CONFIGS["C1"]
    (u, v, r), (tu, tv, tr) = datagen.make(cfg)
    gu, gv, gr, off = _group(mf, cfg.m, u, v, r, nblocks)
    tgu, tgv, tgr, toff = _group(mf, cfg.m, tu, tv, tr, nblocks)
    ref = oracle.Model(cfg.m, cfg.n, cfg.k, ORC[storage], seed=cfg.seed_init)
    with _ctx(mf, cfg, storage, workers=1, count_updates=1, stream_chunk=3_000) as g:
        Ph = np.empty_like(ref.P)
        mf.mf_init_rows_host(g.h, 0, 0, cfg.m, Ph)
        np.testing.assert_array_equal(Ph, ref.P)       # A-7 init bits == the oracle's
        for e in range(2):
            st = mf.mf_epoch_host_blocks(g.h, gu, gv, gr, off, Ph)
            assert st.updates == len(u)
            ref.epoch(gu, gv, gr, oracle.eta(cfg.alpha, cfg.beta, e), cfg.lam)
        Q = np.empty((cfg.n, cfg.k), np.float32)
        mf.mf_get_factors(g.h, None, Q)
        got_rmse = mf.mf_rmse_host_blocks(g.h, tgu, tgv, tgr, toff, Ph)
    Pr, Qr = ref.factors_f32()
    Pg = oracle.widen(Ph, ORC[storage])
    assert np.linalg.norm(Pg - Pr) / np.linalg.norm(Pr) <= TOL[storage]
    assert np.linalg.norm(Q - Qr) / np.linalg.norm(Qr) <= TOL[storage]
    assert got_rmse == pytest.approx(ref.rmse(tgu, tgv, tgr), rel=TOL[storage])


def test_outcore_hogwild_rmse_within_half_percent_pinned(mf):
    """Netflix-degree slice (C2-1pct), fp16, 8 row blocks, default workers, P in pinned host memory: every
    sample once per epoch and the test RMSE after 10 epochs within 0.5% of the oracle over the same order."""
    import torch
    cfg = datagen.CONFIGS["C2-1pct"]
    (u, v, r), (tu, tv, tr) = datagen.make(cfg)
    gu, gv, gr, off = _group(mf, cfg.m, u, v, r, 8)
    tgu, tgv, tgr, toff = _group(mf, cfg.m, tu, tv, tr, 8)
    E = 10
    ref = oracle.Model(cfg.m, cfg.n, cfg.k, oracle.F16, seed=cfg.seed_init)
    for e in range(E):
        ref.epoch(gu, gv, gr, oracle.eta(cfg.alpha, cfg.beta, e), cfg.lam)
    want = ref.rmse(tgu, tgv, tgr)
    with _ctx(mf, cfg, "f16", count_updates=1, stream_chunk=200_000) as g:
        Ph = torch.empty((cfg.m, cfg.k), dtype=torch.int16).pin_memory()
        mf.mf_init_rows_host(g.h, 0, 0, cfg.m, Ph.numpy())
        for _ in range(E):
            assert mf.mf_epoch_host_blocks(g.h, gu, gv, gr, off, Ph).updates == len(u)
        got = mf.mf_rmse_host_blocks(g.h, tgu, tgv, tgr, toff, Ph)
    assert abs(got - want) <= 0.005 * want, (got, want)


def test_outcore_errors(mf):
    cfg = datagen.CONFIGS["C1"]
    (u, v, r), _ = datagen.make(cfg)
    gu, gv, gr, off = _group(mf, cfg.m, u, v, r, 4)
    with _ctx(mf, cfg, "f32") as g:
        Ph = np.zeros((cfg.m, cfg.k), np.float32)
        bad = gu.copy()
        bad[int(off[2]) + 5] = 0                   # a sample of block 2 whose row belongs to block 0
        with pytest.raises(mf.MFError) as ei:
            mf.mf_epoch_host_blocks(g.h, bad, gv, gr, off, Ph)
        assert ei.value.status == mf.MF_EINVAL
        with pytest.raises(mf.MFError) as ei:      # offsets not spanning [0, nnz]
            mf.mf_epoch_host_blocks(g.h, gu, gv, gr, off[:-1], Ph)
        assert ei.value.status == mf.MF_EINVAL
        g.load(u, v, r)
        with pytest.raises(mf.MFError) as ei:      # the device-P entry points refuse
            g.epoch("hogwild")
        assert ei.value.status == mf.MF_ESTATE
        with pytest.raises(mf.MFError) as ei:
            g.factors()
        assert ei.value.status == mf.MF_ESTATE
    with mf.MF(cfg.m, cfg.n, cfg.k, cfg.alpha, cfg.lam, cfg.seed_init) as g:
        with pytest.raises(mf.MFError) as ei:      # without MF_OPT_P_HOST
            mf.mf_epoch_host_blocks(g.h, gu, gv, gr, off, np.zeros((cfg.m, cfg.k), np.float32))
        assert ei.value.status == mf.MF_ESTATE
