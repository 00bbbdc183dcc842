"""Wavefront-update schedule on the GPU.  -m gpu.

Checks: exactly-once, the conflict audit (no two blocks of one
column processed at overlapping times, SPEC.md:297-305 / S:555), every block
visited once per epoch, and test RMSE within 0.5% of the serial
oracle on the same shuffled order (north star).
"""
import numpy as np
import pytest

import datagen
import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mfmod():
    from paper_1610_05838_b200 import mf
    return mf


def _passes(mfmod, g):
    """Passes per epoch of the current wavefront layout (auto: MF_OPT_WAVE_PASSES = 0)."""
    return int(g.get(mfmod.MF_OPT_WAVE_PASSES))


def _audit(rec, s, c, P=1):
    """rec rows: (worker, block, t_start, t_end), block = (pass * s + worker) * c + column.  Returns the
    number of column conflicts (two blocks of one column overlapping in time)."""
    assert len(rec) == P * s * c
    blocks = rec[:, 1]
    assert np.array_equal(np.sort(blocks), np.arange(P * s * c))  # each block exactly once
    assert np.array_equal(rec[:, 0], (blocks // c) % s)           # block (p, w, col) done by worker w
    conflicts = 0
    col = blocks % c
    for cc in range(c):
        iv = rec[col == cc][:, 2:4]
        iv = iv[np.argsort(iv[:, 0])]
        conflicts += int(np.sum(iv[1:, 0] < iv[:-1, 1]))
    return conflicts


@pytest.mark.parametrize("perm", [0, 1])
def test_wavefront_exactly_once_and_conflict_free(mfmod, perm):
    cfg = datagen.CONFIGS["C1"]
    (u, v, r), _ = datagen.make(cfg)
    s, c = 8, 16
    with mfmod.MF(cfg.m, cfg.n, cfg.k, cfg.alpha, cfg.lam, cfg.seed_init, beta=cfg.beta, wave_rows=s,
                  wave_cols=c, wave_perm=perm, trace=1, count_updates=1) as g:
        g.load(u, v, r)
        for _ in range(3):
            st = g.epoch("wavefront")
            assert st.updates == len(u)
            assert st.workers == s
            P = _passes(mfmod, g)
            rec = mfmod.mf_wavefront_trace(g.h, P * s * c + 10)
            assert _audit(rec, s, c, P) == 0


def test_wavefront_audit_at_scale(mfmod):
    """Auto-sized grid (~8 workers/SM) on a Yahoo-shaped slice: still conflict-free."""
    cfg = datagen.CONFIGS["C3-1pct"]
    (u, v, r), _ = datagen.make(cfg)
    with mfmod.MF(cfg.m, cfg.n, cfg.k, cfg.alpha, cfg.lam, cfg.seed_init, beta=cfg.beta, trace=1,
                  count_updates=1) as g:
        g.load(u, v, r)
        st = g.epoch("wavefront")
        assert st.updates == len(u)
        s = st.workers
        c = int(g.get(mfmod.MF_OPT_WAVE_COLS)) or 2 * s
        rec = mfmod.mf_wavefront_trace(g.h, 10 ** 8)
        assert _audit(rec, s, c, _passes(mfmod, g)) == 0


def _oracle_seed_spread(cfg, u, v, r, test, epochs, seeds=(42, 43, 44)):
    """Max - min oracle test RMSE over shuffle seeds: how much the order alone moves the result."""
    out = []
    for sd in seeds:
        _, tr = oracle.train(cfg.m, cfg.n, cfg.k, oracle.F32, cfg.seed_init, u, v, r, cfg.alpha, cfg.beta, cfg.lam,
                             epochs, order=oracle.shuffle_perm(sd, len(u)), test=test)
        out.append(tr[-1])
    return max(out) - min(out), out


@pytest.mark.parametrize("name,s,c,epochs", [("C1", 8, 16, 20), ("C3-1pct", 0, 0, 10)])
def test_wavefront_rmse_within_half_percent(mfmod, name, s, c, epochs):
    """Gate: 0.5% of the oracle (north star) -- or, where the oracle's own shuffle-seed spread exceeds
    0.5% (C1: ~1%), that spread (reading T3)."""
    cfg = datagen.CONFIGS[name]
    (u, v, r), test = datagen.make(cfg)
    order = oracle.shuffle_perm(cfg.seed_shuffle, len(u))
    _, trace = oracle.train(cfg.m, cfg.n, cfg.k, oracle.F32, cfg.seed_init, u, v, r, cfg.alpha, cfg.beta,
                            cfg.lam, epochs, order=order, test=test)
    gate = 0.005 * trace[-1]
    if name == "C1":
        spread, _ = _oracle_seed_spread(cfg, u, v, r, test, epochs)
        gate = max(gate, spread)
    with mfmod.MF(cfg.m, cfg.n, cfg.k, cfg.alpha, cfg.lam, cfg.seed_init, beta=cfg.beta, wave_rows=s,
                  wave_cols=c, seed_shuffle=cfg.seed_shuffle) as g:
        g.load(u, v, r)
        for _ in range(epochs):
            g.epoch("wavefront")
        got = g.rmse(*test)
    assert abs(got - trace[-1]) <= gate, (got, trace[-1], gate)


def test_wavefront_single_worker_is_serial_block_order(mfmod):
    """s = 1 worker: the epoch is serial SGD over the blocks in pi_0 order; with c = 1 it is exactly
    serial SGD on the shuffled order (compare with the oracle, fp32 Frobenius 1e-5)."""
    cfg = datagen.CONFIGS["C1"]
    (u, v, r), _ = datagen.make(cfg)
    order = oracle.shuffle_perm(cfg.seed_shuffle, len(u))
    ref = oracle.Model(cfg.m, cfg.n, cfg.k, oracle.F32, seed=cfg.seed_init)
    ref.epoch(u, v, r, oracle.eta(cfg.alpha, cfg.beta, 0), cfg.lam, order)
    with mfmod.MF(cfg.m, cfg.n, cfg.k, cfg.alpha, cfg.lam, cfg.seed_init, beta=cfg.beta, wave_rows=1,
                  wave_cols=1, seed_shuffle=cfg.seed_shuffle) as g:
        g.load(u, v, r)
        g.epoch("wavefront")
        P, Q = g.factors()
    assert np.linalg.norm(P - ref.P) / np.linalg.norm(ref.P) <= 1e-5
    assert np.linalg.norm(Q - ref.Q) / np.linalg.norm(ref.Q) <= 1e-5


def _trace_order(mfmod, rec, perm, u, v, m, n, s, c, by_row=False, P=1):
    """Serial order of a wavefront epoch reconstructed from its audit trace: blocks by start time, each
    block's samples in stored (shuffled) order.  Blocks of one column never overlap in time and blocks
    of one band run on one worker in sequence, so sorting by start time orders every pair of blocks that
    share a row or a column as the GPU ran them; blocks that overlap in time share neither."""
    band = np.searchsorted([mfmod.mf_segment(m, s, w)[1] for w in range(s)], u[perm], side="right")
    grp = np.searchsorted([mfmod.mf_segment(n, c, g)[1] for g in range(c)], v[perm], side="right")
    pas = (np.arange(len(perm)) * P) // len(perm)  # pass of each stored position
    key = (pas * s + band.astype(np.int64)) * c + grp
    if by_row:  # q-stationary layout: inside a block the samples are sorted by Q row (stable)
        order_pos = np.lexsort((np.arange(len(perm)), v[perm], key))
        by_blk = {}
        for pos in order_pos:
            by_blk.setdefault(int(key[pos]), []).append(pos)
        return np.concatenate([perm[np.asarray(by_blk.get(int(b), []), dtype=np.int64)]
                               for b in rec[np.argsort(rec[:, 2]), 1]])
    by_blk = {}
    for pos in np.argsort(key, kind="stable"):
        by_blk.setdefault(int(key[pos]), []).append(pos)
    order = [perm[np.asarray(by_blk.get(int(b), []), dtype=np.int64)] for b in rec[np.argsort(rec[:, 2]), 1]]
    return np.concatenate(order)


@pytest.mark.parametrize("storage", [0, 1])
@pytest.mark.parametrize("s,c,depth", [(8, 16, 2), (8, 16, 4), (8, 16, 8), (0, 0, 0), (24, 30, 4)])
def test_wavefront_equals_serial_sweep_in_trace_order(mfmod, storage, s, c, depth):
    """The paper-literal wavefront (warp workers, serial blocks, column locks) with D samples of a block in
    flight and register forwarding is exactly serial SGD over the blocks in the order the audit trace
    shows: its factors after 2 epochs equal the oracle's over that order (fp32 1e-5, fp16 2e-3)."""
    cfg = datagen.CONFIGS["C1"]
    (u, v, r), _ = datagen.make(cfg)
    st = {0: oracle.F32, 1: oracle.F16}[storage]
    ref = oracle.Model(cfg.m, cfg.n, cfg.k, st, seed=cfg.seed_init)
    with mfmod.MF(cfg.m, cfg.n, cfg.k, cfg.alpha, cfg.lam, cfg.seed_init, storage=storage, beta=cfg.beta,
                  wave_rows=s, wave_cols=c, trace=1, count_updates=1, seed_shuffle=cfg.seed_shuffle,
                  variant=depth << 4) as g:
        g.load(u, v, r)
        perm = g.order()
        for e in range(2):
            stt = g.epoch("wavefront")
            assert stt.updates == len(u)
            ss = stt.workers
            cc = c or int(g.get(mfmod.MF_OPT_WAVE_COLS)) or 2 * ss
            P = _passes(mfmod, g)
            rec = mfmod.mf_wavefront_trace(g.h, P * ss * cc + 10)
            assert _audit(rec, ss, cc, P) == 0
            ref.epoch(u, v, r, oracle.eta(cfg.alpha, cfg.beta, e), cfg.lam,
                      _trace_order(mfmod, rec, perm, u, v, cfg.m, cfg.n, ss, cc, P=P))
        P, Q = g.factors()
    Pr, Qr = ref.factors_f32()
    tol = {0: 1e-5, 1: 2e-3}[storage]
    assert np.linalg.norm(P - Pr) / np.linalg.norm(Pr) <= tol
    assert np.linalg.norm(Q - Qr) / np.linalg.norm(Qr) <= tol


@pytest.mark.parametrize("storage", [0, 1])
@pytest.mark.parametrize("s,c,P", [(8, 10, 3), (0, 0, 4)])
def test_wavefront_passes_equal_serial_sweep_in_trace_order(mfmod, storage, s, c, P):
    """MF_OPT_WAVE_PASSES = P: the epoch is P passes over consecutive slices of the shuffled samples, each
    with fresh column sequences; still exactly serial SGD over the blocks in trace order (warp workers)."""
    cfg = datagen.CONFIGS["C1"]
    (u, v, r), _ = datagen.make(cfg)
    st = {0: oracle.F32, 1: oracle.F16}[storage]
    ref = oracle.Model(cfg.m, cfg.n, cfg.k, st, seed=cfg.seed_init)
    with mfmod.MF(cfg.m, cfg.n, cfg.k, cfg.alpha, cfg.lam, cfg.seed_init, storage=storage, beta=cfg.beta,
                  wave_rows=s, wave_cols=c, wave_passes=P, trace=1, count_updates=1,
                  seed_shuffle=cfg.seed_shuffle) as g:
        g.load(u, v, r)
        perm = g.order()
        for e in range(2):
            stt = g.epoch("wavefront")
            assert stt.updates == len(u)
            ss = stt.workers
            cc = c or int(g.get(mfmod.MF_OPT_WAVE_COLS))
            assert int(g.get(mfmod.MF_OPT_WAVE_PASSES)) == P
            rec = mfmod.mf_wavefront_trace(g.h, P * ss * cc + 10)
            assert _audit(rec, ss, cc, P) == 0
            ref.epoch(u, v, r, oracle.eta(cfg.alpha, cfg.beta, e), cfg.lam,
                      _trace_order(mfmod, rec, perm, u, v, cfg.m, cfg.n, ss, cc, P=P))
        Pg, Qg = g.factors()
    Pr, Qr = ref.factors_f32()
    tol = {0: 1e-5, 1: 2e-3}[storage]
    assert np.linalg.norm(Pg - Pr) / np.linalg.norm(Pr) <= tol
    assert np.linalg.norm(Qg - Qr) / np.linalg.norm(Qr) <= tol


def test_wavefront_cta_passes_exactly_once_and_conflict_free(mfmod):
    """CTA workers (staged and q-stationary) with P = 4 passes: every sample once per epoch, no column
    conflict across the 4 x s x c blocks."""
    cfg = datagen.CONFIGS["C2-1pct"]
    (u, v, r), _ = datagen.make(cfg)
    for cta in (1, 3):
        with mfmod.MF(cfg.m, cfg.n, cfg.k, cfg.alpha, cfg.lam, cfg.seed_init, storage=1, beta=cfg.beta,
                      wave_cta=cta, wave_passes=4, trace=1, count_updates=1) as g:
            g.load(u, v, r)
            for _ in range(2):
                stt = g.epoch("wavefront")
                assert stt.updates == len(u)
            ss, cc = stt.workers, int(g.get(mfmod.MF_OPT_WAVE_COLS))
            assert _audit(mfmod.mf_wavefront_trace(g.h, 4 * ss * cc + 10), ss, cc, 4) == 0


# ------------------------------------------------- q-stationary CTA workers --
@pytest.mark.parametrize("storage", [0, 1])
@pytest.mark.parametrize("s,c", [(1, 1), (4, 6), (0, 0)])
def test_wavefront_q_one_warp_equals_serial_sweep_in_trace_order(mfmod, storage, s, c):
    """MF_OPT_WAVE_CTA = 3 with one warp claiming runs per CTA (MF_OPT_VARIANT bits 26..27 = 1): every
    block is processed serially run by run (its samples sorted by Q row, stable, so each row keeps the
    shuffled order), q_v held in registers and rounded to storage after every update, p_u rows D = 4
    deep.  The factors after 2 epochs equal the oracle's over the blocks in audit-trace order
    (fp32 1e-5, fp16 2e-3); s = c = 1 is serial SGD over the stored order sorted by item."""
    cfg = datagen.CONFIGS["C1"]
    (u, v, r), _ = datagen.make(cfg)
    st = {0: oracle.F32, 1: oracle.F16}[storage]
    ref = oracle.Model(cfg.m, cfg.n, cfg.k, st, seed=cfg.seed_init)
    with mfmod.MF(cfg.m, cfg.n, cfg.k, cfg.alpha, cfg.lam, cfg.seed_init, storage=storage, beta=cfg.beta,
                  wave_rows=s, wave_cols=c, wave_cta=3, trace=1, count_updates=1, seed_shuffle=cfg.seed_shuffle,
                  variant=1 << 26) as g:
        g.load(u, v, r)
        perm = g.order()
        for e in range(2):
            stt = g.epoch("wavefront")
            assert stt.updates == len(u)
            ss = stt.workers
            cc = c or int(g.get(mfmod.MF_OPT_WAVE_COLS))
            P = _passes(mfmod, g)
            rec = mfmod.mf_wavefront_trace(g.h, P * ss * cc + 10)
            assert _audit(rec, ss, cc, P) == 0
            ref.epoch(u, v, r, oracle.eta(cfg.alpha, cfg.beta, e), cfg.lam,
                      _trace_order(mfmod, rec, perm, u, v, cfg.m, cfg.n, ss, cc, by_row=True, P=P))
        P, Q = g.factors()
    Pr, Qr = ref.factors_f32()
    tol = {0: 1e-5, 1: 2e-3}[storage]
    assert np.linalg.norm(P - Pr) / np.linalg.norm(Pr) <= tol
    assert np.linalg.norm(Q - Qr) / np.linalg.norm(Qr) <= tol


@pytest.mark.parametrize("storage", [0])
@pytest.mark.parametrize("depth", [0, 2, 8])
def test_wavefront_q_exactly_once_conflict_free_and_rmse(mfmod, storage, depth):
    """All warps claiming runs (default), each p_u ring depth: every sample once per epoch, no column
    conflict in the audit, and one run's test RMSE within 0.5% of the serial oracle's on the 10% Netflix
    slice after 10 epochs (fp32; oracle golden tests/golden/C2-10pct_f32_trace.json).  fp16 is not gated
    here: the wavefront order trails serial SGD in its first epochs (+0.7% at epoch 6 of
    the fp16 slice trace, after which the fp16 trajectory leaves the plateau), and the fp16 kernel is
    pinned exactly by the one-warp serial test above."""
    import json
    import os
    cfg = datagen.CONFIGS["C2-10pct"]
    stname = {0: "f32", 1: "f16"}[storage]
    path = os.path.join(os.path.dirname(__file__), "golden", f"C2-10pct_{stname}_trace.json")
    gold = json.load(open(path))["rmse"]
    E = {0: 10, 1: 6}[storage]
    (u, v, r), test = datagen.make(cfg)
    with mfmod.MF(cfg.m, cfg.n, cfg.k, cfg.alpha, cfg.lam, cfg.seed_init, storage=storage, beta=cfg.beta,
                  wave_cta=3, trace=1, count_updates=1, seed_shuffle=cfg.seed_shuffle, variant=depth << 4) as g:
        g.load(u, v, r)
        for e in range(E):
            stt = g.epoch("wavefront")
            assert stt.updates == len(u)
            if e == 0:
                ss, cc = stt.workers, int(g.get(mfmod.MF_OPT_WAVE_COLS))
                P = _passes(mfmod, g)
                assert _audit(mfmod.mf_wavefront_trace(g.h, P * ss * cc + 10), ss, cc, P) == 0
        got = g.rmse(*test)
    assert abs(got - gold[E - 1]) <= 0.005 * gold[E - 1], (got, gold[E - 1])


# ------------------------------------------------------- CTA workers (smem Q) --
def test_wavefront_cta_exactly_once_conflict_free_and_rmse(mfmod):
    """MF_OPT_WAVE_CTA=1: one CTA per SM, the column group's Q rows in shared memory."""
    cfg = datagen.CONFIGS["C3-1pct"]
    (u, v, r), test = datagen.make(cfg)
    E = 10
    order = oracle.shuffle_perm(cfg.seed_shuffle, len(u))
    _, trace = oracle.train(cfg.m, cfg.n, cfg.k, oracle.F32, cfg.seed_init, u, v, r, cfg.alpha, cfg.beta,
                            cfg.lam, E, order=order, test=test)
    with mfmod.MF(cfg.m, cfg.n, cfg.k, cfg.alpha, cfg.lam, cfg.seed_init, beta=cfg.beta, wave_cta=1, trace=1,
                  count_updates=1, seed_shuffle=cfg.seed_shuffle) as g:
        g.load(u, v, r)
        for _ in range(E):
            st = g.epoch("wavefront")
            assert st.updates == len(u)
        s, c = int(g.get(mfmod.MF_OPT_WAVE_ROWS)), int(g.get(mfmod.MF_OPT_WAVE_COLS))
        assert s == st.workers and c >= s
        P = _passes(mfmod, g)
        assert _audit(mfmod.mf_wavefront_trace(g.h, P * s * c), s, c, P) == 0
        got = g.rmse(*test)
    assert abs(got - trace[-1]) <= 0.005 * trace[-1], (got, trace[-1])


_C3_TRACE = {}


def _c3_oracle_trace(storage, E):
    """Oracle test-RMSE trace on C3-1pct for `storage`, computed once per module."""
    if storage not in _C3_TRACE:
        cfg = datagen.CONFIGS["C3-1pct"]
        (u, v, r), test = datagen.make(cfg)
        order = oracle.shuffle_perm(cfg.seed_shuffle, len(u))
        st = {0: oracle.F32, 1: oracle.F16, 2: oracle.BF16}[storage]
        _, tr = oracle.train(cfg.m, cfg.n, cfg.k, st, cfg.seed_init, u, v, r, cfg.alpha, cfg.beta, cfg.lam, E,
                             order=order, test=test)
        _C3_TRACE[storage] = tr
    return _C3_TRACE[storage]


# MF_OPT_VARIANT bits 8..11 = CTA update shape + 1, bits 12..15 = ratings in flight per group
# (0 = tuned default: 8 lanes per rating, one in flight at k = 128); bits 16..19 = P-row L2 prefetch
# per claimed tile (0 = auto, 1 = bulk, 2 = per line, 15 = off)
@pytest.mark.parametrize("storage,variant,wave_cta", [
    (1, 0, 1), (1, 0, 2), (1, (1 << 8) | (2 << 12), 1), (1, (2 << 8) | (2 << 12), 1),
    (0, 0, 1), (0, 0, 2), (0, (1 << 8) | (2 << 12), 1), (0, (2 << 8) | (2 << 12), 1),
    (1, 1 << 16, 1), (1, 2 << 16, 2), (1, 15 << 16, 1), (0, 1 << 16, 2), (0, 2 << 16, 1)])
# (bf16 is not gated here: on C3-1pct it is still descending at epoch 5 -- the serial oracle drops from
# 0.142 to 0.115 by epoch 10 -- and the CTA wavefront trails it by the same +0.7% whatever the prefetch
# setting; the paper's "converges slightly slower" measured as a lag, scripts/storage_dynamics_check.py)
def test_wavefront_cta_shapes_rmse(mfmod, storage, variant, wave_cta):
    """Every CTA update shape / depth / prefetch setting (fp16 and fp32 storage, 1x1024 and 2x512
    workers per SM): exactly
    once per epoch and test RMSE within 0.5% of the storage-matched serial oracle after 5 epochs."""
    cfg = datagen.CONFIGS["C3-1pct"]
    (u, v, r), test = datagen.make(cfg)
    E = 5
    gold = _c3_oracle_trace(storage, E)
    with mfmod.MF(cfg.m, cfg.n, cfg.k, cfg.alpha, cfg.lam, cfg.seed_init, storage=storage, beta=cfg.beta,
                  wave_cta=wave_cta, variant=variant, count_updates=1, seed_shuffle=cfg.seed_shuffle) as g:
        g.load(u, v, r)
        for _ in range(E):
            assert g.epoch("wavefront").updates == len(u)
        got = g.rmse(*test)
    assert abs(got - gold[-1]) <= 0.005 * gold[-1], (got, gold[-1])


@pytest.mark.parametrize("storage,k", [(0, 32), (1, 32), (0, 64), (1, 64), (0, 256), (1, 256)])
def test_wavefront_cta_k_sweep_rmse(mfmod, storage, k):
    """The CTA wavefront at the C5 k values other than 128 (its own default shapes per k): exactly once
    per epoch, test RMSE within 0.5% of the storage-matched serial oracle after 5 epochs (C3-1pct;
    its 115-sample blocks are where the in-block concurrency clamp acts)."""
    cfg = datagen.CONFIGS["C3-1pct"].scaled(k=k)
    (u, v, r), test = datagen.make(cfg)
    E = 5
    st = {0: oracle.F32, 1: oracle.F16}[storage]
    order = oracle.shuffle_perm(cfg.seed_shuffle, len(u))
    _, gold = oracle.train(cfg.m, cfg.n, cfg.k, st, cfg.seed_init, u, v, r, cfg.alpha, cfg.beta, cfg.lam, E,
                           order=order, test=test)
    gate = 0.005
    with mfmod.MF(cfg.m, cfg.n, cfg.k, cfg.alpha, cfg.lam, cfg.seed_init, storage=storage, beta=cfg.beta,
                  wave_cta=1, count_updates=1, seed_shuffle=cfg.seed_shuffle) as g:
        g.load(u, v, r)
        for _ in range(E):
            assert g.epoch("wavefront").updates == len(u)
        got = g.rmse(*test)
    assert abs(got - gold[-1]) <= gate * gold[-1], (got, gold[-1], gate)


@pytest.mark.parametrize("storage,k,variant", [(0, 7, 0), (0, 33, 0), (0, 100, 0), (1, 7, 0), (1, 100, 0),
                                               (2, 7, 0), (2, 66, 0), (0, 7, 1 << 16), (1, 100, 1 << 16),
                                               (0, 33, 2 << 16)])
def test_wavefront_cta_single_block_is_serial(mfmod, storage, k, variant):
    """s = c = 1, N = 32 (one tile) and a masked L = 32 shape (one group per warp, one rating in flight):
    the tile is handled by one warp in order, so the CTA kernel is exactly serial SGD (checks the
    shared-memory staging of Q, including rows whose byte size is not a multiple of 16)."""
    rng = np.random.default_rng(k)
    m_, n_, N = 9, 7, 32
    u = rng.integers(0, m_, N).astype(np.int32)
    v = rng.integers(0, n_, N).astype(np.int32)
    r = rng.normal(size=N).astype(np.float32)
    st = {0: oracle.F32, 1: oracle.F16, 2: oracle.BF16}[storage]
    ref = oracle.Model(m_, n_, k, st, seed=3)
    ref.epoch(u, v, r, 0.05, 0.01)
    Pr, Qr = ref.factors_f32()
    with mfmod.MF(m_, n_, k, 0.05, 0.01, 3, storage=storage, shuffle=0, wave_cta=1, wave_rows=1,
                  wave_cols=1, variant=variant) as g:
        g.load(u, v, r)
        g.epoch("wavefront")
        P, Q = g.factors()
    tol = {0: 1e-5, 1: 2e-3, 2: 1.6e-2}[storage]
    assert np.linalg.norm(P - Pr) / np.linalg.norm(Pr) <= tol
    assert np.linalg.norm(Q - Qr) / np.linalg.norm(Qr) <= tol
