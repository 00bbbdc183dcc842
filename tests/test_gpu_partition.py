"""Partitioned schedule through libmf's loopback transport on one GPU.  -m gpu.

The loopback runs the G partitions of the multi-GPU path on one device and moves Q segments with
device copies following the same round / peer schedule the NCCL transport uses (see
tests/test_partition_host.py for that schedule's algebra over gloo).
"""
import numpy as np
import pytest

import datagen
import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mf():
    from paper_1610_05838_b200 import mf
    return mf


def _block_sweep_order(mf, perm, u, v, m, n, G, seed, e, S=4, split=0):
    """Caller indices in processing order: pass s (stored positions [s N/S, (s+1) N/S)) -> round ->
    partition -> block samples in stored order (split = 1: the lower half of the block's columns, then
    the upper half); pass s of epoch e uses Latin square e*S + s.  split = 2 (unit grid): pass -> round
    -> family h -> partition g -> the samples of unit (sigma_h(g, round), h), the half h of that segment
    (with one worker the two families of a round run one after the other, family 0 first)."""
    us, vs = u[perm], v[perm]
    N = len(perm)
    pas = (np.arange(N) * S) // N
    rs = [mf.mf_segment(m, G, g) for g in range(G)]
    cs = [mf.mf_segment(n, G, c) for c in range(G)]
    out = []

    def half(c, h):
        mid = cs[c][0] + (cs[c][1] - cs[c][0]) // 2
        return (cs[c][0], mid) if h == 0 else (mid, cs[c][1])

    for s in range(S):
        for rnd in range(G):
            if split == 2:
                for h in (0, 1):
                    for g in range(G):
                        lo, hi = half(mf.mf_round_unit(seed, e * S + s, G, rnd, g, h), h)
                        sel = (pas == s) & (us >= rs[g][0]) & (us < rs[g][1]) & (vs >= lo) & (vs < hi)
                        out.append(perm[np.nonzero(sel)[0]])
                continue
            for g in range(G):
                c = mf.mf_round_segment(seed, e * S + s, G, rnd, g)
                for lo, hi in ((half(c, 0), half(c, 1)) if split else ((cs[c][0], cs[c][1]),)):
                    sel = (pas == s) & (us >= rs[g][0]) & (us < rs[g][1]) & (vs >= lo) & (vs < hi)
                    out.append(perm[np.nonzero(sel)[0]])
    return np.concatenate(out)


@pytest.mark.parametrize("split", [0, 1, 2])
@pytest.mark.parametrize("G", [1, 2, 3, 4])
@pytest.mark.parametrize("storage", [0, 1])
def test_loopback_serial_blocks_match_oracle_block_sweep(mf, G, storage, split):
    cfg = datagen.CONFIGS["C1"]
    (u, v, r), test = datagen.make(cfg)
    E = 2
    st = {0: oracle.F32, 1: oracle.F16}[storage]
    with mf.MF(cfg.m, cfg.n, cfg.k, cfg.alpha, cfg.lam, cfg.seed_init, storage=storage, beta=cfg.beta,
               seed_shuffle=cfg.seed_shuffle, partitions=G, workers=1, count_updates=1, part_split=split) as g:
        g.load(u, v, r)
        perm = g.order()
        for _ in range(E):
            s = g.epoch("partitioned")
            assert s.updates == len(u)
        P, Q = g.factors()
        got_rmse = g.rmse(*test)
    ref = oracle.Model(cfg.m, cfg.n, cfg.k, st, seed=cfg.seed_init)
    for e in range(E):
        ref.epoch(u, v, r, oracle.eta(cfg.alpha, cfg.beta, e), cfg.lam,
                  _block_sweep_order(mf, perm, u, v, cfg.m, cfg.n, G, cfg.seed_shuffle, e, split=split))
    Pr, Qr = ref.factors_f32()
    tol = {0: 1e-5, 1: 2e-3}[storage]
    assert np.linalg.norm(P - Pr) / np.linalg.norm(Pr) <= tol
    assert np.linalg.norm(Q - Qr) / np.linalg.norm(Qr) <= tol
    assert got_rmse == pytest.approx(ref.rmse(*test), rel=tol)


@pytest.mark.parametrize("split", [0, 2])
def test_layout_change_between_partitioned_epochs_keeps_q(mf, split):
    """Changing a layout option (MF_OPT_SUBEPOCHS) between partitioned epochs rebuilds the layout; the
    current Q, which lives only in the partitions' segment buffers after an epoch, must be gathered
    first.  Exact mode: epoch 0 with S = 4, epoch 1 with S = 2 equals the oracle over the
    reconstructed orders (fp32, 1e-5)."""
    cfg = datagen.CONFIGS["C1"]
    (u, v, r), test = datagen.make(cfg)
    G = 3
    with mf.MF(cfg.m, cfg.n, cfg.k, cfg.alpha, cfg.lam, cfg.seed_init, beta=cfg.beta, seed_shuffle=cfg.seed_shuffle,
               partitions=G, workers=1, count_updates=1, part_split=split, subepochs=4) as g:
        g.load(u, v, r)
        perm = g.order()
        assert g.epoch("partitioned").updates == len(u)
        g.set(mf.MF_OPT_SUBEPOCHS, 2)
        assert g.epoch("partitioned").updates == len(u)
        P, Q = g.factors()
    ref = oracle.Model(cfg.m, cfg.n, cfg.k, oracle.F32, seed=cfg.seed_init)
    for e, S in ((0, 4), (1, 2)):
        ref.epoch(u, v, r, oracle.eta(cfg.alpha, cfg.beta, e), cfg.lam,
                  _block_sweep_order(mf, perm, u, v, cfg.m, cfg.n, G, cfg.seed_shuffle, e, S=S, split=split))
    assert np.linalg.norm(P - ref.P) / np.linalg.norm(ref.P) <= 1e-5
    assert np.linalg.norm(Q - ref.Q) / np.linalg.norm(ref.Q) <= 1e-5


def test_loopback_hogwild_rmse_within_half_percent(mf):
    cfg = datagen.CONFIGS["C2-1pct"]
    (u, v, r), test = datagen.make(cfg)
    E, G = 10, 4
    order = oracle.shuffle_perm(cfg.seed_shuffle, len(u))
    _, trace = oracle.train(cfg.m, cfg.n, cfg.k, oracle.F32, cfg.seed_init, u, v, r, cfg.alpha, cfg.beta, cfg.lam,
                            E, order=order, test=test)
    with mf.MF(cfg.m, cfg.n, cfg.k, cfg.alpha, cfg.lam, cfg.seed_init, beta=cfg.beta,
               seed_shuffle=cfg.seed_shuffle, partitions=G, count_updates=1) as g:
        g.load(u, v, r)
        for _ in range(E):
            assert g.epoch("partitioned").updates == len(u)
        got = g.rmse(*test)
    assert abs(got - trace[-1]) <= 0.005 * trace[-1], (got, trace[-1])


def test_switching_schedules_keeps_one_consistent_model(mf):
    """partitioned -> hogwild -> partitioned -> set_factors: Q segments and the full Q stay in sync."""
    cfg = datagen.CONFIGS["C1"]
    (u, v, r), test = datagen.make(cfg)
    with mf.MF(cfg.m, cfg.n, cfg.k, cfg.alpha, cfg.lam, cfg.seed_init, beta=cfg.beta, partitions=3,
               workers=1) as g:
        g.load(u, v, r)
        g.epoch("partitioned")
        P1, Q1 = g.factors()
        g.epoch("deterministic")
        g.epoch("partitioned")
        rm = g.rmse(*test)
        g.set_factors(P1, Q1)
        P2, Q2 = g.factors()
        np.testing.assert_array_equal(P2, P1)
        np.testing.assert_array_equal(Q2, Q1)
        g.epoch("partitioned")
        assert g.rmse(*test) < 1.0 and rm < 1.0


def test_nccl_single_rank_path(mf):
    """The NCCL transport with world = 1 (the only size one GPU allows): attach, local-row layout, rotation
    (a no-op), all-gather of Q and the all-reduced RMSE must reproduce the loopback G = 1 result."""
    cfg = datagen.CONFIGS["C1"]
    (u, v, r), test = datagen.make(cfg)
    res = []
    for use_nccl in (False, True):
        g = mf.MF(cfg.m, cfg.n, cfg.k, cfg.alpha, cfg.lam, cfg.seed_init, beta=cfg.beta,
                  seed_shuffle=cfg.seed_shuffle, workers=1, **({} if use_nccl else {"partitions": 1}))
        if use_nccl:
            mf.mf_attach_nccl(g.h, mf.mf_nccl_unique_id(), 0, 1)
        g.load(u, v, r)
        for _ in range(2):
            g.epoch("partitioned")
        res.append(g.factors() + (g.rmse(*test),))
        if use_nccl:
            with pytest.raises(mf.MFError):
                g.epoch("hogwild")  # only the partitioned schedule is collective-safe
        g.close()
    np.testing.assert_array_equal(res[0][0], res[1][0])
    np.testing.assert_array_equal(res[0][1], res[1][1])
    assert res[0][2] == res[1][2]
