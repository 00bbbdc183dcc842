"""Full-size Netflix-shaped parity (BASELINE.json configs[1], N = 99,072,112, k = 128).  -m gpu.

The oracle needs ~2 min (fp32) / ~8 min (fp16) per serial epoch at this size, so its results are
golden files written on the dev box by committed scripts that call only oracle/ and datagen/:
  tests/golden/C2_<st>_trace.json        scripts/make_golden.py       (test RMSE per epoch, 20 epochs)
  tests/golden/C2_<st>_epoch1_rows.npz   scripts/make_golden_rows.py  (sampled rows after epoch 1)
The GPU runs in the launch configuration bench.py times (default workers / variant).
"""
import json
import os

import numpy as np
import pytest

import datagen
import oracle

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")
TOL = {"f32": 1e-5, "f16": 2e-3}


@pytest.fixture(scope="module")
def c2():
    cfg = datagen.CONFIGS["C2"]
    return cfg, datagen.make(cfg)


def _ctx(cfg, storage, **kw):
    from paper_1610_05838_b200 import mf
    variant = 0   # bench.py's default launch configuration (library auto)
    return mf.MF(cfg.m, cfg.n, cfg.k, cfg.alpha, cfg.lam, cfg.seed_init, storage=storage, beta=cfg.beta,
                 seed_shuffle=cfg.seed_shuffle, variant=variant, **kw)


@pytest.mark.parametrize("storage", ["f32", "f16"])
def test_c2_hogwild_rmse_trace_vs_oracle_golden(c2, storage):
    path = os.path.join(GOLD, f"C2_{storage}_trace.json")
    if not os.path.exists(path):
        pytest.skip(f"{path} not generated yet")
    gold = json.load(open(path))["rmse"]
    cfg, ((u, v, r), test) = c2
    with _ctx(cfg, storage, count_updates=1) as g:
        g.load(u, v, r)
        got = []
        for t in range(len(gold)):
            st = g.epoch("hogwild")
            assert st.updates == len(u)
            got.append(g.rmse(*test))
    gate = _gates(storage, gold)
    # north star: every schedule's test RMSE within 0.5% of the oracle's after the same epochs
    assert abs(got[-1] - gold[-1]) <= gate[-1], (got[-1], gold[-1], gate[-1])
    # every earlier epoch of the trace stays within the gate too; after the first epoch (the largest
    # learning rate, where lock-free staleness matters most) batch-Hogwild! is ~1% behind serial
    # (measured +1.07% fp32, +1.09% fp16) and has caught up by the second (+0.01%, +0.16%)
    assert abs(got[0] - gold[0]) <= max(0.02 * gold[0], gate[0]), (got[0], gold[0])
    bad = [(t, a, b, gt) for t, (a, b, gt) in enumerate(zip(got, gold, gate)) if t and abs(a - b) > gt]
    assert not bad, bad


def _gates(storage, gold):
    """Per-epoch gate: 0.5% of the oracle, or the oracle's own spread over shuffle seeds 42/43/44 where
    larger (reading T3).  On the Netflix shape the spread is small (fp32 <= 0.14%, fp16 <= 0.14%
    over 20 epochs, seed 43), so the gate is 0.5% at every epoch."""
    traces = [gold]
    for sd in (43, 44):
        p = os.path.join(GOLD, f"C2_{storage}_seed{sd}_trace.json")
        if os.path.exists(p):
            traces.append(json.load(open(p))["rmse"])
    gates = []
    for t, g in enumerate(gold):
        vals = [tr[t] for tr in traces if len(tr) > t]
        gates.append(max(0.005 * g, max(vals) - min(vals)))
    return gates


@pytest.mark.parametrize("storage", ["f32", "f16"])
def test_c2_wavefront_cta_rmse_trace_vs_oracle_golden(c2, storage):
    """The wavefront schedule with CTA workers (bench.py's throughput configuration) at full size, one run,
    every epoch from the second gated against the oracle's trace (0.5%, or the oracle's own shuffle-seed
    spread where larger: DESIGN.md T3).  Its auto pass count on this shape is 3 (with one
    pass the blocked order trails serial SGD by +265% / +11% after epochs 1 / 2 and wobbles +-0.57% later;
    with three: +1.7% / +0.04% after epochs 1 / 2, then within 0.42% at every epoch to the 20th).  The first
    epoch is checked to be finite and descending, and reported in DESIGN.md, not gated (T6)."""
    path = os.path.join(GOLD, f"C2_{storage}_trace.json")
    if not os.path.exists(path):
        pytest.skip(f"{path} not generated yet")
    gold = json.load(open(path))["rmse"]
    cfg, ((u, v, r), test) = c2
    with _ctx(cfg, storage, count_updates=1, wave_cta=1) as g:
        g.load(u, v, r)
        got = []
        for t in range(len(gold)):
            st = g.epoch("wavefront")
            assert st.updates == len(u)
            got.append(g.rmse(*test))
    assert all(np.isfinite(got)) and got[0] > got[1] > got[2]
    gate = _gates(storage, gold)
    bad = [(t + 1, a, b, gt) for t, (a, b, gt) in enumerate(zip(got, gold, gate)) if t >= 1 and abs(a - b) > gt]
    assert not bad, bad


@pytest.mark.parametrize("storage", ["f32", "f16"])
def test_c2_deterministic_epoch_sampled_rows(c2, storage):
    path = os.path.join(GOLD, f"C2_{storage}_epoch1_rows.npz")
    if not os.path.exists(path):
        pytest.skip(f"{path} not generated yet")
    gold = np.load(path)
    cfg, ((u, v, r), _) = c2
    from paper_1610_05838_b200 import mf
    with _ctx(cfg, storage) as g:
        g.load(u, v, r)
        assert mf.mf_wave_count(g.h) == int(gold["nwaves"])
        g.epoch("deterministic")
        P, Q = g.factors()
    for X, key in ((P, "P"), (Q, "Q")):
        rows = X[gold[f"{key[0].lower()}_idx"]]
        ref = gold[f"{key}_rows"]
        assert np.linalg.norm(rows - ref) / np.linalg.norm(ref) <= TOL[storage]
        assert np.linalg.norm(X.astype(np.float64)) == pytest.approx(float(gold[f"{key}_fro"]), rel=TOL[storage])


def test_c2_rmse_kernel_full_test_set(c2):
    """mf_rmse over the full 1.4M test set == oracle RMSE (fp64 dot) on the same factors."""
    cfg, ((u, v, r), test) = c2
    with _ctx(cfg, "f32") as g:
        g.load(u, v, r)
        g.epoch("hogwild")
        P, Q = g.factors()
        got = g.rmse(*test)
    ref = oracle.Model(cfg.m, cfg.n, cfg.k, oracle.F32, P=P, Q=Q).rmse(*test)
    assert got == pytest.approx(ref, rel=1e-6)


def test_c2_exactly_once_and_order(c2):
    """Full-size load: the A-8 order equals the oracle's permutation; one epoch touches every sample once."""
    cfg, ((u, v, r), _) = c2
    with _ctx(cfg, "f16", count_updates=1) as g:
        g.load(u, v, r)
        np.testing.assert_array_equal(g.order(), oracle.shuffle_perm(cfg.seed_shuffle, len(u)))
        assert g.epoch("hogwild").updates == len(u)
        g.load(u, v, r)  # second load reuses the cached permutation and buffers
        np.testing.assert_array_equal(g.order()[:1000], oracle.shuffle_perm(cfg.seed_shuffle, len(u))[:1000])


# ----------------------------------------------------------- Yahoo!Music shape
# BASELINE.json configs[2]: N = 252,800,275, k = 128, "wavefront-update vs batch-Hogwild!".  Golden
# traces: scripts/make_golden.py C3 <st> 10 (and seed 43 for the order's spread), oracle/ only.
@pytest.fixture(scope="module")
def c3():
    cfg = datagen.CONFIGS["C3"]
    return cfg, datagen.make(cfg)


def _c3_gates(storage, gold):
    traces = [gold]
    p = os.path.join(GOLD, f"C3_{storage}_seed43_trace.json")
    if os.path.exists(p):
        traces.append(json.load(open(p))["rmse"])
    return [max(0.005 * g, max(tr[t] for tr in traces if len(tr) > t) - min(tr[t] for tr in traces if len(tr) > t))
            for t, g in enumerate(gold)]


# fp16 golden: the oracle's -mf16c build (hardware half conversions) at ~7 min per epoch, written late in
# round 2 (scripts/make_golden.py C3 f16 10 [42|43])
@pytest.mark.parametrize("storage", ["f32", "f16"])
@pytest.mark.parametrize("schedule", ["hogwild", "wavefront_cta", "deterministic"])
def test_c3_rmse_trace_vs_oracle_golden(c3, storage, schedule):
    """Yahoo shape, both single-GPU schedules of configs[2], every epoch of the oracle's trace from the
    second on within the gate (0.5%, or the oracle's own shuffle-seed spread where larger).  The first
    epoch (the largest learning rate) is not gated (reading T4): against exact serial SGD it
    is +4.5% for batch-Hogwild! and +34% for the CTA wavefront, whose first epoch walks the matrix
    block by block (the slower start P:256 reports); both are within 0.4% from the second epoch on
    (profiles/r01d_fullsize_traces_vs_serial.jsonl)."""
    path = os.path.join(GOLD, f"C3_{storage}_trace.json")
    if not os.path.exists(path):
        pytest.skip(f"{path} not generated yet")
    gold = json.load(open(path))["rmse"]
    cfg, ((u, v, r), test) = c3
    opts = {"wave_cta": 1} if schedule == "wavefront_cta" else {}
    sched = "wavefront" if opts else schedule
    with _ctx(cfg, storage, count_updates=1, **opts) as g:
        g.load(u, v, r)
        got = []
        for _ in range(len(gold)):
            assert g.epoch(sched).updates == len(u)
            got.append(g.rmse(*test))
    if schedule == "deterministic":  # exact serial SGD (its large-wave execution, 5.3): every epoch at 0.05%
        bad = [(t, a, b) for t, (a, b) in enumerate(zip(got, gold)) if abs(a - b) > 0.0005 * b]
        assert not bad, bad
        return
    gate = _c3_gates(storage, gold)
    bad = [(t, a, b, gt) for t, (a, b, gt) in enumerate(zip(got, gold, gate)) if t >= 1 and abs(a - b) > gt]
    assert not bad, bad


# ------------------------------------------------------------ Hugewiki shape
def test_c4_full_size_exactly_once_beyond_int32():
    """The largest configured problem on one GPU (BASELINE.json configs[3], Hugewiki-shaped: N =
    3,069,817,980 > 2^31 samples, m = 50M rows, P = 12.8 GB in fp16): batch-Hogwild! and the CTA
    wavefront each process every sample exactly once per epoch (64-bit sample counts, offsets and row
    addresses) and the test RMSE improves on the initial factors'."""
    cfg = datagen.CONFIGS["C4"]
    (u, v, r), test = datagen.make(cfg)
    assert len(u) > 2 ** 31
    with _ctx(cfg, "f16", count_updates=1, shuffle=0) as g:
        g.load(u, v, r)
        r0 = g.rmse(*test)
        assert g.epoch("hogwild").updates == len(u)
        r1 = g.rmse(*test)
        from paper_1610_05838_b200 import mf
        g.set(mf.MF_OPT_WAVE_CTA, 1)
        assert g.epoch("wavefront").updates == len(u)
        r2 = g.rmse(*test)
    assert r1 < 0.5 * r0 and r2 < r1, (r0, r1, r2)


def test_c4_full_size_schedules_track_serial_sgd():
    """BASELINE.json configs[3] at FULL size on one GPU (3.07B ratings; the serial CPU oracle would need
    ~2.5 hours per epoch): exact serial SGD is the deterministic schedule (pinned to the oracle's factors at
    1e-5 / 2e-3 on the slices, and to its test RMSE at 0.001% on the C4-rows100 slice), and batch-Hogwild!
    and the partitioned schedule at G = 2 / 4 / 8 loopback partitions -- the per-partition worker counts,
    passes and Latin squares G GPUs would run -- must be within 0.5% of its test RMSE from the 4th epoch
    (fp16).  With the round-1 fixed 4 passes per epoch the partitioned schedule was +59% / +8.7% / +3.5%
    behind after 10 epochs; the auto pass count caps a Q row's updates per visit."""
    from paper_1610_05838_b200 import mf
    cfg = datagen.CONFIGS["C4"]
    (u, v, r), test = datagen.make(cfg)
    E = 5
    traces = {}
    for name, sched, opts in (("serial", "deterministic", {}), ("hogwild", "hogwild", {}),
                              ("G2", "partitioned", {"partitions": 2}), ("G4", "partitioned", {"partitions": 4}),
                              ("G8", "partitioned", {"partitions": 8})):
        with _ctx(cfg, "f16", count_updates=1, shuffle=0, **opts) as g:
            g.load(u, v, r)
            tr = []
            for _ in range(E):
                assert g.epoch(sched).updates == len(u)
                tr.append(g.rmse(*test))
            if sched == "partitioned":  # the auto pass count in use: ceil(N / (n G 1000)) >= 4
                G = opts["partitions"]
                assert int(g.get(mf.MF_OPT_SUBEPOCHS)) == max(4, -(-len(u) // (cfg.n * G * 1000)))
        traces[name] = tr
    ref = traces.pop("serial")
    bad = [(name, t + 1, a, b) for name, tr in traces.items() for t, (a, b) in enumerate(zip(tr, ref))
           if t >= 3 and abs(a - b) > 0.005 * b]
    assert not bad, (bad, traces, ref)


# ------------------------------------------------- Hugewiki shape, parity slice
# the C4 parity config is C4-rows/10 (m = 5,008,260, n = 39,781 kept, N = 306,981,798).
# Golden: scripts/make_golden.py C4-rows10 f32 10 (and seed 43), oracle/ only.
@pytest.fixture(scope="module")
def c4r10():
    cfg = datagen.CONFIGS["C4-rows10"]
    return cfg, datagen.make(cfg)


@pytest.mark.parametrize("storage,schedule,G,split", [
    ("f32", "hogwild", 1, 0), ("f32", "partitioned", 2, 2), ("f32", "partitioned", 4, 2), ("f32", "partitioned", 8, 2),
    ("f32", "partitioned", 2, 0), ("f32", "partitioned", 4, 0), ("f32", "partitioned", 8, 0),
    pytest.param("f32", "partitioned", 4, 1, marks=pytest.mark.xfail(
        strict=False, reason="the pipelined half-segment form (MF_OPT_PART_SPLIT = 1, an option) puts a launch's "
                             "7,674 in-flight ratings on half of a 9,945-column Q segment (kappa 1.5, so the Q rows "
                             "are stored): +0.69..0.74% after 10 epochs (DESIGN.md 5.5, A-20)")),
    ("f16", "hogwild", 1, 0), ("f16", "partitioned", 2, 2), ("f16", "partitioned", 4, 2), ("f16", "partitioned", 8, 2)])
def test_c4_rows10_rmse_vs_oracle_golden(c4r10, storage, schedule, G, split):
    """BASELINE.json configs[3] (R-block grid partition at 2 / 4 / 8 GPUs) at its parity size: the
    partitioned schedule with G partitions (the loopback transport: the same layout, Latin-square
    rounds, passes and unit hand-overs as G GPUs, run on this one) and batch-Hogwild! end the oracle's
    10 epochs within 0.5% of its test RMSE (the north star's gate, "after the same number of epochs"),
    in fp32 and in the paper's half precision.  The model is still descending there (-0.5% per
    epoch), so a schedule's lag shows as its deviation; earlier epochs are reported in DESIGN.md 5.5, not
    gated.  The pipelined half-segment form (an option) doubles the ratings in flight per Q column and
    lags more than the gate at G = 4."""
    path = os.path.join(GOLD, f"C4-rows10_{storage}_trace.json")
    if not os.path.exists(path):
        pytest.skip(f"{path} not generated yet")
    gold = json.load(open(path))["rmse"]
    cfg, ((u, v, r), test) = c4r10
    opts = {"partitions": G, "part_split": split} if schedule == "partitioned" else {}
    with _ctx(cfg, storage, count_updates=1, **opts) as g:
        g.load(u, v, r)
        for _ in range(len(gold)):
            assert g.epoch(schedule).updates == len(u)
        got = g.rmse(*test)
    assert abs(got - gold[-1]) <= 0.005 * gold[-1], (got, gold[-1], (got - gold[-1]) / gold[-1])
