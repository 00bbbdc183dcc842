"""Pins for the CPU oracle (tests -m "not gpu").

Each test checks the oracle against something other than itself: a
hand-worked example (exact rationals), SPEC's printed examples, a finite
difference of the objective, closed forms, brute force, numpy's IEEE
conversions, or a statistical property the mathematics fixes.
"""
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import datagen
import oracle
from oracle import F16, F32, BF16, F64

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _fr(x):
    return Fraction(x)


# ---------------------------------------------------------------- P-1 -----
def _p1():
    with open(os.path.join(GOLD, "p1_worked_example.json")) as f:
        return json.load(f)


def _fractions_sgd(g):
    """Independent exact re-derivation of the worked example."""
    P = [[_fr(x) for x in row] for row in g["P0"]]
    Q = [[_fr(x) for x in row] for row in g["Q0"]]
    eta, lam = _fr(g["eta"]), _fr(g["lambda"])
    steps = []
    for u, v, r in g["samples"]:
        p, q = P[u][:], Q[v][:]
        pred = sum(a * b for a, b in zip(p, q))
        e = _fr(r) - pred
        P[u] = [p[d] + eta * (e * q[d] - lam * p[d]) for d in range(g["k"])]
        Q[v] = [q[d] + eta * (e * p[d] - lam * q[d]) for d in range(g["k"])]
        steps.append((pred, e, P[u][:], Q[v][:]))
    return P, Q, steps


def test_p1_golden_is_consistent_with_exact_rationals():
    g = _p1()
    P, Q, steps = _fractions_sgd(g)
    for (pred, e, pu, qv), s in zip(steps, g["steps"]):
        assert pred == _fr(s["pred"]) and e == _fr(s["err"])
        assert pu == [_fr(x) for x in s["p_u"]] and qv == [_fr(x) for x in s["q_v"]]
    assert P == [[_fr(x) for x in row] for row in g["P_final"]]
    assert Q == [[_fr(x) for x in row] for row in g["Q_final"]]


@pytest.mark.parametrize("storage", [F32, F16, F64])
def test_p1_worked_example_exact(storage):
    g = _p1()
    P0 = np.array([[float(_fr(x)) for x in row] for row in g["P0"]])
    Q0 = np.array([[float(_fr(x)) for x in row] for row in g["Q0"]])
    dt = oracle.STORAGE_DTYPE[storage]
    if storage == F16:
        P0s, Q0s = P0.astype(np.float16).view(np.uint16), Q0.astype(np.float16).view(np.uint16)
    else:
        P0s, Q0s = P0.astype(dt), Q0.astype(dt)
    m = oracle.Model(4, 4, 2, storage, P=P0s, Q=Q0s)
    u = np.array([s[0] for s in g["samples"]], np.int32)
    v = np.array([s[1] for s in g["samples"]], np.int32)
    r = np.array([float(_fr(s[2])) for s in g["samples"]], np.float32)
    assert m.epoch(u, v, r, 0.25, 0.5) == 0
    P, Q = oracle.widen(m.P, storage), oracle.widen(m.Q, storage)
    Pe = np.array([[float(_fr(x)) for x in row] for row in g["P_final"]])
    Qe = np.array([[float(_fr(x)) for x in row] for row in g["Q_final"]])
    np.testing.assert_array_equal(P, Pe)
    np.testing.assert_array_equal(Q, Qe)
    tu = np.array([t[0] for t in g["test"]], np.int32)
    tv = np.array([t[1] for t in g["test"]], np.int32)
    tr = np.array([float(_fr(t[2])) for t in g["test"]], np.float32)
    assert m.rmse(tu, tv, tr) == pytest.approx(math.sqrt(1 / 8), abs=0, rel=1e-15)


def _round_bf16(x: Fraction) -> Fraction:
    """Exact round-to-nearest-even of a rational to bfloat16 (8 significand bits), no float involved."""
    if x == 0:
        return Fraction(0)
    sign = -1 if x < 0 else 1
    a = abs(x)
    e = a.numerator.bit_length() - a.denominator.bit_length()
    if Fraction(2) ** e > a:
        e -= 1
    ulp = Fraction(2) ** (e - 7)
    q, rem = divmod(a, ulp)
    if rem * 2 > ulp or (rem * 2 == ulp and q % 2 == 1):
        q += 1
    return sign * q * ulp


def test_p1_worked_example_bf16_storage():
    """bf16 storage pin: the same three updates in exact rationals, each stored value rounded to bf16
    by an exact nearest-even rule (the dyadic intermediates are exact in the oracle's fp32 math)."""
    g = _p1()
    P0 = [[_round_bf16(_fr(x)) for x in row] for row in g["P0"]]
    Q0 = [[_round_bf16(_fr(x)) for x in row] for row in g["Q0"]]
    P, Q = [row[:] for row in P0], [row[:] for row in Q0]
    eta, lam = _fr(g["eta"]), _fr(g["lambda"])
    for u, v, r in g["samples"]:
        p, q = P[u][:], Q[v][:]
        e = _fr(r) - sum(a * b for a, b in zip(p, q))
        P[u] = [_round_bf16(p[d] + eta * (e * q[d] - lam * p[d])) for d in range(2)]
        Q[v] = [_round_bf16(q[d] + eta * (e * p[d] - lam * q[d])) for d in range(2)]
    bf = lambda rows: (np.array([[float(x) for x in row] for row in rows], np.float32).view(np.uint32) >> 16  # noqa
                       ).astype(np.uint16)
    m = oracle.Model(4, 4, 2, BF16, P=bf(P0), Q=bf(Q0))
    u = np.array([s[0] for s in g["samples"]], np.int32)
    v = np.array([s[1] for s in g["samples"]], np.int32)
    r = np.array([float(_fr(s[2])) for s in g["samples"]], np.float32)
    assert m.epoch(u, v, r, 0.25, 0.5) == 0
    Pw, Qw = oracle.widen(m.P, BF16), oracle.widen(m.Q, BF16)
    np.testing.assert_array_equal(Pw, np.array([[float(x) for x in row] for row in P], np.float32))
    np.testing.assert_array_equal(Qw, np.array([[float(x) for x in row] for row in Q], np.float32))
    assert Qw[1, 1] != float(_fr("1479/2048"))  # bf16 rounding is visible in this example


def test_p1_discriminates_snapshot_reading():
    """Reading A-1: under the sequential reading step 1 would give Q0=[11/16, 67/64]."""
    g = _p1()
    m = oracle.Model(4, 4, 2, F32, P=np.array([[1, .5], [.5, 1], [1, 0], [0, 1]], np.float32),
                     Q=np.array([[.5, 1], [1, .5], [1, 1], [0, .5]], np.float32))
    m.epoch(np.array([0], np.int32), np.array([0], np.int32), np.array([2], np.float32), 0.25, 0.5)
    seq = [float(_fr(x)) for x in g["sequential_reading_Q0_after_step1"]]
    assert list(m.Q[0]) != seq
    assert list(m.Q[0]) == [11 / 16, 1.0]


# ---------------------------------------------------------------- P-2 -----
@pytest.mark.parametrize("lam,pe,qe", [(0.0, [1.0, 0.1], [0.1, 1.0]), (0.05, [0.995, 0.1], [0.1, 0.995])])
def test_p2_spec_examples(lam, pe, qe):
    """SPEC.md:74-75 (core-model sgd_update examples)."""
    m = oracle.Model(1, 1, 2, F64, P=np.array([[1.0, 0.0]]), Q=np.array([[0.0, 1.0]]))
    m.epoch(np.zeros(1, np.int32), np.zeros(1, np.int32), np.ones(1, np.float32), 0.1, lam)
    np.testing.assert_allclose(m.P[0], pe, rtol=0, atol=1e-15)
    np.testing.assert_allclose(m.Q[0], qe, rtol=0, atol=1e-15)


def test_p2_zero_error_zero_lambda_is_identity():
    """err = 0 with lambda = 0 leaves p, q bit-identical."""
    p = np.array([[0.5, 0.25, 0.125, 1.0]], np.float32)
    q = np.array([[1.0, 2.0, 4.0, 0.5]], np.float32)
    r = np.array([float(p[0] @ q[0])], np.float32)
    m = oracle.Model(1, 1, 4, F32, P=p, Q=q)
    m.epoch(np.zeros(1, np.int32), np.zeros(1, np.int32), r, 0.3, 0.0)
    np.testing.assert_array_equal(m.P, p)
    np.testing.assert_array_equal(m.Q, q)


def test_spec_predict_examples():
    """predict([.5]*4, [1,2,3,4]) = 5 (the dot is the rmse residual)."""
    m = oracle.Model(1, 1, 4, F32, P=np.full((1, 4), 0.5, np.float32),
                     Q=np.array([[1, 2, 3, 4]], np.float32))
    assert m.rmse(np.zeros(1, np.int32), np.zeros(1, np.int32), np.zeros(1, np.float32)) == 5.0


# ---------------------------------------------------------------- P-3 -----
def test_p3_update_is_gradient_step_of_objective():
    """Reading A-3: (x' - x)/(-eta) == dL/dx for L = 1/2 e^2 + 1/2 lam (|p|^2+|q|^2),
    checked by central finite differences of the oracle's objective in fp64."""
    rng = np.random.default_rng(3)
    k, lam, eta, h = 6, 0.07, 1e-3, 1e-5
    for _ in range(5):
        p0 = rng.normal(size=(1, k))
        q0 = rng.normal(size=(1, k))
        r = np.array([rng.normal()], np.float32)
        z = np.zeros(1, np.int32)
        m = oracle.Model(1, 1, k, F64, P=p0, Q=q0)
        m.epoch(z, z, r, eta, lam)
        g_upd = np.concatenate([(p0 - m.P)[0], (q0 - m.Q)[0]]) / eta
        g_fd = np.zeros(2 * k)
        for j in range(2 * k):
            for sgn in (+1, -1):
                P, Q = p0.copy(), q0.copy()
                (P if j < k else Q)[0, j % k] += sgn * h
                L = oracle.Model(1, 1, k, F64, P=P, Q=Q).loss(z, z, r, lam)
                g_fd[j] += sgn * L / (2 * h)
        np.testing.assert_allclose(g_upd, g_fd, rtol=1e-6, atol=1e-8)


def test_loss_matches_bruteforce():
    rng = np.random.default_rng(5)
    m_, n_, k = 7, 5, 3
    P, Q = rng.normal(size=(m_, k)), rng.normal(size=(n_, k))
    u, v = rng.integers(0, m_, 20).astype(np.int32), rng.integers(0, n_, 20).astype(np.int32)
    r = rng.normal(size=20).astype(np.float32)
    want = sum(0.5 * (float(r[i]) - P[u[i]] @ Q[v[i]]) ** 2 + 0.5 * 0.1 * (P[u[i]] @ P[u[i]] + Q[v[i]] @ Q[v[i]])
               for i in range(20))
    assert oracle.Model(m_, n_, k, F64, P=P, Q=Q).loss(u, v, r, 0.1) == pytest.approx(want, rel=1e-13)


# ---------------------------------------------------------------- P-4 -----
def test_p4_lr_schedule():
    """SPEC.md:55-57; PAPER.md:388 (§5.1)."""
    assert oracle.lr(0.08, 0.3, 0) == 0.08
    assert oracle.lr(0.08, 0.3, 1) == pytest.approx(0.08 / 1.3, rel=1e-15)
    assert oracle.lr(0.08, 0.3, 1) == pytest.approx(0.0615385, abs=5e-8)
    assert oracle.lr(0.08, 0.2, 4) == pytest.approx(0.08 / 2.6, rel=1e-15)  # t^1.5 = 8
    assert oracle.lr(0.08, 0.2, 4) == pytest.approx(0.0307692, abs=5e-8)
    seq = [oracle.lr(0.08, 0.3, t) for t in range(101)]
    assert all(a > b for a, b in zip(seq, seq[1:]))
    assert all(oracle.lr(0.05, 0.0, t) == 0.05 for t in range(20))
    assert oracle.eta(0.08, 0.3, 1) == np.float32(0.08 / 1.3)


# ---------------------------------------------------------------- P-5 -----
def test_p5_rmse_examples_and_bruteforce():
    """SPEC.md:91-93 and fp64 brute force."""
    z = np.zeros(1, np.int32)
    m = oracle.Model(1, 1, 2, F32, P=np.array([[1, 0]], np.float32), Q=np.array([[1, 0]], np.float32))
    assert m.rmse(z, z, np.ones(1, np.float32)) == 0.0
    m0 = oracle.Model(1, 1, 2, F32, P=np.zeros((1, 2), np.float32), Q=np.zeros((1, 2), np.float32))
    assert m0.rmse(z, z, np.ones(1, np.float32)) == 1.0
    assert m0.rmse(np.zeros(2, np.int32), np.zeros(2, np.int32), np.array([3, 4], np.float32)) == \
        pytest.approx(math.sqrt(12.5), rel=1e-15)
    assert m0.rmse(z[:0], z[:0], np.zeros(0, np.float32)) == -1.0  # empty -> error
    rng = np.random.default_rng(0)
    P, Q = rng.normal(size=(30, 9)).astype(np.float32), rng.normal(size=(20, 9)).astype(np.float32)
    u, v = rng.integers(0, 30, 500).astype(np.int32), rng.integers(0, 20, 500).astype(np.int32)
    r = rng.normal(size=500).astype(np.float32)
    want = math.sqrt(np.mean((r.astype(np.float64) - np.einsum("ij,ij->i", P[u].astype(np.float64),
                                                                 Q[v].astype(np.float64))) ** 2))
    assert oracle.Model(30, 20, 9, F32, P=P, Q=Q).rmse(u, v, r) == pytest.approx(want, rel=1e-12)


# ---------------------------------------------------------------- P-6 -----
@pytest.mark.parametrize("name,gate_sigmas", [("tiny-selfcheck", 1.25), ("C1-selfcheck", 1.5)])
def test_p6_planted_recovery_reaches_noise_floor(name, gate_sigmas):
    """Brute-force recovery of a planted low-rank matrix (k = planted rank), SURVEY §8(c) P-6."""
    cfg = datagen.CONFIGS[name]
    (u, v, r), test = datagen.make(cfg)
    _, trace = oracle.train(cfg.m, cfg.n, cfg.k, F32, cfg.seed_init, u, v, r, cfg.alpha, cfg.beta, cfg.lam,
                            cfg.epochs, test=test)
    assert trace[-1] <= gate_sigmas * cfg.sigma, trace[-5:]


# ---------------------------------------------------------------- P-7 -----
def test_p7_training_loss_monotone_on_decaying_schedule():
    """C1 with Table 3 Netflix parameters: train RMSE strictly decreases per epoch."""
    cfg = datagen.CONFIGS["C1"]
    (u, v, r), _ = datagen.make(cfg)
    m = oracle.Model(cfg.m, cfg.n, cfg.k, F32, seed=cfg.seed_init)
    prev = m.rmse(u, v, r)
    for t in range(cfg.epochs):
        assert m.epoch(u, v, r, oracle.eta(cfg.alpha, cfg.beta, t), cfg.lam) == 0
        cur = m.rmse(u, v, r)
        assert cur < prev, (t, cur, prev)
        prev = cur


# ---------------------------------------------------------------- P-8 -----
def test_p8_fp16_exhaustive_roundtrip_and_numpy_rne():
    L = oracle.lib()
    allh = np.arange(65536, dtype=np.uint32)
    f = np.array([L.orc_f16_to_f32(int(h)) for h in allh], np.float32)
    np.testing.assert_array_equal(f, allh.astype(np.uint16).view(np.float16).astype(np.float32))
    back = np.array([L.orc_f32_to_f16(float(x)) for x in f], np.uint32)
    fin = np.isfinite(f)
    np.testing.assert_array_equal(back[fin], allh[fin])
    # RNE ties (hand cases) and a random fp32 sweep against numpy's IEEE conversion
    assert L.orc_f32_to_f16(1 + 2 ** -11) == 0x3C00
    assert L.orc_f32_to_f16(1 + 3 * 2 ** -11) == np.float16(1 + 2 ** -9).view(np.uint16)
    rng = np.random.default_rng(1)
    bits = rng.integers(0, 2 ** 32, 20000, dtype=np.uint64).astype(np.uint32)
    xs = bits.view(np.float32)
    xs = xs[np.isfinite(xs)]
    got = np.array([L.orc_f32_to_f16(float(x)) for x in xs], np.uint16)
    with np.errstate(over="ignore"):
        np.testing.assert_array_equal(got, xs.astype(np.float16).view(np.uint16))


def _bf16_rne_reference(x):
    """Nearest bf16 by exact distance comparison in fp64, ties to even (independent of the bit recipe)."""
    b = x.view(np.uint32)
    lo = (b & 0xFFFF0000).view(np.float32).astype(np.float64)
    hi = ((b & 0xFFFF0000) + 0x10000).astype(np.uint32).view(np.float32).astype(np.float64)
    xd = x.astype(np.float64)
    dl, dh = np.abs(xd - lo), np.abs(hi - xd)
    even_lo = ((b >> 16) & 1) == 0
    pick_hi = (dh < dl) | ((dh == dl) & ~even_lo)
    return np.where(pick_hi, (b >> 16) + 1, b >> 16).astype(np.uint16)


def test_p8_bf16_exhaustive_roundtrip_and_rne():
    L = oracle.lib()
    for h in range(0, 65536, 7):
        x = L.orc_bf16_to_f32(h)
        if math.isfinite(x):
            assert L.orc_f32_to_bf16(x) == h
    assert L.orc_f32_to_bf16(1 + 2 ** -8) == 0x3F80  # tie -> even
    assert L.orc_f32_to_bf16(1 + 3 * 2 ** -8) == 0x3F82
    rng = np.random.default_rng(2)
    bits = rng.integers(0, 2 ** 32, 20000, dtype=np.uint64).astype(np.uint32)
    xs = bits.view(np.float32)
    xs = xs[np.isfinite(xs) & (np.abs(xs) < 3e38)]
    got = np.array([L.orc_f32_to_bf16(float(x)) for x in xs], np.uint16)
    np.testing.assert_array_equal(got, _bf16_rne_reference(xs))
    assert math.isnan(L.orc_bf16_to_f32(L.orc_f32_to_bf16(float("nan"))))


@pytest.mark.skipif(not oracle.host_has_f16c(), reason="host CPU has no F16C")
def test_f16c_golden_build_is_bitwise_the_plain_build():
    """The golden-writing build (-mf16c: hardware vcvtps2ph / vcvtph2ps for the _Float16 casts) gives
    the plain build's bits: every binary16 pattern widened, sampled fp32 patterns (ties, subnormal
    and overflow ranges) narrowed, and whole fp16 / bf16 epochs on C1 plus the test RMSE."""
    A, B = oracle.load(False), oracle.load(True)
    for h in range(65536):
        x, y = A.orc_f16_to_f32(h), B.orc_f16_to_f32(h)
        assert (x == y) or (math.isnan(x) and math.isnan(y)), h
    rng = np.random.default_rng(3)
    bits = np.concatenate([rng.integers(0, 2 ** 32, 60000, dtype=np.uint64).astype(np.uint32),
                           (np.arange(0x33000000, 0x47800000, 0x1001, dtype=np.uint32))])
    xs = bits.view(np.float32)
    for x in xs[np.isfinite(xs)]:
        assert A.orc_f32_to_f16(float(x)) == B.orc_f32_to_f16(float(x)), float(x)
    cfg = datagen.CONFIGS["C1"]
    (u, v, r), (tu, tv, tr) = datagen.make(cfg)
    order = oracle.shuffle_perm(cfg.seed_shuffle, len(u))
    c = oracle._c
    u, v, r, tu, tv, tr, order = (c(u, np.int32), c(v, np.int32), c(r, np.float32), c(tu, np.int32),
                                  c(tv, np.int32), c(tr, np.float32), c(order, np.int64))
    for st in (F16, BF16):
        fac = []
        for L in (A, B):
            P, Q = oracle.init(cfg.seed_init, cfg.m, cfg.k, 0, st), oracle.init(cfg.seed_init, cfg.n, cfg.k, 1, st)
            for t in range(3):
                assert L.orc_epoch(cfg.k, st, P.ctypes.data, Q.ctypes.data, u.ctypes.data, v.ctypes.data,
                                   r.ctypes.data, order.ctypes.data, len(u), oracle.eta(cfg.alpha, cfg.beta, t),
                                   cfg.lam) == 0
            fac.append((P, Q, L.orc_rmse(cfg.k, st, P.ctypes.data, Q.ctypes.data, tu.ctypes.data, tv.ctypes.data,
                                         tr.ctypes.data, len(tu))))
        np.testing.assert_array_equal(fac[0][0], fac[1][0])
        np.testing.assert_array_equal(fac[0][1], fac[1][1])
        assert fac[0][2] == fac[1][2]


# ------------------------------------------------------- init / shuffle -----
def test_splitmix64_published_vectors():
    """SplitMix64 (Steele, Lea, Flood 2014) from state 1234567: Vigna's reference sequence."""
    L = oracle.lib()
    g = 0x9E3779B97F4A7C15
    want = [6457827717110365317, 3203168211198807973, 9817491932198370423, 4593380528125082431,
            16408922859458223821]
    got = [L.orc_splitmix64((1234567 + i * g) % 2 ** 64) for i in range(5)]
    assert got == want


def test_init_range_determinism_and_moments():
    """A-7: U[0, 1/sqrt(k)) from a counter hash."""
    k = 128
    a = oracle.init(7, 3000, k, 0, F32)
    b = oracle.init(7, 3000, k, 0, F32)
    c = oracle.init(7, 3000, k, 1, F32)
    np.testing.assert_array_equal(a, b)
    assert not np.array_equal(a, c)
    s = 1 / math.sqrt(k)
    assert a.min() >= 0 and a.max() < s
    assert abs(a.mean() - s / 2) < 0.01 * s and abs(a.var() - s * s / 12) < 0.02 * s * s
    h = oracle.init(7, 300, k, 0, F16)
    np.testing.assert_array_equal(h, a[:300].astype(np.float16).view(np.uint16))
    bf = oracle.init(7, 300, k, 0, BF16)
    np.testing.assert_array_equal(bf, _bf16_rne_reference(a[:300].ravel()).reshape(300, k))


def test_shuffle_is_uniform_permutation():
    """A-8 / SPEC.md:182-184: a permutation, deterministic, ~uniform position of each element."""
    p = oracle.shuffle_perm(42, 10000)
    assert np.array_equal(np.sort(p), np.arange(10000))
    assert np.array_equal(p, oracle.shuffle_perm(42, 10000))
    assert not np.array_equal(p, oracle.shuffle_perm(43, 10000))
    pos = np.empty(10000, np.int64)
    pos[p] = np.arange(10000)
    # first half of the indices should land ~evenly in both halves of the order
    frac = np.mean(pos[:5000] < 5000)
    assert abs(frac - 0.5) < 0.03
    assert oracle.shuffle_perm(1, 1).tolist() == [0]


# ------------------------------------------------------------ D-3 waves -----
def test_waves_are_conflict_free_and_reproduce_serial_bitwise():
    """D-3: wave[i] = max(last[u], last[v]) + 1; executing the waves in wave order
    (any order inside a wave) is bit-identical to serial SGD in the original order."""
    rng = np.random.default_rng(9)
    m_, n_, k, N = 60, 50, 8, 1500
    u = rng.integers(0, m_, N).astype(np.int32)
    v = rng.integers(0, n_, N).astype(np.int32)
    r = rng.normal(size=N).astype(np.float32)
    order = oracle.shuffle_perm(5, N)
    w, nw = oracle.waves(m_, n_, u, v, order)
    assert w.min() == 0 and nw == w.max() + 1
    for wv in range(nw):
        sel = order[w == wv]
        assert len(np.unique(u[sel])) == len(sel) and len(np.unique(v[sel])) == len(sel)
    for storage in (F32, F16, BF16):
        a = oracle.Model(m_, n_, k, storage, seed=3)
        b = oracle.Model(m_, n_, k, storage, seed=3)
        a.epoch(u, v, r, 0.05, 0.02, order)
        wave_order = order[np.argsort(w, kind="stable")]
        # inside a wave, reverse the order: still identical (pairwise independent samples)
        rev = np.concatenate([wave_order[(np.sort(w) == wv)][::-1] for wv in range(nw)])
        b.epoch(u, v, r, 0.05, 0.02, rev)
        np.testing.assert_array_equal(a.P, b.P)
        np.testing.assert_array_equal(a.Q, b.Q)


def test_waves_bounds():
    """nw >= max degree (each row/column's samples sit in distinct waves) and <= N."""
    rng = np.random.default_rng(4)
    u = rng.integers(0, 30, 800).astype(np.int32)
    v = rng.integers(0, 20, 800).astype(np.int32)
    _, nw = oracle.waves(30, 20, u, v)
    maxdeg = max(np.bincount(u).max(), np.bincount(v).max())
    assert maxdeg <= nw <= 800


def test_divergence_reported():
    """a non-finite error aborts with a distinct status."""
    m = oracle.Model(1, 1, 2, F32, P=np.array([[1e30, 1e30]], np.float32), Q=np.array([[1e30, 1e30]], np.float32))
    z = np.zeros(1, np.int32)
    assert m.epoch(z, z, np.ones(1, np.float32), 0.1, 0.0) == -5
