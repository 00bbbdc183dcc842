"""bench.py host logic (no GPU): the workload defaults per world size, the roofline object's arithmetic
and the config labels."""
import argparse
import importlib.util
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def bench():
    spec = importlib.util.spec_from_file_location("bench", os.path.join(ROOT, "bench.py"))
    b = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(b)
    return b


def _ns(**kw):
    d = dict(config=None, scaling=None, storage=None, partitioned=False)
    d.update(kw)
    return argparse.Namespace(**d)


def test_defaults_one_gpu_is_netflix_shape(bench):
    a = bench.resolve_defaults(_ns(), 1)
    assert (a.config, a.scaling, a.storage) == ("C2", "weak", "f16")


@pytest.mark.parametrize("world", [2, 4, 8])
def test_defaults_multi_gpu_is_hugewiki_strong_scaling(bench, world):
    a = bench.resolve_defaults(_ns(), world)
    assert (a.config, a.scaling, a.storage) == ("C4", "strong", "f16")
    a = bench.resolve_defaults(_ns(config="C2", scaling="weak"), world)   # explicit choices win
    assert (a.config, a.scaling) == ("C2", "weak")


def test_roofline_arithmetic(bench):
    import datagen
    cfg = datagen.CONFIGS["C2"]
    N, k_s = cfg.n_train, 0.010
    rf = bench.roofline(cfg, "f16", N, k_s, 250.0 * N, "hogwild")
    assert rf["bytes_per_update_alg"] == 12 + 4 * 128 * 2
    assert rf["hbm"]["bytes_per_update"] == pytest.approx(250.0)
    assert rf["hbm"]["frac_compulsory"] == pytest.approx(524 * N / k_s / 1e9 / rf["hbm"]["peak"])
    if rf["l2"]:
        assert rf["l2"]["achieved"] == pytest.approx(1036 * N / k_s / 1e9)
        # the bound is whichever resource the kernel is closer to
        assert rf["frac"] == pytest.approx(max(rf["l2"]["frac"], rf["hbm"]["frac"]))
        assert rf["bound"] == ("l2" if rf["l2"]["frac"] >= rf["hbm"]["frac"] else "hbm")
    assert rf["frac"] == pytest.approx(rf["achieved"] / rf["peak"])
    # the CTA wavefront keeps q_v in shared memory: only 12 + 2kb per update reach L2
    rw = bench.roofline(cfg, "f16", N, k_s, None, "wavefront_cta")
    assert rw["hbm"]["basis"].startswith("compulsory")
    if rw["l2"]:
        assert rw["l2"]["bytes_per_update"] == 524


def test_workload_labels_follow_the_config(bench):
    import datagen
    for name, word in (("C2", "Netflix"), ("C3", "Yahoo"), ("C4", "Hugewiki")):
        w = bench.workload_config(datagen.CONFIGS[name], 1, "f16", "hogwild")["workload"]
        assert word in w and name in w
    w = bench.workload_config(datagen.CONFIGS["C4"], 8, "f16", "partitioned", "strong")["workload"]
    assert "Hugewiki" in w and "strong scaling" in w


def test_reference_arm_prints_the_contract_line():
    """`bench.py --impl reference` (the driver's reference arm: the serial oracle on the host cores, on a
    bounded sample of the same workload) prints ONE JSON line with the contract's keys, and its e2e
    carries no host<->device bytes."""
    import json
    import subprocess
    import sys
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "3", "--ref-sample", "20000"], capture_output=True, text=True, timeout=600,
                         cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "config",
                "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["higher_is_better"] is True and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] == 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["steps"] == 1 and d["warmup"] == 3
