"""The C ABI from plain C (examples/train.c): compiled with gcc against include/mf.h and libmf.so, no
Python or PyTorch in the process.  CPU: the program builds, loads the library and fails loudly with
MF_ECUDA (exit 3) -- there is no CPU fallback.  GPU: every single-GPU schedule trains the planted
problem, each epoch processes every sample once, and the test RMSE falls below half its initial value."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _build(tmp_path):
    exe = str(tmp_path / "mf_train")
    lib = os.path.join(ROOT, "paper_1610_05838_b200")
    subprocess.check_call(["gcc", "-O2", "-std=c11", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                           os.path.join(ROOT, "examples", "train.c"), "-L", lib, "-lmf", f"-Wl,-rpath,{lib}", "-lm",
                           "-o", exe])
    return exe


def test_c_example_builds_and_fails_loudly_without_gpu(tmp_path):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present (the gpu test runs the example)")
    p = subprocess.run([_build(tmp_path)], capture_output=True, text=True, timeout=120)
    assert p.returncode == 3, (p.returncode, p.stderr)
    assert "MF_ECUDA" in p.stderr and "no CPU fallback" in p.stderr


@pytest.mark.gpu
def test_c_example_trains_on_gpu(tmp_path):
    p = subprocess.run([_build(tmp_path)], capture_output=True, text=True, timeout=300)
    assert p.returncode == 0, (p.returncode, p.stdout, p.stderr)
    lines = [ln for ln in p.stdout.splitlines() if ln.strip()]
    assert len(lines) == 3 and lines[0].startswith("hogwild") and lines[1].startswith("deterministic")
