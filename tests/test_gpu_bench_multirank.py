"""bench.py's N > 1 path (the partitioned schedule, one process per GPU) launched the way the driver
launches it -- `python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N` -- as N ranks
on ONE GPU.  -m gpu.

libmf's NCCL calls are served by tests/fake_nccl (LD_PRELOAD; real NCCL refuses two ranks on one
device) and bench.py's own torch.distributed plumbing runs on gloo (MF_BENCH_DIST_BACKEND); everything
else -- data sharding per rank, mf_attach_nccl, partitioned epochs, collective RMSE, max-over-ranks
timing, the rank-0 JSON line -- is the code the 8-GPU run executes.
"""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)


@pytest.fixture(scope="module")
def fake_nccl(tmp_path_factory):
    out = tmp_path_factory.mktemp("fakenccl") / "libfakenccl.so"
    subprocess.check_call(["g++", "-O2", "-std=c++17", "-fPIC", "-shared", "-I/usr/local/cuda/include", "-o", str(out),
                           os.path.join(HERE, "fake_nccl", "fake_nccl.cpp"), "-L/usr/local/cuda/lib64",
                           "-lcudart_static", "-ldl", "-lrt", "-lpthread"])
    return str(out)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("G,scaling", [(2, "weak"), (3, "strong")])
def test_bench_partitioned_multirank_json_line(fake_nccl, G, scaling):
    env = dict(os.environ, LD_PRELOAD=fake_nccl, MF_BENCH_DIST_BACKEND="gloo", MF_BENCH_DEVICE="0",
               PYTHONPATH=ROOT)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={G}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.join(ROOT, "bench.py"),
           "--gpus", str(G), "--config", "C2-1pct", "--steps", "3", "--warmup", "3", "--e2e-steps", "1",
           "--scaling", scaling]
    p = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout[-2000:]  # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == G and d["scaling"] == scaling and d["steps"] == 3
    assert d["config"]["schedule"].startswith("partitioned") and f"over {G} GPUs" in d["config"]["parallelism"]
    assert f"{scaling} scaling" in d["config"]["workload"]
    assert d["value"] > 0 and d["e2e"]["value"] > 0 and d["gpu_launches"] > 0
    # one global planted model (sigma = 0.1): after 6 epochs the collective test RMSE is near the
    # C2-1pct plateau (serial oracle 0.18 after 10 epochs)
    assert 0.1 < d["test_rmse"] < 0.3, d["test_rmse"]
