"""The multi-rank NCCL path of the partitioned schedule, as G processes on ONE GPU.  -m gpu.

Real NCCL refuses two ranks on one device, and this environment gives one GPU per box, so the ranks
run with tests/fake_nccl (LD_PRELOAD), a host-staged stand-in for the NCCL calls libmf makes
(grouped send/recv, all-gather, all-reduce) that keeps their pairing and stream-ordering semantics.
Everything else is the production path: mf_attach_nccl, local-row layout, the hand-over on the comm
stream (whole blocks, the pipelined half-segment form and the unit grid), collective mf_rmse / mf_get_factors.  With one worker per block the
run must equal the serial oracle over the (epoch, pass, round, rank, half) order reconstructed from
the ranks' stored orders and libmf's round schedule.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

import datagen
import oracle

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def fake_nccl(tmp_path_factory):
    out = tmp_path_factory.mktemp("fakenccl") / "libfakenccl.so"
    subprocess.check_call(["g++", "-O2", "-std=c++17", "-fPIC", "-shared", "-I/usr/local/cuda/include", "-o", str(out),
                           os.path.join(HERE, "fake_nccl", "fake_nccl.cpp"), "-L/usr/local/cuda/lib64",
                           "-lcudart_static", "-ldl", "-lrt", "-lpthread"])
    return str(out)


@pytest.mark.parametrize("G,split", [(2, 0), (3, 0), (2, 1), (3, 1), (2, 2), (3, 2)])
def test_multirank_partitioned_matches_oracle_block_sweep(fake_nccl, tmp_path, G, split):
    from paper_1610_05838_b200 import mf
    cfg = datagen.CONFIGS["C1"]
    (u, v, r), (tu, tv, tr) = datagen.make(cfg)
    E = 2
    data = tmp_path / "d.npz"
    np.savez(data, u=u, v=v, r=r, tu=tu, tv=tv, tr=tr, m=cfg.m, n=cfg.n, k=cfg.k, alpha=cfg.alpha, beta=cfg.beta,
             lam=cfg.lam, seed=cfg.seed_init, seed_sh=cfg.seed_shuffle)
    uid_file, out = str(tmp_path / "uid"), str(tmp_path / "out")
    env = dict(os.environ, LD_PRELOAD=fake_nccl, PYTHONPATH=os.path.dirname(HERE))
    procs = [subprocess.Popen([sys.executable, os.path.join(HERE, "_fake_nccl_rank.py"), str(g), str(G), uid_file,
                               str(data), out, str(E), str(split)], env=env) for g in range(G)]
    try:
        rcs = [p.wait(timeout=300) for p in procs]
    finally:
        for p in procs:
            if p.poll() is None:
                p.kill()
        uid = open(uid_file, "rb").read().split(b"\0")[0].decode() if os.path.exists(uid_file) else None
        if uid and os.path.exists(uid):
            os.remove(uid)
    assert rcs == [0] * G
    res = [np.load(f"{out}_{g}.npz") for g in range(G)]
    S = int(res[0]["S"])
    # serial oracle over the reconstructed processing order
    rs = [mf.mf_segment(cfg.m, G, g) for g in range(G)]
    cs = [mf.mf_segment(cfg.n, G, c) for c in range(G)]
    ref = oracle.Model(cfg.m, cfg.n, cfg.k, oracle.F32, seed=cfg.seed_init)
    for e in range(E):
        order = []
        for s in range(S):
            for rnd in range(G):
                for h in ((0, 1) if split == 2 else (None,)):  # unit grid: family 0's sub-blocks, then family 1's
                    for g in range(G):
                        o = res[g]["order"]  # this rank's stored order, as indices into the global arrays
                        pos = np.arange(len(o))
                        if split == 2:
                            c = mf.mf_round_unit(cfg.seed_shuffle, e * S + s, G, rnd, g, h)
                        else:
                            c = mf.mf_round_segment(cfg.seed_shuffle, e * S + s, G, rnd, g)
                        mid = cs[c][0] + (cs[c][1] - cs[c][0]) // 2
                        if split == 2:
                            ranges = ((cs[c][0], mid),) if h == 0 else ((mid, cs[c][1]),)
                        else:
                            ranges = ((cs[c][0], mid), (mid, cs[c][1])) if split else ((cs[c][0], cs[c][1]),)
                        for lo, hi in ranges:
                            sel = ((pos * S) // len(o) == s) & (v[o] >= lo) & (v[o] < hi)
                            order.append(o[sel])
        order = np.concatenate(order)
        assert len(order) == len(u) and len(np.unique(order)) == len(u)
        ref.epoch(u, v, r, oracle.eta(cfg.alpha, cfg.beta, e), cfg.lam, order)
    P = np.concatenate([res[g]["P"] for g in range(G)])
    for g in range(G):
        np.testing.assert_array_equal(res[g]["Q"], res[0]["Q"])      # every rank gathered the same Q
        assert float(res[g]["rmse"]) == float(res[0]["rmse"])         # and the same global RMSE
    assert np.linalg.norm(P - ref.P) / np.linalg.norm(ref.P) <= 1e-5
    assert np.linalg.norm(res[0]["Q"] - ref.Q) / np.linalg.norm(ref.Q) <= 1e-5
    assert float(res[0]["rmse"]) == pytest.approx(ref.rmse(tu, tv, tr), rel=1e-5)


def test_collective_status_agreement(fake_nccl, tmp_path):
    """mf_epoch / mf_rmse / mf_get_factors with NCCL attached are collective: a call that is invalid on
    one rank only returns the same status on every rank and leaves no rank blocked;
    a rank with an empty test shard still joins the global RMSE."""
    from paper_1610_05838_b200 import mf
    G = 2
    cfg = datagen.CONFIGS["C1"]
    (u, v, r), (tu, tv, tr) = datagen.make(cfg)
    data = tmp_path / "d.npz"
    np.savez(data, u=u, v=v, r=r, tu=tu, tv=tv, tr=tr, m=cfg.m, n=cfg.n, k=cfg.k)
    uid_file, out = str(tmp_path / "uid"), str(tmp_path / "out")
    env = dict(os.environ, LD_PRELOAD=fake_nccl, PYTHONPATH=os.path.dirname(HERE))
    procs = [subprocess.Popen([sys.executable, os.path.join(HERE, "_fake_nccl_status.py"), str(g), str(G), uid_file,
                               str(data), out], env=env) for g in range(G)]
    try:
        rcs = [p.wait(timeout=120) for p in procs]
    finally:
        for p in procs:
            if p.poll() is None:
                p.kill()
        uid = open(uid_file, "rb").read().split(b"\0")[0].decode() if os.path.exists(uid_file) else None
        if uid and os.path.exists(uid):
            os.remove(uid)
    assert rcs == [0] * G
    res = [np.load(f"{out}_{g}.npz") for g in range(G)]
    want = [mf.MF_ESTATE, mf.MF_EINVAL, 0, mf.MF_EINVAL]
    for g in range(G):
        assert list(res[g]["codes"]) == want, (g, list(res[g]["codes"]))
    # the global RMSE with rank 1's test shard empty is rank 0's shard's RMSE, on both ranks
    assert float(res[0]["rmse"][0]) == float(res[1]["rmse"][0])
    np.testing.assert_array_equal(res[0]["Q"], res[1]["Q"])
