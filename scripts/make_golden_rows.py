"""Golden sampled rows after ONE serial epoch at full size (deterministic-mode parity at full scale).

Calls only oracle/ and datagen/.  Writes tests/golden/<cfg>_<storage>_epoch1_rows.npz with
256 sampled rows of P and of Q (indices drawn with numpy seed 0), ||P||_F, ||Q||_F and the wave
count of the A-8 order (D-3), for tests/test_gpu_fullsize.py.
    python scripts/make_golden_rows.py C2 f32
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import datagen  # noqa: E402
import oracle  # noqa: E402


def main():
    name, storage = sys.argv[1], sys.argv[2]
    cfg = datagen.CONFIGS[name]
    st = oracle.STORAGE_NAME[storage]
    (u, v, r), _ = datagen.make(cfg)
    order = oracle.shuffle_perm(cfg.seed_shuffle, len(u))
    _, nw = oracle.waves(cfg.m, cfg.n, u, v, order)
    m = oracle.Model(cfg.m, cfg.n, cfg.k, st, seed=cfg.seed_init)
    assert m.epoch(u, v, r, oracle.eta(cfg.alpha, cfg.beta, 0), cfg.lam, order) == 0
    P, Q = m.factors_f32()
    rng = np.random.default_rng(0)
    pi = np.sort(rng.choice(cfg.m, 256, replace=False))
    qi = np.sort(rng.choice(cfg.n, 256, replace=False))
    out = os.path.join(ROOT, "tests", "golden", f"{name}_{storage}_epoch1_rows.npz")
    np.savez_compressed(out, p_idx=pi, q_idx=qi, P_rows=P[pi], Q_rows=Q[qi],
                        P_fro=np.linalg.norm(P.astype(np.float64)), Q_fro=np.linalg.norm(Q.astype(np.float64)),
                        nwaves=nw, what="oracle factors after 1 serial epoch on the A-8 order; "
                                        "written by scripts/make_golden_rows.py (oracle/ + datagen/ only)")
    print(out, nw)


if __name__ == "__main__":
    main()
