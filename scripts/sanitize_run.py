"""One small run of every kernel family, for `compute-sanitizer --tool memcheck`.

    compute-sanitizer --tool memcheck --error-exitcode 1 python scripts/sanitize_run.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import datagen  # noqa: E402
from paper_1610_05838_b200 import mf  # noqa: E402


def main():
    cfg = datagen.CONFIGS["C1"]
    (u, v, r), test = datagen.make(cfg)
    for storage in ("f32", "f16", "bf16"):
        for k in (cfg.k, 7, 64, 128):
            for sched, opts in (("hogwild", {}), ("hogwild", {"variant": 1 << 16}),
                                ("deterministic", {}), ("deterministic", {"variant": 1 << 24}),
                                ("deterministic", {"variant": 2 << 24}), ("wavefront", {}),
                                ("wavefront", {"wave_cta": 1}), ("wavefront", {"wave_cta": 1, "variant": 1 << 16}),
                                ("wavefront", {"wave_cta": 1, "variant": 2 << 16}),
                                ("wavefront", {"wave_cta": 1, "variant": 2 << 20}), ("wavefront", {"wave_cta": 2}),
                                ("wavefront", {"wave_cta": 3}), ("wavefront", {"wave_cta": 3, "variant": 8 << 4}),
                                ("wavefront", {"variant": 4 << 4}), ("wavefront", {"variant": 8 << 4}),
                                ("hogwild", {"r_staging": 2}), ("hogwild", {"r_staging": 2, "batch_f": 96}),
                                ("deterministic", {"variant": 1 << 22}),
                                ("partitioned", {"partitions": 3}), ("partitioned", {"partitions": 3, "part_split": 0}),
                                ("partitioned", {"partitions": 3, "part_split": 1}),
                                ("hogwild", {"q_update": 1}), ("hogwild", {"q_update": 1, "r_staging": 2}),
                                ("partitioned", {"partitions": 3, "q_update": 1}),
                                ("deterministic", {"det_flow": 1}), ("deterministic", {"det_flow": 1, "variant": 2 << 24})):
                g = mf.MF(cfg.m, cfg.n, k, cfg.alpha, cfg.lam, cfg.seed_init, storage=storage, beta=cfg.beta,
                          count_updates=1, trace=1, **opts)
                g.load(u, v, r)
                for _ in range(4):  # epochs 0-2 are the auto-prefetch trials, 3 runs the pick
                    st = g.epoch(sched)
                    assert st.updates == len(u), (storage, k, sched, opts, st.updates)
                g.rmse(*test)
                P, Q = g.factors()
                assert np.isfinite(P).all() and np.isfinite(Q).all()
                g.close()
            g = mf.MF(cfg.m, cfg.n, k, cfg.alpha, cfg.lam, cfg.seed_init, storage=storage, stream_chunk=7000)
            g.epoch_host(u, v, r)
            g.close()
            # out-of-core factors: P in host memory, 5 row blocks
            ends = np.array([mf.mf_segment(cfg.m, 5, b)[1] for b in range(5)])
            blk = np.searchsorted(ends, u, side="right")
            o = np.argsort(blk, kind="stable")
            off = np.concatenate([[0], np.cumsum(np.bincount(blk, minlength=5))]).astype(np.int64)
            g = mf.MF(cfg.m, cfg.n, k, cfg.alpha, cfg.lam, cfg.seed_init, storage=storage, stream_chunk=7000, p_host=1)
            Ph = np.zeros((cfg.m, k), np.float32 if storage == "f32" else np.uint16)
            mf.mf_init_rows_host(g.h, 0, 0, cfg.m, Ph)
            mf.mf_epoch_host_blocks(g.h, u[o], v[o], r[o], off, Ph)
            mf.mf_rmse_host_blocks(g.h, u[o], v[o], r[o], off, Ph)
            g.close()
    print("sanitize run ok")


if __name__ == "__main__":
    main()
