"""C4 (Hugewiki shape) oracle timing: the serial C++ oracle over the first `n` samples of the
stored order with FULL-size P / Q (50M x 128 and 39,781 x 128), on one core; extrapolated to one epoch
(3.07B samples) and labelled so.  Test infrastructure (calls only oracle/ and datagen/).

python scripts/oracle_c4_timing.py [n_samples] [storage]
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import datagen  # noqa: E402
import oracle  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 20_000_000
    storage = sys.argv[2] if len(sys.argv) > 2 else "f16"
    cfg = datagen.CONFIGS["C4"]
    m_rows = cfg.m
    # the first n samples of the generator stream are the first n stored samples (MF_OPT_SHUFFLE = 0 reading,
    # i.i.d. draws); generated as a row segment covering every row
    (u, v, r), _ = datagen.make_segment(cfg, m_rows, 0, m_rows, n, 1, 0)
    t0 = time.perf_counter()
    mdl = oracle.Model(cfg.m, cfg.n, cfg.k, oracle.STORAGE_NAME[storage], seed=cfg.seed_init)
    init_s = time.perf_counter() - t0
    t0 = time.perf_counter()
    mdl.epoch(u, v, r, oracle.eta(cfg.alpha, cfg.beta, 0), cfg.lam)
    dt = time.perf_counter() - t0
    rate = n / dt
    cpu = "unknown"
    for line in open("/proc/cpuinfo"):
        if line.startswith("model name"):
            cpu = line.split(":", 1)[1].strip()
            break
    print(json.dumps({"cfg": "C4", "storage": storage, "samples_timed": n, "seconds": dt, "updates_per_s": rate,
                      "epoch_seconds_extrapolated": cfg.n_train / rate, "init_seconds_full_size_factors": init_s,
                      "cores": 1, "cpu_model": cpu, "host_cpus": os.cpu_count(),
                      "note": "extrapolated from the first samples of the stored order, full-size P / Q"}))


if __name__ == "__main__":
    main()
