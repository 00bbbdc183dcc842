"""Throughput probe (development tool): batch-Hogwild! variants on the Netflix-shaped config.

python scripts/probe.py [--cfg C2] [--epochs 3] [--storage f32,f16] [--variants 0,16,32,64,1,17,2]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import datagen  # noqa: E402
from paper_1610_05838_b200 import mf  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", default="C2")
    ap.add_argument("--epochs", type=int, default=3)
    ap.add_argument("--storage", default="f32,f16")
    ap.add_argument("--variants", default="-1", help="-1 = bench.py's default for the storage")
    ap.add_argument("--workers", default="0")
    ap.add_argument("--batch", default="256")
    ap.add_argument("--k", type=int, default=0)
    ap.add_argument("--sched", default="hogwild")
    ap.add_argument("--opt", action="append", default=[], help="extra MF option, e.g. wave_cta=1")
    a = ap.parse_args()
    cfg = datagen.CONFIGS[a.cfg]
    if a.k:
        cfg = cfg.scaled(k=a.k)
    t0 = time.time()
    (u, v, r), test = datagen.make(cfg)
    print(f"gen {cfg.name} N={len(u)} in {time.time() - t0:.1f}s", flush=True)
    peak = 6551.4e9
    for storage in a.storage.split(","):
        b = 4 if storage == "f32" else 2
        B = 12 + 4 * cfg.k * b
        extra = {"shuffle": 0}
        extra.update({kv.split("=")[0]: float(kv.split("=")[1]) for kv in a.opt})
        g = mf.MF(cfg.m, cfg.n, cfg.k, cfg.alpha, cfg.lam, cfg.seed_init, storage=storage, beta=cfg.beta, **extra)
        g.load(u, v, r)
        for var in [int(x) for x in a.variants.split(",")]:
            for w in [int(x) for x in a.workers.split(",")]:
                for f in [int(x) for x in a.batch.split(",")]:
                    g.set(mf.MF_OPT_VARIANT, var if var >= 0 else 0)
                    g.set(mf.MF_OPT_WORKERS, w)
                    g.set(mf.MF_OPT_BATCH_F, f)
                    ks = []
                    for e in range(a.epochs):
                        st = g.epoch(a.sched)
                        ks.append(st.kernel_seconds)
                    kb = min(ks[1:]) if len(ks) > 1 else ks[0]
                    U = len(u) / kb
                    print(f"{storage} var={var:3d} workers={st.workers:6d} f={f:5d} kernel {kb*1e3:7.2f} ms "
                          f"U={U/1e9:6.3f} G/s  alg {U*B/1e9:7.1f} GB/s frac={U*B/peak:.3f} "
                          f"rmse={g.rmse(*test):.4f}", flush=True)
        g.close()


if __name__ == "__main__":
    main()
