"""Hogwild concurrency study (A-10): throughput and test RMSE vs worker count at full size,
against the oracle's golden trace (tests/golden/C2_<st>_trace.json).

python scripts/worker_sweep.py [--storage f32] [--epochs 10] [--workers 0,20000,40000,0x]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import datagen  # noqa: E402
from paper_1610_05838_b200 import mf  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", default="C2")
    ap.add_argument("--storage", default="f32")
    ap.add_argument("--epochs", type=int, default=10)
    ap.add_argument("--workers", default="0,20000,40000,80000")
    ap.add_argument("--variants", default="-1")
    a = ap.parse_args()
    cfg = datagen.CONFIGS[a.cfg]
    (u, v, r), test = datagen.make(cfg)
    gold = None
    gp = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                      f"{cfg.name}_{a.storage}_trace.json")
    if os.path.exists(gp):
        gold = json.load(open(gp))["rmse"]
    for var in [int(x) for x in a.variants.split(",")]:
        variant = var if var >= 0 else 0
        for w in [int(x) for x in a.workers.split(",")]:
            g = mf.MF(cfg.m, cfg.n, cfg.k, cfg.alpha, cfg.lam, cfg.seed_init, storage=a.storage, beta=cfg.beta,
                      seed_shuffle=cfg.seed_shuffle, workers=w, variant=variant)
            g.load(u, v, r)
            ks, rm = [], []
            for t in range(a.epochs):
                st = g.epoch("hogwild")
                ks.append(st.kernel_seconds)
                rm.append(g.rmse(*test))
            kb = sorted(ks)[len(ks) // 2]
            ref = gold[a.epochs - 1] if gold and len(gold) >= a.epochs else None
            rel = (rm[-1] - ref) / ref if ref else float("nan")
            print(json.dumps({"storage": a.storage, "variant": variant, "workers": st.workers,
                              "kernel_ms": kb * 1e3, "updates_per_s": len(u) / kb, "rmse": rm[-1],
                              "oracle_rmse": ref, "rel_diff": rel}), flush=True)
            g.close()


if __name__ == "__main__":
    main()
