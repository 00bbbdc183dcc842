"""Test RMSE of the partitioned schedule vs the single-GPU schedules (development tool).

PAPER.md:518-521 states the convergence condition of Hogwild! inside partitioned blocks,
s << min(m/i, n/j), empirically s < min(m/i, n/j)/20.  This runs every schedule for E epochs on
one GPU (partitioned via the loopback transport, G partitions) with the default worker count and
with the paper's bound, and prints test RMSE.

python scripts/partition_convergence.py C3-1pct C4-rows10 [--epochs 10] [--G 2,4,8]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import datagen  # noqa: E402
from paper_1610_05838_b200 import mf  # noqa: E402


def run(cfg, data, storage, sched, E, **opts):
    (u, v, r), test = data
    with mf.MF(cfg.m, cfg.n, cfg.k, cfg.alpha, cfg.lam, cfg.seed_init, storage=storage, beta=cfg.beta,
               seed_shuffle=cfg.seed_shuffle, **opts) as g:
        g.load(u, v, r)
        for _ in range(E):
            st = g.epoch(sched)
        return g.rmse(*test), st.workers


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("cfgs", nargs="+")
    ap.add_argument("--epochs", type=int, default=10)
    ap.add_argument("--G", default="2,4,8")
    ap.add_argument("--storage", default="f32")
    a = ap.parse_args()
    for name in a.cfgs:
        cfg = datagen.CONFIGS[name]
        data = datagen.make(cfg)
        rec = {"cfg": name, "m": cfg.m, "n": cfg.n, "N": len(data[0][0]), "epochs": a.epochs}
        rec["hogwild"] = run(cfg, data, a.storage, "hogwild", a.epochs)
        rec["wavefront_cta"] = run(cfg, data, a.storage, "wavefront", a.epochs, wave_cta=1)
        for G in map(int, a.G.split(",")):
            rec[f"part{G}"] = run(cfg, data, a.storage, "partitioned", a.epochs, partitions=G)
            s_paper = max(1, min(cfg.m // G, cfg.n // G) // 20)
            rec[f"part{G}_paper_s{s_paper}"] = run(cfg, data, a.storage, "partitioned", a.epochs, partitions=G,
                                                   workers=s_paper)
        print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
