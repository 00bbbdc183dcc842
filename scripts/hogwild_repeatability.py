"""Development check: run-to-run spread of batch-Hogwild! (fp16, C2-1pct, 10 epochs) against the serial oracle, per prefetch setting."""
import os, sys
sys.path.insert(0, os.getcwd())
import datagen
from paper_1610_05838_b200 import mf
cfg = datagen.CONFIGS["C2-1pct"]
(u, v, r), test = datagen.make(cfg)
gold = 0.18419947582160215
for var in (1 << 16, 0, 15 << 16):
    devs = []
    for rep in range(6):
        with mf.MF(cfg.m, cfg.n, cfg.k, cfg.alpha, cfg.lam, cfg.seed_init, storage=1, beta=cfg.beta,
                   seed_shuffle=cfg.seed_shuffle, variant=var) as g:
            g.load(u, v, r)
            for _ in range(10):
                g.epoch("hogwild")
            devs.append(100 * (g.rmse(*test) - gold) / gold)
    print(var, " ".join(f"{d:+.3f}" for d in devs), flush=True)
