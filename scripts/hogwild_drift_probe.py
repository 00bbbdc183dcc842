"""Development probe: does batch-Hogwild!'s epoch time follow the factor values (reset them) or the epoch count?"""
import json, sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, datagen
from paper_1610_05838_b200 import mf
cfg = datagen.CONFIGS["C2"]
(u, v, r), test = datagen.make(cfg)
g = mf.MF(cfg.m, cfg.n, cfg.k, cfg.alpha, cfg.lam, cfg.seed_init, storage="f16", beta=cfg.beta, seed_shuffle=cfg.seed_shuffle)
g.load(u, v, r)
P0, Q0 = g.factors()
ks = []
for e in range(30):
    ks.append(g.epoch("hogwild").kernel_seconds * 1e3)
print("train 30:", [round(x, 2) for x in ks], flush=True)
P1, Q1 = g.factors()
g.set_factors(P0, Q0)  # back to the initial values, epoch index keeps counting
ks2 = [g.epoch("hogwild").kernel_seconds * 1e3 for _ in range(6)]
print("reset to init:", [round(x, 2) for x in ks2], flush=True)
g.set_factors(P1, Q1)
ks3 = [g.epoch("hogwild").kernel_seconds * 1e3 for _ in range(6)]
print("back to epoch-30 values:", [round(x, 2) for x in ks3], flush=True)
print("fraction of |P| < 6.1e-5:", float((np.abs(P1) < 6.1e-5).mean()), "Q:", float((np.abs(Q1) < 6.1e-5).mean()))
print("P0 small:", float((np.abs(P0) < 6.1e-5).mean()))
