"""Per-launch overhead of k_hogwild: one epoch over the first n samples of the Netflix-shaped set
(full-size P/Q) for decreasing n; kernel time vs n / steady-state rate."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen
from paper_1610_05838_b200 import mf

cfg = datagen.CONFIGS["C2"]
(u, v, r), test = datagen.make(cfg)
for st in ("f16", "f32"):
    g = mf.MF(cfg.m, cfg.n, cfg.k, cfg.alpha, cfg.lam, cfg.seed_init, storage=st, beta=cfg.beta, shuffle=0,
              variant=0, workers=9907)
    for n in (99_072_112, 12_384_014, 1_548_001, 774_000, 387_000, 100_000):
        g.load(u[:n], v[:n], r[:n])
        ks = []
        for _ in range(5):
            ks.append(g.epoch("hogwild").kernel_seconds)
        kb = min(ks[1:])
        print(f"{st} n={n:10d} kernel {kb*1e6:9.1f} us  rate {n/kb/1e9:6.2f} G/s", flush=True)
    g.close()
