"""Development check: test-RMSE traces of every single-GPU schedule and prefetch setting on C3-1pct for
bf16 / fp16 / fp32 storage (10 epochs, one line per run)."""
import sys, os
sys.path.insert(0, os.getcwd())
import datagen
from paper_1610_05838_b200 import mf
cfg = datagen.CONFIGS["C3-1pct"]
(u, v, r), test = datagen.make(cfg)
for storage in (2, 1, 0):
    for sched, opts in (("wavefront", dict(wave_cta=1, variant=15 << 16)), ("wavefront", dict(wave_cta=1, variant=2 << 16)),
                        ("wavefront", dict(wave_cta=1, variant=1 << 16)),
                        ("hogwild", dict(variant=15 << 16)), ("deterministic", {})):
        with mf.MF(cfg.m, cfg.n, cfg.k, cfg.alpha, cfg.lam, cfg.seed_init, storage=storage, beta=cfg.beta,
                   seed_shuffle=cfg.seed_shuffle, **opts) as g:
            g.load(u, v, r)
            tr = []
            for e in range(10):
                g.epoch(sched)
                tr.append(g.rmse(*test))
            print(storage, sched, opts, " ".join(f"{x:.5f}" for x in tr), flush=True)
