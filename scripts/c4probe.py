"""Hugewiki-shaped (C4) and other large-shape probe on one B200: batch-Hogwild! and CTA wavefront.

python scripts/c4probe.py C4 f16
"""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import datagen
from paper_1610_05838_b200 import mf
cfg = datagen.CONFIGS[sys.argv[1]]
st = sys.argv[2]
t0 = time.time()
(u, v, r), test = datagen.make(cfg)
print("gen", len(u), time.time() - t0, flush=True)
g = mf.MF(cfg.m, cfg.n, cfg.k, cfg.alpha, cfg.lam, cfg.seed_init, storage=st, beta=cfg.beta, shuffle=0,
          variant=0)
t0 = time.time(); g.load(u, v, r); print("load", time.time() - t0, flush=True)
for sched, opts in (("hogwild", {}), ("wavefront", {"wave_cta": 1})):
    for kk, vv in opts.items(): g.set(getattr(mf, "MF_OPT_" + kk.upper()), vv)
    ks = []
    for e in range(5):  # epochs 0-2 are the auto-prefetch trials; report the picked setting's epochs
        s = g.epoch(sched); ks.append(s.kernel_seconds)
    B = 12 + 4 * cfg.k * (4 if st == "f32" else 2)
    kb = min(ks[3:])
    print(json.dumps({"cfg": cfg.name, "N": len(u), "storage": st, "schedule": sched, "opts": opts, "kernel_s": kb,
                      "updates_per_s": len(u) / kb, "frac_alg": len(u) / kb * B / 6551.4e9,
                      "variant": int(g.get(mf.MF_OPT_VARIANT)), "rmse": g.rmse(*test)}), flush=True)
