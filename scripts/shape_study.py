"""Throughput across the BASELINE.json configs (development / reporting tool, one B200).

C3 (Yahoo!Music-shaped): batch-Hogwild! vs wavefront (CTA workers) vs deterministic waves.
C5 (k sweep on the Netflix shape): k in {32, 64, 128, 256}, fp32 and fp16 storage.
Each line: updates/s from the event-timed update kernel (median of the timed epochs), algorithmic
GB/s (12 + 4kb bytes per update) and its fraction of the measured HBM copy bandwidth, and test RMSE.

    python scripts/shape_study.py --what c3,c5 > profiles/<round>_shapes.jsonl
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import datagen  # noqa: E402
from paper_1610_05838_b200 import mf  # noqa: E402

PEAK = 6551.4e9


def run(cfg, storage, schedule, epochs, data, **opts):
    (u, v, r), test = data
    g = mf.MF(cfg.m, cfg.n, cfg.k, cfg.alpha, cfg.lam, cfg.seed_init, storage=storage, beta=cfg.beta,
              seed_shuffle=cfg.seed_shuffle, variant=0, **opts)
    t0 = time.time()
    g.load(u, v, r)
    if schedule == "deterministic":
        nw = mf.mf_wave_count(g.h)
    load_s = time.time() - t0
    ks = []
    for _ in range(epochs):
        st = g.epoch(schedule)
        ks.append(st.kernel_seconds)
    rm = g.rmse(*test)
    g_variant = g.get(mf.MF_OPT_VARIANT)
    g.close()
    # epochs 0-2 of the hogwild / CTA-wavefront schedules are the auto L2-prefetch trials: time the
    # epochs after them (median)
    tail = ks[3:] if len(ks) > 3 else (ks[1:] if len(ks) > 1 else ks)
    kb = sorted(tail)[len(tail) // 2]
    B = 12 + 4 * cfg.k * (4 if storage == "f32" else 2)
    U = len(u) / kb
    out = {"config": cfg.name, "k": cfg.k, "storage": storage, "schedule": schedule,
           "opts": opts, "N": len(u), "epochs": epochs, "kernel_ms": kb * 1e3, "updates_per_s": U,
           "alg_GBps": U * B / 1e9, "frac_alg": U * B / PEAK, "test_rmse": rm, "workers": st.workers,
           "layout_s": load_s, "variant": int(g_variant)}
    if schedule == "deterministic":
        out["waves"] = nw
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--what", default="c3,c5")
    ap.add_argument("--epochs", type=int, default=6)
    a = ap.parse_args()
    if "c5" in a.what:
        base = datagen.CONFIGS["C2"]
        data = datagen.make(base)
        for k in (32, 64, 128, 256):
            cfg = base.scaled(k=k)
            for st in ("f32", "f16"):
                run(cfg, st, "hogwild", a.epochs, data)
                run(cfg, st, "wavefront", a.epochs, data, wave_cta=1)
    if "c3" in a.what:
        cfg = datagen.CONFIGS["C3"]
        data = datagen.make(cfg)
        for st in ("f32", "f16"):
            run(cfg, st, "hogwild", a.epochs, data)
            run(cfg, st, "wavefront", a.epochs, data, wave_cta=1)
            run(cfg, st, "wavefront", 2, data)
        run(cfg, "f16", "deterministic", 2, data)


if __name__ == "__main__":
    main()
