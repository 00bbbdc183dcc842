"""Development tool: per-epoch test RMSE of every single-GPU schedule on a full-size shape.

The deterministic schedule reproduces serial SGD over the stored order (D-3; pinned to the
oracle at 1e-5 on the slices the oracle can run), so at sizes where the CPU oracle would take hours its
trace shows where the parallel schedules stand relative to serial SGD.

python scripts/trace_compare.py [--cfg C3] [--storage f16] [--epochs 20]
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
    ap.add_argument("--cfg", default="C3")
    ap.add_argument("--storage", default="f16")
    ap.add_argument("--epochs", type=int, default=20)
    ap.add_argument("--shuffle", type=int, default=1, help="MF_OPT_SHUFFLE (0 for the full Hugewiki shape: i.i.d. draws)")
    ap.add_argument("--scheds", default="deterministic,hogwild,wavefront_cta",
                    help="comma list; partitioned:G runs G loopback partitions")
    a = ap.parse_args()
    cfg = datagen.CONFIGS[a.cfg]
    (u, v, r), test = datagen.make(cfg)
    for spec in a.scheds.split(","):
        # schedule[@option=value@...]: extra MF options, e.g. wavefront_cta@variant=134217728
        sch, *extra = spec.split("@")
        opts = {"wave_cta": 1} if sch.startswith("wavefront_cta") else {}
        name = "wavefront" if sch.startswith("wavefront_cta") else sch
        if sch.startswith("wavefront_cta:"):  # wavefront_cta:c -- c column groups
            opts["wave_cols"] = int(sch.split(":")[1])
        if sch.startswith("partitioned:"):  # loopback partitions, e.g. partitioned:8 or partitioned:8:16 (S)
            f = sch.split(":")
            name, opts = "partitioned", {"partitions": int(f[1])}
            if len(f) > 2 and f[2]:
                opts["subepochs"] = int(f[2])
            if len(f) > 3 and f[3]:  # partitioned:G:S:workers
                opts["workers"] = int(f[3])
            if len(f) > 4:  # partitioned:G:S:workers:split
                opts["part_split"] = int(f[4])
        for kv in extra:
            opts[kv.split("=")[0]] = int(kv.split("=")[1])
        with mf.MF(cfg.m, cfg.n, cfg.k, cfg.alpha, cfg.lam, cfg.seed_init, storage=a.storage, beta=cfg.beta,
                   seed_shuffle=cfg.seed_shuffle, shuffle=a.shuffle, **opts) as g:
            g.load(u, v, r)
            tr, ks = [], []
            for _ in range(a.epochs):
                ks.append(g.epoch(name).kernel_seconds)
                tr.append(g.rmse(*test))
        print(json.dumps({"cfg": cfg.name, "storage": a.storage, "schedule": spec, "rmse": tr,
                          "kernel_s": ks}), flush=True)


if __name__ == "__main__":
    main()
