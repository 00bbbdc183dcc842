"""Timeline of the partitioned schedule's stream graph (development tool, one GPU, loopback partitions).

Runs partitioned epochs under torch.profiler (CUPTI activity records of every kernel and copy in the
process, libmf's included) and reports, per hand-over mode (MF_OPT_PART_SPLIT), how much of the Q-unit
hand-over time (the device-to-device copies the loopback transport issues on the comm stream, where
the NCCL transport issues ncclSend/ncclRecv) overlaps an update kernel, and how long each stream
sits idle between its update launches.

python scripts/partition_timeline.py [--cfg C4-rows100] [--G 4] [--storage f16] [--epochs 2]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import datagen  # noqa: E402


def intervals(events, pred):
    return sorted((e["ts"], e["ts"] + e["dur"], e.get("args", {}).get("stream")) for e in events if pred(e))


def overlap(a, bs):
    """Length of interval a covered by the union of intervals bs."""
    s, e = a
    cov, cur = 0.0, s
    for b0, b1 in bs:
        if b1 <= cur or b0 >= e:
            continue
        b0 = max(b0, cur)
        b1 = min(b1, e)
        if b1 > b0:
            cov += b1 - b0
            cur = b1
    return cov


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", default="C4-rows100")
    ap.add_argument("--G", type=int, default=4)
    ap.add_argument("--storage", default="f16")
    ap.add_argument("--epochs", type=int, default=2)
    ap.add_argument("--modes", default="0,2")
    ap.add_argument("--out", default="gpurun_out")
    a = ap.parse_args()
    import torch
    from torch.profiler import ProfilerActivity, profile

    from paper_1610_05838_b200 import mf
    cfg = datagen.CONFIGS[a.cfg]
    (u, v, r), test = datagen.make(cfg)
    for mode in [int(x) for x in a.modes.split(",")]:
        g = mf.MF(cfg.m, cfg.n, cfg.k, cfg.alpha, cfg.lam, cfg.seed_init, storage=a.storage, beta=cfg.beta,
                  seed_shuffle=cfg.seed_shuffle, partitions=a.G, part_split=mode)
        g.load(u, v, r)
        g.epoch("partitioned")  # layout + warm-up
        torch.cuda.synchronize()
        path = os.path.join(a.out, f"partition_timeline_{a.cfg}_G{a.G}_mode{mode}.json")
        ks = []
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            for _ in range(a.epochs):
                ks.append(g.epoch("partitioned").kernel_seconds)
            torch.cuda.synchronize()
        prof.export_chrome_trace(path)
        g.close()
        ev = json.load(open(path))["traceEvents"]
        kern = intervals(ev, lambda e: e.get("cat") == "kernel" and "k_hogwild" in e.get("name", ""))
        copies = intervals(ev, lambda e: e.get("cat") in ("gpu_memcpy",) and "DtoD" in e.get("name", "")
                           or (e.get("cat") == "gpu_memcpy" and e.get("args", {}).get("kind") == "DtoD"))
        kspans = [(s, e) for s, e, _ in kern]
        cp_total = sum(e - s for s, e, _ in copies)
        cp_hidden = sum(overlap((s, e), kspans) for s, e, _ in copies)
        streams = sorted({st for _, _, st in kern})
        gaps = {}
        for st in streams:
            ivs = [(s, e) for s, e, x in kern if x == st]
            gaps[str(st)] = sum(max(0.0, ivs[i + 1][0] - ivs[i][1]) for i in range(len(ivs) - 1))
        span = (max(e for _, e, _ in kern) - min(s for s, _, _ in kern)) if kern else 0.0
        busy = 0.0
        cur = None
        for s, e in sorted(kspans):  # union of kernel time
            if cur is None or s > cur[1]:
                if cur:
                    busy += cur[1] - cur[0]
                cur = [s, e]
            else:
                cur[1] = max(cur[1], e)
        if cur:
            busy += cur[1] - cur[0]
        print(json.dumps({"cfg": a.cfg, "G": a.G, "storage": a.storage, "part_split": mode, "epochs": a.epochs,
                          "epoch_kernel_ms": [x * 1e3 for x in ks], "update_launches": len(kern),
                          "compute_streams": len(streams), "handover_copies": len(copies),
                          "handover_us": cp_total, "handover_us_overlapped_by_updates": cp_hidden,
                          "handover_overlap_frac": cp_hidden / cp_total if cp_total else None,
                          "update_span_us": span, "update_busy_us": busy,
                          "idle_frac_no_update_running": 1 - busy / span if span else None,
                          "idle_us_between_launches_per_stream": gaps, "trace": path}), flush=True)


if __name__ == "__main__":
    main()
