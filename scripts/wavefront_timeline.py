"""Development tool: where a CTA-wavefront epoch's time goes, from the audit trace (MF_OPT_TRACE).

For every worker (CTA): busy = sum over its blocks of (t_end - t_start) (after the Q-group copy-in,
before the copy-out), span = last t_end - first t_start; the rest of the kernel time is lock waits,
Q staging, barriers and the launch ramp.  Also reports per-block sample counts and time per sample.

python scripts/wavefront_timeline.py [--cfg C2] [--storage f16]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import datagen  # noqa: E402
from paper_1610_05838_b200 import mf  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", default="C2")
    ap.add_argument("--storage", default="f16")
    ap.add_argument("--epochs", type=int, default=4)
    ap.add_argument("--variant", type=int, default=0)
    ap.add_argument("--wave-cta", type=int, default=1, help="0 = warp workers, 1 = staged CTA, 3 = q-stationary CTA")
    a = ap.parse_args()
    cfg = datagen.CONFIGS[a.cfg]
    (u, v, r), test = datagen.make(cfg)
    with mf.MF(cfg.m, cfg.n, cfg.k, cfg.alpha, cfg.lam, cfg.seed_init, storage=a.storage, beta=cfg.beta, shuffle=0,
               wave_cta=a.wave_cta, trace=1, variant=a.variant) as g:
        g.load(u, v, r)
        for e in range(a.epochs):
            st = g.epoch("wavefront")
        s = int(g.get(mf.MF_OPT_WAVE_ROWS)) if hasattr(mf, "MF_OPT_WAVE_ROWS") else 0
        tr = mf.mf_wavefront_trace(g.h, 50_000_000)
    w, blk, t0, t1 = tr.T
    kern_ns = st.kernel_seconds * 1e9
    start = t0.min()
    busy = np.zeros(w.max() + 1)
    first = np.full(w.max() + 1, np.inf)
    last = np.zeros(w.max() + 1)
    np.add.at(busy, w, t1 - t0)
    np.minimum.at(first, w, t0)
    np.maximum.at(last, w, t1)
    dur = (t1 - t0)
    print(f"{cfg.name} {a.storage}: kernel {kern_ns / 1e6:.2f} ms, {len(tr)} blocks, {w.max() + 1} workers")
    print(f"  per worker busy (in-block)   mean {busy.mean() / 1e6:.2f} ms  = {busy.mean() / kern_ns:.1%} of the kernel")
    print(f"  per worker first start       mean {(first - start).mean() / 1e3:.1f} us (launch ramp + first lock)")
    print(f"  per worker finish            max {(last - start).max() / 1e6:.2f} ms, min {(last - start).min() / 1e6:.2f} ms")
    print(f"  block duration               median {np.median(dur) / 1e3:.1f} us, p99 {np.percentile(dur, 99) / 1e3:.1f} us")
    nb = len(tr) / (w.max() + 1)
    gaps = (last - first - busy) / np.maximum(1, nb - 1)
    print(f"  gap between blocks (lock + Q out/in + barriers)  mean {gaps.mean() / 1e3:.2f} us x {nb:.0f} blocks")


if __name__ == "__main__":
    main()
