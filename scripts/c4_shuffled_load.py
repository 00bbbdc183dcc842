"""Footprint check (development tool): the whole Hugewiki shape (3.07B ratings) loaded WITH the A-8 shuffle
(MF_OPT_SHUFFLE = 1: 64-bit hash keys, radix sort, gather) on one B200, then one batch-Hogwild! epoch;
prints the device memory in use after the load and the peak the caching allocator never sees (libmf
allocates with cudaMalloc / cudaMallocAsync, so the numbers come from cudaMemGetInfo).

python scripts/c4_shuffled_load.py
"""
import json
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import datagen  # noqa: E402
from paper_1610_05838_b200 import mf  # noqa: E402


def main():
    cfg = datagen.CONFIGS["C4"]
    t0 = time.time()
    (u, v, r), test = datagen.make(cfg)
    gen_s = time.time() - t0
    free0, total = torch.cuda.mem_get_info()
    with mf.MF(cfg.m, cfg.n, cfg.k, cfg.alpha, cfg.lam, cfg.seed_init, storage="f16", beta=cfg.beta,
               seed_shuffle=cfg.seed_shuffle, shuffle=1, count_updates=1) as g:
        peak = [0]
        done = threading.Event()

        def poll():  # device memory in use, sampled during the load (libmf's own allocations included)
            while not done.is_set():
                f, _ = torch.cuda.mem_get_info()
                peak[0] = max(peak[0], total - f)
                time.sleep(0.02)
        th = threading.Thread(target=poll, daemon=True)
        th.start()
        t0 = time.time()
        g.load(u, v, r)
        load_s = time.time() - t0
        done.set()
        th.join()
        free1, _ = torch.cuda.mem_get_info()
        st = g.epoch("hogwild")
        assert st.updates == len(u)
        rm = g.rmse(*test)
        order_head = g.order()[:8].tolist() if len(u) < 2 ** 31 else None
    print(json.dumps({"cfg": "C4", "N": len(u), "gen_s": gen_s, "load_shuffled_s": load_s,
                      "device_GB_total": total / 1e9, "device_GB_used_before": (total - free0) / 1e9,
                      "device_GB_used_after_load": (total - free1) / 1e9, "device_GB_peak_during_load_sampled": peak[0] / 1e9, "epoch_kernel_s": st.kernel_seconds,
                      "rmse_after_1_epoch": rm, "order_head": order_head}), flush=True)


if __name__ == "__main__":
    main()
