"""Host vs device time of partitioned epochs on one GPU (1 loopback partition, S passes): how far the
host stays ahead of the launches.  Development tool."""
import os
import sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen
from paper_1610_05838_b200 import mf
cfg = datagen.CONFIGS["C2"]
(u, v, r), test = datagen.make(cfg)
for S in (4, 64):
    g = mf.MF(cfg.m, cfg.n, cfg.k, cfg.alpha, cfg.lam, cfg.seed_init, storage="f16", beta=cfg.beta, shuffle=0,
              variant=0, partitions=1, subepochs=S)
    g.load(u, v, r)
    g.epoch("partitioned")
    for _ in range(3):
        t0 = time.perf_counter(); st = g.epoch("partitioned"); t1 = time.perf_counter()
        print(S, "host wall ms %.2f" % ((t1 - t0) * 1e3), "device epoch ms %.2f" % (st.seconds * 1e3),
              "kernel-span ms %.2f" % (st.kernel_seconds * 1e3), "launches", st.launches, flush=True)
    g.close()
