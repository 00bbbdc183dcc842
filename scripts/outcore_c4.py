"""Out-of-core factors at the Hugewiki shape (development tool): P (50M x 128 fp16, 12.8 GB) and the 3.07B
ratings live in pinned host memory; each epoch streams 64 row blocks (the paper's 64 x 1 blocks)
through the GPU with mf_epoch_host_blocks -- P segment and ratings in, batch-Hogwild!, P segment back --
while Q stays resident.  Prints updates/s end to end (host-to-host per epoch) and the test RMSE.

python scripts/outcore_c4.py [epochs] [nblocks]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import datagen  # noqa: E402
from paper_1610_05838_b200 import mf  # noqa: E402


def main():
    E = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    B = int(sys.argv[2]) if len(sys.argv) > 2 else 64
    cfg = datagen.CONFIGS["C4"]
    t0 = time.time()
    n_tr, n_te = cfg.n_train // B, cfg.n_test // B
    N, NT = n_tr * B, n_te * B
    U = torch.empty(N, dtype=torch.int32, pin_memory=True)
    V = torch.empty(N, dtype=torch.int32, pin_memory=True)
    R = torch.empty(N, dtype=torch.float32, pin_memory=True)
    tu, tv, tr, off, toff = [], [], [], [0], [0]
    for b in range(B):  # block b's ratings are draws of the same planted model restricted to its rows
        lo, hi = mf.mf_segment(cfg.m, B, b)
        (u, v, r), (a, c_, d) = datagen.make_segment(cfg, cfg.m, lo, hi, n_tr, n_te, b)
        U[b * n_tr:(b + 1) * n_tr] = torch.from_numpy(u)
        V[b * n_tr:(b + 1) * n_tr] = torch.from_numpy(v)
        R[b * n_tr:(b + 1) * n_tr] = torch.from_numpy(r)
        tu.append(a), tv.append(c_), tr.append(d)
        off.append((b + 1) * n_tr)
        toff.append((b + 1) * n_te)
    tu, tv, tr = np.concatenate(tu), np.concatenate(tv), np.concatenate(tr)
    gen_s = time.time() - t0
    with mf.MF(cfg.m, cfg.n, cfg.k, cfg.alpha, cfg.lam, cfg.seed_init, storage="f16", beta=cfg.beta, p_host=1,
               stream_chunk=1 << 24) as g:
        Ph = torch.empty((cfg.m, cfg.k), dtype=torch.int16, pin_memory=True)
        mf.mf_init_rows_host(g.h, 0, 0, cfg.m, Ph.numpy())
        free, total = torch.cuda.mem_get_info()
        ep = []
        for _ in range(E):
            t1 = time.time()
            st = mf.mf_epoch_host_blocks(g.h, U, V, R, off, Ph)
            ep.append({"wall_s": time.time() - t1, "device_s": st.seconds, "kernel_s": st.kernel_seconds,
                       "updates": st.updates})
        rm = mf.mf_rmse_host_blocks(g.h, tu, tv, tr, toff, Ph)
    best = min(e["device_s"] for e in ep[1:]) if E > 1 else ep[0]["device_s"]
    print(json.dumps({"cfg": "C4", "N": N, "nblocks": B, "storage": "f16", "gen_s": gen_s,
                      "device_GB_used": (total - free) / 1e9, "epochs": ep,
                      "updates_per_s_end_to_end": N / best, "test_rmse": rm,
                      "note": "P (12.8 GB) and R (36.8 GB) in pinned host memory; per epoch 62 GB cross the host link"}))


if __name__ == "__main__":
    main()
