"""One rank of the multi-process partitioned run used by tests/test_gpu_nccl_fake.py.

Runs under LD_PRELOAD=libfakenccl.so (tests/fake_nccl/), so several ranks can share one GPU.
argv: rank world uid_file data.npz out_prefix epochs [part_split]
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    rank, world, uid_file, data, out, epochs = sys.argv[1:7]
    split = int(sys.argv[7]) if len(sys.argv) > 7 else 0
    rank, world, epochs = int(rank), int(world), int(epochs)
    from paper_1610_05838_b200 import mf
    d = np.load(data)
    u, v, r = d["u"], d["v"], d["r"]
    tu, tv, tr = d["tu"], d["tv"], d["tr"]
    m, n, k = int(d["m"]), int(d["n"]), int(d["k"])
    alpha, beta, lam, seed, seed_sh = (float(d["alpha"]), float(d["beta"]), float(d["lam"]), int(d["seed"]),
                                       int(d["seed_sh"]))
    if rank == 0:
        uid = mf.mf_nccl_unique_id()
        with open(uid_file + ".tmp", "wb") as f:
            f.write(uid)
        os.rename(uid_file + ".tmp", uid_file)
    else:
        while not os.path.exists(uid_file):
            time.sleep(0.01)
        uid = open(uid_file, "rb").read()
    g = mf.MF(m, n, k, alpha, lam, seed, beta=beta, seed_shuffle=seed_sh, workers=1, count_updates=1,
              part_split=split)
    mf.mf_attach_nccl(g.h, uid, rank, world)
    pb, pe = mf.mf_segment(m, world, rank)
    mine = (u >= pb) & (u < pe)
    idx = np.nonzero(mine)[0]
    g.load(u[idx], v[idx], r[idx])
    order_local = g.order()  # stored position -> index into this rank's shard
    for _ in range(epochs):
        st = g.epoch("partitioned")
        assert st.updates == len(idx), (st.updates, len(idx))
    tm = (tu >= pb) & (tu < pe)
    rm = g.rmse(tu[tm], tv[tm], tr[tm])  # collective: global RMSE on every rank
    P = np.empty((pe - pb, k), np.float32)
    Q = np.empty((n, k), np.float32)
    mf.mf_get_factors(g.h, P, Q)      # collective: local P rows, full Q
    S = int(mf.mf_get_option(g.h, mf.MF_OPT_SUBEPOCHS))
    g.close()
    np.savez(f"{out}_{rank}.npz", P=P, Q=Q, rmse=rm, order=idx[order_local], S=S)


if __name__ == "__main__":
    main()
