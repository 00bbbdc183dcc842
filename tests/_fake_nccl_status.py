"""One rank of the collective-status test (tests/test_gpu_nccl_fake.py), under LD_PRELOAD=libfakenccl.so.

Every collective call must return the same status on all ranks, and a rank whose own call is invalid
must still enter the collective (its peers would otherwise block in NCCL):
  1. mf_epoch before any rank loaded (ESTATE everywhere);
  2. mf_rmse where only rank 1 passes an out-of-range test index (EINVAL everywhere);
  3. mf_rmse where rank 1 holds an empty test shard (OK, the global RMSE of rank 0's shard);
  4. mf_epoch with a non-partitioned schedule on rank 1 only (EINVAL everywhere).
argv: rank world uid_file data.npz out_prefix
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    rank, world, uid_file, data, out = sys.argv[1:]
    rank, world = int(rank), int(world)
    from paper_1610_05838_b200 import mf
    d = np.load(data)
    u, v, r, tu, tv, tr = (d[x] for x in ("u", "v", "r", "tu", "tv", "tr"))
    m, n, k = int(d["m"]), int(d["n"]), int(d["k"])
    if rank == 0:
        uid = mf.mf_nccl_unique_id()
        with open(uid_file + ".tmp", "wb") as f:
            f.write(uid)
        os.rename(uid_file + ".tmp", uid_file)
    else:
        while not os.path.exists(uid_file):
            time.sleep(0.01)
        uid = open(uid_file, "rb").read()
    g = mf.MF(m, n, k, 0.05, 0.01, 7)
    mf.mf_attach_nccl(g.h, uid, rank, world)
    codes = []

    def status(fn):
        try:
            fn()
            return 0
        except mf.MFError as e:
            return e.status

    codes.append(status(lambda: g.epoch("partitioned")))                      # 1: nobody loaded
    pb, pe = mf.mf_segment(m, world, rank)
    mine = (u >= pb) & (u < pe)
    g.load(u[mine], v[mine], r[mine])
    assert g.epoch("partitioned").updates == int(mine.sum())
    tm = (tu >= pb) & (tu < pe)
    bu = tu[tm].copy()
    if rank == 1:
        bu[0] = m + 5  # out of range
    codes.append(status(lambda: g.rmse(bu, tv[tm], tr[tm])))                # 2: rank 1 invalid
    got = []
    if rank == 1:
        codes.append(status(lambda: got.append(g.rmse(tu[:0], tv[:0], tr[:0]))))  # 3: empty shard
    else:
        codes.append(status(lambda: got.append(g.rmse(tu[tm], tv[tm], tr[tm]))))
    sched = "hogwild" if rank == 1 else "partitioned"
    codes.append(status(lambda: g.epoch(sched)))                             # 4: rank 1 wrong schedule
    P = np.empty((pe - pb, k), np.float32)
    Q = np.empty((n, k), np.float32)
    mf.mf_get_factors(g.h, P, Q)
    g.close()
    np.savez(f"{out}_{rank}.npz", codes=np.array(codes), rmse=np.array(got), P=P, Q=Q)


if __name__ == "__main__":
    main()
