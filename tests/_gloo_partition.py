"""Worker for tests/test_partition_host.py: the partitioned schedule's host algebra over gloo (CPU).

Each of G processes owns P row segment g and the samples of that segment, holds one Q column
segment at a time as libmf's schedule says (mf_round_segment), updates its block with the serial
oracle, and passes Q segments to the peers libmf names (mf_round_peers) with torch.distributed
send/recv.  Rank 0 gathers P and Q at the end and writes them to `out` for comparison with a
single-process oracle sweep over the same block order.
"""
import os
import sys

import numpy as np


def run(rank, G, port, data, out, epochs, seed, mode="seg"):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=G)
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import oracle
    from paper_1610_05838_b200 import mf

    d = np.load(data)
    u, v, r, P0, Q0 = d["u"], d["v"], d["r"], d["P0"], d["Q0"]
    m, n, k = P0.shape[0], Q0.shape[0], P0.shape[1]
    lam, alpha = float(d["lam"]), float(d["alpha"])
    pb, pe = mf.mf_segment(m, G, rank)
    mine = (u >= pb) & (u < pe)          # samples of my row segment, stored order kept
    P = P0[pb:pe].copy()
    seg = [mf.mf_segment(n, G, c) for c in range(G)]
    if mode == "unit":
        P, Qfull = _run_units(dist, torch, oracle, mf, rank, G, u, v, r, P, Q0, mine, pb, pe, k, lam, alpha, epochs,
                              seed, n)
        Ps = [torch.zeros((e_ - b_, k)) for b_, e_ in (mf.mf_segment(m, G, g) for g in range(G))]
        _gather_var(dist, torch, P, Ps)
        if rank == 0:
            np.savez(out, P=np.concatenate([p.numpy() for p in Ps]), Q=Qfull)
        dist.destroy_process_group()
        return
    held = mf.mf_round_segment(seed, 0, G, 0, rank)
    Q = Q0[seg[held][0]:seg[held][1]].copy()
    for e in range(epochs):
        eta = oracle.eta(alpha, 0.0, e)
        for rnd in range(G):
            c = mf.mf_round_segment(seed, e, G, rnd, rank)
            assert c == held, "holding the wrong Q segment"
            qb, qe = seg[c]
            dst, src = mf.mf_round_peers(seed, e, G, rnd, rank)
            nxt_e, nxt_r = (e, rnd + 1) if rnd + 1 < G else (e + 1, 0)
            want = mf.mf_round_segment(seed, nxt_e, G, nxt_r, rank)
            buf = np.empty((seg[want][1] - seg[want][0], k), np.float32)
            # libmf's round: the block's lower-half columns, hand over that half of Q, then the upper half
            for h in (0, 1):
                mid = (qe - qb) // 2
                lo, hi = (qb, qb + mid) if h == 0 else (qb + mid, qe)
                sel = mine & (v >= lo) & (v < hi)
                mdl = oracle.Model(pe - pb, qe - qb, k, oracle.F32, P=P, Q=Q)
                mdl.epoch(u[sel] - pb, v[sel] - qb, r[sel], eta, lam)
                P, Q = mdl.P, mdl.Q
                wl = len(buf) // 2
                rows_out = slice(0, mid) if h == 0 else slice(mid, qe - qb)
                rows_in = slice(0, wl) if h == 0 else slice(wl, len(buf))
                if dst == rank:
                    assert src == rank
                    buf[rows_in] = Q[rows_out]
                else:
                    recv = np.empty_like(buf[rows_in])
                    reqs = [dist.isend(torch.from_numpy(np.ascontiguousarray(Q[rows_out])), dst),
                            dist.irecv(torch.from_numpy(recv), src)]
                    for q in reqs:
                        q.wait()
                    buf[rows_in] = recv
            Q, held = buf, want
    # gather: P segments and the Q segment each rank holds
    Ps = [torch.zeros((e_ - b_, k)) for b_, e_ in (mf.mf_segment(m, G, g) for g in range(G))]
    dist.all_gather(Ps, torch.from_numpy(P)) if len({p.shape for p in Ps}) == 1 else _gather_var(dist, torch, P, Ps)
    helds = [torch.zeros(1, dtype=torch.int64) for _ in range(G)]
    dist.all_gather(helds, torch.tensor([held]))
    Qfull = np.zeros_like(Q0)
    for g in range(G):
        h = int(helds[g])
        t = torch.zeros((seg[h][1] - seg[h][0], k))
        if g == rank:
            t = torch.from_numpy(Q)
        dist.broadcast(t, g)
        Qfull[seg[h][0]:seg[h][1]] = t.numpy()
    if rank == 0:
        np.savez(out, P=np.concatenate([p.numpy() for p in Ps]), Q=Qfull)
    dist.destroy_process_group()


def _unit(seg, c, h):
    mid = (seg[c][1] - seg[c][0]) // 2
    return (seg[c][0], seg[c][0] + mid) if h == 0 else (seg[c][0] + mid, seg[c][1])


def _run_units(dist, torch, oracle, mf, rank, G, u, v, r, P, Q0, mine, pb, pe, k, lam, alpha, epochs, seed, n):
    """Unit grid (MF_OPT_PART_SPLIT = 2, one pass per epoch): the rank holds one unit of each family (the
    half h of segment mf_round_unit(.., h)), updates its rows x unit h block for h = 0, 1 and hands unit
    h to the peer mf_unit_peers names."""
    seg = [mf.mf_segment(n, G, c) for c in range(G)]
    held = [mf.mf_round_unit(seed, 0, G, 0, rank, h) for h in (0, 1)]
    Qh = [Q0[slice(*_unit(seg, held[h], h))].copy() for h in (0, 1)]
    for e in range(epochs):
        eta = oracle.eta(alpha, 0.0, e)
        for rnd in range(G):
            for h in (0, 1):
                c = mf.mf_round_unit(seed, e, G, rnd, rank, h)
                assert c == held[h], "holding the wrong unit"
                lo, hi = _unit(seg, c, h)
                sel = mine & (v >= lo) & (v < hi)
                mdl = oracle.Model(pe - pb, hi - lo, k, oracle.F32, P=P, Q=Qh[h])
                mdl.epoch(u[sel] - pb, v[sel] - lo, r[sel], eta, lam)
                P, Qh[h] = mdl.P, mdl.Q
                dst, src = mf.mf_unit_peers(seed, e, G, rnd, rank, h)
                nxt_e, nxt_r = (e, rnd + 1) if rnd + 1 < G else (e + 1, 0)
                want = mf.mf_round_unit(seed, nxt_e, G, nxt_r, rank, h)
                wlo, whi = _unit(seg, want, h)
                if dst == rank:
                    assert src == rank and want == c
                else:
                    recv = np.empty((whi - wlo, k), np.float32)
                    reqs = [dist.isend(torch.from_numpy(np.ascontiguousarray(Qh[h])), dst),
                            dist.irecv(torch.from_numpy(recv), src)]
                    for q in reqs:
                        q.wait()
                    Qh[h] = recv
                held[h] = want
    Qfull = np.zeros_like(Q0)
    for h in (0, 1):
        helds = [torch.zeros(1, dtype=torch.int64) for _ in range(G)]
        dist.all_gather(helds, torch.tensor([held[h]]))
        for g in range(G):
            lo, hi = _unit(seg, int(helds[g]), h)
            t = torch.from_numpy(Qh[h]) if g == rank else torch.zeros((hi - lo, k))
            dist.broadcast(t, g)
            Qfull[lo:hi] = t.numpy()
    return P, Qfull


def _gather_var(dist, torch, P, Ps):
    rank = dist.get_rank()
    for g in range(len(Ps)):
        t = torch.from_numpy(P) if g == rank else Ps[g]
        dist.broadcast(t, g)
        Ps[g] = t


if __name__ == "__main__":
    rank, G, port, data, out, epochs, seed = sys.argv[1:8]
    run(int(rank), int(G), int(port), data, out, int(epochs), int(seed), sys.argv[8] if len(sys.argv) > 8 else "seg")
