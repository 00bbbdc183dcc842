"""Host logic of the partitioned multi-GPU schedule (no GPU): Latin-square rounds, exchange peers,
the paper's 8-of-24 count, and a world-size-2/3 gloo run of the exchange pattern that must equal a
serial oracle sweep over the same block order."""
import itertools
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

import oracle

HERE = os.path.dirname(os.path.abspath(__file__))


def _mf():
    from paper_1610_05838_b200 import mf
    return mf


@pytest.mark.parametrize("G", [1, 2, 3, 4, 8])
def test_rounds_form_latin_squares(G):
    mf = _mf()
    for e in range(4):
        sq = np.array([[mf.mf_round_segment(42, e, G, r, g) for r in range(G)] for g in range(G)])
        for g in range(G):
            assert sorted(sq[g]) == list(range(G))      # each rank sees every column segment once per epoch
        for r in range(G):
            assert sorted(sq[:, r]) == list(range(G))   # a round's blocks share no column segment


@pytest.mark.parametrize("G", [2, 3, 5, 8])
def test_peers_move_every_segment_where_it_is_needed(G):
    mf = _mf()
    for e in range(3):
        for r in range(G):
            ne, nr = (e, r + 1) if r + 1 < G else (e + 1, 0)
            held = [mf.mf_round_segment(7, e, G, r, g) for g in range(G)]
            want = [mf.mf_round_segment(7, ne, G, nr, g) for g in range(G)]
            peers = [mf.mf_round_peers(7, e, G, r, g) for g in range(G)]
            for g, (dst, src) in enumerate(peers):
                assert want[dst] == held[g] and held[src] == want[g]
                assert peers[dst][1] == g                   # send/recv pairs match
            if r + 1 < G:
                assert all(dst == (g - 1) % G for g, (dst, _) in enumerate(peers))  # ring shift inside an epoch


@pytest.mark.parametrize("G", [1, 2, 3, 4, 8])
def test_unit_grid_is_a_latin_rectangle(G):
    """Unit grid (MF_OPT_PART_SPLIT = 2): over the G rounds of a pass every rank visits all 2G column units
    (segment c's lower half in family 0, its upper half in family 1) exactly once, a round's units are
    pairwise distinct across ranks, family 0 is the whole-segment Latin square, and the pair of units a
    rank holds is not fixed (the families' squares are drawn independently)."""
    mf = _mf()
    pairs = set()
    for p in range(6):
        sq = np.array([[[mf.mf_round_unit(42, p, G, r, g, h) for h in (0, 1)] for r in range(G)] for g in range(G)])
        for g in range(G):
            units = {(int(sq[g, r, h]), h) for r in range(G) for h in (0, 1)}
            assert units == {(c, h) for c in range(G) for h in (0, 1)}
            for r in range(G):
                assert sq[g, r, 0] == mf.mf_round_segment(42, p, G, r, g)
                pairs.add(int(sq[g, r, 1] - sq[g, r, 0]) % G)
        for r in range(G):
            for h in (0, 1):
                assert sorted(sq[:, r, h]) == list(range(G))
        for r in range(G):
            for g in range(G):
                for h in (0, 1):
                    dst, src = mf.mf_unit_peers(42, p, G, r, g, h)
                    ne, nr = (p, r + 1) if r + 1 < G else (p + 1, 0)
                    assert mf.mf_round_unit(42, ne, G, nr, dst, h) == sq[g, r, h]
                    assert mf.mf_unit_peers(42, p, G, r, dst, h)[1] == g
    if G > 1:
        assert len(pairs) > 1  # the two families are not locked to the same segment


def _feasible(order, G=2):
    """Orders of the 2x2 grid's blocks executable by 2 workers: consecutive pairs run concurrently and
    must share no row or column (Fig. 16)."""
    blk = lambda b: divmod(b, G)  # noqa: E731
    for i in range(0, len(order), 2):
        (r1, c1), (r2, c2) = blk(order[i]), blk(order[i + 1])
        if r1 == r2 or c1 == c2:
            return False
    return True


def test_eight_of_24_orders_feasible_and_schedule_inside_them():
    orders = list(itertools.permutations(range(4)))
    feas = [o for o in orders if _feasible(o)]
    assert len(orders) == 24 and len(feas) == 8
    mf = _mf()
    seen = set()
    for e in range(40):
        for firsts in itertools.product((0, 1), repeat=2):  # concurrent blocks of a round in either order
            o = []
            for r in range(2):
                gs = (firsts[r], 1 - firsts[r])
                o += [g * 2 + mf.mf_round_segment(3, e, 2, r, g) for g in gs]
            assert tuple(o) in feas
            seen.add(tuple(o))
    assert len(seen) == 8                              # the randomized Latin square reaches all of them


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("G,mode", [(2, "seg"), (3, "seg"), (2, "unit"), (3, "unit")])
def test_gloo_exchange_equals_serial_block_sweep(tmp_path, G, mode):
    rng = np.random.default_rng(G)
    m_, n_, k, N, epochs, seed = 60, 45, 8, 3000, 2, 11
    u = rng.integers(0, m_, N).astype(np.int32)
    v = rng.integers(0, n_, N).astype(np.int32)
    r = rng.normal(size=N).astype(np.float32)
    P0 = oracle.init(5, m_, k, 0, oracle.F32)
    Q0 = oracle.init(5, n_, k, 1, oracle.F32)
    data = tmp_path / "d.npz"
    out = tmp_path / "o.npz"
    np.savez(data, u=u, v=v, r=r, P0=P0, Q0=Q0, lam=0.02, alpha=0.05)
    port = _free_port()
    env = dict(os.environ, PYTHONPATH=os.path.dirname(HERE))
    procs = [subprocess.Popen([sys.executable, os.path.join(HERE, "_gloo_partition.py"), str(g), str(G), str(port),
                               str(data), str(out), str(epochs), str(seed), mode], env=env) for g in range(G)]
    assert all(p.wait(timeout=240) == 0 for p in procs)
    got = np.load(out)
    # serial sweep: epoch -> round -> (family ->) rank -> block samples in stored order
    mf = _mf()
    ref = oracle.Model(m_, n_, k, oracle.F32, P=P0, Q=Q0)
    rs = [mf.mf_segment(m_, G, g) for g in range(G)]
    cs = [mf.mf_segment(n_, G, c) for c in range(G)]

    def half(c, h):
        mid = cs[c][0] + (cs[c][1] - cs[c][0]) // 2
        return (cs[c][0], mid) if h == 0 else (mid, cs[c][1])

    for e in range(epochs):
        order = []
        for rnd in range(G):
            if mode == "unit":
                for h in (0, 1):
                    for g in range(G):
                        lo, hi = half(mf.mf_round_unit(seed, e, G, rnd, g, h), h)
                        sel = (u >= rs[g][0]) & (u < rs[g][1]) & (v >= lo) & (v < hi)
                        order.append(np.nonzero(sel)[0])
                continue
            for g in range(G):
                c = mf.mf_round_segment(seed, e, G, rnd, g)
                for lo, hi in (half(c, 0), half(c, 1)):  # lower-half columns first, as libmf
                    sel = (u >= rs[g][0]) & (u < rs[g][1]) & (v >= lo) & (v < hi)
                    order.append(np.nonzero(sel)[0])
        ref.epoch(u, v, r, oracle.eta(0.05, 0.0, e), 0.02, np.concatenate(order))
    np.testing.assert_array_equal(got["P"], ref.P)
    np.testing.assert_array_equal(got["Q"], ref.Q)
