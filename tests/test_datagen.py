"""The shared input generator (datagen/): determinism, shapes and the planted-model statistics."""
import numpy as np

import datagen


def test_deterministic_and_in_range():
    a = datagen.planted_coo(5, 300, 200, 8, 0.1, 5000)
    b = datagen.planted_coo(5, 300, 200, 8, 0.1, 5000)
    for x, y in zip(a, b):
        np.testing.assert_array_equal(x, y)
    u, v, r = a
    assert u.min() >= 0 and u.max() < 300 and v.min() >= 0 and v.max() < 200
    assert np.isfinite(r).all()


def test_without_replacement_distinct_cells():
    u, v, _ = datagen.planted_coo(1, 100, 80, 8, 0.01, 4000, with_replacement=False)
    cells = u.astype(np.int64) * 80 + v
    assert len(np.unique(cells)) == 4000


def test_planted_statistics():
    """r = P*_u.Q*_v + sigma*g with var(P*), var(Q*) = rank^-1/2: std(r) ~ 1, residual std = sigma."""
    m, n, rank, sigma = 2000, 1500, 8, 0.1
    u, v, r = datagen.planted_coo(3, m, n, rank, sigma, 200_000)
    P, Q = datagen.planted_factors(3, m, n, rank)
    assert abs(P.var() - rank ** -0.5) < 0.02 and abs(Q.var() - rank ** -0.5) < 0.02
    resid = r.astype(np.float64) - np.einsum("ij,ij->i", P[u], Q[v])
    assert abs(resid.std() - sigma) < 0.005 and abs(resid.mean()) < 0.002
    assert abs(r.std() - 1.0) < 0.1
    # uniform degrees (with replacement): Poisson around N/m
    deg = np.bincount(u, minlength=m)
    assert abs(deg.mean() - 100) < 1e-9 and deg.std() < 15


def test_zipf_degrees_follow_the_power_law():
    """NEXT-4 generator: column ids ~ Zipf(s) (scrambled): the k-th most frequent id has frequency
    ~ k^-s / H_n(s); ratings keep the planted model."""
    n, s, N = 2000, 0.8, 400_000
    u, v, r = datagen.zipf_coo(9, 5000, n, 8, 0.1, N, 0.0, s)
    freq = np.sort(np.bincount(v, minlength=n))[::-1] / N
    H = np.sum(np.arange(1, n + 1) ** -s)
    for kk in (1, 10, 100):
        assert abs(freq[kk - 1] - kk ** -s / H) < 0.1 * kk ** -s / H + 3e-4
    assert np.argmax(np.bincount(v)) != 0  # hot ids are scrambled, not clustered at 0
    du = np.bincount(u, minlength=5000) / N  # s_u = 0: uniform rows
    assert du.max() < 3 / 5000
    P, Q = datagen.planted_factors(9, 5000, n, 8)
    resid = r.astype(np.float64) - np.einsum("ij,ij->i", P[u], Q[v])
    assert abs(resid.std() - 0.1) < 0.005


def test_configs_table2_shapes():
    """PAPER.md:373-377 Table 2."""
    c = datagen.CONFIGS
    assert (c["C2"].m, c["C2"].n, c["C2"].n_train, c["C2"].n_test) == (480190, 17771, 99072112, 1408395)
    assert (c["C3"].m, c["C3"].n, c["C3"].n_train, c["C3"].n_test) == (1000990, 624961, 252800275, 4003960)
    assert (c["C4"].m, c["C4"].n, c["C4"].n_train, c["C4"].n_test) == (50082604, 39781, 3069817980, 31327899)
    assert all(c[x].k == 128 for x in ("C2", "C3", "C4"))


def test_planted_segment_is_a_slice_of_the_global_model():
    """make_segment (multi-GPU bench shards): rows stay in the segment, every rank sees the same global
    planted model (residual std = sigma against the global P*, Q*), streams are disjoint per rank."""
    cfg = datagen.CONFIGS["C2-1pct"]
    G, m_glob = 3, 3 * 1000
    shards = [datagen.make_segment(cfg, m_glob, g * 1000, (g + 1) * 1000, 20_000, 2_000, g) for g in range(G)]
    P, Q = datagen.planted_factors(cfg.seed_data, m_glob, cfg.n, cfg.rank)
    for g, ((u, v, r), (tu, tv, tr)) in enumerate(shards):
        assert u.min() >= g * 1000 and u.max() < (g + 1) * 1000 and tu.min() >= g * 1000
        assert v.min() >= 0 and v.max() < cfg.n
        resid = r.astype(np.float64) - np.einsum("ij,ij->i", P[u], Q[v])
        assert abs(resid.std() - cfg.sigma) < 0.005
    assert not np.array_equal(shards[0][0][1], shards[1][0][1])
    again = datagen.make_segment(cfg, m_glob, 1000, 2000, 20_000, 2_000, 1)
    np.testing.assert_array_equal(again[0][2], shards[1][0][2])
