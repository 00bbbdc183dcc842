"""Workload shapes (BASELINE.json `configs`).

Shapes (m, n, train, test) are the paper's Table 2;
alpha/beta/lambda are Table 3 except Yahoo's lambda
(reading A-18).  Data are synthetic planted rank-8 ratings.
"""
from __future__ import annotations

from dataclasses import dataclass, replace


@dataclass(frozen=True)
class Config:
    name: str
    m: int
    n: int
    n_train: int
    n_test: int
    k: int
    alpha: float
    beta: float
    lam: float
    sigma: float
    rank: int = 8
    seed_data: int = 1
    seed_shuffle: int = 42
    seed_init: int = 7
    with_replacement: bool = True
    epochs: int = 20
    zipf: tuple | None = None  # (s_u, s_v): Zipf-skewed row / column popularity (NEXT-4)

    def scaled(self, **kw) -> "Config":
        return replace(self, **kw)


CONFIGS = {
    # configs[0]: planted rank-8, parity config
    "C1": Config("C1", 1000, 800, 50_000, 5_000, 32, 0.08, 0.3, 0.05, 0.01,
                 seed_data=1, with_replacement=False, epochs=20),
    # P-6 planted-recovery self-check (k = planted rank)
    "C1-selfcheck": Config("C1-selfcheck", 1000, 800, 50_000, 5_000, 8, 0.05, 0.0, 0.0, 0.01,
                           seed_data=1, with_replacement=False, epochs=50),
    "tiny-selfcheck": Config("tiny-selfcheck", 200, 150, 15_000, 1_500, 4, 0.05, 0.0, 0.0, 0.01,
                             rank=4, seed_data=11, with_replacement=False, epochs=20),
    # configs[1]: Netflix-shaped (Table 2 Netflix column, Table 3 Netflix row)
    "C2": Config("C2", 480_190, 17_771, 99_072_112, 1_408_395, 128, 0.08, 0.3, 0.05, 0.1,
                 seed_data=2, epochs=20),
    # Netflix-shaped 1% slice: rows and columns /100, samples /100 -> same degrees as C2
    "C2-1pct": Config("C2-1pct", 4_802, 178, 990_721, 14_084, 128, 0.08, 0.3, 0.05, 0.1,
                      seed_data=2, epochs=20),
    # Netflix-scaled 10% (SURVEY §8(c) [SIM] instance): same degrees as C2
    "C2-10pct": Config("C2-10pct", 48_019, 1_777, 9_907_211, 140_840, 128, 0.08, 0.3, 0.05, 0.1,
                       seed_data=2, epochs=20),
    # NEXT-4: Netflix shape with power-law degrees (top item ~0.4% of the ratings, as real data is
    # heavy-tailed) and its 1% slice for oracle-sized parity
    "C2-zipf": Config("C2-zipf", 480_190, 17_771, 99_072_112, 1_408_395, 128, 0.08, 0.3, 0.05, 0.1,
                      seed_data=5, epochs=20, zipf=(0.3, 0.5)),
    "C2-zipf-1pct": Config("C2-zipf-1pct", 4_802, 178, 990_721, 14_084, 128, 0.08, 0.3, 0.05, 0.1,
                           seed_data=5, epochs=20, zipf=(0.3, 0.5)),
    # its 10% slice: on the 1% slice the shuffle order alone moves the oracle's test RMSE by 0.75% after 10
    # epochs, more than the 0.5% gate; the 10% slice keeps the skew with ten times the ratings per column
    "C2-zipf-10pct": Config("C2-zipf-10pct", 48_019, 1_777, 9_907_211, 140_840, 128, 0.08, 0.3, 0.05, 0.1,
                            seed_data=5, epochs=10, zipf=(0.3, 0.5)),
    # configs[2]: Yahoo!Music-shaped, lambda per reading A-18
    "C3": Config("C3", 1_000_990, 624_961, 252_800_275, 4_003_960, 128, 0.08, 0.2, 0.05, 0.1,
                 seed_data=3, epochs=10),
    "C3-1pct": Config("C3-1pct", 10_010, 6_250, 2_528_003, 40_040, 128, 0.08, 0.2, 0.05, 0.1,
                      seed_data=3, epochs=10),
    # Yahoo-shaped 10% slice: rows, columns and samples /10 -> same degrees as C3 (fp16 / fp32 goldens)
    "C3-10pct": Config("C3-10pct", 100_099, 62_496, 25_280_028, 400_396, 128, 0.08, 0.2, 0.05, 0.1,
                       seed_data=3, epochs=10),
    # configs[3]: Hugewiki-shaped
    "C4": Config("C4", 50_082_604, 39_781, 3_069_817_980, 31_327_899, 128, 0.08, 0.3, 0.03, 0.1,
                 seed_data=4, epochs=10),
    "C4-rows10": Config("C4-rows10", 5_008_260, 39_781, 306_981_798, 3_132_790, 128, 0.08, 0.3, 0.03, 0.1,
                        seed_data=4, epochs=10),
    # rows and samples /100, n kept (per-segment c / n_seg of the partitioned path as at full size)
    "C4-rows100": Config("C4-rows100", 500_826, 39_781, 30_698_180, 313_279, 128, 0.08, 0.3, 0.03, 0.1,
                         seed_data=4, epochs=10),
    "C4-rows1000": Config("C4-rows1000", 50_083, 398, 3_069_818, 31_328, 128, 0.08, 0.3, 0.03, 0.1,
                          seed_data=4, epochs=10),
}
