"""The C-ABI library loads and exports every symbol include/mf.h declares; host-only logic (no GPU)."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "mf.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|void|const char \*)\s*(mf_\w+)\s*\(", src, re.M)))


def test_header_symbols_exported():
    from paper_1610_05838_b200 import mf
    names = _declared()
    assert len(names) >= 15
    lib = ctypes.CDLL(mf.LIB_PATH)
    for nm in names:
        assert hasattr(lib, nm), nm
    assert set(names) == set(mf.EXPORTS)


def test_create_validates_arguments_without_device():
    from paper_1610_05838_b200 import mf
    for bad in [(0, 5, 4, 0.1, 0.0), (5, 0, 4, 0.1, 0.0), (5, 5, 0, 0.1, 0.0), (5, 5, 2000, 0.1, 0.0),
                (5, 5, 4, 0.0, 0.0), (5, 5, 4, 0.1, -1.0), (2 ** 31, 5, 4, 0.1, 0.0)]:
        with pytest.raises(mf.MFError) as e:
            mf.mf_create(*bad, 1)
        assert e.value.status == mf.MF_EINVAL
    h = mf.mf_create(10, 8, 4, 0.1, 0.01, 3)
    try:
        mf.mf_set_option(h, mf.MF_OPT_BETA, 0.3)
        assert mf.mf_get_option(h, mf.MF_OPT_BETA) == 0.3
        assert mf.mf_get_option(h, mf.MF_OPT_Q_UPDATE) == 2  # default: auto by kappa (A-20)
        assert mf.mf_get_option(h, mf.MF_OPT_Q_KAPPA) == -1
        assert mf.mf_get_option(h, mf.MF_OPT_DET_FLOW) == 0
        mf.mf_set_option(h, mf.MF_OPT_Q_UPDATE, 0)
        assert mf.mf_get_option(h, mf.MF_OPT_Q_UPDATE) == 0
        with pytest.raises(mf.MFError):
            mf.mf_set_option(h, mf.MF_OPT_Q_UPDATE, 3)
        with pytest.raises(mf.MFError):
            mf.mf_set_option(h, mf.MF_OPT_STORAGE, 7)
        with pytest.raises(mf.MFError):
            mf.mf_set_option(h, mf.MF_OPT_BATCH_F, 100)
        with pytest.raises(mf.MFError) as e:
            mf.mf_epoch(h, "hogwild")
        assert e.value.status == mf.MF_ESTATE
    finally:
        mf.mf_destroy(h)


def test_no_cpu_fallback_without_device():
    """On a box without a GPU, compute calls fail loudly (MF_ECUDA) instead of falling back."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    from paper_1610_05838_b200 import mf
    h = mf.mf_create(10, 8, 4, 0.1, 0.01, 3)
    try:
        with pytest.raises(mf.MFError) as e:
            mf.mf_load_coo(h, np.zeros(3, np.int32), np.zeros(3, np.int32), np.ones(3, np.float32))
        assert e.value.status == mf.MF_ECUDA
    finally:
        mf.mf_destroy(h)


def test_segments_partition_the_extent():
    from paper_1610_05838_b200 import mf
    for extent, G in [(10, 3), (50082604, 8), (17771, 8), (5, 5), (7, 1)]:
        segs = [mf.mf_segment(extent, G, g) for g in range(G)]
        assert segs[0][0] == 0 and segs[-1][1] == extent
        assert all(a[1] == b[0] for a, b in zip(segs, segs[1:]))
        assert all(e - b in (extent // G, extent // G + 1) for b, e in segs)


def test_feasibility_rule_matches_the_papers_pair():
    """mf_feasibility against the paper's printed example: Hugewiki, min(m, n) = 40k,
    s = 768 workers -- converges at j = 2 (bound 40000/2/20 = 1000 > 768), fails at j = 4 (500 < 768);
    s = 1 on a 21 x 21 matrix passes (1 < 21/20: the comparison is exact, SPEC.md's trivial example);
    non-positive arguments are rejected."""
    from paper_1610_05838_b200 import mf
    m_hw, n_hw = 50_082_604, 40_000
    assert mf.mf_feasibility(m_hw, n_hw, 1, 2, 768) == (True, 1000)
    assert mf.mf_feasibility(m_hw, n_hw, 1, 4, 768) == (False, 500)
    assert mf.mf_feasibility(21, 21, 1, 1, 1) == (True, 1)
    assert mf.mf_feasibility(20, 20, 1, 1, 1) == (False, 1)
    assert mf.mf_feasibility(40, 40, 1, 1, 1) == (True, 2)
    # the Netflix shape at the library's default worker count fails the paper's rule (A-10 replaces it)
    assert mf.mf_feasibility(480_190, 17_771, 1, 1, 9_472) == (False, 888)
    with pytest.raises(mf.MFError):
        mf.mf_feasibility(0, 10, 1, 1, 1)
