"""Pin the CPU oracle against golden vectors produced by the reference itself
(tests/golden/gen_golden.py)."""
import numpy as np
import pytest

from oracle import ptq_oracle as O
from paper_2202_05048_b200.config import CACHE_SIZES, GENERIC, enumerate_space

SCHEMES = ("Asymmetric", "Symmetric", "SymmetricUint8", "SymmetricPower2")


@pytest.mark.parametrize("scheme", SCHEMES)
def test_scheme_params(golden, scheme):
    arrs, _ = golden
    sc, zp = [], []
    for lo, hi in arrs["kat_ranges"]:
        p = O.params_for_range(scheme, lo, hi)
        sc.append(np.float32(p.scale))
        zp.append(int(p.zp))
    assert np.array_equal(np.asarray(sc, np.float32).view(np.uint32), arrs[f"kat_scale_{scheme}"].view(np.uint32))
    assert np.array_equal(np.asarray(zp), arrs[f"kat_zp_{scheme}"])


@pytest.mark.parametrize("scheme", SCHEMES)
def test_quantize_array(golden, scheme):
    arrs, _ = golden
    p = O.params_for_range(scheme, -2.0, 3.0)
    assert np.array_equal(O.quantize_array(arrs["kat_q_x"], p), arrs[f"kat_q_codes_{scheme}"])


def test_requantize(golden):
    arrs, _ = golden
    out = np.asarray([O.requantize(a, m, int(z)) for a, m, z in
                      zip(arrs["kat_rq_acc"], arrs["kat_rq_m"], arrs["kat_rq_zp"])], dtype=np.int8)
    assert np.array_equal(out, arrs["kat_rq_out"])


def _hist(arrs, meta, key, i):
    lo, hi = arrs[f"cache_range/{key}"][i]
    return O.Hist(meta["cache_tensors"][key][i], float(lo), float(hi),
                  arrs[f"cache_counts/{key}"][i], int(arrs[f"cache_nsamp/{key}"][i]))


@pytest.mark.parametrize("rec", ["lenet-ish", "resnet-toy", "mobile-toy"])
def test_calibration_caches(golden, ds, toys, rec):
    arrs, meta = golden
    for sc in ("S1", "S2"):
        key = f"{rec}/{sc}"
        cache = O.build_cache(toys[rec], ds, sc, 0)
        assert list(cache) == meta["cache_tensors"][key]
        rng = np.asarray([[h.lo, h.hi] for h in cache.values()], dtype=np.float32)
        assert np.array_equal(rng, arrs[f"cache_range/{key}"])
        assert np.array_equal(np.stack([h.counts for h in cache.values()]), arrs[f"cache_counts/{key}"])


@pytest.mark.parametrize("rec", ["lenet-ish", "resnet-toy", "mobile-toy"])
def test_kl_ranges(golden, rec):
    arrs, meta = golden
    for sc in CACHE_SIZES:
        key = f"{rec}/{sc}"
        want = arrs[f"kl_range/{key}"]
        for i in range(len(meta["cache_tensors"][key])):
            assert O.clip_range_kl(_hist(arrs, meta, key, i)) == tuple(want[i])


def test_kl_canary(golden, ds, toys):
    _, meta = golden
    cache = O.build_cache(toys["mobile-toy"], ds, "S1", 0)
    assert list(O.clip_range_kl(cache["t_avgp11"])) == meta["kl_canary"]["range"]


@pytest.mark.parametrize("rec", ["lenet-ish", "resnet-toy", "mobile-toy"])
def test_grid_subset(golden, ds, toys, rec):
    """Every 5th config of the 96-grid, caches injected from the golden file."""
    arrs, meta = golden
    caches = {}
    for sc in CACHE_SIZES:
        key = f"{rec}/{sc}"
        caches[sc] = {meta["cache_tensors"][key][i]: _hist(arrs, meta, key, i)
                      for i in range(len(meta["cache_tensors"][key]))}
    ev = O.make_accuracy_evaluator(toys[rec], ds, 0, caches=caches)
    space = enumerate_space(GENERIC)
    want = arrs[f"grid/{rec}"]
    for ci in range(0, 96, 5):
        assert ev(space[ci]) == want[ci], (rec, ci, space[ci])
