"""The reference's own search drivers (ptqtune.tuner, from the offline install in
baseline/_ref -- skipped when it is absent) calling the GPU evaluator as their
`evaluate` callable: the drop-in claim of SURVEY.md 8(b) exercised through the
reference's code, not a mirror of it.  Caches are the reference's own (golden), so the
grid must reproduce the reference's App. B accuracies (bit-exact for Mixed=Off)."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def RT():
    if not os.path.isdir(os.path.join(REF, "ptqtune")):
        pytest.skip("reference install baseline/_ref absent")
    sys.path.insert(0, REF)
    try:
        from ptqtune import tuner
    finally:
        sys.path.remove(REF)
    return tuner


@pytest.mark.parametrize("rec", ["lenet-ish", "resnet-toy"])
@pytest.mark.parametrize("workers", [1, 8])
def test_reference_tune_grid_drives_gpu_evaluator(RT, golden, ds, toys, rec, workers):
    from paper_2202_05048_b200.evaluator import GpuEvaluator
    from test_gpu_parity import golden_caches
    arrs, meta = golden
    ev = GpuEvaluator(toys[rec], ds, 0, None, calibrate=False)
    try:
        _, ranges, counts, nsamp, _ = golden_caches(golden, rec)
        ev.install_caches(ranges, counts, nsamp)
        space = RT.enumerate_space(RT.TargetProfile("Generic"))
        res = RT.tune_grid(None, space, ev, budget=len(space), workers=workers)
        got = np.asarray([t.top1 for t in res.trials])
        assert not any(t.error for t in res.trials)
        want = arrs[f"grid/{rec}"]
        off = np.asarray([c.mixed == "Off" for c in space])
        assert np.array_equal(got[off], want[off])
        assert np.max(np.abs(got[~off] - want[~off])) <= 0.01
        assert abs(res.best_top1 - meta["grids"][rec]["best_top1"]) <= 0.01
    finally:
        ev.close()


def test_reference_tune_xgb_drives_gpu_evaluator(RT, golden, ds, toys):
    """Sequential XGBoost-guided search (tuner.py:251-281) through the GPU evaluator
    takes the same trajectory as through a table of the reference's own accuracies,
    up to the first config whose GPU top-1 differs from the reference's (only
    FirstLastFp32 configs may, by fp32 ulps)."""
    from paper_2202_05048_b200.evaluator import GpuEvaluator
    from test_gpu_parity import golden_caches
    sys.path.insert(0, REF)
    try:
        from ptqtune.ir import extract_features
    finally:
        sys.path.remove(REF)
    arrs, _ = golden
    rec = "resnet-toy"
    space = RT.enumerate_space(RT.TargetProfile("Generic"))
    want = arrs[f"grid/{rec}"]
    index = {c: i for i, c in enumerate(space)}
    feats = extract_features(toys[rec])
    ref = RT.tune_xgb(feats, space, lambda c: float(want[index[c]]), budget=30, seed=0)
    ev = GpuEvaluator(toys[rec], ds, 0, None, calibrate=False)
    try:
        _, ranges, counts, nsamp, _ = golden_caches(golden, rec)
        ev.install_caches(ranges, counts, nsamp)
        res = RT.tune_xgb(feats, space, ev, budget=30, seed=0)
    finally:
        ev.close()
    assert len(res.trials) == len(ref.trials) == 30
    for a, b in zip(res.trials, ref.trials):
        assert a.config == b.config
        if a.top1 != b.top1:
            assert a.config.mixed == "FirstLastFp32" and abs(a.top1 - b.top1) <= 0.01
            break
