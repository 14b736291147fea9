"""Full-size (BASELINE.json configs[1]: ResNet-50 IR, 224x224, 1000 eval images) GPU
properties.  The numpy oracle cannot run this size in test time, so these check
size-independent invariants of the path on the exact workload the bench measures:

* histogram count conservation: every cache/tensor histogram holds n_images x elems
  samples (calibration.py:81-93 bins every value; lo == hi puts all in bin 0);
* the optimised A-operand paths (TMA tiles, kw-reuse slabs) and the fused epilogues
  (relu / residual-add tables) give exactly the top-1 counts of the plain cp.async
  gather path without fusion;
* the tcgen05 conv equals a CUDA-core reference conv of the same contract on two
  configurations (one with weight zero points) over the whole evaluation set.

Every int8 tensor is already bit-exact against the oracle at 64x64
(test_gpu_imagenet.py); these tests tie the full-size measurement to those paths.
"""
import numpy as np
import pytest

from paper_2202_05048_b200 import GENERIC, build_model, enumerate_space, make_dataset

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ev224():
    from paper_2202_05048_b200.evaluator import GpuEvaluator
    g = build_model("resnet50", 0)
    d = make_dataset(n_calib=300, n_eval=1000, seed=0, shape=(3, 224, 224))
    ev = GpuEvaluator(g, d, 0, GENERIC)
    yield ev
    ev.close()


def test_histogram_count_conservation(ev224):
    counts = ev224.cache_counts.sum(axis=-1)
    assert np.array_equal(counts, ev224.cache_nsamp)
    lo, hi = ev224.cache_ranges[..., 0], ev224.cache_ranges[..., 1]
    assert np.all(lo <= hi)


def test_batched_histograms_equal_per_tensor_launches(ev224):
    """The batched work-list histogram launch (k_histogram_multi, chunks of 2^20 values over
    every cache/tensor) bins every calibration value exactly like one k_histogram launch per
    histogram (the per-tensor kernel is pinned bin-exact against np.histogram in
    test_gpu_parity.py)."""
    from paper_2202_05048_b200 import dist
    from paper_2202_05048_b200.config import CACHE_SIZES, select_images
    ids = [select_images(ev224.n_calib, sc, 0) for sc in CACHE_SIZES]
    sizes = np.asarray([len(i) for i in ids], dtype=np.int32)
    flat = np.concatenate(ids).astype(np.int64)
    got = {}
    for mode in (1, 0):
        ev224.set_option("hist_multi", mode)
        ranges = ev224.forward_minmax(sizes, flat)
        got[mode] = ev224.histogram(ranges)
    ev224.set_option("hist_multi", 1)
    assert np.array_equal(got[0], got[1])
    assert np.array_equal(got[1], ev224.cache_counts)
    del dist


def test_fast_paths_equal_plain_path(ev224):
    space = enumerate_space(GENERIC)
    picks = [space[i] for i in (0, 2, 12, 20, 45, 54, 67, 90)]   # Off + FirstLastFp32, zw = 0 / != 0
    fast = ev224.correct_counts(picks)
    try:
        ev224.set_option("tma", 0)
        ev224.set_option("kwr", -1)
        ev224.set_option("fusion", 0)
        ev224.set_option("subsample", 0)
        plain = ev224.correct_counts(picks)
    finally:
        ev224.set_option("tma", 1)
        ev224.set_option("kwr", 0)
        ev224.set_option("fusion", 1)
        ev224.set_option("subsample", 1)
    assert np.array_equal(fast, plain)
    assert np.all((fast >= 0) & (fast <= 1000))


def test_tc_conv_equals_reference_conv_fullsize(ev224):
    space = enumerate_space(GENERIC)
    picks = [space[12], space[2]]                  # Sym/KL/Tensor and Asym/Max/Channel (zw != 0)
    tc = ev224.correct_counts(picks)
    try:
        ev224.set_option("conv_ref", 1)
        ref = ev224.correct_counts(picks)
    finally:
        ev224.set_option("conv_ref", 0)
    assert np.array_equal(tc, ref)


def test_strided_1x1_subsample_codes_bit_exact(ev224):
    """The downsample shortcuts (1x1, stride 2) run as subsample + pointwise TMA GEMM; their
    output codes must equal the direct strided gather path bit for bit (zw = 0 and != 0)."""
    space = enumerate_space(GENERIC)
    g = ev224.graph
    shortcuts = [n for n in g.nodes if n.kind == "conv2d" and int(n.attrs.get("kernel", 0) or
                 np.asarray(g.weights[n.inputs[1]]).shape[-1]) == 1 and int(n.attrs.get("stride", 1)) > 1]
    assert len(shortcuts) == 3
    def after_add(t):                      # the shortcut feeds an add (+ relu): probe its end
        add = next(m for m in g.nodes if m.kind == "add" and t in m.inputs)
        relu = [m for m in g.nodes if m.kind == "relu" and m.inputs[0] == add.output]
        return relu[0].output if relu else add.output

    for ci in (0, 2):
        for n in shortcuts:
            for fusion, t in ((0, n.output), (1, after_add(n.output))):
                ev224.set_option("fusion", fusion)
                try:
                    fast = ev224.probe_codes(space[ci], t)
                    ev224.set_option("subsample", 0)
                    plain = ev224.probe_codes(space[ci], t)
                finally:
                    ev224.set_option("subsample", 1)
                    ev224.set_option("fusion", 1)
                assert np.array_equal(fast, plain), (ci, n.id, fusion)


def test_mma_row_sums_equal_row_sum_warp(ev224):
    """Asymmetric weights: the row sums Σx the tensor core computes through the K-indicator
    rows of the bn <= 128 weight tiles (rs_mma) must give the same int32 accumulators and
    codes as the row-sum warp / pixel-sum / stem window-sum sources (rs_mma=0), on every
    A-operand mode the bench runs (s2d stem slab, kw-reuse 3x3, TMA 1x1, strided gather)."""
    space = enumerate_space(GENERIC)
    g = ev224.graph
    comp = [n for n in g.nodes if n.kind in ("conv2d", "pointwise_conv2d")]
    by_id = {n.id: n for n in comp}
    probe = [nid for nid in ("conv0", "conv5", "poin25", "conv27", "poin33") if nid in by_id]
    assert len(probe) == 5
    imgs = np.array([0, 137, 421, 999], dtype=np.int32)

    def materialised(t):                         # a relu-fused conv output: probe the relu
        relu = [m for m in g.nodes if m.kind == "relu" and m.inputs[0] == t]
        return relu[0].output if relu else t
    outs = [materialised(by_id[nid].output) for nid in probe]
    for ci in (0, 2):                            # Asymmetric per-tensor / per-channel, Mixed=Off
        cfg = space[ci]
        assert cfg.to_dict()["scheme"] == "Asymmetric"
        got = {}
        for mode in (1, 0):
            ev224.set_option("rs_mma", mode)
            try:
                acc = {nid: ev224.probe_acc(cfg, nid, imgs) for nid in probe}
                codes = ev224.probe_tensors(cfg, outs, imgs)
                counts = ev224.correct_counts([cfg])
            finally:
                ev224.set_option("rs_mma", 1)
            got[mode] = (acc, codes, counts)
        for nid in probe:
            assert np.array_equal(got[1][0][nid], got[0][0][nid]), (ci, nid)
        assert set(got[1][1]) == set(got[0][1]) and len(got[1][1]) >= 3, sorted(got[1][1])
        for t in got[1][1]:
            assert np.array_equal(got[1][1][t], got[0][1][t]), (ci, t)
        assert np.array_equal(np.asarray(got[1][2]), np.asarray(got[0][2])), ci
