"""Oracle parity at BASELINE.json's sizes: 224x224 inputs, 1000 eval images, the exact
evaluator the bench times (ResNet-50 = C4, ResNet-18 = C2, MobileNet-v2 = C3).

The GPU evaluates the whole 1000-image eval split -- so every BN >= 64 tcgen05 launch runs
many tiles per CTA through both TMEM accumulators and every A-operand mode (TMA 64/128,
stem slab, kw-reuse, subsample, gather) -- and the probes copy out 8 images spread over the
batch.  The oracle (oracle/ptq_oracle.py, pinned to the reference's golden vectors) is
handed the GPU's calibration caches (staged parity P3) and runs those 8
images through run_quantized (ref intexec.py:148-351).  Checked bit-exact:

* every int8 tensor's codes, fusion off (all tensors materialised) and on (fused relu /
  residual-add epilogues; the tensors still materialised);
* the int32-saturated accumulators acc + bias of every int8 compute node
  (intexec.py:177-190), read from the same tcgen05 / depthwise launches;
* run_quantized's return value: dequantized output logits (schemes.py:153-155).

FirstLastFp32 (intexec.py:304-334): the fp32 first-layer output and the fp32 logits of the
last layer (given the GPU's own int8 input codes of that layer) within 1e-5 relative.

P4 at 224^2: the GPU's own fp32 calibration forward of a 2-image cache against the
oracle's calibrate() on the same images (ranges within 1e-5 relative; histograms of the
GPU's activations binned with the oracle's ranges: at most 1e-3 of a tensor's samples move to a
neighbouring bin, the same bound as the toy-size P4 test).
"""
import numpy as np
import pytest

from oracle import ptq_oracle as O
from paper_2202_05048_b200 import GENERIC, build_model, enumerate_space, make_dataset

pytestmark = pytest.mark.gpu

SHAPE = (3, 224, 224)
IMGS = [0, 3, 137, 250, 421, 600, 871, 999]
# Asym/Max/Channel (zw != 0), Sym/KL/Tensor, S2 Uint8/Max/Channel, S3 Pow2/KL/Tensor
CFGS = (2, 12, 50, 92)
MIXED_CFG = 3                       # S1 / Asym / Max / Channel / FirstLastFp32


@pytest.fixture(scope="module")
def ds224():
    return make_dataset(n_calib=300, n_eval=1000, seed=0, shape=SHAPE)


_CACHE = {}


def setup(name, ds224):
    if name in _CACHE:
        return _CACHE[name]
    from paper_2202_05048_b200.evaluator import GpuEvaluator
    g = build_model(name, seed=0, shape=SHAPE)
    ev = GpuEvaluator(g, ds224, 0, GENERIC)
    caches = {}
    for k, sc in enumerate(("S1", "S2", "S3")):
        caches[sc] = {t: O.Hist(t, float(ev.cache_ranges[k, i, 0]), float(ev.cache_ranges[k, i, 1]),
                                ev.cache_counts[k, i], int(ev.cache_nsamp[k, i]))
                      for i, t in enumerate(ev.lowered.tensor_names)}
        for i, t in enumerate(ev.lowered.tensor_names):   # seed the oracle's KL memo with the
            caches[sc][t].memo["KL"] = tuple(ev.kl_ranges[k, i])   # device choice (checked below)
    for old in list(_CACHE.values()):            # one 224^2 evaluator alive at a time
        old[1].close()
    _CACHE.clear()
    _CACHE[name] = (g, ev, caches)
    return _CACHE[name]


def oracle_run(g, caches, cfg, imgs):
    qm = O.quantize_model(g, caches[cfg.cache], cfg)
    seen, accs = {}, {}
    seen["input"] = O.quantize_array(imgs, qm.act["input"]).astype(np.int64) if "input" in qm.act else None
    out = O.run_quantized(qm, imgs, sink=lambda t, v: seen.__setitem__(t, v), accs=accs)
    return qm, seen, accs, out


@pytest.mark.parametrize("name", ["resnet50", "resnet18", "mobilenet_v2"])
def test_codes_accs_logits_224(name, ds224):
    g, ev, caches = setup(name, ds224)
    space = enumerate_space(GENERIC)
    imgs = ds224.eval_images[IMGS]
    for ci in CFGS:
        cfg = space[ci]
        assert cfg.mixed == "Off"
        qm, seen, accs, out = oracle_run(g, caches, cfg, imgs)
        tensors = [t for t in seen if t in qm.act]
        for fusion in (0, 1):
            ev.set_option("fusion", fusion)
            try:
                got = ev.probe_tensors(cfg, tensors, IMGS)
            finally:
                ev.set_option("fusion", 1)
            if fusion == 0:
                assert set(got) == set(tensors), (name, ci)
            else:
                assert len(got) < len(tensors) or name == "squeezenet"
            for t, v in got.items():
                assert np.array_equal(v, seen[t].astype(np.int8).reshape(v.shape)), (name, ci, fusion, t)
        # dequantized output logits (run_quantized's return value)
        logits = ev.probe_output(cfg, IMGS)
        assert np.array_equal(logits, np.asarray(out, dtype=np.float32)), (name, ci)
        # int32 accumulators of every int8 compute node, for the zw != 0 config and one zw == 0
        if ci in (2, 12):
            for n in g.nodes:
                if n.id not in accs:
                    continue
                a = ev.probe_acc(cfg, n.id, IMGS)
                assert np.array_equal(a, accs[n.id].reshape(a.shape)), (name, ci, n.id)


@pytest.mark.parametrize("name", ["resnet50", "mobilenet_v2"])
def test_first_last_fp32_224(name, ds224):
    g, ev, caches = setup(name, ds224)
    cfg = enumerate_space(GENERIC)[MIXED_CFG]
    assert cfg.mixed == "FirstLastFp32"
    imgs = ds224.eval_images[IMGS]
    comp = [n for n in g.nodes if n.kind in O.COMPUTE_KINDS]
    first, last = comp[0], comp[-1]
    # fp32 first layer (config-invariant prefix) vs the oracle's fp32 conv (ref fp32.py:41-51)
    f = ev.probe_f32(cfg, first.output, IMGS)
    w = g.weights[first.inputs[1]]
    b = g.weights[first.inputs[2]] if len(first.inputs) > 2 else None
    ref = O.conv2d(imgs.astype(np.float32), w, b, int(first.attrs.get("stride", 1)),
                   int(first.attrs.get("padding", 0))).astype(np.float32)
    assert f.shape == ref.shape
    np.testing.assert_allclose(f, ref, rtol=1e-5, atol=1e-5 * float(np.abs(ref).max()))
    # fp32 last layer given the GPU's own int8 input codes: dequantize + fp32 fc + bias
    qm = O.quantize_model(g, caches[cfg.cache], cfg)
    xin = last.inputs[0]
    codes = ev.probe_tensors(cfg, [xin], IMGS)[xin]
    x = O.dequantize_array(codes.astype(np.int8), qm.act[xin])
    wl = g.weights[last.inputs[1]]
    want = x.reshape(len(IMGS), -1).astype(np.float32) @ wl.T
    if len(last.inputs) > 2:
        want = want + g.weights[last.inputs[2]]
    got = ev.probe_output(cfg, IMGS)
    np.testing.assert_allclose(got, want, rtol=1e-5, atol=1e-5 * float(np.abs(want).max()))
    # the int8 network between the fp32 layers, on identical inputs: the boundary codes are
    # quantize_array of the GPU's own fp32 first-layer output (exact), and with those codes
    # injected the oracle reproduces every downstream int8 tensor bit for bit
    ev.set_option("fusion", 0)
    try:
        tensors = [t for t in qm.act if t != "input"]
        got = ev.probe_tensors(cfg, tensors, IMGS)
    finally:
        ev.set_option("fusion", 1)
    boundary = O.quantize_array(f, qm.act[first.output]).astype(np.int8)
    assert np.array_equal(got[first.output], boundary), name
    seen = {}
    logits = O.run_quantized(qm, imgs, sink=lambda t, v: seen.__setitem__(t, v),
                             inject={first.output: got[first.output].astype(np.int64)})
    for t, v in got.items():
        assert np.array_equal(v, seen[t].astype(np.int8).reshape(v.shape)), (name, t)
    np.testing.assert_allclose(ev.probe_output(cfg, IMGS), logits, rtol=1e-5,
                               atol=1e-5 * float(np.abs(logits).max()))


def test_kl_ranges_match_oracle_224(ds224):
    """The device KL sweep + host tie re-rank choose the oracle's window for every histogram
    of the three ResNet-50 caches (clipping.py:55-86)."""
    g, ev, _ = setup("resnet50", ds224)
    for k in range(3):
        for i, t in enumerate(ev.lowered.tensor_names):
            h = O.Hist(t, float(ev.cache_ranges[k, i, 0]), float(ev.cache_ranges[k, i, 1]),
                       ev.cache_counts[k, i], int(ev.cache_nsamp[k, i]))
            assert O.clipped_range(h, "KL") == tuple(ev.kl_ranges[k, i]), (k, t)


@pytest.mark.parametrize("name", ["resnet50", "mobilenet_v2"])
def test_own_calibration_p4_224(name, ds224):
    """P4: the GPU's fp32 observer forward + F1 kernels on 2 calibration images against the
    oracle's calibrate() (calibration.py:57-106) on the same images."""
    from paper_2202_05048_b200.evaluator import GpuEvaluator
    g = build_model(name, seed=0, shape=SHAPE)
    ev = GpuEvaluator(g, ds224, 0, GENERIC, calibrate=False)
    try:
        ids = np.array([17, 204], dtype=np.int64)
        local = ev.forward_minmax(np.array([2], dtype=np.int32), ids)[0]
        want = O.calibrate(g, ds224.images[ids])
        names = ev.lowered.tensor_names
        ranges = np.array([[want[t].lo, want[t].hi] for t in names], dtype=np.float32)
        for i, t in enumerate(names):
            for j in range(2):
                a, b = float(local[i, j]), float(ranges[i, j])
                assert abs(a - b) <= 1e-5 * max(abs(a), abs(b)) + 1e-30, (name, t, j, a, b)
        # histograms of the GPU's own activations binned with the oracle's ranges
        counts = ev.histogram(ranges[None])[0]
        for i, t in enumerate(names):
            # (a GPU value just outside the oracle's range is dropped, as np.histogram does)
            moved = int(np.abs(counts[i] - want[t].counts).sum()) // 2
            assert moved <= max(4, int(1e-3 * counts[i].sum())), (name, t, moved)
    finally:
        ev.close()


def test_minmax_kernel_identical_inputs():
    """P1 for minmax_sink (calibration.py:67-76): the F1a kernels over identical fp32 arrays
    give numpy's exact min / max, for odd sizes, unaligned tails, signed zeros, subnormals and
    extreme magnitudes."""
    from paper_2202_05048_b200 import generate_fixture
    from paper_2202_05048_b200.evaluator import GpuEvaluator
    g = generate_fixture("lenet-ish", 1)
    d = make_dataset(n_calib=8, n_eval=4, seed=0)
    ev = GpuEvaluator(g, d, 0, GENERIC, calibrate=False)
    rng = np.random.default_rng(5)
    try:
        for n_img, elems in ((1, 1), (3, 7), (5, 4099), (2, 1 << 20), (7, 802816)):
            x = (rng.standard_normal((n_img, elems)) * 10.0 ** rng.integers(-40, 38)).astype(np.float32)
            x.ravel()[rng.integers(0, x.size, 3)] = np.float32(-0.0)
            x.ravel()[rng.integers(0, x.size, 2)] = np.float32(1e-45)
            assert ev.minmax_array(x) == (float(x.min()), float(x.max())), (n_img, elems)
        x = np.full((3, 33), -0.0, dtype=np.float32)
        assert ev.minmax_array(x) == (0.0, 0.0)
    finally:
        ev.close()
