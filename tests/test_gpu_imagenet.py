"""GPU parity on the ImageNet-shaped models (ResNet-50 / ResNet-18 / MobileNet-v2 /
SqueezeNet IR) at a reduced 64x64 input so the numpy oracle finishes in seconds.

These exercise what the 32x32 toys do not: bottleneck blocks with fused
residual adds and downsample convs, BN=256 tiles and multi-stage K loops
(K up to 4608), stride-2 3x3 convs, the packed-im2col RGB stem, 17 depthwise
layers (MobileNet-v2) and fire-module concats (SqueezeNet).

Staged parity P3: the GPU calibrates; the oracle is handed the GPU's caches
and must reproduce every int8 tensor bit-exactly for Mixed=Off configs.
"""
import numpy as np
import pytest

from oracle import ptq_oracle as O
from paper_2202_05048_b200 import GENERIC, build_model, enumerate_space, make_dataset

pytestmark = pytest.mark.gpu
SHAPE = (3, 64, 64)


@pytest.fixture(scope="module")
def ds64():
    return make_dataset(n_calib=300, n_eval=12, seed=0, shape=SHAPE)


def gpu_and_oracle(name, ds64):
    from paper_2202_05048_b200.evaluator import GpuEvaluator
    g = build_model(name, seed=0, shape=SHAPE)
    ev = GpuEvaluator(g, ds64, 0, GENERIC)
    caches = {}
    for k, sc in enumerate(("S1", "S2", "S3")):
        caches[sc] = {t: O.Hist(t, float(ev.cache_ranges[k, i, 0]), float(ev.cache_ranges[k, i, 1]),
                                ev.cache_counts[k, i], int(ev.cache_nsamp[k, i]))
                      for i, t in enumerate(ev.lowered.tensor_names)}
        for i, t in enumerate(ev.lowered.tensor_names):      # device KL == oracle KL sweep
            h = caches[sc][t]
            assert O.clipped_range(h, "KL") == tuple(ev.kl_ranges[k, i]), (name, sc, t)
    return g, ev, caches


@pytest.mark.parametrize("name", ["resnet50", "mobilenet_v2", "squeezenet", "resnet18"])
def test_codes_bit_exact(name, ds64):
    g, ev, caches = gpu_and_oracle(name, ds64)
    space = enumerate_space(GENERIC)
    ev.set_option("fusion", 0)
    try:
        for ci in (2, 20, 54):                    # Asym/Channel, Sym/KL/Tensor, S2 Uint8/Channel
            cfg = space[ci]
            assert cfg.mixed == "Off"
            qm = O.quantize_model(g, caches[cfg.cache], cfg)
            seen = {"input": O.quantize_array(ds64.eval_images, qm.act["input"]).astype(np.int64)}
            O.run_quantized(qm, ds64.eval_images, sink=lambda t, v: seen.__setitem__(t, v))
            for t, v in seen.items():
                if t not in qm.act:
                    continue
                got = ev.probe_codes(cfg, t).reshape(v.shape)
                assert np.array_equal(got, v.astype(np.int8)), (name, ci, t)
    finally:
        ev.set_option("fusion", 1)
    # fused epilogues (relu / residual add folded into the conv): every tensor that is still
    # materialised must carry the same codes
    for ci in (2, 20):
        cfg = space[ci]
        qm = O.quantize_model(g, caches[cfg.cache], cfg)
        seen = {}
        O.run_quantized(qm, ds64.eval_images, sink=lambda t, v: seen.__setitem__(t, v))
        fused_away = 0
        for t, v in seen.items():
            if t not in qm.act:
                continue
            try:
                got = ev.probe_codes(cfg, t).reshape(v.shape)
            except Exception as e:  # noqa: BLE001 - the library reports fused-away tensors
                assert "fused away" in str(e)
                fused_away += 1
                continue
            assert np.array_equal(got, v.astype(np.int8)), (name, ci, t, "fused")
        assert fused_away > 0 or name == "squeezenet"
    ev.close()


@pytest.mark.parametrize("name", ["resnet50", "mobilenet_v2", "squeezenet"])
def test_top1_matches_oracle(name, ds64):
    g, ev, caches = gpu_and_oracle(name, ds64)
    space = enumerate_space(GENERIC)
    picks = [0, 2, 7, 13, 22, 31, 40, 47, 58, 66, 77, 95]
    got = ev.correct_counts([space[i] for i in picks])
    oev = O.make_accuracy_evaluator(g, ds64, 0, caches=caches)
    for i, c in zip(picks, got):
        want = round(oev(space[i]) * len(ds64.eval_labels))
        if space[i].mixed == "Off":
            assert int(c) == want, (name, space[i])
        else:                                     # fp32 first/last layer: ulp-level drift allowed
            assert abs(int(c) - want) <= 1, (name, space[i])
    ev.close()


def test_input_quantizer_at_rounding_boundaries():
    """The s2d input quantizer runs on the fp32 pipe with an fp64 guard: eval images whose
    values sit exactly on, and one fp32 ulp either side of, the reference's RHA rounding
    points (x/s + zp = k + 0.5) must quantize exactly like quantize_array (schemes.py:145-150)."""
    from paper_2202_05048_b200.dataset import Dataset
    from paper_2202_05048_b200.evaluator import GpuEvaluator
    base = make_dataset(n_calib=300, n_eval=12, seed=0, shape=SHAPE)
    g = build_model("resnet50", seed=0, shape=SHAPE)
    space = enumerate_space(GENERIC)
    cfg = space[2]                                 # Asym / Max / Channel, Mixed=Off
    ev = GpuEvaluator(g, base, 0, GENERIC)
    caches = {sc: {t: O.Hist(t, float(ev.cache_ranges[k, i, 0]), float(ev.cache_ranges[k, i, 1]),
                             ev.cache_counts[k, i], int(ev.cache_nsamp[k, i]))
                   for i, t in enumerate(ev.lowered.tensor_names)}
              for k, sc in enumerate(("S1", "S2", "S3"))}
    ev.close()
    qp = O.quantize_model(g, caches[cfg.cache], cfg).act["input"]
    s, z = float(qp.scale), float(qp.zp)
    rng = np.random.default_rng(1)
    n_img = 12
    k = rng.integers(-140, 140, size=(n_img,) + SHAPE)
    x = ((k + 0.5 - z) * s).astype(np.float32)     # on (or next to) the rounding points
    step = rng.integers(-1, 2, size=x.shape)
    x = np.where(step > 0, np.nextafter(x, np.float32(np.inf)),
                 np.where(step < 0, np.nextafter(x, np.float32(-np.inf)), x)).astype(np.float32)
    imgs = np.concatenate([base.images[:base.n_calib], x]).astype(np.float32)
    d = Dataset(images=imgs, labels=np.concatenate([base.labels[:base.n_calib], base.labels[:n_img]]),
                n_calib=base.n_calib)
    ev = GpuEvaluator(g, d, 0, GENERIC)
    ev.set_option("fusion", 0)
    got = ev.probe_codes(cfg, "input").reshape(x.shape)
    want = O.quantize_array(x, qp).astype(np.int8)
    assert np.array_equal(got, want)
    ev.close()


def test_integer_only_profile(ds64):
    """IntegerOnly profile (power-of-two scales, per-tensor, Mixed=Off, optional fusion;
    tuner.py:75-80): the requant multiplier is 2^-s, so the fp64 epilogue equals the
    reference's shift form (intexec.py:80-84).  Every code bit-exact for two configs and the
    top-1 of the whole 12-config IntegerOnly space equal to the oracle's."""
    from paper_2202_05048_b200 import INTEGER_ONLY
    from paper_2202_05048_b200.evaluator import GpuEvaluator
    g = build_model("resnet50", seed=0, shape=SHAPE)
    ev = GpuEvaluator(g, ds64, 0, INTEGER_ONLY)
    caches = {sc: {t: O.Hist(t, float(ev.cache_ranges[k, i, 0]), float(ev.cache_ranges[k, i, 1]),
                             ev.cache_counts[k, i], int(ev.cache_nsamp[k, i]))
                   for i, t in enumerate(ev.lowered.tensor_names)}
              for k, sc in enumerate(("S1", "S2", "S3"))}
    space = enumerate_space(INTEGER_ONLY)
    assert len(space) == 12 and all(c.scheme.value == "SymmetricPower2" for c in space)
    ev.set_option("fusion", 0)
    try:
        for cfg in (space[0], space[-1]):
            qm = O.quantize_model(g, caches[cfg.cache], cfg)
            seen = {}
            O.run_quantized(qm, ds64.eval_images, sink=lambda t, v: seen.__setitem__(t, v))
            for t, v in seen.items():
                if t in qm.act:
                    assert np.array_equal(ev.probe_codes(cfg, t).reshape(v.shape), v.astype(np.int8)), (cfg, t)
    finally:
        ev.set_option("fusion", 1)
    got = ev.correct_counts(space)
    oev = O.make_accuracy_evaluator(g, ds64, 0, caches=caches)
    want = [round(oev(c) * len(ds64.eval_labels)) for c in space]
    assert [int(x) for x in got] == want
    ev.close()


def test_grid_batch_equals_isolated_configs(ds64):
    """evaluate_many reorders a batch by (mixed, cache, scheme, clipping) and reuses the
    quantized graph input / folded FirstLastFp32 prefix across configs that share them: the
    whole grid in one batch must count exactly like every config evaluated on its own right
    after a config of a different parameter variant (nothing left to reuse)."""
    from paper_2202_05048_b200.evaluator import GpuEvaluator
    g = build_model("resnet50", seed=0, shape=SHAPE)
    ev = GpuEvaluator(g, ds64, 0, GENERIC)
    space = enumerate_space(GENERIC)
    batch = ev.correct_counts(space)
    for i, cfg in enumerate(space):
        other = next(c for c in space if (c.cache, c.scheme, c.clipping) != (cfg.cache, cfg.scheme, cfg.clipping)
                     and c.mixed == cfg.mixed)
        ev.correct_counts([other])
        assert int(ev.correct_counts([cfg])[0]) == int(batch[i]), cfg
    ev.close()


def test_dwconv_vectorized_equals_scalar(ds64):
    """k_dwconv_i8_v4 (4 channels per thread) vs the scalar k_dwconv_i8: every depthwise
    output of MobileNet-v2 bit-identical, for zw = 0 and zw != 0 configs."""
    from paper_2202_05048_b200.evaluator import GpuEvaluator
    g = build_model("mobilenet_v2", seed=0, shape=SHAPE)
    ev = GpuEvaluator(g, ds64, 0, GENERIC)
    try:
        ev.set_option("fusion", 0)
        dw = [n.output for n in g.nodes if n.kind == "depthwise_conv2d"]
        assert len(dw) == 17
        for ci in (0, 2, 14):
            cfg = enumerate_space(GENERIC)[ci]
            got = {}
            try:
                for mode in (2, 1, 0):          # register-weight k x k, 4-channel, scalar
                    ev.set_option("dwconv_v4", mode)
                    got[mode] = [ev.probe_codes(cfg, t) for t in dw]
            finally:
                ev.set_option("dwconv_v4", 2)
            for mode in (2, 1):
                for t, a, b in zip(dw, got[mode], got[0]):
                    assert np.array_equal(a, b), (ci, mode, t)
    finally:
        ev.set_option("fusion", 1)
        ev.close()


def test_concat_lut_equals_scalar(ds64):
    """k_concat_codes_v16 (per-block 256-entry requant table, 16 codes per thread) vs the
    per-byte fp64 k_concat_codes: every SqueezeNet concat output bit-identical."""
    from paper_2202_05048_b200.evaluator import GpuEvaluator
    g = build_model("squeezenet", seed=0, shape=SHAPE)
    ev = GpuEvaluator(g, ds64, 0, GENERIC)
    try:
        ev.set_option("fusion", 0)
        cat = [n.output for n in g.nodes if n.kind == "concat"]
        assert len(cat) == 8
        for ci in (0, 2, 14, 30):
            cfg = enumerate_space(GENERIC)[ci]
            fast = [ev.probe_codes(cfg, t) for t in cat]
            ev.set_option("concat_v16", 0)
            try:
                slow = [ev.probe_codes(cfg, t) for t in cat]
            finally:
                ev.set_option("concat_v16", 1)
            for t, a, b in zip(cat, fast, slow):
                assert np.array_equal(a, b), (ci, t)
    finally:
        ev.set_option("fusion", 1)
        ev.close()
