"""GPU parity: the CUDA path (through the C-ABI) vs the CPU oracle and the
reference's golden vectors.  Staged protocol of SURVEY.md 8(c):

  P1  histogram binning / min-max given identical fp32 values -> bit-exact
  P2  given identical caches: Max ranges, KL thresholds, scales/zero-points -> exact
  P3  given identical caches: every int8 tensor's codes and the top-1 -> bit-exact
      (Mixed=Off); mixed configs within the fp32-forward tolerance
  P4  end to end with the GPU's own fp32 calibration forward: ranges within
      1e-5 relative, identical chosen configuration.
"""
import numpy as np
import pytest

from oracle import ptq_oracle as O
from paper_2202_05048_b200.config import (CACHE_SIZES, GENERIC, SCHEME_IDS, Scheme,
                                          enumerate_space)

pytestmark = pytest.mark.gpu

TOYS = ("lenet-ish", "resnet-toy", "mobile-toy")


def golden_caches(golden, rec):
    arrs, meta = golden
    T = len(meta["cache_tensors"][f"{rec}/S1"])
    ranges = np.stack([arrs[f"cache_range/{rec}/{sc}"] for sc in CACHE_SIZES])
    counts = np.stack([arrs[f"cache_counts/{rec}/{sc}"] for sc in CACHE_SIZES])
    nsamp = np.stack([arrs[f"cache_nsamp/{rec}/{sc}"] for sc in CACHE_SIZES])
    kl = np.stack([arrs[f"kl_range/{rec}/{sc}"] for sc in CACHE_SIZES])
    return T, ranges, counts, nsamp, kl


def oracle_caches(golden, rec):
    arrs, meta = golden
    out = {}
    for sc in CACHE_SIZES:
        key = f"{rec}/{sc}"
        tids = meta["cache_tensors"][key]
        out[sc] = {t: O.Hist(t, float(arrs[f"cache_range/{key}"][i, 0]), float(arrs[f"cache_range/{key}"][i, 1]),
                             arrs[f"cache_counts/{key}"][i], int(arrs[f"cache_nsamp/{key}"][i]))
                   for i, t in enumerate(tids)}
    return out


@pytest.fixture(scope="module")
def injected(golden, ds, toys):
    """GPU evaluators with the reference's caches injected (device KL sweep)."""
    from paper_2202_05048_b200.evaluator import GpuEvaluator
    evs = {}
    for rec in TOYS:
        ev = GpuEvaluator(toys[rec], ds, 0, GENERIC, calibrate=False)
        T, ranges, counts, nsamp, _ = golden_caches(golden, rec)
        ev.install_caches(ranges, counts, nsamp)
        evs[rec] = ev
    yield evs
    for ev in evs.values():
        ev.close()


# ------------------------------------------------------------------ P1
def test_histogram_exact_adversarial(injected):
    ev = injected["lenet-ish"]
    rng = np.random.default_rng(5)
    for trial in range(40):
        lo = np.float32(rng.normal() * 10 ** rng.uniform(-3, 3))
        hi = np.float32(lo + abs(rng.normal()) * 10 ** rng.uniform(-6, 3) + 1e-30)
        if not lo < hi:
            continue
        edges = np.linspace(float(lo), float(hi), 2049)
        pts = np.concatenate([edges, np.nextafter(edges, -np.inf), np.nextafter(edges, np.inf)])
        x = np.concatenate([rng.uniform(float(lo), float(hi), 20000), pts]).astype(np.float32)
        x = x[(x >= lo) & (x <= hi)]
        x = np.concatenate([x, [lo, hi]]).astype(np.float32)
        want = O.histogram_counts(x, float(lo), float(hi))
        got = ev.histogram_array(x, float(lo), float(hi))
        assert np.array_equal(got, want), trial


def test_histogram_exact_adversarial_large(injected):
    """Arrays large enough for the 16-value batched binning loop (every thread runs several
    4 x float4 rounds): edge points, their fp32 neighbours, exact zeros and the range ends
    mixed into uniform values; counts must equal numpy's histogram exactly."""
    ev = injected["lenet-ish"]
    rng = np.random.default_rng(11)
    for lo, hi in ((-1.3, 2.7), (0.0, 5.0e-3), (-40.0, -0.5)):
        lo, hi = np.float32(lo), np.float32(hi)
        edges = np.linspace(float(lo), float(hi), 2049)
        pts = np.concatenate([edges, np.nextafter(edges, -np.inf), np.nextafter(edges, np.inf)]).astype(np.float32)
        n = 9_000_004
        x = rng.uniform(float(lo), float(hi), n).astype(np.float32)
        x[rng.integers(0, n, 600_000)] = rng.choice(pts, 600_000)
        if lo <= 0 <= hi:
            x[rng.integers(0, n, 2_000_000)] = 0.0
        x[:2] = lo, hi
        x = np.clip(x, lo, hi)
        for m in (n, n - 1):                       # float4 path and scalar path
            want = O.histogram_counts(x[:m], float(lo), float(hi))
            got = ev.histogram_array(x[:m], float(lo), float(hi))
            assert np.array_equal(got, want), (lo, hi, m)


def test_histogram_degenerate(injected):
    ev = injected["lenet-ish"]
    x = np.full(1000, 3.5, np.float32)
    got = ev.histogram_array(x, 3.5, 3.5)
    assert got[0] == 1000 and got[1:].sum() == 0


# ------------------------------------------------------------------ P2
@pytest.mark.parametrize("rec", TOYS)
def test_kl_ranges_match_reference(injected, golden, rec):
    ev = injected[rec]
    _, _, _, _, kl = golden_caches(golden, rec)
    assert np.array_equal(ev.kl_ranges, kl), np.argwhere(ev.kl_ranges != kl)[:5]


@pytest.mark.parametrize("rec", TOYS)
def test_kl_values_match_oracle(injected, golden, rec):
    """Device KL per window == numpy's within a few ulps (and inf where numpy is inf)."""
    ev = injected[rec]
    oc = oracle_caches(golden, rec)
    for k, sc in enumerate(CACHE_SIZES):
        for t, h in enumerate(oc[sc].values()):
            if h.lo == h.hi:
                continue
            _, _, want = O.kl_sweep(h)
            got = ev.kl_values[k, t]
            fin = np.isfinite(want)
            assert np.array_equal(fin, np.isfinite(got))
            assert np.allclose(got[fin], want[fin], rtol=1e-13, atol=0)


def test_kl_canary(injected, golden, ds, toys):
    """SURVEY App. A.K 1-ulp near tie (mobile-toy S1 t_avgp11): with the
    reference's cache the device sweep + host re-rank picks numpy's window
    exactly; with the GPU's own fp32 calibration the threshold stays within
    the 1e-5 relative contract."""
    from paper_2202_05048_b200.evaluator import GpuEvaluator
    _, meta = golden
    want = meta["kl_canary"]["range"]
    ev = injected["mobile-toy"]
    t = ev.lowered.tensor_ids["t_avgp11"]
    assert list(ev.kl_ranges[0, t]) == want
    ev2 = GpuEvaluator(toys["mobile-toy"], ds, 0, GENERIC)
    assert np.allclose(ev2.kl_ranges[0, t], want, rtol=1e-5, atol=0)
    ev2.close()


@pytest.mark.parametrize("rec", TOYS)
def test_act_params_exact(injected, golden, rec):
    ev = injected[rec]
    oc = oracle_caches(golden, rec)
    for k, sc in enumerate(CACHE_SIZES):
        for s in Scheme:
            for ci, clip in enumerate(("Max", "KL")):
                scale, zp = ev.act_params(k, SCHEME_IDS[s], ci)
                for t, h in enumerate(oc[sc].values()):
                    lo, hi = O.clipped_range(h, clip)
                    p = O.params_for_range(s.value, lo, hi)
                    assert np.float32(p.scale).view(np.uint32) == scale[t].view(np.uint32), (sc, s, clip, t)
                    assert int(p.zp) == int(zp[t])


# ------------------------------------------------------------------ P3
def _oracle_codes(qm, ds):
    seen = {}
    O.run_quantized(qm, ds.eval_images, sink=lambda t, v: seen.__setitem__(t, v))
    return seen


@pytest.mark.parametrize("rec", TOYS)
@pytest.mark.parametrize("ci", [0, 2, 6, 10, 14, 17, 22, 26, 30, 45, 63, 90])
def test_codes_every_tensor_bit_exact(injected, golden, ds, toys, rec, ci):
    ev = injected[rec]
    cfg = enumerate_space(GENERIC)[ci]
    oc = oracle_caches(golden, rec)
    qm = O.quantize_model(toys[rec], oc[cfg.cache], cfg)
    want = _oracle_codes(qm, ds)
    if cfg.mixed == "Off":
        want["input"] = O.quantize_array(ds.eval_images, qm.act["input"]).astype(np.int64)
    ev.set_option("fusion", 0)
    try:
        for t, v in want.items():
            if t not in qm.act:
                continue
            got = ev.probe_codes(cfg, t).reshape(v.shape)
            if cfg.mixed == "Off":
                assert np.array_equal(got, v.astype(np.int8)), (rec, cfg, t)
            else:
                # first-layer fp32 output differs from OpenBLAS in the last ulps
                assert np.mean(got != v.astype(np.int8)) < 1e-3, (rec, cfg, t)
    finally:
        ev.set_option("fusion", 1)


@pytest.mark.parametrize("rec", TOYS)
@pytest.mark.parametrize("ci", [2, 12, 50, 92])
def test_accumulators_and_logits_bit_exact(injected, golden, ds, toys, rec, ci):
    """int32-saturated accumulators acc + bias of every int8 compute node (intexec.py:177-190),
    read from the tcgen05 / depthwise launches' accumulator epilogue, and run_quantized's
    dequantized output (intexec.py:346-348, schemes.py:153-155): bit-exact on all eval images
    with the reference's caches (zw != 0 and zw == 0, per-tensor and per-channel)."""
    ev = injected[rec]
    cfg = enumerate_space(GENERIC)[ci]
    qm = O.quantize_model(toys[rec], oracle_caches(golden, rec)[cfg.cache], cfg)
    accs = {}
    out = O.run_quantized(qm, ds.eval_images, accs=accs)
    imgs = np.arange(len(ds.eval_images))
    assert accs
    for node_id, want in accs.items():
        got = ev.probe_acc(cfg, node_id, imgs)
        assert np.array_equal(got, want.reshape(got.shape)), (rec, ci, node_id)
    assert np.array_equal(ev.probe_output(cfg, imgs), np.asarray(out, dtype=np.float32)), (rec, ci)


@pytest.mark.parametrize("rec", TOYS)
def test_grid_matches_reference(injected, golden, rec):
    """Full 96-config grid with the reference's caches: top-1 bit-exact vs App. B."""
    arrs, _ = golden
    ev = injected[rec]
    space = enumerate_space(GENERIC)
    got = np.asarray(ev.evaluate_many(space))
    want = arrs[f"grid/{rec}"]
    off = np.asarray([c.mixed == "Off" for c in space])
    assert np.array_equal(got[off], want[off])
    assert np.max(np.abs(got[~off] - want[~off])) <= 0.01
    assert space[int(np.argmax(got))] == space[int(np.argmax(want))]


def test_tc_conv_equals_reference_conv(injected):
    ev = injected["resnet-toy"]
    space = enumerate_space(GENERIC)
    a = ev.correct_counts(space)
    ev.set_option("conv_ref", 1)
    try:
        b = ev.correct_counts(space)
    finally:
        ev.set_option("conv_ref", 0)
    assert np.array_equal(a, b)


# ------------------------------------------------------------------ P4
@pytest.mark.parametrize("rec", TOYS)
def test_end_to_end_gpu_calibration(golden, ds, toys, rec):
    from paper_2202_05048_b200 import make_accuracy_evaluator
    arrs, meta = golden
    ev = make_accuracy_evaluator(toys[rec], ds, 0, GENERIC)
    T, ranges, counts, nsamp, kl = golden_caches(golden, rec)
    assert np.allclose(ev.cache_ranges, ranges, rtol=1e-5, atol=1e-6)
    assert np.array_equal(ev.cache_nsamp, nsamp)
    # histogram counts differ only where the fp32 forward moved a value across a bin edge
    moved = np.abs(ev.cache_counts - counts).sum() / counts.sum()
    assert moved < 1e-3
    space = enumerate_space(GENERIC)
    got = np.asarray(ev.evaluate_many(space))
    want = arrs[f"grid/{rec}"]
    assert np.max(np.abs(got - want)) <= 0.02
    assert got.max() == want.max()
    ev.close()


@pytest.mark.parametrize("rec", TOYS)
def test_save_cache_matches_reference_file(injected, rec, tmp_path):
    """GpuEvaluator.save_cache writes the evaluator's caches as the
    reference's .qcal, byte-identical to ptqtune.save_cache (tests/golden/ref_qcal.json)."""
    import hashlib
    import json
    import os
    ref = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "ref_qcal.json")))
    ev = injected[rec]
    for sc in ("S1", "S2", "S3"):
        path = tmp_path / f"{sc}.qcal"
        ev.save_cache(str(path), sc)
        assert hashlib.sha256(path.read_bytes()).hexdigest() == ref["qcal"][f"{rec}/{sc}/plain"]["sha256"]


@pytest.mark.parametrize("rec", TOYS)
def test_save_qtm8_matches_reference_file(injected, rec, tmp_path):
    """The quantized model of a config written from device state (artifacts.save_qtm8:
    weight codes / params and int32 bias codes via ptq_export_layer, activation params
    from the device table) is byte-identical to ptqtune.save_quantized
    (tests/golden/ref_qcal.json "qtm8": Generic configs incl. FirstLastFp32 and an
    IntegerOnly config with fusion)."""
    import hashlib
    import json
    import os

    from paper_2202_05048_b200.artifacts import save_qtm8
    from paper_2202_05048_b200.config import QuantConfig
    ref = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "ref_qcal.json")))
    ev = injected[rec]
    keys = [k for k in ref["qtm8"] if k.startswith(rec + "/")]
    assert keys
    for key in keys:
        cfg = QuantConfig.from_dict(ref["qtm8"][key]["config"])
        path = tmp_path / "m.qtm8"
        save_qtm8(str(path), ev, cfg)
        blob = path.read_bytes()
        assert len(blob) == ref["qtm8"][key]["bytes"], key
        assert hashlib.sha256(blob).hexdigest() == ref["qtm8"][key]["sha256"], key


@pytest.mark.parametrize("rec", TOYS)
def test_percentile_matches_oracle(injected, golden, ds, toys, rec):
    """EXTENSION (the reference rejects "Percentile", clipping.py:91-92; parity unpinned):
    the device percentile clipping equals oracle.percentile_range bit-for-bit on the
    reference's histograms, and top-1 with those ranges equals the oracle's (Mixed=Off);
    the KL slot the extension borrows is restored afterwards."""
    arrs, meta = golden
    ev = injected[rec]
    T, ranges, counts, _, _ = golden_caches(golden, rec)
    for pct in (90.0, 99.0, 99.9, 99.99, 100.0):
        got = ev.percentile_ranges(pct)
        for k in range(3):
            for i in range(T):
                want = O.percentile_range(counts[k, i], ranges[k, i, 0], ranges[k, i, 1], pct)
                assert (float(got[k, i, 0]), float(got[k, i, 1])) == want, (pct, k, i)
    space = [c for c in enumerate_space(GENERIC) if c.clipping == "KL" and c.mixed == "Off"]
    kl_before = ev.correct_counts(space)
    pr = ev.percentile_ranges(99.9)
    caches = oracle_caches(golden, rec)
    for k, sc in enumerate(CACHE_SIZES):
        for i, t in enumerate(meta["cache_tensors"][f"{rec}/{sc}"]):
            caches[sc][t].memo["KL"] = (float(pr[k, i, 0]), float(pr[k, i, 1]))
    oev = O.make_accuracy_evaluator(toys[rec], ds, 0, caches=caches)
    got = ev.correct_counts_percentile(space, 99.9)
    n = len(ds.eval_labels)
    for c, g in zip(space[::4], got[::4]):
        assert int(g) == round(oev(c) * n), c
    assert np.array_equal(ev.correct_counts(space), kl_before)
