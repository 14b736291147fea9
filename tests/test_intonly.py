"""Integer-only executor (SURVEY.md 8(f) row 2; reference intexec.py:40-145, :354-359).

CPU: the oracle's strict integer program and the host trace/check mirror against
golden vectors the reference itself produced (tests/golden/gen_intonly_golden.py).
GPU: the device codes against the same golden codes (acceptance criterion 3,
tests/test_acceptance.py:85-100), zero float categories in the trace, and the
reference's rejections.
"""
import hashlib
import json
import os

import numpy as np
import pytest

from oracle import ptq_oracle as O
from paper_2202_05048_b200.config import QuantConfig, Scheme
from paper_2202_05048_b200.intonly import (IntegerOnlyError, OpTrace, check_integer_only,
                                           integer_program_trace)

GOLD = os.path.join(os.path.dirname(__file__), "golden")
TOYS = ("lenet-ish", "resnet-toy", "mobile-toy")


@pytest.fixture(scope="module")
def intgold():
    with open(os.path.join(GOLD, "ref_intonly.json")) as f:
        meta = json.load(f)
    return np.load(os.path.join(GOLD, "ref_intonly.npz")), meta


def _cfg(fusion=False, **kw):
    base = dict(cache="S2", scheme=Scheme.SymmetricPower2, clipping="Max", granularity="Tensor",
                mixed="Off", fusion=fusion)
    base.update(kw)
    return QuantConfig(**base)


def _sha(s: str) -> str:
    return hashlib.sha256(s.encode()).hexdigest()[:16]


def _oracle_s2(golden, rec):
    arrs, meta = golden
    key = f"{rec}/S2"
    return {t: O.Hist(t, float(arrs[f"cache_range/{key}"][i, 0]), float(arrs[f"cache_range/{key}"][i, 1]),
                      arrs[f"cache_counts/{key}"][i], int(arrs[f"cache_nsamp/{key}"][i]))
            for i, t in enumerate(meta["cache_tensors"][key])}


@pytest.mark.parametrize("fusion", [False, True])
@pytest.mark.parametrize("rec", TOYS)
def test_oracle_integer_only_matches_reference(golden, intgold, ds, toys, rec, fusion):
    arrs, meta = intgold
    cfg = _cfg(fusion)
    qm = O.quantize_model(toys[rec], _oracle_s2(golden, rec), cfg)
    if fusion:
        qm.graph = O.fuse_graph(qm.graph)
    tr = O.OpTrace()
    codes = O.run_integer_only(qm, ds.eval_images, tr)
    key = f"{rec}/fusion{int(fusion)}"
    assert np.array_equal(codes, arrs[f"codes/{key}"])
    assert tr.float_ops() == 0
    assert _sha(tr.to_csv()) == meta["cases"][key]["trace_sha"]
    # criterion 3: identical to the simulated (multiplier) path
    sim = O.run_quantized(O.quantize_model(toys[rec], _oracle_s2(golden, rec), cfg), ds.eval_images)
    assert np.array_equal(O.dequantize_array(codes, qm.act[O._output_tensor(qm.graph)]), sim)


@pytest.mark.parametrize("fusion", [False, True])
@pytest.mark.parametrize("rec", TOYS)
def test_host_trace_matches_reference(intgold, toys, rec, fusion):
    _, meta = intgold
    tr = OpTrace()
    integer_program_trace(toys[rec], _cfg(fusion), tr)
    case = meta["cases"][f"{rec}/fusion{int(fusion)}"]
    assert _sha(tr.to_csv()) == case["trace_sha"]
    assert len(tr.events) == case["trace_events"] and tr.float_ops() == 0


@pytest.mark.parametrize("rec", TOYS)
def test_rejections_match_reference(intgold, toys, rec):
    _, meta = intgold
    for bad, msg in [(dict(scheme=Scheme.Symmetric), "scheme=Symmetric"),
                     (dict(granularity="Channel"), "granularity=Channel"),
                     (dict(mixed="FirstLastFp32"), "mixed=FirstLastFp32")]:
        with pytest.raises(IntegerOnlyError) as e:
            check_integer_only(toys[rec], _cfg(**bad))
        assert str(e.value) == meta["rejects"][f"{rec}/{msg}"]


def test_exact_log2():
    from paper_2202_05048_b200.intonly import exact_log2
    assert exact_log2(0.25) == -2 and exact_log2(1.0) == 0 and exact_log2(2.0 ** -30) == -30
    with pytest.raises(IntegerOnlyError):
        exact_log2(0.3)


# ------------------------------------------------------------------ GPU
@pytest.mark.gpu
@pytest.mark.parametrize("fusion", [False, True])
@pytest.mark.parametrize("rec", TOYS)
def test_gpu_integer_only_codes_bit_exact(golden, intgold, ds, toys, rec, fusion):
    from paper_2202_05048_b200.evaluator import GpuEvaluator
    from test_gpu_parity import golden_caches
    arrs, meta = intgold
    ev = GpuEvaluator(toys[rec], ds, 0, None, calibrate=False)
    try:
        _, ranges, counts, nsamp, _ = golden_caches(golden, rec)
        ev.install_caches(ranges, counts, nsamp)
        tr = OpTrace()
        codes = ev.run_integer_only(_cfg(fusion), trace=tr)
        key = f"{rec}/fusion{int(fusion)}"
        assert codes.dtype == np.int8
        assert np.array_equal(codes, arrs[f"codes/{key}"])
        assert tr.float_ops() == 0 and _sha(tr.to_csv()) == meta["cases"][key]["trace_sha"]
        assert np.array_equal(ev.run_quantized_codes(_cfg(fusion)), codes)
        with pytest.raises(IntegerOnlyError):
            ev.run_integer_only(_cfg(fusion, scheme=Scheme.Symmetric))
    finally:
        ev.close()
