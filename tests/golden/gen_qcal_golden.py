"""Golden hashes of the reference's artifact files: calibration caches (.qcal) and
quantized models (.qtm8).

Run in the build container (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/gen_qcal_golden.py

For every toy fixture and cache size class, the reference builds the cache
(calibration.py:109-112) and writes it with its own save_cache
(calibration.py:115-134); the sha256 and length of those bytes go to
tests/golden/ref_qcal.json.  paper_2202_05048_b200.artifacts must reproduce them
byte for byte from the same cache content (tests/test_artifacts.py) and from the
GPU evaluator's device state (tests/test_gpu_parity.py).  For the .qtm8 files the
reference quantizes a few configurations of each toy (quantize_model,
quantize.py:133-211) with those caches and writes them with save_quantized
(quantize.py:254-300); the GPU evaluator must write the same bytes from its device
state (tests/test_gpu_parity.py).
"""

from __future__ import annotations

import hashlib
import json
import os
import tempfile

import ptqtune as R
from ptqtune import calibration as RCAL
from ptqtune import quantize as RQ

QTM8_CONFIGS = (0, 2, 7, 30)          # Generic-space indices (Asym/Tensor, Asym/Channel, mixed, Pow2/KL)

OUT = os.path.dirname(os.path.abspath(__file__))
TOYS = ("lenet-ish", "resnet-toy", "mobile-toy")


def main() -> None:
    ds = R.make_dataset(seed=0)
    out = {"model_name": {}, "qcal": {}}
    with tempfile.TemporaryDirectory() as tmp:
        for rec in TOYS:
            g = R.generate_fixture(rec, 1)
            out["model_name"][rec] = g.name
            for sc in RQ.CACHE_SIZES:
                cache = R.build_cache(g, ds, sc, seed=0)
                for tag, meta in (("plain", None), ("meta", {"seed": 0, "tool": "ptqtune"})):
                    path = os.path.join(tmp, f"{rec}_{sc}_{tag}.qcal")
                    RCAL.save_cache(cache, path, meta=meta)
                    blob = open(path, "rb").read()
                    out["qcal"][f"{rec}/{sc}/{tag}"] = {"sha256": hashlib.sha256(blob).hexdigest(),
                                                        "bytes": len(blob)}
    out["qtm8"] = {}
    space = R.enumerate_space(R.TargetProfile("Generic"))
    io_space = R.enumerate_space(R.TargetProfile("IntegerOnly"))
    with tempfile.TemporaryDirectory() as tmp:
        for rec in TOYS:
            g = R.generate_fixture(rec, 1)
            caches = {sc: R.build_cache(g, ds, sc, seed=0) for sc in RQ.CACHE_SIZES}
            picks = [("g%d" % i, space[i]) for i in QTM8_CONFIGS] + [("io_last", io_space[-1])]
            for tag, cfg in picks:
                qg = RQ.quantize_model(g, caches[cfg.cache], cfg)
                path = os.path.join(tmp, f"{rec}_{tag}.qtm8")
                RQ.save_quantized(qg, path)
                blob = open(path, "rb").read()
                out["qtm8"][f"{rec}/{tag}"] = {"config": cfg.to_dict(), "bytes": len(blob),
                                               "sha256": hashlib.sha256(blob).hexdigest()}
    with open(os.path.join(OUT, "ref_qcal.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
