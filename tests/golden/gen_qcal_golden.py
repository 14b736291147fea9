"""Golden hashes of the reference's calibration-cache files (.qcal).

Run in the build container (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/gen_qcal_golden.py

For every toy fixture and cache size class, the reference builds the cache
(calibration.py:109-112) and writes it with its own save_cache
(calibration.py:115-134); the sha256 and length of those bytes go to
tests/golden/ref_qcal.json.  paper_2202_05048_b200.artifacts must reproduce them
byte for byte from the same cache content (tests/test_artifacts.py) and from the
GPU evaluator's device state (tests/test_gpu_parity.py).
"""

from __future__ import annotations

import hashlib
import json
import os
import tempfile

import ptqtune as R
from ptqtune import calibration as RCAL
from ptqtune import quantize as RQ

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
    with open(os.path.join(OUT, "ref_qcal.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
