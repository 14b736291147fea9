"""Golden vectors for the integer-only executor, produced by
running the REFERENCE's run_integer_only / OpTrace (intexec.py:48-64, :132-145,
:354-359) in the build container:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/gen_intonly_golden.py

Writes tests/golden/ref_intonly.npz (output codes) + ref_intonly.json (trace CSV
hashes, event counts, rejection messages).  Acceptance criterion 3
(tests/test_acceptance.py:85-100) is the case recorded for fusion=False.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

import ptqtune as R
from ptqtune import intexec as RI
from ptqtune import quantize as RQ

OUT = os.path.dirname(os.path.abspath(__file__))
TOYS = ("lenet-ish", "resnet-toy", "mobile-toy")


def main() -> None:
    ds = R.make_dataset(seed=0)
    arrays, meta = {}, {"reference": "/root/reference/pkg/src/ptqtune", "cases": {}, "rejects": {}}
    for rec in TOYS:
        g = R.generate_fixture(rec, 1)
        cache = R.build_cache(g, ds, "S2", seed=0)
        for fusion in (False, True):
            cfg = RQ.QuantConfig(cache="S2", scheme=R.Scheme.SymmetricPower2, clipping="Max",
                                 granularity="Tensor", mixed="Off", fusion=fusion)
            qg = RQ.quantize_model(g, cache, cfg)
            tr = RI.OpTrace()
            codes = RI.run_integer_only(qg, ds.eval_images, trace=tr)
            sim = RI.run_quantized(qg, ds.eval_images, return_codes=True)
            assert np.array_equal(codes, sim)
            ftr = RI.OpTrace()
            RI.run_quantized(qg, ds.eval_images, trace=ftr)
            key = f"{rec}/fusion{int(fusion)}"
            arrays[f"codes/{key}"] = codes
            csv = tr.to_csv()
            meta["cases"][key] = {
                "trace_sha": hashlib.sha256(csv.encode()).hexdigest()[:16],
                "trace_events": len(tr.events), "float_ops": tr.float_ops(),
                "sim_trace_sha": hashlib.sha256(ftr.to_csv().encode()).hexdigest()[:16],
                "sim_float_ops": ftr.float_ops(), "sim_trace_events": len(ftr.events)}
        for bad in (dict(scheme=R.Scheme.Symmetric), dict(granularity="Channel"),
                    dict(mixed="FirstLastFp32")):
            cfg = RQ.QuantConfig(**{**dict(cache="S2", scheme=R.Scheme.SymmetricPower2, clipping="Max",
                                           granularity="Tensor", mixed="Off"), **bad})
            qg = RQ.quantize_model(g, cache, cfg)
            try:
                RI.run_integer_only(qg, ds.eval_images[:2])
                msg = None
            except RI.IntegerOnlyError as e:
                msg = str(e)
            meta["rejects"][f"{rec}/{'/'.join(f'{k}={getattr(v, 'value', v)}' for k, v in bad.items())}"] = msg
    np.savez_compressed(os.path.join(OUT, "ref_intonly.npz"), **arrays)
    with open(os.path.join(OUT, "ref_intonly.json"), "w") as f:
        json.dump(meta, f, indent=1, sort_keys=True)
    print(json.dumps(meta, indent=1))


if __name__ == "__main__":
    sys.exit(main())
