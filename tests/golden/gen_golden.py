"""Generate golden vectors by running the REFERENCE implementation.

Run in the build container (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/gen_golden.py

Writes tests/golden/ref_golden.npz + ref_golden.json.  Everything in them is
produced by /root/reference/pkg/src/ptqtune itself (never by the oracle), so
tests/test_oracle_golden.py can pin the oracle and the host mirror against
the reference, and the GPU tests can pin the CUDA path against the same
numbers.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

import ptqtune as R
from ptqtune import clipping as RC
from ptqtune import intexec as RI
from ptqtune import quantize as RQ
from ptqtune import schemes as RS

OUT = os.path.dirname(os.path.abspath(__file__))
TOYS = ("lenet-ish", "resnet-toy", "mobile-toy")


def sha(a) -> str:
    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.tobytes() + str(a.dtype).encode() + str(a.shape).encode()).hexdigest()[:16]


def main() -> None:
    arrays: dict[str, np.ndarray] = {}
    meta: dict = {"numpy": np.__version__, "reference": "/root/reference/pkg/src/ptqtune"}

    # ---- host mirror: dataset + fixture hashes (dataset.py / fixtures.py)
    ds = R.make_dataset(seed=0)
    meta["dataset_seed0"] = {"images": sha(ds.images), "labels": sha(ds.labels)}
    meta["fixtures"] = {}
    for rec in TOYS:
        g = R.generate_fixture(rec, 1)
        meta["fixtures"][rec] = {k: sha(v) for k, v in g.weights.items()}

    # ---- scheme KATs (schemes.py:81-131): a grid of ranges incl. degenerate ones
    rng = np.random.default_rng(11)
    ranges = [(0.0, 25.5), (-12.7, 12.7), (-1.0, 1.0), (0.0, 0.0), (-3.0, 0.0), (0.0, 100.0),
              (-0.001, 5.0), (1e-30, 2e-30), (-7.25, 3.5), (2.0, 2.0), (-2.0, -2.0)]
    ranges += [tuple(sorted(rng.normal(0, 10 ** rng.uniform(-4, 3), 2).tolist())) for _ in range(200)]
    ranges += [(0.0, float(v)) for v in 10 ** rng.uniform(-6, 4, 100)]
    rr = np.asarray(ranges, dtype=np.float64)
    arrays["kat_ranges"] = rr
    for s in R.Scheme:
        sc, zp = [], []
        for lo, hi in ranges:
            p = RS.params_for_range(s, lo, hi)
            sc.append(np.float32(p.scale))
            zp.append(int(p.zero_point))
        arrays[f"kat_scale_{s.value}"] = np.asarray(sc, dtype=np.float32)
        arrays[f"kat_zp_{s.value}"] = np.asarray(zp, dtype=np.int64)

    # quantize_array / requantize KATs
    xs = np.concatenate([rng.normal(0, 3, 5000), np.arange(-20, 20) * 0.05, [0.5, -0.5, 1.5, -1.5]])
    arrays["kat_q_x"] = xs.astype(np.float32)
    for s in R.Scheme:
        p = RS.params_for_range(s, -2.0, 3.0)
        arrays[f"kat_q_codes_{s.value}"] = RS.quantize_array(xs.astype(np.float32), p)
    accs = rng.integers(-2 ** 31, 2 ** 31 - 1, 4000)
    mults = 10 ** rng.uniform(-9, 0, 4000)
    zps = rng.integers(-128, 128, 4000)
    arrays["kat_rq_acc"], arrays["kat_rq_m"], arrays["kat_rq_zp"] = accs, mults, zps
    arrays["kat_rq_out"] = np.asarray([RI.requantize(a, multiplier=m, zero_point=int(z))
                                       for a, m, z in zip(accs, mults, zps)], dtype=np.int8)

    # ---- calibration caches + KL picks + the 96-config grids (App. B)
    meta["grids"] = {}
    for rec in TOYS:
        g = R.generate_fixture(rec, 1)
        ev = R.make_accuracy_evaluator(g, ds, seed=0)
        caches = {sc: R.build_cache(g, ds, sc, seed=0) for sc in RQ.CACHE_SIZES}
        for sc, cache in caches.items():
            tids = list(cache.histograms)
            h = [cache.histograms[t] for t in tids]
            key = f"{rec}/{sc}"
            meta.setdefault("cache_tensors", {})[key] = tids
            meta.setdefault("cache_ids", {})[key] = [int(i) for i in cache.image_ids]
            arrays[f"cache_range/{key}"] = np.asarray([[x.min_seen, x.max_seen] for x in h], dtype=np.float32)
            arrays[f"cache_counts/{key}"] = np.stack([x.bin_counts for x in h]).astype(np.int64)
            arrays[f"cache_nsamp/{key}"] = np.asarray([x.n_samples for x in h], dtype=np.int64)
            arrays[f"kl_range/{key}"] = np.asarray([RC.clip_range_kl(x) for x in h], dtype=np.float64)
        space = R.enumerate_space(R.TargetProfile("Generic"))
        res = R.tune_grid(None, space, ev, budget=len(space))
        accs = np.asarray([r.top1 for r in res.trials], dtype=np.float64)
        arrays[f"grid/{rec}"] = accs
        meta["grids"][rec] = {"sha_f64": hashlib.sha256(accs.tobytes()).hexdigest()[:16],
                              "best": res.best_config.to_dict(), "best_top1": res.best_top1,
                              "trials_to_best": res.trials_to_best}
        # per-node code hashes for two configs (staged parity P3)
        for ci in (2, 45):
            cfg = space[ci]
            qg = RQ.quantize_model(g, caches[cfg.cache], cfg)
            seen = {}
            RI.run_quantized(qg, ds.eval_images, sink=lambda t, v: seen.__setitem__(t, sha(np.asarray(v))))
            meta.setdefault("node_sha", {})[f"{rec}/{ci}"] = seen
        print(rec, "grid", accs.min(), accs.max(), flush=True)

    # KL near-tie canary (SURVEY App. A.K): mobile-toy seed 1, S1, t_avgp11
    g = R.generate_fixture("mobile-toy", 1)
    h = R.build_cache(g, ds, "S1", seed=0).histograms["t_avgp11"]
    meta["kl_canary"] = {"range": list(RC.clip_range_kl(h))}

    np.savez_compressed(os.path.join(OUT, "ref_golden.npz"), **arrays)
    with open(os.path.join(OUT, "ref_golden.json"), "w") as f:
        json.dump(meta, f, indent=1, sort_keys=True)
    print("wrote", len(arrays), "arrays")


if __name__ == "__main__":
    sys.exit(main())
