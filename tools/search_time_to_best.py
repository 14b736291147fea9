"""BASELINE config C5: the reference's own search drivers (ptqtune.tuner.tune_grid /
tune_xgb / tune_random, from the offline install in baseline/_ref) driving the GPU
evaluator as their `evaluate` callable -- time-to-best-config of the XGBoost-guided
search vs the grid, on the SqueezeNet IR (ShuffleNet is not expressible in the
reference IR) and on ResNet-18.

    python tools/search_time_to_best.py [--models squeezenet resnet18] [--n-eval 1000]

Prints one JSON line per (model, strategy).  Times are host wall clock around the
driver call (the driver itself is host Python); the evaluator is built once per model after one warm-up
construction (its calibration time is reported separately).
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--models", nargs="+", default=["squeezenet", "resnet18"])
    ap.add_argument("--n-eval", type=int, default=1000)
    ap.add_argument("--budget", type=int, default=96)
    ap.add_argument("--cpu-samples", type=int, default=2, help="reference CPU samples per model (0: skip)")
    ap.add_argument("--cpu-imgs", type=int, default=8)
    args = ap.parse_args()

    import ptqtune as R                                   # the reference driver
    from ptqtune import tuner as RT

    from paper_2202_05048_b200 import build_model, make_accuracy_evaluator, make_dataset
    from paper_2202_05048_b200.fixtures import IMAGENET_SHAPE

    d = make_dataset(n_calib=300, n_eval=args.n_eval, seed=0, shape=IMAGENET_SHAPE)
    space = RT.enumerate_space(RT.TargetProfile("Generic"))
    for name in args.models:
        g = build_model(name, seed=0)
        make_accuracy_evaluator(g, d, 0).close()        # warm-up: CUDA context, library, allocator
        t0 = time.perf_counter()
        ev = make_accuracy_evaluator(g, d, 0)
        t_cal = time.perf_counter() - t0
        stamps = []

        def timed(cfg, _ev=ev, _st=stamps):
            v = _ev(cfg)
            _st.append((time.perf_counter(), v))
            return v

        feats = R.extract_features(g)
        runs = {
            "grid": lambda: RT.tune_grid(None, space, timed, budget=args.budget),
            "xgb": lambda: RT.tune_xgb(feats, space, timed, budget=args.budget, seed=0),
            "random": lambda: RT.tune_random(None, space, timed, budget=args.budget, seed=0),
            # measure_many's thread pool (tuner.py:192-203): concurrent calls coalesce
            "grid-workers8": lambda: RT.tune_grid(None, space, timed, budget=args.budget, workers=8),
        }
        trials = {}
        for strat, fn in runs.items():
            stamps.clear()
            t0 = time.perf_counter()
            res = fn()
            t_all = time.perf_counter() - t0
            best = res.best_top1
            t_best = next(t for t, v in stamps if v == best) - t0
            print(json.dumps({"model": name, "strategy": strat, "n_eval": args.n_eval,
                              "budget": args.budget, "calibrate_s": round(t_cal, 4),
                              "search_s": round(t_all, 4), "time_to_best_s": round(t_best, 4),
                              "trials_to_best": res.trials_to_best, "best_top1": best,
                              "best_config": res.best_config.to_dict(),
                              "evaluator": "paper_2202_05048_b200 GPU (tcgen05 int8)",
                              "driver": "ptqtune.tuner (reference, baseline/_ref)"}), flush=True)
            trials[strat] = (res.trials_to_best, t_all)
        ev.close()
        if args.cpu_samples:
            # the same searches with the reference's own CPU evaluator: the trajectory is the
            # same (identical accuracies), so time-to-best = trials_to_best x the reference's
            # per-config cost (calibration + KL reported separately, as for the GPU lines), measured on a bounded sample (bench.py's sampler:
            # calibrate() of 2 images, clip_range_kl of 1 histogram, quantize_model of 1 config and
            # run_quantized of `cpu_imgs` eval images per sample) and extrapolated linearly
            from bench import ReferenceSampler
            smp = ReferenceSampler(g, d, args.cpu_imgs)
            for _ in range(args.cpu_samples):
                smp.step()
            T = len(g.nodes) + 1
            t_cal_cpu = smp.n_union() * smp.t_cal / smp.n_cal + 3 * T * smp.t_kl / smp.n_kl
            t_cfg_cpu = smp.t_q / smp.n_q + args.n_eval * smp.t_ev / smp.n_ev
            for strat in ("grid", "xgb"):
                n_best = trials[strat][0]
                print(json.dumps({"model": name, "strategy": strat, "n_eval": args.n_eval, "budget": args.budget,
                                  "evaluator": f"reference ptqtune CPU ({smp.kind}, {os.cpu_count()} threads), "
                                               "extrapolated from a bounded sample",
                                  "calibrate_s": round(t_cal_cpu, 1), "per_config_s": round(t_cfg_cpu, 2),
                                  "trials_to_best": n_best,
                                  "time_to_best_s": round(n_best * t_cfg_cpu, 1),
                                  "search_s": round(args.budget * t_cfg_cpu, 1),
                                  "sample": f"{smp.calls} samples: {smp.n_cal} calibration images, {smp.n_kl} KL "
                                            f"sweeps, {smp.n_q} quantize_model, {smp.n_ev} eval images"}), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
