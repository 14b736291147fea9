"""Benchmark: quant configs evaluated/sec (calibration + int8 eval, ResNet-50,
1k synthetic 224^2 images), BASELINE.json's headline metric.

One step = one full-grid PTQ campaign, exactly what the reference's
``make_accuracy_evaluator`` + ``tune_grid(budget=96)`` does
(ptqtune/tuner.py:434-444, :225-245): calibrate the S1/S2/S3 caches (fp32
forward over the 289 sampled calibration images, exact min/max, 2048-bin
histograms), KL threshold sweep of every histogram, weight/activation
quantization for every variant, and the int8 forward + top-1 of all 96
configurations over the 1000 eval images.  metric = 96 / step time.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

Under torchrun (N>1) calibration images and configurations are sharded over
ranks (paper_2202_05048_b200/dist.py); time = max over ranks.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "quant configs evaluated/sec (calib+int8 eval, ResNet-50, 1k imgs)"
UNIT = "configs/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--model", default="resnet50")
    ap.add_argument("--n-eval", type=int, default=1000)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-imgs", type=int, default=4)
    ap.add_argument("--configs", type=int, default=96, help="profiling only: first N configs")
    return ap.parse_args()


def workload(model: str, n_eval: int):
    from paper_2202_05048_b200 import build_model, make_dataset
    from paper_2202_05048_b200.fixtures import IMAGENET_SHAPE
    g = build_model(model, seed=0)
    d = make_dataset(n_calib=300, n_eval=n_eval, seed=0, shape=IMAGENET_SHAPE)
    return g, d


# ---------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.samples = []
        self.proc = None
        self.index = index

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            self.proc.wait(timeout=5)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 3 + i and s[3 + i].lower().startswith("active")})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


# ---------------------------------------------------------------- CPU baseline (oracle port)
def cpu_baseline(g, d, n_imgs: int) -> dict:
    """Time the numpy port of the reference on a bounded sample and extrapolate
    to the full workload (289 calibration images x 2 passes, 3 x T KL sweeps,
    96 x (quantize_model + 1000-image int8 forward))."""
    from oracle import ptq_oracle as O
    from paper_2202_05048_b200 import GENERIC, enumerate_space
    space = enumerate_space(GENERIC)
    n_union = len(set(np.concatenate([O.select_images(d.n_calib, sc, 0) for sc in ("S1", "S2", "S3")])))
    t0 = time.perf_counter()
    cache = O.calibrate(g, d.images[:n_imgs])               # two observer passes (calibration.py:57-106)
    t_cal_img = (time.perf_counter() - t0) / n_imgs
    hs = [h for h in cache.values() if h.lo != h.hi][:6]
    t0 = time.perf_counter()
    for h in hs:
        O.clip_range_kl(h)
    t_kl = (time.perf_counter() - t0) / max(1, len(hs))
    T = len(cache)
    full_cache = {t: h for t, h in cache.items()}
    for h in full_cache.values():                            # avoid the KL sweep inside quantize_model
        h.memo["KL"] = (h.lo, h.hi)
    cfg = space[2]                                           # S1 / Asymmetric / Max / Channel / Off
    t0 = time.perf_counter()
    qm = O.quantize_model(g, full_cache, cfg)
    t_q = time.perf_counter() - t0
    t0 = time.perf_counter()
    O.run_quantized(qm, d.eval_images[:n_imgs])
    t_eval_img = (time.perf_counter() - t0) / n_imgs
    n_eval = len(d.eval_images)
    total = n_union * t_cal_img + 3 * T * t_kl + len(space) * (t_q + n_eval * t_eval_img)
    return {"value": len(space) / total, "unit": UNIT, "cores": os.cpu_count(), "kind": "port",
            "sample": (f"oracle/ptq_oracle.py numpy port (OpenBLAS, {os.cpu_count()} threads): calibration "
                       f"of {n_imgs} images ({t_cal_img:.2f} s/img), KL sweep of {len(hs)} histograms "
                       f"({t_kl:.3f} s each), quantize_model of 1 config ({t_q:.2f} s), int8 forward "
                       f"of {n_imgs} eval images ({t_eval_img:.3f} s/img); extrapolated linearly to "
                       f"{n_union} calibration images, {3 * T} histograms, {len(space)} configs x "
                       f"{n_eval} images = {total:.0f} s per full grid"),
            "extrapolated_step_s": total}


def _reference_pkg():
    """The unmodified reference (ptqtune) from the offline install in baseline/_ref, or None."""
    ref = os.path.join(os.path.dirname(os.path.abspath(__file__)), "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "ptqtune")):
        return None
    if ref not in sys.path:
        sys.path.insert(0, ref)
    import ptqtune
    return ptqtune


def cpu_baseline_reference(g, d, n_imgs: int) -> dict | None:
    """The same bounded sample as cpu_baseline, run through the REFERENCE's own functions
    (ptqtune.calibration.calibrate, clipping.clip_range_kl, quantize.quantize_model,
    intexec.run_quantized) from baseline/_ref, extrapolated the same way."""
    R = _reference_pkg()
    if R is None:
        return None
    from ptqtune import calibration as RC
    from ptqtune import clipping as RK
    from ptqtune import intexec as RI
    from ptqtune import quantize as RQ
    from ptqtune import tuner as RT
    space = RT.enumerate_space(RT.TargetProfile("Generic"))
    n_union = len(set(np.concatenate([RC.select_images(d.calib_images, sc, 0) for sc in ("S1", "S2", "S3")])))
    t0 = time.perf_counter()
    cache = RC.calibrate(g, d.images[:n_imgs], model_name=g.name)
    t_cal_img = (time.perf_counter() - t0) / n_imgs
    hs = [h for h in cache.histograms.values() if h.min_seen != h.max_seen][:6]
    t0 = time.perf_counter()
    for h in hs:
        RK.clip_range_kl(h)
    t_kl = (time.perf_counter() - t0) / max(1, len(hs))
    T = len(cache.histograms)
    cfg = space[2]                                           # S1 / Asymmetric / Max / Channel / Off
    t0 = time.perf_counter()
    qg = RQ.quantize_model(g, cache, cfg)
    t_q = time.perf_counter() - t0
    t0 = time.perf_counter()
    RI.run_quantized(qg, d.eval_images[:n_imgs])
    t_eval_img = (time.perf_counter() - t0) / n_imgs
    n_eval = len(d.eval_images)
    total = n_union * t_cal_img + 3 * T * t_kl + len(space) * (t_q + n_eval * t_eval_img)
    return {"value": len(space) / total, "unit": UNIT, "cores": os.cpu_count(), "kind": "reference",
            "sample": (f"reference ptqtune (baseline/_ref, numpy/OpenBLAS, {os.cpu_count()} threads): "
                       f"calibrate() of {n_imgs} images ({t_cal_img:.2f} s/img), clip_range_kl of "
                       f"{len(hs)} histograms ({t_kl:.3f} s each), quantize_model of 1 config "
                       f"({t_q:.2f} s), run_quantized of {n_imgs} eval images ({t_eval_img:.3f} s/img); "
                       f"extrapolated linearly to {n_union} calibration images, {3 * T} histograms, "
                       f"{len(space)} configs x {n_eval} images = {total:.0f} s per full grid"),
            "extrapolated_step_s": total}


# ---------------------------------------------------------------- reference arm
def run_reference(args):
    import torch.distributed as dist
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    g, d = workload(args.model, args.n_eval)
    vals = []
    for _ in range(max(1, args.steps)):
        vals.append(cpu_baseline_reference(g, d, args.cpu_sample_imgs)
                    or cpu_baseline(g, d, args.cpu_sample_imgs))
    v = float(np.median([x["value"] for x in vals]))
    cb = dict(vals[-1])
    cb["value"] = v
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1000.0 * float(np.median([x["extrapolated_step_s"] for x in vals])),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "int8/fp64",
            "data": "synthetic (make_dataset seed 0, 224^2) + random-init ResNet-50 IR (seed 0)",
            "config": {"workload": f"{args.model} full 96-config grid, 1k eval imgs, 289 calib imgs",
                       "model": args.model, "n_eval": args.n_eval, "n_configs": 96},
            "cpu_baseline": cb,
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- B200 arm
def run_b200(args):
    import torch
    import torch.distributed as dist

    from paper_2202_05048_b200 import GENERIC, enumerate_space, make_accuracy_evaluator
    from paper_2202_05048_b200.evaluator import GpuEvaluator

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    g, d = workload(args.model, args.n_eval)
    space = enumerate_space(GENERIC)[: args.configs]
    ev = GpuEvaluator(g, d, 0, GENERIC, device=local, calibrate=False)
    stream = torch.cuda.ExternalStream(ev.stream_handle(), device=torch.device("cuda", local))

    def barrier():
        if world > 1:
            dist.barrier()

    phases = {}

    def step():
        t0 = time.perf_counter()
        ev.calibrate_all()                  # fp32 forward, min/max, histograms, KL, prepare
        t1 = time.perf_counter()
        out = ev.evaluate_grid(space)       # 96 configs (sharded over ranks)
        t2 = time.perf_counter()
        phases["calibrate_prepare_s"] = round(t1 - t0, 4)
        phases["eval_configs_s"] = round(t2 - t1, 4)
        return out

    for _ in range(args.warmup):
        step()
    ev.set_option("time_conv", 4)           # CUDA events around the conv launches of 4 configs/step
    times, counts = [], None
    launches = 0
    conv_ms = conv_ops = 0.0
    conv_n = conv_total = 0
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            barrier()
            torch.cuda.synchronize()
            ev.set_option("reset_stats", 1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            counts = step()
            e1.record(stream)
            torch.cuda.synchronize()
            barrier()
            st = ev.stats()
            launches, conv_ms, conv_ops, conv_n = st["launches"], st["conv_ms"], st["conv_ops"], st["conv_launches"]
            conv_total = st["conv_launches_total"]
            times.append(e0.elapsed_time(e1))
    ev.set_option("time_conv", 0)
    t_ms = float(np.median(times))
    if world > 1:
        tt = torch.tensor([t_ms], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_ms = float(tt.item())
    value = len(space) / (t_ms / 1000.0)

    # roofline of the dominant kernel (F4 tcgen05 int8 conv), per launch, measured live
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    bf16 = peaks.get("bf16_tflops")
    peak = 2.0 * bf16 if bf16 else 2.0 * 1590.0
    achieved = (conv_ops / (conv_ms / 1000.0)) / 1e12 if conv_ms > 0 else 0.0
    # DRAM traffic per k_conv_tc launch from the committed ncu capture of one config's 54
    # conv launches (profiles/r1/conv_dram_per_launch.csv), mean over launches
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "r1", "conv_dram_per_launch.csv")
    if os.path.exists(tpath):
        rows = [ln.split(",") for ln in open(tpath).read().strip().splitlines()[1:]]
        if rows:
            traffic = sum(int(r[2]) + int(r[3]) for r in rows) / len(rows)
    roofline = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TOP/s",
                "frac": achieved / peak if peak else None, "traffic": traffic,
                "traffic_unit": "bytes per launch (ncu dram__bytes_read+write, mean of one config's 54 launches)",
                "kernel": "k_conv_tc (tcgen05.mma.kind::i8)",
                "timed_launches": conv_n, "timed_ms": conv_ms,
                "avg_launch_ms": conv_ms / conv_n if conv_n else None,
                "launches_per_step": conv_total,
                "kernel_ms_per_step": conv_ms * conv_total / conv_n if conv_n else None,
                "share_of_step": (conv_ms * conv_total / conv_n) / t_ms if conv_n and t_ms else None,
                "peak_basis": ("int8 dense = 2 x measured bf16 burst (MEASURED_PEAKS.json bf16_tflops)"
                               if bf16 else "int8 dense = 2 x fallback bf16 1.59 PF")}

    # end-to-end through the public API, host buffers in / host results out
    e2e_times = []
    h2d = d.images.nbytes + d.eval_labels.nbytes + sum(w.nbytes for w in g.weights.values())
    T = len(g.nodes) + 1
    d2h = 3 * T * 2048 * 8 + 3 * T * 1921 * 8 + 3 * T * 2 * 4 + len(space) * 8
    ev.close()
    for _ in range(args.e2e_steps):
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ev2 = make_accuracy_evaluator(g, d, 0, GENERIC, device=local)
        acc = ev2.evaluate_many(space) if world == 1 else ev2.evaluate_grid(space)
        torch.cuda.synchronize()
        e2e_times.append(time.perf_counter() - t0)
        ev2.close()
    e2e_s = float(np.median(e2e_times))
    if world > 1:
        tt = torch.tensor([e2e_s], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_s = float(tt.item())

    if rank == 0:
        cb = None
        if world == 1 and not args.no_cpu_baseline:
            cb = cpu_baseline_reference(g, d, args.cpu_sample_imgs) or cpu_baseline(g, d, args.cpu_sample_imgs)
            cb.pop("extrapolated_step_s", None)
        best = int(np.argmax(counts))
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": t_ms, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "int8 (s32 acc, fp64 requant)",
                "data": "synthetic (make_dataset seed 0, 224^2) + random-init ResNet-50 IR (seed 0)",
                "config": {"workload": f"{args.model} full 96-config grid (calib S1/S2/S3 + KL + 96 x int8 eval), "
                                       f"{args.n_eval} eval imgs, 289 calib imgs",
                           "model": args.model, "n_eval": args.n_eval, "n_configs": len(space),
                           "l2": "inputs larger than L2 (783 MB images, 30 GB calibration activations)",
                           "parallelism": f"configs+calib images sharded over {world} GPU(s)"},
                "roofline": roofline, "cpu_baseline": cb,
                "e2e": {"value": len(space) / e2e_s, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                        "d2h_bytes_per_step": int(d2h)},
                "gpu_launches": int(launches), "clocks": clk.summary(), "phases_wall": phases,
                "best_config": space[best].to_dict(), "best_top1": int(counts[best]) / args.n_eval}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
