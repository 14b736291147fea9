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
MODEL_LABEL = {"resnet50": "ResNet-50", "resnet18": "ResNet-18", "mobilenet_v2": "MobileNet-v2",
               "squeezenet": "SqueezeNet"}


def metric_for(model: str) -> str:
    """BASELINE.json's metric for the headline ResNet-50; the same metric on C2 / C3 models."""
    return METRIC.replace("ResNet-50", MODEL_LABEL.get(model, model))
UNIT = "configs/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--model", default="resnet50", help="resnet50 (C4, headline), resnet18 (C2), mobilenet_v2 (C3)")
    ap.add_argument("--n-eval", type=int, default=1000)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-imgs", type=int, default=8, help="eval images per reference sample")
    ap.add_argument("--configs", type=int, default=96, help="profiling only: first N configs")
    return ap.parse_args()


def workload(model: str, n_eval: int):
    from paper_2202_05048_b200 import build_model, make_dataset
    from paper_2202_05048_b200.fixtures import IMAGENET_SHAPE
    g = build_model(model, seed=0)
    d = make_dataset(n_calib=300, n_eval=n_eval, seed=0, shape=IMAGENET_SHAPE)
    return g, d


def config_dict(args, world: int) -> dict:
    """The `config` object of the JSON line -- identical for the B200 arm and the reference arm."""
    return {"workload": f"{args.model} full 96-config grid (calib S1/S2/S3 + KL + 96 x int8 eval), "
                        f"{args.n_eval} eval imgs, 289 calib imgs",
            "model": args.model, "n_eval": args.n_eval, "n_configs": args.configs,
            "l2": "inputs larger than L2 (783 MB images, 30 GB calibration activations)",
            "parallelism": f"configs+calib images sharded over {world} GPU(s)"}


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


# ---------------------------------------------------------------- CPU baseline / reference arm
def _reference_pkg():
    """The unmodified reference (ptqtune) from the offline install in baseline/_ref, or None."""
    ref = os.path.join(os.path.dirname(os.path.abspath(__file__)), "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "ptqtune")):
        return None
    if ref not in sys.path:
        sys.path.insert(0, ref)
    import ptqtune
    return ptqtune


class ReferenceSampler:
    """Times the reference's own CPU implementation (ptqtune from baseline/_ref: calibrate,
    clip_range_kl, quantize_model, run_quantized) on bounded samples of the workload and
    extrapolates linearly to the full grid.  Samples are pooled over calls: call i times
    config i % 2 of {S1/Asym/Max/Channel, S2/Sym/KL/Tensor} (Mixed=Off) on the next `imgs`
    eval images, calibrates the next 2 calibration images and sweeps the next histogram, so
    K steps together cover 2 configs x K*imgs/2 eval images (2 configs x 64
    images).  Falls back to the oracle port (kind "port") when baseline/_ref is absent."""

    def __init__(self, g, d, imgs: int = 8):
        self.g, self.d, self.imgs = g, d, imgs
        self.R = _reference_pkg()
        self.kind = "reference" if self.R is not None else "port"
        self.t_cal, self.n_cal, self.t_kl, self.n_kl = 0.0, 0, 0.0, 0
        self.t_q, self.n_q, self.t_ev, self.n_ev = 0.0, 0, 0.0, 0
        self.calls = 0
        self.hists = None
        self.cache = None

    def step(self) -> float:
        """One bounded sample; returns the extrapolated full-grid time (s) so far."""
        g, d, i = self.g, self.d, self.calls
        if self.R is not None:
            from ptqtune import calibration as RC
            from ptqtune import clipping as RK
            from ptqtune import intexec as RI
            from ptqtune import quantize as RQ
            from ptqtune import tuner as RT
            space = RT.enumerate_space(RT.TargetProfile("Generic"))
            calib = lambda imgs: RC.calibrate(g, imgs, model_name=g.name)          # noqa: E731
            hist_of = lambda c: [h for h in c.histograms.values() if h.min_seen != h.max_seen]   # noqa: E731
            kl = RK.clip_range_kl
            qmodel = RQ.quantize_model
            run = RI.run_quantized
        else:
            from oracle import ptq_oracle as O
            from paper_2202_05048_b200 import GENERIC, enumerate_space
            space = enumerate_space(GENERIC)
            calib = lambda imgs: O.calibrate(g, imgs)                               # noqa: E731
            hist_of = lambda c: [h for h in c.values() if h.lo != h.hi]              # noqa: E731
            kl = O.clip_range_kl
            qmodel = O.quantize_model
            run = O.run_quantized
        j = (2 * i) % d.n_calib
        t0 = time.perf_counter()
        cache = calib(d.images[j:j + 2])                       # two observer passes per image
        self.t_cal += time.perf_counter() - t0
        self.n_cal += 2
        if self.cache is None:
            self.cache = cache
            self.hists = hist_of(cache)
            for h in (self.cache.histograms.values() if self.R is not None else self.cache.values()):
                if self.R is None:
                    h.memo["KL"] = (h.lo, h.hi)                 # KL is timed separately below
        h = self.hists[i % len(self.hists)]
        t0 = time.perf_counter()
        kl(h)
        self.t_kl += time.perf_counter() - t0
        self.n_kl += 1
        cfg = space[(2, 12)[i % 2]]
        if self.R is not None and cfg.clipping == "KL":
            cfg = space[(2, 10)[i % 2]]                        # S1 / Symmetric / Max / Tensor
        t0 = time.perf_counter()
        qm = qmodel(g, self.cache, cfg)
        self.t_q += time.perf_counter() - t0
        self.n_q += 1
        e0 = (i * self.imgs) % len(d.eval_images)
        t0 = time.perf_counter()
        run(qm, d.eval_images[e0:e0 + self.imgs])
        self.t_ev += time.perf_counter() - t0
        self.n_ev += self.imgs
        self.calls += 1
        return self.extrapolated()

    def n_union(self) -> int:
        from paper_2202_05048_b200.config import select_images
        return len(set(np.concatenate([select_images(self.d.n_calib, sc, 0) for sc in ("S1", "S2", "S3")])))

    def extrapolated(self) -> float:
        T = len(self.g.nodes) + 1
        n_eval = len(self.d.eval_images)
        return (self.n_union() * self.t_cal / self.n_cal + 3 * T * self.t_kl / self.n_kl +
                96 * (self.t_q / self.n_q + n_eval * self.t_ev / self.n_ev))

    def summary(self) -> dict:
        total = self.extrapolated()
        who = ("reference ptqtune (baseline/_ref, numpy/OpenBLAS" if self.kind == "reference"
               else "oracle/ptq_oracle.py numpy port (OpenBLAS")
        return {"value": 96 / total, "unit": UNIT, "cores": os.cpu_count(), "kind": self.kind,
                "sample": (f"{who}, {os.cpu_count()} threads), pooled over {self.calls} samples: calibrate() of "
                           f"{self.n_cal} images ({self.t_cal / self.n_cal:.2f} s/img), clip_range_kl of {self.n_kl} "
                           f"histograms ({self.t_kl / self.n_kl:.3f} s each), quantize_model of {self.n_q} configs "
                           f"({self.t_q / self.n_q:.2f} s), run_quantized of {self.n_ev} eval images over 2 configs "
                           f"({self.t_ev / self.n_ev:.3f} s/img); extrapolated linearly to {self.n_union()} "
                           f"calibration images, {3 * (len(self.g.nodes) + 1)} histograms, 96 configs x "
                           f"{len(self.d.eval_images)} images = {total:.0f} s per full grid"),
                "extrapolated_step_s": total}


# ---------------------------------------------------------------- reference arm
def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    g, d = workload(args.model, args.n_eval)
    sampler = ReferenceSampler(g, d, args.cpu_sample_imgs)
    steps = []
    for _ in range(max(1, args.steps)):
        steps.append(sampler.step())
    cb = sampler.summary()
    v = cb["value"]
    line = {"impl": "reference", "metric": metric_for(args.model), "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * cb["extrapolated_step_s"],
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "int8/fp64",
            "data": f"synthetic (make_dataset seed 0, 224^2) + random-init {MODEL_LABEL.get(args.model, args.model)} IR (seed 0)",
            "config": config_dict(args, args.gpus),
            "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
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

    # roofline of the dominant kernel (F4 tcgen05 int8 conv), per launch, measured live;
    # denominator: the int8 tensor-pipe rate measured on this pool (tools/int8_peak.cu,
    # profiles/r2/int8_peak.json), else 2 x the measured bf16 burst
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    i8 = os.path.join(ROOT, "profiles", "r2", "int8_peak.json")
    if os.path.exists(i8):
        peak = float(json.load(open(i8))["peak_int8_tops"])
        basis = ("measured int8 tensor-pipe rate (tools/int8_peak.cu mma_only, max of burst/sustained, "
                 "profiles/r2/int8_peak.json)")
    else:
        bf16 = peaks.get("bf16_tflops") or 1590.0
        peak, basis = 2.0 * bf16, "int8 dense = 2 x bf16 burst (MEASURED_PEAKS.json or fallback)"
    achieved = (conv_ops / (conv_ms / 1000.0)) / 1e12 if conv_ms > 0 else 0.0
    # DRAM traffic per k_conv_tc launch from the committed ncu capture of one config's 54
    # conv launches, mean over launches
    traffic = None
    for tpath in (os.path.join(ROOT, "profiles", "r2", "conv_dram_per_launch.csv"),
                  os.path.join(ROOT, "profiles", "r1", "conv_dram_per_launch.csv")):
        if os.path.exists(tpath):
            rows = [ln.split(",") for ln in open(tpath).read().strip().splitlines()[1:]]
            if rows:
                traffic = sum(int(r[2]) + int(r[3]) for r in rows) / len(rows)
                break
    roofline = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TOP/s",
                "frac": achieved / peak if peak else None, "traffic": traffic,
                "traffic_unit": "bytes per launch (ncu dram__bytes_read+write, mean of one config's 54 launches)",
                "kernel": "k_conv_tc (tcgen05.mma.kind::i8)",
                "timed_launches": conv_n, "timed_ms": conv_ms,
                "avg_launch_ms": conv_ms / conv_n if conv_n else None,
                "launches_per_step": conv_total,
                "kernel_ms_per_step": conv_ms * conv_total / conv_n if conv_n else None,
                "share_of_step": (conv_ms * conv_total / conv_n) / t_ms if conv_n and t_ms else None,
                "peak_basis": basis}
    # whole-path roofline: the int8 forward of one config is HBM-bound as a
    # whole; minimal traffic = every layer reads its int8 input / writes its output once
    from paper_2202_05048_b200.fixtures import int8_traffic_per_image
    hbm = float(peaks.get("hbm_gbs") or 6650.0)
    bytes_cfg = float(int8_traffic_per_image(g)) * args.n_eval
    roofline_path = {"bound": "hbm", "bytes_per_config": bytes_cfg,
                     "achieved": bytes_cfg * value / 1e9, "peak": hbm, "unit": "GB/s",
                     "frac": bytes_cfg * value / 1e9 / hbm,
                     "configs_per_s_at_roof": hbm * 1e9 / bytes_cfg,
                     "note": "algorithmic int8 activation bytes of one config x configs/s (whole step, "
                             "calibration included) vs measured HBM copy bandwidth"}

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
            sampler = ReferenceSampler(g, d, args.cpu_sample_imgs)
            for _ in range(2):
                sampler.step()
            cb = sampler.summary()
            cb.pop("extrapolated_step_s", None)
        best = int(np.argmax(counts))
        line = {"metric": metric_for(args.model), "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": t_ms, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "int8 (s32 acc, exact int64 fixed-point requant of the fp64 reference)",
                "data": f"synthetic (make_dataset seed 0, 224^2) + random-init {MODEL_LABEL.get(args.model, args.model)} IR (seed 0)",
                "config": config_dict(args, world),
                "roofline": roofline, "roofline_path": roofline_path, "cpu_baseline": cb,
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
