"""Conv time (CUDA events around every k_conv_tc launch) and eval wall time of each config of
the 96-config grid: which configurations dominate the bench step.
Usage: python tools/grid_conv_times.py [model] [n_eval] [key=value runtime options ...]"""
import sys
import time

sys.path.insert(0, ".")
from paper_2202_05048_b200 import GENERIC, build_model, enumerate_space, make_dataset  # noqa: E402
from paper_2202_05048_b200.evaluator import GpuEvaluator  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "resnet50"
n_eval = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
g = build_model(name, 0)
d = make_dataset(n_calib=300, n_eval=n_eval, seed=0, shape=(3, 224, 224))
ev = GpuEvaluator(g, d, 0, GENERIC)
for kv in sys.argv[3:]:
    k, v = kv.split("=")
    ev.set_option(k, int(v))
ev.set_option("time_conv", 1)
space = enumerate_space(GENERIC)
ev.correct_counts(space[:4])
tot_conv = tot_wall = 0.0
for i, cfg in enumerate(space):
    t0 = time.perf_counter()
    ev.correct_counts([cfg])
    wall = (time.perf_counter() - t0) * 1e3
    conv = float(ev.conv_timings().sum())
    tot_conv += conv
    tot_wall += wall
    c = cfg.to_dict()
    print(f"{i:2d} {c['cache']} {c['scheme'][:6]:6s} {c['clipping']:3s} {c['granularity'][:4]:4s} {c['mixed'][:5]:5s}"
          f"  conv {conv:7.3f} ms  wall {wall:7.3f} ms")
print(f"mean conv {tot_conv / len(space):.3f} ms  mean wall {tot_wall / len(space):.3f} ms per config")
