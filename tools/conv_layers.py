"""Per-layer timing of the tcgen05 conv kernel on one config (CUDA events around each
launch).  Usage: python tools/conv_layers.py [model] [config_index] [n_eval] [ablate]
[key=value runtime options ...]"""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2202_05048_b200 import GENERIC, build_model, enumerate_space, make_dataset  # noqa: E402
from paper_2202_05048_b200.evaluator import GpuEvaluator  # noqa: E402
from paper_2202_05048_b200.ir import tensor_shapes  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "resnet50"
ci = int(sys.argv[2]) if len(sys.argv) > 2 else 0
n_eval = int(sys.argv[3]) if len(sys.argv) > 3 else 1000
g = build_model(name, 0)
d = make_dataset(n_calib=300, n_eval=n_eval, seed=0, shape=(3, 224, 224))
ev = GpuEvaluator(g, d, 0, GENERIC)
cfg = enumerate_space(GENERIC)[ci]
ev.set_option("time_conv", 1)
ablate = int(sys.argv[4]) if len(sys.argv) > 4 else 0
ev.set_option("ablate", ablate)
for kv in sys.argv[5:]:
    k, v = kv.split("=")
    ev.set_option(k, int(v))
for _ in range(3):
    ev.correct_counts([cfg])
t0 = time.perf_counter()
ev.correct_counts([cfg])
wall = time.perf_counter() - t0
ms = ev.conv_timings()
sh = tensor_shapes(g)
rows = []
fp32 = set()
comp = [n for n in g.nodes if n.kind in ("conv2d", "pointwise_conv2d", "fully_connected")]
if cfg.mixed != "Off":
    fp32 = {comp[0].id, comp[-1].id}
layers = [n for n in comp if n.id not in fp32]
tot_ops = 0.0
print(f"{name} cfg {ci} {cfg.to_dict()}  eval wall {wall*1e3:.1f} ms, conv sum {ms.sum():.1f} ms")
for n, t in zip(layers, ms):
    o = sh[n.output]
    w = g.weights[n.inputs[1]]
    K = int(np.prod(w.shape[1:]))
    M = n_eval * (o[1] * o[2] if len(o) == 3 else 1)
    N = o[0]
    ops = 2.0 * M * N * K
    tot_ops += ops
    print(f"{n.id:8s} {n.kind[:5]:5s} k={w.shape[-1] if w.ndim == 4 else 1} M={M:9d} N={N:5d} K={K:5d}"
          f"  {t:7.3f} ms  {ops / t / 1e9:7.1f} TOP/s  {M * N / t / 1e6:7.1f} Gout/s")
print(f"total {tot_ops / ms.sum() / 1e9:.1f} TOP/s over {len(ms)} launches")
