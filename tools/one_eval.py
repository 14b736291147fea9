"""Profiling helper: one warm eval of one config on ResNet-50 (1k images) bracketed by
cudaProfilerStart/Stop, for `ncu --profile-from-start off`.
Usage: python tools/one_eval.py [model] [config_index] [n_eval]"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2202_05048_b200 import GENERIC, build_model, enumerate_space, make_dataset  # noqa: E402
from paper_2202_05048_b200.evaluator import GpuEvaluator  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "resnet50"
ci = int(sys.argv[2]) if len(sys.argv) > 2 else 12
n_eval = int(sys.argv[3]) if len(sys.argv) > 3 else 1000
g = build_model(name, 0)
d = make_dataset(n_calib=300, n_eval=n_eval, seed=0, shape=(3, 224, 224))
ev = GpuEvaluator(g, d, 0, GENERIC)
cfg = enumerate_space(GENERIC)[ci]
for _ in range(2):
    ev.correct_counts([cfg])
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
ev.correct_counts([cfg])
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("done", cfg)
