"""Driver for the per-family ncu captures (F1 min/max + histogram, F2 KL sweep, F3 quantize /
weight variants / subsample): full-size ResNet-50 calibration (289 images, three caches)
plus two config evaluations, then exit.  Run under ncu with a -k regex per family, e.g.

    ncu --set full --clock-control none -k regex:k_histogram -s 20 -c 3 \\
        -o gpurun_out/f1 python tools/ncu_families.py
"""
import sys

sys.path.insert(0, ".")
from paper_2202_05048_b200 import GENERIC, build_model, enumerate_space, make_dataset  # noqa: E402
from paper_2202_05048_b200.evaluator import GpuEvaluator  # noqa: E402

g = build_model("resnet50", 0)
d = make_dataset(n_calib=300, n_eval=1000, seed=0, shape=(3, 224, 224))
ev = GpuEvaluator(g, d, 0, GENERIC)
space = enumerate_space(GENERIC)
print(ev.correct_counts([space[0], space[2]]))
ev.close()
