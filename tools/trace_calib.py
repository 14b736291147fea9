"""Phase timing of calibration + prepare on ResNet-50 (PTQ_TRACE=1 prints the runtime's
device-synchronised phase times).  Usage: PTQ_TRACE=1 python tools/trace_calib.py"""
import sys
import time

sys.path.insert(0, ".")
from paper_2202_05048_b200 import GENERIC, build_model, enumerate_space, make_dataset  # noqa: E402
from paper_2202_05048_b200.evaluator import GpuEvaluator  # noqa: E402

g = build_model("resnet50", 0)
d = make_dataset(n_calib=300, n_eval=1000, seed=0, shape=(3, 224, 224))
ev = GpuEvaluator(g, d, 0, GENERIC)
cfg = enumerate_space(GENERIC)[0]
import os  # noqa: E402

import torch  # noqa: E402

for it in range(3):
    prof = os.environ.get("PROFILE") and it == 2
    if prof:
        torch.cuda.synchronize()
        torch.cuda.cudart().cudaProfilerStart()
    t0 = time.perf_counter()
    ev.calibrate_all()
    if prof:
        torch.cuda.synchronize()
        torch.cuda.cudart().cudaProfilerStop()
    ev.correct_counts([cfg])
    print(f"iter {it}: calibrate_all + 1 config {time.perf_counter() - t0:.3f} s, "
          f"KL windows re-ranked on the host: {ev.kl_reranked}", file=sys.stderr)
    if it == 0:
        import numpy as np
        from paper_2202_05048_b200.evaluator import TIE_BAND
        kl = ev.kl_values.reshape(-1, ev.kl_values.shape[-1])
        best = kl.min(axis=1)
        band = (kl <= best[:, None] + np.abs(best)[:, None] * TIE_BAND).sum(axis=1)
        print("band sizes > 1:", sorted(band[band > 1].tolist())[-20:], "zero-best:", int((best == 0).sum()),
              file=sys.stderr)
