"""Debug helper: compare every materialised int8 tensor of one config (GPU, fusion on)
with the oracle handed the GPU's caches.  Usage: python tools/debug_codes.py model cfg_idx"""
import sys

import numpy as np

sys.path.insert(0, ".")
from oracle import ptq_oracle as O  # noqa: E402
from paper_2202_05048_b200 import GENERIC, build_model, enumerate_space, make_dataset  # noqa: E402
from paper_2202_05048_b200.evaluator import GpuEvaluator  # noqa: E402

name, ci = sys.argv[1], int(sys.argv[2])
fusion = int(sys.argv[3]) if len(sys.argv) > 3 else 1
SHAPE = (3, 64, 64)
ds = make_dataset(n_calib=300, n_eval=12, seed=0, shape=SHAPE)
g = build_model(name, seed=0, shape=SHAPE)
ev = GpuEvaluator(g, ds, 0, GENERIC)
ev.set_option("fusion", fusion)
import os
ev.set_option("ablate", int(os.environ.get("ABLATE", "0")))
ev.set_option("tma", int(os.environ.get("TMA", "1")))
caches = {}
for k, sc in enumerate(("S1", "S2", "S3")):
    caches[sc] = {t: O.Hist(t, float(ev.cache_ranges[k, i, 0]), float(ev.cache_ranges[k, i, 1]),
                            ev.cache_counts[k, i], int(ev.cache_nsamp[k, i]))
                  for i, t in enumerate(ev.lowered.tensor_names)}
cfg = enumerate_space(GENERIC)[ci]
print(cfg)
qm = O.quantize_model(g, caches[cfg.cache], cfg)
seen = {}
O.run_quantized(qm, ds.eval_images, sink=lambda t, v: seen.__setitem__(t, v))
for t, v in seen.items():
    if t not in qm.act:
        continue
    try:
        got = ev.probe_codes(cfg, t).reshape(v.shape).astype(np.int64)
    except Exception as e:  # noqa: BLE001
        print(f"{t:12s} not probed ({str(e)[:60]})")
        continue
    d = got != v
    print(f"{t:12s} mismatches {int(d.sum()):8d} / {d.size}  maxdiff {int(np.abs(got - v).max())}")

if len(sys.argv) > 4:
    t = sys.argv[4]
    v = seen[t]
    got = ev.probe_codes(cfg, t).reshape(v.shape).astype(np.int64)
    d = got != v                                    # [N, C, H, W]
    print("bad per channel (first 64):", d.sum(axis=(0, 2, 3))[:64].tolist())
    print("bad per image:", d.sum(axis=(1, 2, 3)).tolist())
    print("bad per row h:", d.sum(axis=(0, 1, 3)).tolist())
    idx = np.argwhere(d)[:10]
    for n, c, h, w in idx:
        print(n, c, h, w, "got", got[n, c, h, w], "want", v[n, c, h, w])
    ev.set_option("fusion", 0)
    u = ev.probe_codes(cfg, t).reshape(v.shape).astype(np.int64)
    print("fusion0 vs fused mismatches", int((u != got).sum()), "fusion0 vs oracle", int((u != v).sum()))
    if len(sys.argv) > 6:
        ta, tb = sys.argv[5], sys.argv[6]
        A = ev.probe_codes(cfg, ta).reshape(v.shape).astype(np.int64)
        Bv = ev.probe_codes(cfg, tb).reshape(v.shape).astype(np.int64)
        for n, c, h, w in idx:
            print("a", A[n, c, h, w], "b", Bv[n, c, h, w], "got", got[n, c, h, w], "want", v[n, c, h, w])
        bad = d
        print("hist of got among bad:", np.unique(got[bad], return_counts=True))
        print("hist of want among bad:", np.unique(v[bad], return_counts=True)[0][:20])
