"""Multi-GPU sharding of the evaluator (one process per GPU, torch.distributed).

SURVEY.md 8(e): every configuration is independent and every calibration
statistic is an order-independent reduction, so

* calibration images of each cache are split across ranks; the per-cache
  (min, max) are combined with an allreduce MIN/MAX (exact), then every rank
  bins its own images with the global range and the int64 histograms are
  combined with an allreduce SUM (exact) -- bit-identical to one GPU;
* the KL sweep is replicated (deterministic, milliseconds);
* grid configurations are dealt round-robin and the int64 correct-counts are
  all-gathered.

The protocol functions take a small "backend" object so the same code runs
with the CUDA library (GpuEvaluator) on NCCL and with the CPU oracle on gloo
in the tests (tests/test_dist_gloo.py).
"""

from __future__ import annotations

import numpy as np

from .config import CACHE_SIZES, N_BINS, select_images


def world():
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(), dist.get_world_size()
    return 0, 1


def shard(seq, rank: int, n: int):
    """Round-robin shard (rank r takes items r, r+n, ...)."""
    return list(seq)[rank::n]


def eval_slice(n_eval: int, rank: int, n: int) -> tuple[int, int]:
    """Contiguous [lo, hi) share of the eval split for image-sharded evaluation
    (the sequential xgb / GA searches, tuner.py:251-281, evaluate one
    config at a time, so their ranks split the eval images and SUM the correct
    counts)."""
    lo, hi = n_eval * rank // n, n_eval * (rank + 1) // n
    if hi <= lo:
        raise ValueError(f"rank {rank} of {n} has no eval images (n_eval={n_eval})")
    return lo, hi


def _tensor(a: np.ndarray):
    import torch
    import torch.distributed as dist
    t = torch.from_numpy(np.ascontiguousarray(a))
    if dist.get_backend() == "nccl":
        t = t.cuda()
    return t


def allreduce(a: np.ndarray, op: str) -> np.ndarray:
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return a
    t = _tensor(a)
    dist.all_reduce(t, op={"min": dist.ReduceOp.MIN, "max": dist.ReduceOp.MAX,
                           "sum": dist.ReduceOp.SUM}[op])
    return t.cpu().numpy()


def sharded_calibration(backend, n_calib: int, seed: int, T: int):
    """Run the two-phase calibration over this rank's share of every cache.

    backend.forward_minmax(sizes int32[3], ids int64[...]) -> ranges f32 [3][T][2]
    backend.histogram(ranges f32 [3][T][2]) -> counts int64 [3][T][2048]
    Returns (ranges, counts, n_samples-per-cache-image-count)."""
    rank, n = world()
    ids = [select_images(n_calib, sc, seed) for sc in CACHE_SIZES]
    mine = [np.asarray(shard(i, rank, n), dtype=np.int64) for i in ids]
    sizes = np.asarray([len(m) for m in mine], dtype=np.int32)
    flat = np.concatenate(mine) if sizes.sum() else np.zeros(0, np.int64)
    local = backend.forward_minmax(sizes, flat).reshape(3, T, 2)
    lo = allreduce(np.ascontiguousarray(local[..., 0]), "min")
    hi = allreduce(np.ascontiguousarray(local[..., 1]), "max")
    ranges = np.stack([lo, hi], axis=-1).astype(np.float32)
    counts = allreduce(backend.histogram(ranges).reshape(3, T, N_BINS), "sum")
    return ranges, counts, np.asarray([len(i) for i in ids], dtype=np.int64)


def gather_counts(local_counts: np.ndarray, n_total: int) -> np.ndarray:
    """Reassemble round-robin config shards: rank r's j-th result is config r + j*n."""
    rank, n = world()
    full = np.zeros(n_total, dtype=np.int64)
    full[rank::n] = local_counts
    return allreduce(full, "sum")
