"""Multi-GPU sharding of the evaluator (one process per GPU, torch.distributed).

SURVEY.md 8(e): every configuration is independent and every calibration
statistic is an order-independent reduction, so

* calibration images of each cache are split across ranks; the per-cache
  (min, max) are combined with an allreduce MIN/MAX (exact), then every rank
  bins its own images with the global range and the int64 histograms are
  combined with an allreduce SUM (exact) -- bit-identical to one GPU;
* the KL sweep is sharded by histogram: each rank sweeps a contiguous share of the
  3 x T histograms and the chosen (lo, hi) windows are SUM-allreduced (each slot is
  written by exactly one rank, so the sum is exact);
* grid configurations are split into contiguous blocks of whole parameter variants
  (cache, scheme, clipping) in (cache, scheme, clipping, mixed, granularity) order,
  so every rank holds the same mix of Mixed=Off / FirstLastFp32 and per-tensor /
  per-channel configs (equal cost) and the variant's quantized graph input and
  folded prefix codes are reused inside the rank; the int64 correct-counts are
  reassembled with one SUM allreduce.

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
    """Round-robin shard (rank r takes items r, r+n, ...): calibration image ids."""
    return list(seq)[rank::n]


def _variant_key(cfg):
    from .config import config_key
    c = config_key(cfg)
    return (c[0], c[1], c[2]), (c[4], c[3])        # (cache, scheme, clipping), (mixed, granularity)


def config_cost(cfg) -> float:
    """Relative evaluation cost used to balance config shards: FirstLastFp32 skips the int8
    first and last layers; weight zero points (Asymmetric / SymmetricUint8 per-channel) add
    the row-sum correction."""
    from .config import config_key
    cache, scheme, clip, gran, mixed, _ = config_key(cfg)
    return (0.94 if mixed else 1.0) + (0.03 if scheme in (0, 2) and gran == 1 else 0.0)


def shard_plan(cfgs, n: int) -> list[list[int]]:
    """Config indices of every rank: contiguous blocks of whole (cache, scheme, clipping)
    variants in variant order, cut where the cumulative cost crosses k / n of the total."""
    cfgs = list(cfgs)
    order = sorted(range(len(cfgs)), key=lambda i: _variant_key(cfgs[i]))
    groups: list[list[int]] = []
    for i in order:
        if groups and _variant_key(cfgs[groups[-1][0]])[0] == _variant_key(cfgs[i])[0]:
            groups[-1].append(i)
        else:
            groups.append([i])
    total = sum(config_cost(cfgs[i]) for i in order) or 1.0
    plan: list[list[int]] = [[] for _ in range(n)]
    acc = 0.0
    for grp in groups:
        c = sum(config_cost(cfgs[i]) for i in grp)
        plan[min(n - 1, int((acc + c / 2) * n / total))].extend(grp)   # the rank owning the group's midpoint
        acc += c
    return plan


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


def gather_counts(local_counts: np.ndarray, idx, n_total: int) -> np.ndarray:
    """Reassemble config shards: this rank's results belong at positions ``idx``."""
    full = np.zeros(n_total, dtype=np.int64)
    full[np.asarray(idx, dtype=np.int64)] = local_counts
    return allreduce(full, "sum")


def kl_slice(n_hist: int, rank: int, n: int) -> tuple[int, int]:
    """Contiguous [lo, hi) share of the 3 x T histograms whose KL sweep this rank runs."""
    return n_hist * rank // n, n_hist * (rank + 1) // n
