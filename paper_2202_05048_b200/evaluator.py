"""GPU drop-in for the reference's measured evaluator.

``make_accuracy_evaluator(g, d, seed, profile=None)`` has the signature and
contract of ``ptqtune.tuner.make_accuracy_evaluator``
(/root/reference/pkg/src/ptqtune/tuner.py:434-444): building it calibrates
the three cache size classes once; the returned callable maps a QuantConfig
to its top-1 accuracy on the eval split (a Python float, correct / n_eval).
Errors surface as exceptions, which the reference's ``_Campaign._safe_eval``
(tuner.py:173-177) records as failed trials.

Everything numeric runs in libptq_b200.so on the GPU; the host only draws the
calibration image ids (numpy RNG parity with calibration.py:44-54), picks the
KL window from the device-computed divergences and, for the handful of
windows whose device KL is within 1e-9 of the best (mathematically tied
windows whose order is decided by the last ulp of numpy's log), re-ranks
them with numpy's own arithmetic so the chosen threshold is the reference's
(SURVEY.md App. A.K).
"""

from __future__ import annotations

import ctypes as C
import math
import os
import sys
import threading
import time

import numpy as np

from . import _lib
from .config import (CACHE_SIZES, N_BINS, QuantConfig, TargetProfile, config_key,
                     select_images)
from .lowering import LoweredGraph

TIE_BAND = 1e-9


class _trace:
    """PTQ_TRACE=1: wall time of host-side evaluator phases on stderr."""

    def __init__(self, name):
        self.name = name

    def __enter__(self):
        self.t0 = time.perf_counter()

    def __exit__(self, *a):
        if os.environ.get("PTQ_TRACE"):
            print(f"[ptq-trace] py:{self.name:25s} {1e3 * (time.perf_counter() - self.t0):9.3f} ms",
                  file=sys.stderr, flush=True)


# ---------------------------------------------------------------- KL window choice (host side)

def kl_window_bounds(lo: float, hi: float, i: int) -> tuple[int, int]:
    """Window [start, end) of width i (ref clipping.py:72-76)."""
    if lo < 0.0:
        zero_bin = int((0.0 - lo) / ((hi - lo) / N_BINS))
        start = min(max(zero_bin - i // 2, 0), N_BINS - i)
    else:
        start = 0
    return start, start + i


_AR128 = np.arange(128)
_AR2048 = np.arange(N_BINS)


def _numpy_window_kl(counts: np.ndarray, lo: float, hi: float, i: int, _pre=None) -> float:
    """numpy evaluation of one window's KL in the reference's op order
    (clipping.py:38-52, :77-81) -- used only to break near-ties.  `_pre` carries the
    per-histogram (float64 counts, total, cumsum) when several windows are ranked."""
    c, total, cum = _pre if _pre is not None else _kl_pre(counts)
    start, end = kl_window_bounds(lo, hi, i)
    win = c[start:end]
    ref = win.copy()
    if start > 0:
        ref[0] += cum[start - 1]
    ref[-1] += total - cum[end - 1]
    m = i // 128
    starts = _AR128 * m
    sums = np.add.reduceat(win, starts)
    nz = ref > 0
    nzg = np.add.reduceat(nz.astype(np.float64), starts)
    gidx = np.minimum(_AR2048[:i] // m, 127)
    q = np.zeros(i)
    q[nz] = sums[gidx[nz]] / nzg[gidx[nz]]
    if np.any(nz & (q == 0.0)):
        return math.inf
    p = ref[nz]
    return float(np.sum(p * (np.log(p) - np.log(q[nz]))) / ref.sum())


def _kl_pre(counts: np.ndarray):
    c = counts.astype(np.float64)
    return c, c.sum(), np.cumsum(c)


def choose_kl_range(counts: np.ndarray, lo: float, hi: float, kl: np.ndarray) -> tuple[tuple[float, float], int]:
    """(lo, hi) clip range from the device KLs; returns (range, n_reranked)."""
    lo, hi = float(lo), float(hi)
    if lo == hi or int(counts.sum()) <= 0:
        return (lo, hi), 0
    best = int(kl.argmin())                 # first minimum == strict '<' sweep (clipping.py:82)
    reranked = 0
    kb = float(kl[best])
    if math.isfinite(kb):
        band = np.flatnonzero(kl <= kb + abs(kb) * TIE_BAND)
        if band.size > 1:
            reranked = int(band.size)
            best_kl = math.inf
            pre = _kl_pre(counts)
            for w in band:
                v = _numpy_window_kl(counts, lo, hi, int(w) + 128, pre)
                if v < best_kl:
                    best_kl, best = v, int(w)
        start, end = kl_window_bounds(lo, hi, best + 128)
    else:
        start, end = 0, N_BINS
    return (_linspace_edge(lo, hi, start), _linspace_edge(lo, hi, end)), reranked


def _linspace_edge(lo: float, hi: float, k: int) -> float:
    """np.linspace(lo, hi, N_BINS + 1)[k] without building the array (numpy
    function_base.linspace: fl(k * fl(delta / div)) + lo, last = hi, and the
    step == 0 branch (k / div) * delta + lo)."""
    if k >= N_BINS:
        return hi
    delta = hi - lo
    step = delta / N_BINS
    if step == 0:
        return (k / N_BINS) * delta + lo
    return k * step + lo


# ---------------------------------------------------------------- call coalescing
class Coalescer:
    """Batches concurrent single-item calls: the first caller becomes the leader and runs
    ``batch_fn`` on everything queued (repeating while new requests arrive); the others
    wait for their slot.  Results and exceptions go back to the caller that asked: when a
    batch raises, its items are re-run one at a time, so only the offending caller sees the
    error (the reference's _safe_eval fails one trial, not its neighbours, tuner.py:173-177)."""

    def __init__(self, batch_fn):
        self._fn = batch_fn
        self._cv = threading.Condition()
        self._queue: list = []
        self._busy = False
        self.batches: list[int] = []          # sizes of the batches run (for tests / stats)

    def __call__(self, item):
        slot = {"done": False}
        with self._cv:
            self._queue.append((item, slot))
            if self._busy:
                while not slot["done"]:
                    self._cv.wait()
                return self._result(slot)
            self._busy = True
        try:
            while True:
                with self._cv:
                    batch, self._queue = self._queue, []
                    if not batch:
                        self._busy = False
                        self._cv.notify_all()
                        break
                try:
                    res = [(r, None) for r in self._fn([b[0] for b in batch])]
                except Exception as e:  # noqa: BLE001 - isolate the failing item(s)
                    if len(batch) == 1:
                        res = [(None, e)]
                    else:
                        res = []
                        for item, _ in batch:
                            try:
                                res.append((self._fn([item])[0], None))
                            except Exception as e1:  # noqa: BLE001 - this caller's error
                                res.append((None, e1))
                with self._cv:
                    self.batches.append(len(batch))
                    for (_, sl), (r, err) in zip(batch, res):
                        sl.update(done=True, value=r, error=err)
                    self._cv.notify_all()
        finally:
            with self._cv:
                if self._busy and not self._queue:
                    self._busy = False
                self._cv.notify_all()
        return self._result(slot)

    @staticmethod
    def _result(slot):
        if slot.get("error") is not None:
            raise slot["error"]
        return slot["value"]


# ---------------------------------------------------------------- evaluator

class GpuEvaluator:
    """Callable ``QuantConfig -> top-1`` backed by one B200 context."""

    def __init__(self, g, d, seed: int, profile: TargetProfile | None = None, *, device: int = 0,
                 eval_chunk: int | None = None, calibrate: bool = True, image_sharded: bool = False):
        self.lib = _lib.load()
        self.graph, self.profile, self.seed = g, profile, seed
        self.lowered = LoweredGraph(g)
        self.T = self.lowered.n_tensors
        self.n_calib = int(d.n_calib)
        self.n_eval = int(len(d.images) - d.n_calib)
        if self.n_eval <= 0:
            raise ValueError("empty evaluation set")
        self._lock = threading.RLock()
        self._coalescer = None
        imgs = np.ascontiguousarray(np.asarray(d.images, dtype=np.float32))
        labels = np.ascontiguousarray(np.asarray(d.labels[d.n_calib:], dtype=np.int64))
        # image-sharded mode (sequential xgb / GA search): every rank keeps all
        # calibration images and a contiguous slice of the eval split; correct counts are
        # SUM-allreduced per config, so each config costs 1/world of the images per GPU
        self.image_sharded = False
        if image_sharded:
            from . import dist
            rank, world = dist.world()
            if world > 1:
                lo, hi = dist.eval_slice(self.n_eval, rank, world)
                imgs = np.ascontiguousarray(np.concatenate([imgs[: self.n_calib],
                                                            imgs[self.n_calib + lo: self.n_calib + hi]]))
                labels = np.ascontiguousarray(labels[lo:hi])
                self.image_sharded = True
        self.n_eval_local = int(len(labels))
        if tuple(imgs.shape[1:]) != tuple(int(v) for v in g.input_shape):
            raise ValueError(f"dataset shape {imgs.shape[1:]} does not match graph input {g.input_shape}")
        self._ctx = C.c_void_p()
        _lib.check(self.lib.ptq_create(C.byref(self._ctx), device, C.byref(self.lowered.desc),
                                       _lib.ptr(imgs), _lib.ptr(labels), len(imgs), self.n_calib))
        # ptq_create returns once the calibration images are resident; the evaluation images keep
        # uploading from this buffer while calibration runs, so it must outlive the context
        self._host_imgs = imgs
        if eval_chunk:
            self.set_option("eval_chunk", int(eval_chunk))
        self.kl_reranked = 0
        if calibrate:
            self.calibrate_all()

    # ------------------------------------------------------------ calibration (tuner.py:438)
    def calibrate_all(self) -> None:
        """Build the S1/S2/S3 caches; under torch.distributed the images of each
        cache are sharded across ranks (dist.sharded_calibration)."""
        from . import dist
        with _trace("sharded_calibration"):
            ranges, counts, n_img = dist.sharded_calibration(self, self.n_calib, self.seed, self.T)
        elems = self.tensor_elems()
        nsamp = n_img[:, None] * elems[None, :]
        self.image_ids = [select_images(self.n_calib, sc, self.seed) for sc in CACHE_SIZES]
        self.install_caches(ranges, counts, nsamp)

    # backend protocol of dist.sharded_calibration
    def forward_minmax(self, sizes: np.ndarray, ids: np.ndarray) -> np.ndarray:
        sizes = np.ascontiguousarray(sizes, dtype=np.int32)
        ids = np.ascontiguousarray(ids, dtype=np.int64)
        out = np.zeros((len(sizes), self.T, 2), dtype=np.float32)
        _lib.check(self.lib.ptq_calib_forward(self._ctx, len(sizes), _lib.ptr(sizes),
                                              _lib.ptr(ids) if ids.size else None, _lib.ptr(out)))
        return out

    def histogram(self, ranges: np.ndarray, lo=None, hi=None) -> np.ndarray:
        if lo is not None:                       # single host array (parity probe)
            return self.histogram_array(ranges, lo, hi)
        ranges = np.ascontiguousarray(ranges, dtype=np.float32)
        out = np.zeros((ranges.shape[0], self.T, N_BINS), dtype=np.int64)
        _lib.check(self.lib.ptq_calib_histogram(self._ctx, _lib.ptr(ranges), _lib.ptr(out)))
        return out

    def tensor_elems(self) -> np.ndarray:
        from .ir import tensor_shapes
        shapes = tensor_shapes(self.graph)
        return np.asarray([int(np.prod(shapes[t])) for t in self.lowered.tensor_names], dtype=np.int64)

    def install_caches(self, ranges: np.ndarray, counts: np.ndarray, nsamp: np.ndarray | None = None,
                       kl_ranges: np.ndarray | None = None) -> None:
        """Set the three caches (device KL sweep unless kl_ranges is given)."""
        T = self.T
        ranges = np.ascontiguousarray(ranges, dtype=np.float32).reshape(3, T, 2)
        counts = np.ascontiguousarray(counts, dtype=np.int64).reshape(3, T, N_BINS)
        self.cache_ranges, self.cache_counts = ranges, counts
        self.cache_nsamp = nsamp
        if kl_ranges is None:
            # under torch.distributed each rank sweeps a contiguous share of the 3 x T
            # histograms; every (lo, hi) slot is written by one rank, so a SUM allreduce
            # assembles the exact table (dist.py)
            from . import dist
            rank, world = dist.world()
            lo, hi = dist.kl_slice(3 * T, rank, world)
            flat_c = counts.reshape(3 * T, N_BINS)
            flat_r = ranges.reshape(3 * T, 2)
            kl = np.full((3 * T, _lib.PTQ_NWINDOWS), np.inf, dtype=np.float64)
            if hi > lo:
                part = np.zeros((hi - lo, _lib.PTQ_NWINDOWS), dtype=np.float64)
                _lib.check(self.lib.ptq_kl_sweep(self._ctx, hi - lo, _lib.ptr(np.ascontiguousarray(flat_c[lo:hi])),
                                                 _lib.ptr(np.ascontiguousarray(flat_r[lo:hi])), _lib.ptr(part)))
                kl[lo:hi] = part
            self.kl_values = kl.reshape(3, T, -1)
            chosen = np.zeros((3 * T, 2), dtype=np.float64)
            self.kl_reranked = 0
            with _trace("choose_kl_ranges"):
                # vectorised first pass: histograms whose best window is unique within the tie
                # band (and finite) need no numpy re-rank; only the rest go through
                # choose_kl_range one by one
                if hi > lo:
                    sub = kl[lo:hi]
                    best = sub.argmin(axis=1)
                    kb = sub[np.arange(hi - lo), best]
                    band = (sub <= (kb + np.abs(kb) * TIE_BAND)[:, None]).sum(axis=1)
                    lo_r, hi_r = flat_r[lo:hi, 0].astype(np.float64), flat_r[lo:hi, 1].astype(np.float64)
                    simple = np.isfinite(kb) & (band == 1) & (lo_r < hi_r) & (flat_c[lo:hi].sum(axis=1) > 0)
                    for k in range(hi - lo):
                        h = lo + k
                        if simple[k]:
                            start, end = kl_window_bounds(float(lo_r[k]), float(hi_r[k]), int(best[k]) + 128)
                            chosen[h] = (_linspace_edge(float(lo_r[k]), float(hi_r[k]), start),
                                         _linspace_edge(float(lo_r[k]), float(hi_r[k]), end))
                        else:
                            (a, b), nr = choose_kl_range(flat_c[h], flat_r[h, 0], flat_r[h, 1], kl[h])
                            chosen[h] = (a, b)
                            self.kl_reranked += nr
            kl_ranges = dist.allreduce(chosen, "sum") if world > 1 else chosen
        self.kl_ranges = np.ascontiguousarray(kl_ranges, dtype=np.float64).reshape(3, T, 2)
        for k in range(3):
            mx = np.ascontiguousarray(ranges[k].astype(np.float64))
            _lib.check(self.lib.ptq_set_clip_ranges(self._ctx, k, 0, _lib.ptr(mx)))
            kr = np.ascontiguousarray(self.kl_ranges[k])
            _lib.check(self.lib.ptq_set_clip_ranges(self._ctx, k, 1, _lib.ptr(kr)))
        with _trace("prepare"):
            _lib.check(self.lib.ptq_prepare(self._ctx))

    # ------------------------------------------------------------ extension: percentile clipping
    def percentile_ranges(self, pct: float) -> np.ndarray:
        """EXTENSION, not in the reference (clipped_range rejects "Percentile",
        clipping.py:91-92; parity unpinned, checked against oracle.percentile_range): the
        device percentile clipping of every cache/tensor histogram, [3, T, 2] fp64."""
        out = np.zeros((3 * self.T, 2), dtype=np.float64)
        _lib.check(self.lib.ptq_percentile_ranges(self._ctx, 3 * self.T, _lib.ptr(self.cache_counts),
                                                  _lib.ptr(self.cache_ranges), float(pct), _lib.ptr(out)))
        return out.reshape(3, self.T, 2)

    def correct_counts_percentile(self, cfgs, pct: float) -> np.ndarray:
        """EXTENSION: evaluate configs with percentile-clipped activation ranges in place of
        the clipping each config names (the KL slot is borrowed and restored afterwards)."""
        import dataclasses
        pr = self.percentile_ranges(pct)
        cfgs = [dataclasses.replace(c, clipping="KL") for c in cfgs]
        with self._lock:          # no other thread may evaluate KL configs while the slot is borrowed
            try:
                for k in range(3):
                    _lib.check(self.lib.ptq_set_clip_ranges(self._ctx, k, 1, _lib.ptr(np.ascontiguousarray(pr[k]))))
                return self.correct_counts(cfgs)
            finally:
                for k in range(3):
                    _lib.check(self.lib.ptq_set_clip_ranges(self._ctx, k, 1,
                                                            _lib.ptr(np.ascontiguousarray(self.kl_ranges[k]))))

    # ------------------------------------------------------------ evaluation
    def _check_cfg(self, cfg) -> None:
        if not isinstance(cfg, QuantConfig):
            cfg = QuantConfig.from_dict(cfg.to_dict())
        if self.profile is not None and not self.profile.contains(cfg):
            raise ValueError(f"config {cfg} not allowed by profile {self.profile.name}")

    def correct_counts(self, cfgs) -> np.ndarray:
        cfgs = list(cfgs)
        for cfg in cfgs:
            self._check_cfg(cfg)
        arr = (_lib.ConfigDesc * max(1, len(cfgs)))()
        for i, cfg in enumerate(cfgs):
            arr[i] = _lib.ConfigDesc(*config_key(cfg))
        out = np.zeros(max(1, len(cfgs)), dtype=np.int64)
        with self._lock:
            _lib.check(self.lib.ptq_eval_configs(self._ctx, arr, len(cfgs), _lib.ptr(out)))
        return out[: len(cfgs)]

    def evaluate_many(self, cfgs) -> list[float]:
        counts = self.correct_counts(cfgs)
        if self.image_sharded:
            from . import dist
            counts = dist.allreduce(counts, "sum")
        return [int(c) / float(self.n_eval) for c in counts]

    def __call__(self, cfg) -> float:
        # an invalid config fails its own caller only, before it can join a batch
        self._check_cfg(cfg)
        if self.image_sharded:
            # every rank must all-reduce the same configs in the same order: no coalescing
            # (batches would form differently on each rank)
            with self._lock:
                return self.evaluate_many([cfg])[0]
        # concurrent callers (measure_many's thread pool, tuner.py:192-203) are coalesced
        # into one evaluate_many batch
        if self._coalescer is None:
            self._coalescer = Coalescer(self.evaluate_many)
        return self._coalescer(cfg)

    # ------------------------------------------------------------ probes / options
    def set_option(self, key: str, value: int) -> None:
        _lib.check(self.lib.ptq_set_option(self._ctx, key.encode(), int(value)))

    def probe_codes(self, cfg, tensor: str) -> np.ndarray:
        tid = self.lowered.tensor_ids[tensor]
        cd = _lib.ConfigDesc(*config_key(cfg))
        n = C.c_int64()
        _lib.check(self.lib.ptq_probe_codes(self._ctx, C.byref(cd), tid, None, C.byref(n)))
        out = np.zeros(n.value, dtype=np.int8)
        with self._lock:
            _lib.check(self.lib.ptq_probe_codes(self._ctx, C.byref(cd), tid, _lib.ptr(out), C.byref(n)))
        return out

    # ------------------------------------------------------------ parity probes (image subsets)
    def _imgs(self, imgs) -> np.ndarray:
        return np.ascontiguousarray(np.asarray(imgs, dtype=np.int64).ravel())

    def probe_tensors(self, cfg, tensors, imgs) -> dict:
        """int8 codes {tensor: [n_imgs, C, H, W]} of every requested tensor the evaluation of
        ``cfg`` materialises, for eval images ``imgs`` (one device evaluation)."""
        from .ir import tensor_shapes
        shapes = tensor_shapes(self.graph)
        imgs = self._imgs(imgs)
        tids = np.asarray([self.lowered.tensor_ids[t] for t in tensors], dtype=np.int32)
        sizes = [len(imgs) * int(np.prod(shapes[t])) for t in tensors]
        out = np.zeros(max(1, sum(sizes)), dtype=np.int8)
        found = np.zeros(len(tids), dtype=np.int32)
        cd = _lib.ConfigDesc(*config_key(cfg))
        with self._lock:
            _lib.check(self.lib.ptq_probe_tensors(self._ctx, C.byref(cd), len(tids), _lib.ptr(tids), len(imgs),
                                                  _lib.ptr(imgs), _lib.ptr(out), _lib.ptr(found)))
        res, off = {}, 0
        for t, n, f in zip(tensors, sizes, found):
            if f:
                res[t] = out[off:off + n].reshape((len(imgs),) + tuple(shapes[t]))
            off += n
        return res

    def probe_acc(self, cfg, node_id: str, imgs) -> np.ndarray:
        """Clipped int32 accumulators of one int8 compute node, [n_imgs, Cout, OH, OW]."""
        from .ir import tensor_shapes
        node = next(i for i, n in enumerate(self.graph.nodes) if n.id == node_id)
        shape = tuple(tensor_shapes(self.graph)[self.graph.nodes[node].output])
        imgs = self._imgs(imgs)
        out = np.zeros((len(imgs),) + shape, dtype=np.int32)
        cd = _lib.ConfigDesc(*config_key(cfg))
        with self._lock:
            _lib.check(self.lib.ptq_probe_acc(self._ctx, C.byref(cd), node, len(imgs), _lib.ptr(imgs),
                                              _lib.ptr(out)))
        return out

    def probe_output(self, cfg, imgs) -> np.ndarray:
        """run_quantized's return value for eval images ``imgs`` (intexec.py:337-351)."""
        imgs = self._imgs(imgs)
        out = np.zeros((len(imgs), int(self.graph.output_classes)), dtype=np.float32)
        cd = _lib.ConfigDesc(*config_key(cfg))
        with self._lock:
            _lib.check(self.lib.ptq_probe_output(self._ctx, C.byref(cd), len(imgs), _lib.ptr(imgs), _lib.ptr(out)))
        return out

    def probe_f32(self, cfg, tensor: str, imgs) -> np.ndarray:
        """An fp32-domain tensor of ``cfg`` (FirstLastFp32 layers), [n_imgs, C, H, W]."""
        from .ir import tensor_shapes
        shape = tuple(tensor_shapes(self.graph)[tensor])
        imgs = self._imgs(imgs)
        out = np.zeros((len(imgs),) + shape, dtype=np.float32)
        cd = _lib.ConfigDesc(*config_key(cfg))
        with self._lock:
            _lib.check(self.lib.ptq_probe_f32(self._ctx, C.byref(cd), self.lowered.tensor_ids[tensor], len(imgs),
                                              _lib.ptr(imgs), _lib.ptr(out)))
        return out

    def minmax_array(self, x: np.ndarray) -> tuple[float, float]:
        """Device min/max of a host array [n_img, ...] through the calibration kernels."""
        x = np.ascontiguousarray(np.asarray(x, dtype=np.float32))
        x = x.reshape(x.shape[0], -1)
        r = np.zeros(2, dtype=np.float32)
        _lib.check(self.lib.ptq_minmax_host(self._ctx, _lib.ptr(x), x.shape[0], x.shape[1], _lib.ptr(r)))
        return float(r[0]), float(r[1])

    def run_quantized_codes(self, cfg) -> np.ndarray:
        """Output codes of the eval set (intexec.run_quantized(..., return_codes=True))."""
        from .intonly import run_quantized_codes
        return run_quantized_codes(self, cfg)

    def run_integer_only(self, cfg, trace=None) -> np.ndarray:
        """intexec.run_integer_only (intexec.py:354-359) from device state; see intonly.py."""
        from .intonly import run_integer_only
        return run_integer_only(self, cfg, trace)

    def save_cache(self, path: str, size_class: str, meta: dict | None = None) -> None:
        """Write one calibration cache of this evaluator as the reference's ``.qcal``
        (calibration.py:115-134), byte-identical to ptqtune.save_cache of the same cache."""
        from .artifacts import save_qcal
        k = CACHE_SIZES.index(size_class)
        ids = self.image_ids[k] if getattr(self, "image_ids", None) else select_images(self.n_calib, size_class, self.seed)
        save_qcal(path, getattr(self.graph, "name", "model"), size_class, ids, self.lowered.tensor_names,
                  self.cache_ranges[k], self.cache_counts[k], self.cache_nsamp[k], meta)

    def act_params(self, cache: int, scheme: int, clipping: int):
        s = np.zeros(self.T, dtype=np.float32)
        z = np.zeros(self.T, dtype=np.int32)
        _lib.check(self.lib.ptq_probe_act_params(self._ctx, cache, scheme, clipping, _lib.ptr(s), _lib.ptr(z)))
        return s, z

    def evaluate_grid(self, cfgs) -> np.ndarray:
        """Correct counts of every config; under torch.distributed each rank evaluates its
        block of whole parameter variants (dist.shard_plan) and one SUM allreduce
        reassembles the counts in the caller's order."""
        from . import dist
        cfgs = list(cfgs)
        if self.image_sharded:
            return dist.allreduce(self.correct_counts(cfgs), "sum")
        rank, n = dist.world()
        if n == 1:
            return self.correct_counts(cfgs)
        idx = dist.shard_plan(cfgs, n)[rank]
        mine = self.correct_counts([cfgs[i] for i in idx]) if idx else np.zeros(0, np.int64)
        return dist.gather_counts(mine, idx, len(cfgs))

    def histogram_array(self, x: np.ndarray, lo: float, hi: float) -> np.ndarray:
        x = np.ascontiguousarray(np.asarray(x, dtype=np.float32).ravel())
        out = np.zeros(N_BINS, dtype=np.int64)
        _lib.check(self.lib.ptq_histogram_host(self._ctx, _lib.ptr(x), x.size, float(lo), float(hi),
                                               _lib.ptr(out)))
        return out

    def stats(self) -> dict:
        n, ms, ops, nc, nt = C.c_int64(), C.c_double(), C.c_double(), C.c_int64(), C.c_int64()
        _lib.check(self.lib.ptq_last_stats(self._ctx, C.byref(n), C.byref(ms), C.byref(ops), C.byref(nc),
                                           C.byref(nt)))
        return {"launches": n.value, "conv_ms": ms.value, "conv_ops": ops.value,
                "conv_launches": nc.value, "conv_launches_total": nt.value}

    def conv_timings(self) -> np.ndarray:
        n = C.c_int64()
        _lib.check(self.lib.ptq_conv_timings(self._ctx, None, 0, C.byref(n)))
        out = np.zeros(n.value, dtype=np.float32)
        _lib.check(self.lib.ptq_conv_timings(self._ctx, _lib.ptr(out), n.value, C.byref(n)))
        return out

    def stream_handle(self) -> int:
        s = C.c_void_p()
        _lib.check(self.lib.ptq_stream(self._ctx, C.byref(s)))
        return s.value or 0

    def close(self) -> None:
        if getattr(self, "_ctx", None) and self._ctx.value:
            self.lib.ptq_destroy(self._ctx)
            self._ctx = C.c_void_p()
        self._host_imgs = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def make_accuracy_evaluator(g, d, seed: int, profile: TargetProfile | None = None, *,
                            device: int = 0, eval_chunk: int | None = None,
                            image_sharded: bool = False) -> GpuEvaluator:
    """Drop-in for ptqtune.tuner.make_accuracy_evaluator (tuner.py:434-444).
    ``image_sharded=True`` under torch.distributed splits the eval images over the ranks
    (for the one-config-at-a-time xgb / GA searches); every rank must then evaluate the
    same configs in the same order."""
    return GpuEvaluator(g, d, seed, profile, device=device, eval_chunk=eval_chunk,
                        image_sharded=image_sharded)
