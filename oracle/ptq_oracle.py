"""CPU oracle: numpy restatement of the reference's PTQ evaluator hot path.

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs may import this module, and
only as the checker or the timed CPU baseline -- never as part of the
product path (the GPU evaluator fails loudly when its CUDA library is
missing; it has no CPU fallback).

Parity is PINNED: tests/test_oracle_golden.py checks every function here
against golden vectors that tests/golden/gen_golden.py produced by importing
the reference itself (/root/reference/pkg/src/ptqtune) in the build
container (scheme / quantize / requantize known answers, caches, KL windows
and the App. B grids of the three fixtures).

Each function cites the reference file:line it restates ("ref:" below is
/root/reference/pkg/src/ptqtune/).  Graph and dataset arguments are
duck-typed (anything with the reference's Graph/Dataset attributes).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
from numpy.lib.stride_tricks import sliding_window_view

QMIN, QMAX = -128, 127
INT32_MIN, INT32_MAX = -(2 ** 31), 2 ** 31 - 1
N_BINS = 2048
SIZE_CLASSES = {"S1": 1, "S2": 32, "S3": 256}
INPUT = "input"
CONV_KINDS = ("conv2d", "depthwise_conv2d", "pointwise_conv2d")
COMPUTE_KINDS = CONV_KINDS + ("fully_connected",)


def _ins(n):
    return list(n.inputs[:1]) if n.kind in COMPUTE_KINDS else list(n.inputs)


def _consumers(g, t):
    return [n for n in g.nodes if t in _ins(n)]


def _output_tensor(g):
    used = {t for n in g.nodes for t in _ins(n)}
    outs = [n.output for n in g.nodes if n.output not in used]
    assert len(outs) == 1
    return outs[0]


def _scheme_name(s) -> str:
    return getattr(s, "value", s)


# ---------------------------------------------------------------- schemes
# ref: schemes.py:61-131

def rha(x):
    """Round half away from zero (ref: schemes.py:61-64)."""
    x = np.asarray(x, dtype=np.float64)
    return np.sign(x) * np.floor(np.abs(x) + 0.5)


def rhu(x):
    """Round half up (ref: intexec.py:67-69)."""
    return np.floor(np.asarray(x, dtype=np.float64) + 0.5)


def ceil_log2(x: float) -> int:
    """ref: schemes.py:67-72 (frexp based, exact)."""
    if not (x > 0 and math.isfinite(x)):
        raise ValueError(f"ceil_log2 needs a positive finite value, got {x}")
    m, e = math.frexp(x)
    return e - 1 if m == 0.5 else e


@dataclass
class Params:
    scale: object          # np.float32 scalar or float32 array (per channel)
    zp: object             # int or int64 array
    axis: int | None = None


def params_for_range(scheme, vmin: float, vmax: float) -> Params:
    """(scale, zero_point) for a range; ref: schemes.py:81-131."""
    scheme = _scheme_name(scheme)
    vmin, vmax = float(vmin), float(vmax)
    for v in (vmin, vmax):
        if not math.isfinite(v):
            raise ValueError("non-finite range value")
    max_abs = max(abs(vmin), abs(vmax))

    def sym(m):
        if m == 0.0:
            return Params(np.float32(1.0), 0)
        return Params(np.float32(abs(m) / 127), 0)

    if scheme == "Asymmetric":                      # ref: schemes.py:81-93
        if vmin > vmax:
            raise ValueError("min > max")
        lo, hi = min(vmin, 0.0), max(vmax, 0.0)
        if lo == hi:
            return Params(np.float32(1.0), 0)
        s64 = (hi - lo) / 255
        return Params(np.float32(s64), int(-rha(lo / s64)) - 128)
    if scheme == "Symmetric":                       # ref: schemes.py:96-101
        return sym(max_abs)
    if scheme == "SymmetricUint8":                  # ref: schemes.py:104-111
        if vmin < 0.0:
            return sym(max_abs)
        if max_abs == 0.0:
            return Params(np.float32(1.0), -128)
        return Params(np.float32(abs(max_abs) / 255), -128)
    if scheme == "SymmetricPower2":                 # ref: schemes.py:114-117
        k = ceil_log2(float(sym(max_abs).scale))
        return Params(np.float32(2.0 ** k), 0)
    raise ValueError(f"unknown scheme {scheme!r}")


def _bcast(p: Params, ndim: int, axis: int):
    s = np.asarray(p.scale, dtype=np.float64)
    z = np.asarray(p.zp, dtype=np.float64)
    if p.axis is not None:
        shape = [1] * ndim
        shape[axis] = -1
        s, z = s.reshape(shape), z.reshape(shape)
    return s, z


def quantize_array(x, p: Params, axis: int = 0) -> np.ndarray:
    """ref: schemes.py:145-150 -- clip(RHA(x64 / s64 + zp), -128, 127)."""
    x = np.asarray(x, dtype=np.float64)
    s, z = _bcast(p, x.ndim, axis)
    return np.clip(rha(x / s + z), QMIN, QMAX).astype(np.int8)


def dequantize_array(c, p: Params, axis: int = 0) -> np.ndarray:
    """ref: schemes.py:153-155 -- f32((c - zp) * s)."""
    c = np.asarray(c, dtype=np.float64)
    s, z = _bcast(p, c.ndim, axis)
    return ((c - z) * s).astype(np.float32)


# ---------------------------------------------------------------- fp32 forward
# ref: fp32.py:33-114

def _win(x, k, s, p):
    if p:
        x = np.pad(x, ((0, 0), (0, 0), (p, p), (p, p)))
    return sliding_window_view(x, (k, k), axis=(2, 3))[:, :, ::s, ::s]


def conv2d(x, w, b, s, p):
    """im2col + GEMM (ref: fp32.py:41-51)."""
    win = _win(x, w.shape[2], s, p)
    n, _, oh, ow = win.shape[:4]
    cols = np.ascontiguousarray(win.transpose(0, 2, 3, 1, 4, 5).reshape(n * oh * ow, -1))
    y = cols @ w.reshape(w.shape[0], -1).T
    if b is not None:
        y = y + b
    return y.reshape(n, oh, ow, -1).transpose(0, 3, 1, 2)


def dwconv2d(x, w, b, s, p):
    """ref: fp32.py:54-60."""
    y = np.einsum("nchwij,cij->nchw", _win(x, w.shape[2], s, p), w[:, 0], dtype=x.dtype)
    return y if b is None else y + b[None, :, None, None]


def _softmax(x):
    z = np.exp(x - x.max(axis=-1, keepdims=True))
    return z / z.sum(axis=-1, keepdims=True)


def _fp32_node(g, n, env):
    x = env[n.inputs[0]]
    k = n.kind
    if k in COMPUTE_KINDS:
        w = g.weights[n.inputs[1]]
        b = g.weights[n.inputs[2]] if len(n.inputs) > 2 else None
        if k == "fully_connected":
            y = x.reshape(x.shape[0], -1) @ w.T
            return y if b is None else y + b
        s, p = int(n.attrs.get("stride", 1)), int(n.attrs.get("padding", 0))
        return (dwconv2d if k == "depthwise_conv2d" else conv2d)(x, w, b, s, p)
    if k == "relu":
        return np.maximum(x, np.float32(0))
    if k in ("maxpool", "avgpool"):
        ks = int(n.attrs["kernel"])
        win = _win(x, ks, int(n.attrs.get("stride", ks)), 0)
        return win.max(axis=(-1, -2)) if k == "maxpool" else win.mean(axis=(-1, -2), dtype=x.dtype)
    if k == "add":
        return x + env[n.inputs[1]]
    if k == "concat":
        return np.concatenate([env[t] for t in n.inputs], axis=1)
    if k == "softmax":
        return _softmax(x)
    raise ValueError(k)


def run_fp32(g, batch, sink=None):
    """ref: fp32.py:77-114; sink(tensor_id, values) sees input + every node."""
    batch = np.asarray(batch, dtype=np.float32)
    if batch.ndim == 3:
        batch = batch[None]
    env = {INPUT: batch}
    if sink is not None:
        sink(INPUT, batch)
    for n in g.nodes:
        env[n.output] = _fp32_node(g, n, env).astype(np.float32, copy=False)
        if sink is not None:
            sink(n.output, env[n.output])
    return env[_output_tensor(g)]


def observe_activations(g, images, sink):
    """One image at a time (ref: fp32.py:138-148)."""
    images = np.asarray(images, dtype=np.float32)
    if images.ndim == 3:
        images = images[None]
    for i in range(images.shape[0]):
        run_fp32(g, images[i:i + 1], sink)


def top1_count(scores, labels) -> int:
    """argmax with lowest index on ties (ref: fp32.py:123-128)."""
    return int(np.sum(np.argmax(scores, axis=-1) == np.asarray(labels)))


# ---------------------------------------------------------------- calibration
# ref: calibration.py:19-112

@dataclass
class Hist:
    tensor_id: str
    lo: float                   # float32 value (min_seen)
    hi: float                   # float32 value (max_seen)
    counts: np.ndarray          # int64[2048]
    n_samples: int
    memo: dict = field(default_factory=dict, repr=False)

    def edges(self):
        return np.linspace(float(self.lo), float(self.hi), N_BINS + 1)


def select_images(n_pool: int, size_class: str, seed: int) -> np.ndarray:
    """ref: calibration.py:44-54."""
    n = SIZE_CLASSES[size_class]
    return np.sort(np.random.default_rng(seed).choice(n_pool, size=n, replace=False))


def histogram_counts(values, lo: float, hi: float) -> np.ndarray:
    """One tensor's contribution (ref: calibration.py:81-91)."""
    flat = np.asarray(values).ravel().astype(np.float64)
    out = np.zeros(N_BINS, dtype=np.int64)
    if lo == hi:
        out[0] += flat.size
    else:
        out += np.histogram(flat, bins=N_BINS, range=(lo, hi))[0]
    return out


def calibrate_from_activations(per_image: list[dict]) -> dict[str, Hist]:
    """Two-pass calibration over recorded per-image activations.

    ``per_image[i][tensor_id]`` is the fp32 tensor image i produced; the
    insertion order of the first image gives the tensor order.  Restates
    ref: calibration.py:57-106 with the activations injected (staged parity
    P1: the GPU is fed the very same fp32 activations)."""
    order = list(per_image[0].keys())
    mins = {t: math.inf for t in order}
    maxs = {t: -math.inf for t in order}
    for acts in per_image:                         # pass 1 (ref: :67-76)
        for t in order:
            v = acts[t]
            mins[t] = min(mins[t], float(v.min()))
            maxs[t] = max(maxs[t], float(v.max()))
    counts = {t: np.zeros(N_BINS, dtype=np.int64) for t in order}
    nsamp = {t: 0 for t in order}
    for acts in per_image:                         # pass 2 (ref: :81-93)
        for t in order:
            counts[t] += histogram_counts(acts[t], mins[t], maxs[t])
            nsamp[t] += acts[t].size
    return {t: Hist(t, float(np.float32(mins[t])), float(np.float32(maxs[t])), counts[t], nsamp[t])
            for t in order}


def calibrate(g, images) -> dict[str, Hist]:
    """ref: calibration.py:57-106 (fp32 forward one image at a time)."""
    images = np.asarray(images, dtype=np.float32)
    per_image = []
    for i in range(images.shape[0]):
        acts = {}
        run_fp32(g, images[i:i + 1], lambda t, v: acts.__setitem__(t, v))
        per_image.append(acts)
    return calibrate_from_activations(per_image)


def build_cache(g, d, size_class: str, seed: int) -> dict[str, Hist]:
    """ref: calibration.py:109-112."""
    idx = select_images(d.n_calib, size_class, seed)
    return calibrate(g, d.images[: d.n_calib][idx])


# ---------------------------------------------------------------- clipping
# ref: clipping.py:34-96

def window_kl(win: np.ndarray, ref: np.ndarray, levels: int = 128) -> float:
    """KL(P || Q) of one candidate window (ref: clipping.py:38-52)."""
    i = win.size
    m = i // levels
    starts = np.arange(levels) * m
    gsum = np.add.reduceat(win, starts)
    nz = ref > 0
    gnz = np.add.reduceat(nz.astype(np.float64), starts)
    grp = np.minimum(np.arange(i) // m, levels - 1)
    q = np.zeros(i)
    q[nz] = gsum[grp[nz]] / gnz[grp[nz]]
    if np.any(nz & (q == 0.0)):
        return math.inf
    p = ref[nz]
    return float(np.sum(p * (np.log(p) - np.log(q[nz]))) / ref.sum())


def kl_windows(h: Hist):
    """Yield (i, start, end, win, ref) for every candidate (ref: clipping.py:55-81)."""
    lo, hi = float(h.lo), float(h.hi)
    counts = np.asarray(h.counts, dtype=np.float64)
    total = counts.sum()
    signed = lo < 0.0
    zero_bin = int((0.0 - lo) / ((hi - lo) / N_BINS)) if signed else 0
    cum = np.cumsum(counts)
    for i in range(128, N_BINS + 1):
        start = min(max(zero_bin - i // 2, 0), N_BINS - i) if signed else 0
        end = start + i
        win = counts[start:end]
        ref = win.copy()
        if start > 0:
            ref[0] += cum[start - 1]
        ref[-1] += total - cum[end - 1]
        yield i, start, end, win, ref


def kl_sweep(h: Hist) -> tuple[int, int, np.ndarray]:
    """All 1921 candidate KLs plus the chosen (start, end) (ref: clipping.py:55-86)."""
    kls = np.full(N_BINS + 1 - 128, np.inf)
    best, best_kl = (0, N_BINS), math.inf
    for i, start, end, win, ref in kl_windows(h):
        kl = window_kl(win, ref)
        kls[i - 128] = kl
        if kl < best_kl:                          # strict: ties keep smaller window
            best_kl, best = kl, (start, end)
    return best[0], best[1], kls


def clip_range_kl(h: Hist) -> tuple[float, float]:
    """ref: clipping.py:55-86."""
    if h.n_samples <= 0:
        raise ValueError("empty histogram")
    lo, hi = float(h.lo), float(h.hi)
    if lo == hi or float(np.asarray(h.counts, dtype=np.float64).sum()) <= 0:
        return lo, hi
    start, end, _ = kl_sweep(h)
    e = h.edges()
    return float(e[start]), float(e[end])


def clipped_range(h: Hist, mode: str) -> tuple[float, float]:
    """Memoised Max/KL dispatch (ref: clipping.py:89-96)."""
    if mode not in h.memo:
        h.memo[mode] = (float(h.lo), float(h.hi)) if mode == "Max" else clip_range_kl(h)
    return h.memo[mode]


def percentile_range(counts, lo: float, hi: float, pct: float) -> tuple[float, float]:
    """EXTENSION, not a restatement: the reference rejects "Percentile" clipping
    (clipping.py:91-92), so this definition is ours and parity is unpinned (include/ptq_b200.h,
    ptq_percentile_ranges).  With N = sum(counts), q = pct / 100 and cum the running count:
    hi_idx = first bin with cum >= q N, lo_idx = first bin with cum > (1 - q) N; the range is
    (edge[lo_idx], edge[hi_idx + 1]) on numpy's histogram edges (calibration.py:81-91).
    Histograms the KL sweep skips (lo == hi or empty) keep (lo, hi)."""
    counts = np.asarray(counts, dtype=np.int64).ravel()
    lo, hi = float(lo), float(hi)
    total = int(counts.sum())
    if total == 0 or not lo < hi:
        return (lo, hi)
    q = float(pct) / 100.0
    cum = np.cumsum(counts).astype(np.float64)
    li = np.flatnonzero(cum > (1.0 - q) * float(total))
    hj = np.flatnonzero(cum >= q * float(total))
    li = int(li[0]) if li.size else N_BINS - 1
    hj = int(hj[0]) if hj.size else N_BINS - 1
    edges = np.linspace(lo, hi, N_BINS + 1)
    return (float(edges[li]), float(edges[hj + 1]))


# ---------------------------------------------------------------- quantize_model
# ref: quantize.py:99-211

def quantize_weights(w, scheme, granularity):
    """ref: quantize.py:99-113."""
    w = np.asarray(w, dtype=np.float32)
    if granularity == "Channel" and w.ndim >= 2:
        ps = [params_for_range(scheme, float(w[o].min()), float(w[o].max()))
              for o in range(w.shape[0])]
        p = Params(np.asarray([q.scale for q in ps], dtype=np.float32),
                   np.asarray([q.zp for q in ps], dtype=np.int64), axis=0)
    else:
        p = params_for_range(scheme, float(w.min()), float(w.max()))
    return quantize_array(w, p, axis=0), p


@dataclass
class QModel:
    graph: object
    cfg: object
    act: dict            # tensor -> Params
    wcodes: dict         # weight id -> int8 codes
    wparams: dict        # weight id -> Params
    bias: dict           # bias id -> int32 codes
    fp32_nodes: set


def _narrowed(g, n):
    """ref: quantize.py:125-130."""
    cons = _consumers(g, n.output)
    return cons[0].output if len(cons) == 1 and cons[0].kind == "relu" else n.output


def quantize_model(g, cache: dict, cfg) -> QModel:
    """ref: quantize.py:133-211 (Generic profile; fusion is numerics-neutral)."""
    scheme = _scheme_name(cfg.scheme)

    def ap(t):
        lo, hi = clipped_range(cache[t], cfg.clipping)
        return params_for_range(scheme, lo, hi)

    comp = [n for n in g.nodes if n.kind in COMPUTE_KINDS]
    fp32_nodes = {comp[0].id, comp[-1].id} if cfg.mixed == "FirstLastFp32" else set()
    act, wc, wp, bias = {}, {}, {}, {}
    dom = {INPUT: cfg.mixed == "Off"}
    if dom[INPUT]:
        act[INPUT] = ap(INPUT)
    for n in g.nodes:
        ind = [dom[t] for t in _ins(n)]
        if n.kind in COMPUTE_KINDS:
            if n.id in fp32_nodes:
                if n.id == comp[-1].id:
                    dom[n.output] = False
                else:
                    act[n.output] = ap(_narrowed(g, n))
                    dom[n.output] = True
                continue
            assert all(ind)
            codes, p = quantize_weights(g.weights[n.inputs[1]], scheme, cfg.granularity)
            wc[n.inputs[1]], wp[n.inputs[1]] = codes, p
            if len(n.inputs) > 2:                  # ref: quantize.py:177-182
                s_b = float(act[n.inputs[0]].scale) * np.asarray(p.scale, dtype=np.float64)
                bq = rha(np.asarray(g.weights[n.inputs[2]], dtype=np.float64) / s_b)
                bias[n.inputs[2]] = np.clip(bq, INT32_MIN, INT32_MAX).astype(np.int32)
            act[n.output] = ap(_narrowed(g, n))
            dom[n.output] = True
        elif n.kind in ("add", "concat"):
            if all(ind):
                act[n.output] = ap(_narrowed(g, n) if n.kind == "add" else n.output)
                dom[n.output] = True
            else:
                assert not any(ind)
                dom[n.output] = False
        else:
            dom[n.output] = dom[n.inputs[0]]
            if dom[n.output]:
                act[n.output] = act[n.inputs[0]]
    return QModel(g, cfg, act, wc, wp, bias, fp32_nodes)


# ---------------------------------------------------------------- int8 execution
# ref: intexec.py:72-351

def requantize(acc, m, zp):
    """ref: intexec.py:72-85 (multiplier path)."""
    acc = np.asarray(acc, dtype=np.int64)
    return np.clip(rhu(acc * np.asarray(m, dtype=np.float64)) + zp, QMIN, QMAX).astype(np.int8)


def requantize_shift(acc, shift, zp):
    """ref: intexec.py:80-84 (shift path)."""
    acc = np.asarray(acc, dtype=np.int64)
    if shift > 0:
        v = (acc + (1 << (shift - 1))) >> shift
    elif shift == 0:
        v = acc
    else:
        v = acc << (-shift)
    return np.clip(v + zp, QMIN, QMAX).astype(np.int8)


def int_conv(kind, xs, ws, stride, pad):
    """Exact integer conv via a float64 carrier (ref: intexec.py:95-105)."""
    xf, wf = xs.astype(np.float64), ws.astype(np.float64)
    if kind in ("conv2d", "pointwise_conv2d"):
        y = conv2d(xf, wf, None, stride, pad)
    elif kind == "depthwise_conv2d":
        y = dwconv2d(xf, wf, None, stride, pad)
    else:
        y = xf.reshape(xf.shape[0], -1) @ wf.T
    return y.astype(np.int64)


def _pc(v, ndim):
    shape = [1] * ndim
    shape[1] = -1
    return np.asarray(v).reshape(shape)


def run_quantized(qm: QModel, batch, sink=None, accs=None, inject=None):
    """Simulated-int8 forward (ref: intexec.py:148-351).

    Returns fp32 scores (dequantized output codes, or fp32 logits when the
    last layer is kept in fp32).  ``sink(t, v)`` sees codes (int64) for
    quantized tensors and fp32 values otherwise; ``accs`` (dict) collects
    each int8 compute node's clipped int32 accumulator.  ``inject`` (test
    staging only) replaces a node's output by the given values, e.g. the
    device's codes at the boundary after an fp32 first layer, so everything
    downstream is compared on identical int8 inputs."""
    g = qm.graph
    batch = np.asarray(batch, dtype=np.float32)
    env = {}
    env[INPUT] = quantize_array(batch, qm.act[INPUT]).astype(np.int64) if INPUT in qm.act else batch
    for n in g.nodes:
        x = env[n.inputs[0]]
        k = n.kind
        if k in COMPUTE_KINDS and n.id in qm.fp32_nodes:
            out = _run_fp32_layer(qm, n, env)
        elif k in COMPUTE_KINDS:
            wid = n.inputs[1]
            pw, pin, pout = qm.wparams[wid], qm.act[n.inputs[0]], qm.act[n.output]
            xs = x - int(pin.zp)
            ws = qm.wcodes[wid].astype(np.int64)
            ws = ws - np.atleast_1d(np.asarray(pw.zp, dtype=np.int64)).reshape((-1,) + (1,) * (ws.ndim - 1))
            acc = int_conv(k, xs, ws, int(n.attrs.get("stride", 1)), int(n.attrs.get("padding", 0)))
            if len(n.inputs) > 2:
                b = qm.bias[n.inputs[2]].astype(np.int64)
                acc = acc + (_pc(b, acc.ndim) if acc.ndim == 4 else b)
            acc = np.clip(acc, INT32_MIN, INT32_MAX)
            if accs is not None:
                accs[n.id] = acc
            m = float(pin.scale) * np.asarray(pw.scale, dtype=np.float64) / float(pout.scale)
            if pw.axis is not None and acc.ndim == 4:
                m = _pc(m, acc.ndim)
            out = requantize(acc, m, int(pout.zp))
            if n.attrs.get("fused_relu"):
                out = np.maximum(out, np.int8(pout.zp))
            out = out.astype(np.int64)
        elif k == "relu":
            out = np.maximum(x, int(qm.act[n.output].zp)) if n.output in qm.act else np.maximum(x, np.float32(0))
        elif k == "maxpool":
            ks = int(n.attrs["kernel"])
            out = _win(x, ks, int(n.attrs.get("stride", ks)), 0).max(axis=(-1, -2))
        elif k == "avgpool":
            ks = int(n.attrs["kernel"])
            s = int(n.attrs.get("stride", ks))
            if n.output in qm.act:
                zp = int(qm.act[n.output].zp)
                tot = _win(x, ks, s, 0).sum(axis=(-1, -2))
                out = requantize(tot - zp * ks * ks, 1.0 / (ks * ks), zp).astype(np.int64)
            else:
                out = _win(x, ks, s, 0).mean(axis=(-1, -2), dtype=x.dtype)
        elif k == "add":
            y = env[n.inputs[1]]
            if n.output in qm.act:                 # ref: intexec.py:245-276
                po, pa, pb = qm.act[n.output], qm.act[n.inputs[0]], qm.act[n.inputs[1]]
                so = float(po.scale)
                acc = (x - int(pa.zp)) * (float(pa.scale) / so) + (y - int(pb.zp)) * (float(pb.scale) / so)
                out = np.clip(rhu(acc) + int(po.zp), QMIN, QMAX).astype(np.int64)
            else:
                out = x + y
        elif k == "concat":
            if n.output in qm.act:                 # ref: intexec.py:115-129, :281-289
                po = qm.act[n.output]
                parts = [requantize(env[t] - int(qm.act[t].zp),
                                    float(qm.act[t].scale) / float(po.scale), int(po.zp)).astype(np.int64)
                         for t in n.inputs]
                out = np.concatenate(parts, axis=1)
            else:
                out = np.concatenate([env[t] for t in n.inputs], axis=1)
        elif k == "softmax":
            out = x if n.output in qm.act else _softmax(x)
        else:
            raise ValueError(k)
        if inject is not None and n.output in inject:
            out = np.asarray(inject[n.output]).astype(out.dtype if hasattr(out, "dtype") else np.int64)
        env[n.output] = out
        if sink is not None:
            sink(n.output, out)
    t = _output_tensor(g)
    if t in qm.act:
        return dequantize_array(env[t].astype(np.int8), qm.act[t])
    return env[t]


def _run_fp32_layer(qm: QModel, n, env):
    """Mixed-precision layer (ref: intexec.py:304-334)."""
    g = qm.graph
    x = env[n.inputs[0]]
    if n.inputs[0] in qm.act:
        x = dequantize_array(x.astype(np.int8), qm.act[n.inputs[0]])
    w = g.weights[n.inputs[1]]
    b = g.weights[n.inputs[2]] if len(n.inputs) > 2 else None
    if n.kind in CONV_KINDS:
        s, p = int(n.attrs.get("stride", 1)), int(n.attrs.get("padding", 0))
        out = (dwconv2d if n.kind == "depthwise_conv2d" else conv2d)(x.astype(np.float32), w, b, s, p)
    else:
        out = x.reshape(x.shape[0], -1).astype(np.float32) @ w.T
        if b is not None:
            out = out + b
    if n.attrs.get("fused_relu"):
        out = np.maximum(out, np.float32(0))
    if n.output in qm.act:
        out = quantize_array(out, qm.act[n.output]).astype(np.int64)
    return out


# ---------------------------------------------------------------- evaluator
# ref: tuner.py:434-444

def make_accuracy_evaluator(g, d, seed: int, caches: dict | None = None):
    """Returns evaluate(cfg) -> top-1 (ref: tuner.py:434-444).

    ``caches`` may inject prebuilt {size_class: {tensor: Hist}} (staged
    parity P2)."""
    if caches is None:
        caches = {sc: build_cache(g, d, sc, seed) for sc in ("S1", "S2", "S3")}

    def evaluate(cfg) -> float:
        qm = quantize_model(g, caches[cfg.cache], cfg)
        scores = run_quantized(qm, d.images[d.n_calib:])
        return top1_count(scores, d.labels[d.n_calib:]) / float(len(d.labels) - d.n_calib)

    evaluate.caches = caches
    return evaluate


# ---------------------------------------------------------------- integer-only executor
# ref: intexec.py:40-64 (OpTrace), :88-92 (_exact_log2), :115-145, :354-359,
# :369-398 (fuse_conv_relu); pinned by tests/golden/gen_intonly_golden.py

FLOAT_CATS = ("float_mul", "float_add", "float_kernel")


class IntegerOnlyError(ValueError):
    """ref: intexec.py:43."""


@dataclass
class OpTrace:
    """(node id, op category) events in execution order (ref: intexec.py:47-64)."""
    events: list = field(default_factory=list)

    def add(self, node_id, *cats):
        self.events.extend((node_id, c) for c in cats)

    def float_ops(self) -> int:
        return sum(1 for _, c in self.events if c in FLOAT_CATS)

    def to_csv(self) -> str:
        return "\n".join(["node,category"] + [f"{n},{c}" for n, c in self.events]) + "\n"


@dataclass
class _N:
    id: str
    kind: str
    inputs: list
    output: str
    attrs: dict


@dataclass
class _G:
    nodes: list
    weights: dict


def fuse_graph(g):
    """Compute -> sole-relu pairs merged into one node with fused_relu (ref: intexec.py:369-398)."""
    fuse = {}
    for n in g.nodes:
        if n.kind in COMPUTE_KINDS:
            cons = _consumers(g, n.output)
            if len(cons) == 1 and cons[0].kind == "relu":
                fuse[n.id] = cons[0]
    drop = {r.id for r in fuse.values()}
    nodes = [_N(n.id, n.kind, list(n.inputs), fuse[n.id].output if n.id in fuse else n.output,
                {**dict(n.attrs), **({"fused_relu": True} if n.id in fuse else {})})
             for n in g.nodes if n.id not in drop]
    return _G(nodes, g.weights)


def exact_log2(scale: float) -> int:
    """ref: intexec.py:88-92."""
    k = ceil_log2(scale)
    if 2.0 ** k != scale:
        raise IntegerOnlyError(f"scale {scale} is not a power of two")
    return k


def check_integer_only(qm: QModel) -> None:
    """ref: intexec.py:132-145."""
    cfg = qm.cfg
    scheme = _scheme_name(cfg.scheme)
    if scheme != "SymmetricPower2" or cfg.granularity != "Tensor" or cfg.mixed != "Off":
        raise IntegerOnlyError(
            "integer-only execution requires scheme=SymmetricPower2, granularity=Tensor, mixed=Off; "
            f"got {scheme}/{cfg.granularity}/{cfg.mixed}")
    for n in qm.graph.nodes:
        if n.kind == "avgpool":
            area = int(n.attrs["kernel"]) ** 2
            if area & (area - 1):
                raise IntegerOnlyError(f"avgpool {n.id}: area {area} not a power of two")


def run_integer_only(qm: QModel, batch, trace: OpTrace | None = None) -> np.ndarray:
    """Strict integer program: mul/add/shift/clamp only (ref: intexec.py:148-359 with
    integer_only=True).  ``qm.graph`` is the graph as executed (pass a fuse_graph()
    graph for fusion=True).  Returns int8 output codes."""
    check_integer_only(qm)
    g = qm.graph
    tr = trace if trace is not None else OpTrace()
    env = {INPUT: quantize_array(np.asarray(batch, dtype=np.float32), qm.act[INPUT]).astype(np.int64)}
    for n in g.nodes:
        x = env[n.inputs[0]]
        k = n.kind
        if k in COMPUTE_KINDS:                         # ref: intexec.py:170-211
            wid = n.inputs[1]
            pw, pin, pout = qm.wparams[wid], qm.act[n.inputs[0]], qm.act[n.output]
            ws = qm.wcodes[wid].astype(np.int64) - int(np.asarray(pw.zp))
            acc = int_conv(k, x - int(pin.zp), ws, int(n.attrs.get("stride", 1)), int(n.attrs.get("padding", 0)))
            tr.add(n.id, "int_mul", "int_add")
            if len(n.inputs) > 2:
                b = qm.bias[n.inputs[2]].astype(np.int64)
                acc = acc + (_pc(b, acc.ndim) if acc.ndim == 4 else b)
                tr.add(n.id, "int_add")
            acc = np.clip(acc, INT32_MIN, INT32_MAX)
            s = exact_log2(float(pout.scale)) - exact_log2(float(pin.scale)) - exact_log2(float(pw.scale))
            out = requantize_shift(acc, s, int(pout.zp))
            tr.add(n.id, "int_add", "shift", "clamp")
            if n.attrs.get("fused_relu"):
                out = np.maximum(out, np.int8(pout.zp))
                tr.add(n.id, "clamp")
            out = out.astype(np.int64)
        elif k == "relu":
            out = np.maximum(x, int(qm.act[n.output].zp))
            tr.add(n.id, "clamp")
        elif k == "maxpool":
            ks = int(n.attrs["kernel"])
            out = _win(x, ks, int(n.attrs.get("stride", ks)), 0).max(axis=(-1, -2))
        elif k == "avgpool":                           # ref: intexec.py:225-243
            ks = int(n.attrs["kernel"])
            zp = int(qm.act[n.output].zp)
            tot = _win(x, ks, int(n.attrs.get("stride", ks)), 0).sum(axis=(-1, -2))
            out = requantize_shift(tot - zp * ks * ks, exact_log2(float(ks * ks)), zp).astype(np.int64)
            tr.add(n.id, "int_add", "shift", "clamp")
        elif k == "add":                               # ref: intexec.py:256-265
            y = env[n.inputs[1]]
            po, pa, pb = qm.act[n.output], qm.act[n.inputs[0]], qm.act[n.inputs[1]]
            ka, kb, ko = exact_log2(float(pa.scale)), exact_log2(float(pb.scale)), exact_log2(float(po.scale))
            kmin = min(ka, kb)
            acc = ((x - int(pa.zp)) << (ka - kmin)) + ((y - int(pb.zp)) << (kb - kmin))
            out = requantize_shift(acc, ko - kmin, int(po.zp)).astype(np.int64)
            tr.add(n.id, "int_add", "shift", "int_add", "shift", "int_add", "shift", "clamp")
        elif k == "concat":                            # ref: intexec.py:115-129
            po = qm.act[n.output]
            parts = []
            for t in n.inputs:
                s = exact_log2(float(po.scale)) - exact_log2(float(qm.act[t].scale))
                parts.append(requantize_shift(env[t] - int(qm.act[t].zp), s, int(po.zp)).astype(np.int64))
                tr.add(n.id, "int_add", "shift", "clamp")
            out = np.concatenate(parts, axis=1)
        elif k == "softmax":
            out = x
        else:
            raise ValueError(k)
        env[n.output] = out
    return env[_output_tensor(g)].astype(np.int8)
