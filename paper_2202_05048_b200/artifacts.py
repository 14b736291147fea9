"""Artifact emitters: calibration caches written from the GPU
evaluator's state in the reference's `.qcal` file format, byte for byte.

The container (ptqtune/container.py:1-52) is: the magic line ``QTM1``, a line
``HDR <n>`` with the byte length of the header, the header as canonical JSON
(sorted keys, no whitespace, UTF-8) carrying a ``buffers`` table of
``{dtype, shape}``, then the raw little-endian buffers in that order.  A
calibration cache (calibration.py:115-134) lists its tensors sorted by name and
stores float32 ranges [T, 2] and int64 counts [T, 2048].

Parity: tests/test_artifacts.py (CPU, golden hashes of the reference's own
files: tests/golden/ref_qcal.json) and tests/test_gpu_parity.py (from device
state).
"""

from __future__ import annotations

import json

import numpy as np

CONTAINER_MAGIC = b"QTM1\n"


def _canonical(obj) -> bytes:
    return json.dumps(obj, sort_keys=True, separators=(",", ":")).encode("utf-8")


def write_container(path: str, header: dict, buffers) -> None:
    """QTM1 container: magic, header length line, canonical JSON header, raw buffers."""
    if "buffers" in header:
        raise ValueError("the 'buffers' header key is reserved")
    little = [np.ascontiguousarray(b).astype(np.asarray(b).dtype.newbyteorder("<"), copy=False) for b in buffers]
    full = dict(header)
    full["buffers"] = [{"dtype": b.dtype.name, "shape": list(b.shape)} for b in little]
    head = _canonical(full)
    with open(path, "wb") as f:
        f.write(CONTAINER_MAGIC)
        f.write(b"HDR %d\n" % len(head))
        f.write(head)
        for b in little:
            f.write(b.tobytes())


def save_qcal(path: str, model_name: str, size_class: str, image_ids, names, ranges, counts, n_samples,
              meta: dict | None = None) -> None:
    """One calibration cache as ``.qcal``: tensors in name order (calibration.py:116)."""
    names = list(names)
    order = sorted(range(len(names)), key=lambda i: names[i])
    rng = np.asarray(ranges, dtype=np.float32).reshape(len(names), 2)[order]
    cnt = np.asarray(counts, dtype=np.int64).reshape(len(names), -1)[order]
    header = {
        "format": "qcal",
        "version": 1,
        "model_name": model_name,
        "size_class": size_class,
        "image_ids": [int(i) for i in image_ids],
        "tensors": [names[i] for i in order],
        "n_samples": [int(np.asarray(n_samples).reshape(-1)[i]) for i in order],
    }
    if meta:
        header["meta"] = meta
    write_container(path, header, [rng, cnt])


# ---------------------------------------------------------------- quantized model (.qtm8)
class _P:
    """One activation-parameter object: computed params are distinct objects, ops that
    adopt their input's params share the object (quantize.py:198-202) -- save_quantized
    records that sharing in act_sources."""

    def __init__(self, hist: str):
        self.hist = hist


def _plan(g, cfg):
    """Domains, activation-param objects and fp32 nodes exactly as quantize_model walks the
    graph (quantize.py:133-205), without any values."""
    from .ir import COMPUTE_KINDS, INPUT_TENSOR, consumers, data_inputs

    def narrowed(n):                                  # quantize.py:125-130
        cons = consumers(g, n.output)
        return cons[0].output if len(cons) == 1 and cons[0].kind == "relu" else n.output

    compute = [n for n in g.nodes if n.kind in COMPUTE_KINDS]
    fp32 = {compute[0].id, compute[-1].id} if cfg.mixed == "FirstLastFp32" else set()
    last = compute[-1].id
    act = {}
    domain = {INPUT_TENSOR: cfg.mixed == "Off"}
    if domain[INPUT_TENSOR]:
        act[INPUT_TENSOR] = _P(INPUT_TENSOR)
    int8_compute = []
    for n in g.nodes:
        ins = [domain[t] for t in data_inputs(n)]
        if n.kind in COMPUTE_KINDS:
            if n.id in fp32:
                if n.id == last:
                    domain[n.output] = False
                else:
                    act[n.output] = _P(narrowed(n))
                    domain[n.output] = True
                continue
            int8_compute.append(n)
            act[n.output] = _P(narrowed(n))
            domain[n.output] = True
        elif n.kind in ("add", "concat"):
            if all(ins):
                act[n.output] = _P(narrowed(n) if n.kind == "add" else n.output)
                domain[n.output] = True
            else:
                domain[n.output] = False
        else:
            src = data_inputs(n)[0]
            domain[n.output] = domain[src]
            if domain[src]:
                act[n.output] = act[src]
    return act, fp32, int8_compute


def _fuse(g, nodes_attrs):
    """fuse_conv_relu (intexec.py:369-398): compute -> sole-relu pairs merged."""
    from .ir import COMPUTE_KINDS, INPUT_TENSOR, consumers, data_inputs
    fuse = {}
    for n in g.nodes:
        if n.kind in COMPUTE_KINDS:
            cons = consumers(g, n.output)
            if len(cons) == 1 and cons[0].kind == "relu":
                fuse[n.id] = cons[0]
    drop = {r.id for r in fuse.values()}
    out = []
    for n in g.nodes:
        if n.id in drop:
            continue
        if n.id in fuse:
            out.append({"id": n.id, "kind": n.kind, "inputs": list(n.inputs), "output": fuse[n.id].output,
                        "attrs": {**dict(n.attrs), "fused_relu": True}})
        else:
            out.append({"id": n.id, "kind": n.kind, "inputs": list(n.inputs), "output": n.output,
                        "attrs": dict(n.attrs)})
    live = {INPUT_TENSOR} | {d["output"] for d in out} | \
        {t for d in out for t in (d["inputs"][:1] if d["kind"] in COMPUTE_KINDS else d["inputs"])}
    return out, live, bool(fuse)


def save_qtm8(path: str, ev, cfg, meta: dict | None = None) -> None:
    """The quantized model of `cfg` from the GPU evaluator's device state, written as the
    reference's .qtm8 (save_quantized, quantize.py:254-300): weight codes / params and
    int32 bias codes come from ptq_export_layer, activation params from the device
    parameter table, the container layout from write_container."""
    import ctypes as C

    from . import _lib
    from .config import CACHE_SIZES, Scheme, config_key

    g = ev.graph
    act, fp32, int8_compute = _plan(g, cfg)
    nodes = [{"id": n.id, "kind": n.kind, "inputs": list(n.inputs), "output": n.output, "attrs": dict(n.attrs)}
             for n in g.nodes]
    fused = False
    if cfg.fusion:
        f_nodes, live, any_fused = _fuse(g, None)
        if any_fused:
            nodes, fused = f_nodes, True
            act = {t: p for t, p in act.items() if t in live}
    # activation values: the device table of this (cache, scheme, clipping)
    schemes = [s.value for s in Scheme]
    scheme_v = cfg.scheme.value if hasattr(cfg.scheme, "value") else str(cfg.scheme)
    a_s, a_z = ev.act_params(CACHE_SIZES.index(cfg.cache), schemes.index(scheme_v),
                             ("Max", "KL").index(cfg.clipping))
    tid = ev.lowered.tensor_ids
    act_ids = sorted(act)
    shared, act_src, uniq = {}, [], []
    for t in act_ids:
        p = act[t]
        if id(p) in shared:
            act_src.append(shared[id(p)])
        else:
            shared[id(p)] = t
            act_src.append(t)
            uniq.append(t)
    act_scales = np.asarray([float(a_s[tid[act[t].hist]]) for t in uniq], dtype=np.float32)
    act_zps = np.asarray([int(a_z[tid[act[t].hist]]) for t in uniq], dtype=np.int32)
    # weights of the int8 layers
    cd = _lib.ConfigDesc(*config_key(cfg))
    wcodes, wparams, bcodes = {}, {}, {}
    node_index = {n.id: i for i, n in enumerate(g.nodes)}
    for n in int8_compute:
        w = np.asarray(g.weights[n.inputs[1]])
        cout = w.shape[0]
        codes = np.zeros(w.size, dtype=np.int8)
        sc = np.zeros(cout, dtype=np.float32)
        zp = np.zeros(cout, dtype=np.int32)
        bias = np.zeros(cout, dtype=np.int32)
        _lib.check(ev.lib.ptq_export_layer(ev._ctx, C.byref(cd), node_index[n.id], _lib.ptr(codes), _lib.ptr(sc),
                                           _lib.ptr(zp), _lib.ptr(bias)))
        wcodes[n.inputs[1]] = codes.reshape(w.shape)
        per_ch = cfg.granularity == "Channel"
        wparams[n.inputs[1]] = (sc if per_ch else sc[:1], zp if per_ch else zp[:1], 0 if per_ch else None)
        if len(n.inputs) > 2:
            bcodes[n.inputs[2]] = bias
    wq_ids, bias_ids = sorted(wcodes), sorted(bcodes)
    fp32_w = sorted(set(g.weights) - set(wcodes) - set(bcodes))
    buffers = [act_scales, act_zps]
    wp_meta = []
    for t in wq_ids:
        s, z, axis = wparams[t]
        buffers += [wcodes[t], s.astype(np.float32), z.astype(np.int32)]
        wp_meta.append({"id": t, "axis": axis})
    buffers += [bcodes[t] for t in bias_ids]
    buffers += [np.asarray(g.weights[t]) for t in fp32_w]
    header = {
        "format": "qtm8",
        "version": 1,
        "name": g.name,
        "input_shape": list(g.input_shape),
        "output_classes": g.output_classes,
        "nodes": nodes,
        "config": cfg.to_dict(),
        "fp32_nodes": sorted(fp32),
        "fused": fused,
        "act_tensors": act_ids,
        "act_sources": act_src,
        "act_unique": uniq,
        "weight_tensors": wp_meta,
        "bias_tensors": bias_ids,
        "fp32_weight_tensors": fp32_w,
    }
    if meta:
        header["meta"] = meta
    write_container(path, header, buffers)
