"""Integer-only executor on the GPU path.

Mirrors the reference's strict integer program (ptqtune/intexec.py): ``OpTrace``
(:47-64), ``IntegerOnlyError`` (:43), ``_exact_log2`` (:88-92),
``check_integer_only`` (:132-145) and ``run_integer_only`` (:354-359), served from
the GPU evaluator's device state (codes of the graph output over its eval images).

What the device executes: every shift of the integer program is a requantization
by m = 2^-s with s an integer (all scales are powers of two, checked below).
The conv epilogue is the exact fixed-point requant of k_conv_tc (LayerRt::fx):
code = hi32(acc * M + B) >> (S - 32), integer multiply-add and shift only; for
m = 2^-s the solved M is a power of two and B the rounding constant, i.e. the
reference's (acc + 2^(s-1)) >> s.  (Layers whose constants cannot be solved fall back
to floor(acc * m + 0.5) in fp64, also exact for m = 2^-s and |acc| < 2^31.)  The
residual add goes through the per-config add table, whose entries
xs*2^(ka-ko) + ys*2^(kb-ko) are exact in fp64 and equal the reference's
(xs << (ka-kmin)) + (ys << (kb-kmin)) shifted by ko-kmin.  The codes
are therefore bit-identical to run_integer_only (tests/test_intonly.py checks
them against the reference's own output).  The ``OpTrace`` returned here is the
trace of the integer PROGRAM (the reference's categories, derived from the executed
graph); it is not a record of sm_100a instructions.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .config import CACHE_SIZES, Scheme, config_key
from .ir import COMPUTE_KINDS, output_tensor

FLOAT_CATS = ("float_mul", "float_add", "float_kernel")


class IntegerOnlyError(ValueError):
    """A quantized model cannot run on the strict integer path (intexec.py:43)."""


@dataclass
class OpTrace:
    """(node id, op category) events in program order (intexec.py:47-64)."""
    events: list = field(default_factory=list)

    def add(self, node_id: str, *categories: str) -> None:
        for c in categories:
            self.events.append((node_id, c))

    def count(self, *categories: str) -> int:
        return sum(1 for _, c in self.events if c in categories)

    def float_ops(self) -> int:
        return self.count(*FLOAT_CATS)

    def to_csv(self) -> str:
        return "\n".join(["node,category"] + [f"{n},{c}" for n, c in self.events]) + "\n"


def exact_log2(scale: float) -> int:
    """intexec.py:88-92 (ceil_log2 via frexp, schemes.py:67-72)."""
    m, e = math.frexp(float(scale))
    k = e - 1 if m == 0.5 else e
    if 2.0 ** k != scale:
        raise IntegerOnlyError(f"scale {scale} is not a power of two")
    return k


def check_integer_only(graph, cfg) -> None:
    """intexec.py:132-145: SymmetricPower2 / Tensor / Off and power-of-two avgpool areas."""
    scheme = cfg.scheme.value if hasattr(cfg.scheme, "value") else str(cfg.scheme)
    if scheme != Scheme.SymmetricPower2.value or cfg.granularity != "Tensor" or cfg.mixed != "Off":
        raise IntegerOnlyError(
            "integer-only execution requires scheme=SymmetricPower2, "
            f"granularity=Tensor, mixed=Off; got {scheme}/{cfg.granularity}/{cfg.mixed}")
    for n in graph.nodes:
        if n.kind == "avgpool":
            area = int(n.attrs["kernel"]) ** 2
            if area & (area - 1):
                raise IntegerOnlyError(f"avgpool {n.id}: area {area} not a power of two")


def _executed_nodes(graph, cfg):
    """The node list as executed: fuse_conv_relu (intexec.py:369-398) when cfg.fusion."""
    if not cfg.fusion:
        return [(n.id, n.kind, list(n.inputs), n.output, dict(n.attrs)) for n in graph.nodes]
    from .artifacts import _fuse
    nodes, _, _ = _fuse(graph, None)
    return [(d["id"], d["kind"], d["inputs"], d["output"], d["attrs"]) for d in nodes]


def integer_program_trace(graph, cfg, trace: OpTrace) -> None:
    """The op categories of the integer program, in the order _execute emits them
    (intexec.py:166-292 with integer_only=True; the input quantization is host-side
    and untraced, :158-160)."""
    for nid, kind, inputs, _out, attrs in _executed_nodes(graph, cfg):
        if kind in COMPUTE_KINDS:
            trace.add(nid, "int_mul", "int_add")
            if len(inputs) > 2:
                trace.add(nid, "int_add")
            trace.add(nid, "int_add", "shift", "clamp")
            if attrs.get("fused_relu"):
                trace.add(nid, "clamp")
        elif kind == "relu":
            trace.add(nid, "clamp")
        elif kind == "avgpool":
            trace.add(nid, "int_add", "shift", "clamp")
        elif kind == "add":
            trace.add(nid, "int_add", "shift", "int_add", "shift", "int_add", "shift", "clamp")
        elif kind == "concat":
            for _ in inputs:
                trace.add(nid, "int_add", "shift", "clamp")


def _check_scales(ev, cfg) -> None:
    """Every activation and weight scale of the config must be an exact power of two
    (the _exact_log2 calls of intexec.py:116-121, :196, :235, :257-259)."""
    from .artifacts import _plan
    schemes = [s.value for s in Scheme]
    scheme_v = cfg.scheme.value if hasattr(cfg.scheme, "value") else str(cfg.scheme)
    a_s, _ = ev.act_params(CACHE_SIZES.index(cfg.cache), schemes.index(scheme_v),
                           ("Max", "KL").index(cfg.clipping))
    act, _, int8_compute = _plan(ev.graph, cfg)
    tid = ev.lowered.tensor_ids
    for t, p in act.items():
        exact_log2(float(a_s[tid[p.hist]]))
    cd = _lib.ConfigDesc(*config_key(cfg))
    node_index = {n.id: i for i, n in enumerate(ev.graph.nodes)}
    for n in int8_compute:
        w = np.asarray(ev.graph.weights[n.inputs[1]])
        codes = np.zeros(w.size, dtype=np.int8)
        sc = np.zeros(w.shape[0], dtype=np.float32)
        zp = np.zeros(w.shape[0], dtype=np.int32)
        bias = np.zeros(w.shape[0], dtype=np.int32)
        with ev._lock:
            _lib.check(ev.lib.ptq_export_layer(ev._ctx, C.byref(cd), node_index[n.id], _lib.ptr(codes),
                                               _lib.ptr(sc), _lib.ptr(zp), _lib.ptr(bias)))
        exact_log2(float(sc[0]))


def run_quantized_codes(ev, cfg) -> np.ndarray:
    """int8 output codes of the eval set for ``cfg`` (run_quantized(..., return_codes=True),
    intexec.py:337-351), read from the device."""
    ev._check_cfg(cfg)
    t = output_tensor(ev.graph)
    if cfg.mixed != "Off":
        raise ValueError("graph output is fp32; no codes to return")
    out = ev.probe_codes(cfg, t)
    return out.reshape(ev.n_eval_local, -1)


def run_integer_only(ev, cfg, trace: OpTrace | None = None) -> np.ndarray:
    """intexec.py:354-359 on the GPU evaluator: the strict integer program's int8 output
    codes over the evaluator's eval images.  Raises IntegerOnlyError exactly where the
    reference does."""
    check_integer_only(ev.graph, cfg)
    _check_scales(ev, cfg)
    if trace is not None:
        integer_program_trace(ev.graph, cfg, trace)
    return run_quantized_codes(ev, cfg)
