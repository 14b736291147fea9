"""Host-side model IR consumed by the GPU evaluator.

Mirrors the reference's ``Graph``/``Node`` contract
(/root/reference/pkg/src/ptqtune/ir.py:29-92) so a reference graph object can
be handed to :func:`paper_2202_05048_b200.make_accuracy_evaluator` unchanged
(duck-typed: ``name``, ``nodes``, ``weights``, ``input_shape``,
``output_classes``).  Shape propagation follows ir.py:95-171 (conv output
``(h + 2p - k)//s + 1``; pooling has no padding, ir.py:150).

This module is host plumbing, not the hot path: the lowering in
:mod:`paper_2202_05048_b200.lowering` turns a Graph into the flat POD arrays
that cross the C-ABI.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Any

import numpy as np

INPUT_TENSOR = "input"
CONV_KINDS = ("conv2d", "depthwise_conv2d", "pointwise_conv2d")
COMPUTE_KINDS = CONV_KINDS + ("fully_connected",)
NODE_KINDS = COMPUTE_KINDS + ("relu", "maxpool", "avgpool", "add", "concat", "softmax")


class GraphError(ValueError):
    """Malformed graph (same role as reference ir.py:36-37)."""


@dataclass
class Node:
    id: str
    kind: str
    inputs: list[str]
    output: str
    attrs: dict[str, Any] = field(default_factory=dict)

    @property
    def weight_id(self) -> str | None:
        return self.inputs[1] if self.kind in COMPUTE_KINDS and len(self.inputs) > 1 else None

    @property
    def bias_id(self) -> str | None:
        return self.inputs[2] if self.kind in COMPUTE_KINDS and len(self.inputs) > 2 else None

    @property
    def data_inputs(self) -> list[str]:
        return list(self.inputs[:1]) if self.kind in COMPUTE_KINDS else list(self.inputs)


@dataclass
class Graph:
    name: str
    nodes: list[Node]
    weights: dict[str, np.ndarray]
    input_shape: tuple[int, int, int]
    output_classes: int

    def consumers(self, tensor_id: str) -> list[Node]:
        return consumers(self, tensor_id)

    def output_tensor(self) -> str:
        return output_tensor(self)

    def compute_nodes(self) -> list[Node]:
        return [n for n in self.nodes if n.kind in COMPUTE_KINDS]


# free functions work on any duck-typed graph (reference Graph objects too)

def data_inputs(n) -> list[str]:
    return list(n.inputs[:1]) if n.kind in COMPUTE_KINDS else list(n.inputs)


def consumers(g, tensor_id: str) -> list:
    return [n for n in g.nodes if tensor_id in data_inputs(n)]


def output_tensor(g) -> str:
    used = {t for n in g.nodes for t in data_inputs(n)}
    outs = [n.output for n in g.nodes if n.output not in used]
    if len(outs) != 1:
        raise GraphError(f"graph must have exactly one output, found {outs}")
    return outs[0]


def conv_out_hw(h: int, w: int, k: int, stride: int, pad: int) -> tuple[int, int]:
    oh, ow = (h + 2 * pad - k) // stride + 1, (w + 2 * pad - k) // stride + 1
    if oh < 1 or ow < 1:
        raise GraphError(f"kernel {k} stride {stride} pad {pad} does not fit {h}x{w}")
    return oh, ow


def tensor_shapes(g) -> dict[str, tuple[int, ...]]:
    """Per-tensor shapes without the batch dim (CHW, or (F,) after fc)."""
    shapes: dict[str, tuple[int, ...]] = {INPUT_TENSOR: tuple(int(v) for v in g.input_shape)}
    for n in g.nodes:
        ins = data_inputs(n)
        for t in ins:
            if t not in shapes:
                raise GraphError(f"node {n.id}: input {t!r} used before definition")
        x = shapes[ins[0]]
        if n.kind in CONV_KINDS:
            w = g.weights[n.inputs[1]]
            o, ci, kh, kw = w.shape
            if kh != kw:
                raise GraphError(f"node {n.id}: only square kernels are supported")
            if n.kind == "depthwise_conv2d":
                if ci != 1 or o != x[0]:
                    raise GraphError(f"node {n.id}: depthwise weight must be (C,1,k,k)")
            elif ci != x[0]:
                raise GraphError(f"node {n.id}: weight expects {ci} channels, input has {x[0]}")
            s, p = int(n.attrs.get("stride", 1)), int(n.attrs.get("padding", 0))
            shapes[n.output] = (o,) + conv_out_hw(x[1], x[2], kh, s, p)
        elif n.kind == "fully_connected":
            w = g.weights[n.inputs[1]]
            if w.shape[1] != int(np.prod(x)):
                raise GraphError(f"node {n.id}: fc expects {w.shape[1]} inputs, got {x}")
            shapes[n.output] = (w.shape[0],)
        elif n.kind in ("maxpool", "avgpool"):
            k = int(n.attrs["kernel"])
            s = int(n.attrs.get("stride", k))
            shapes[n.output] = (x[0],) + conv_out_hw(x[1], x[2], k, s, 0)
        elif n.kind in ("relu", "softmax"):
            shapes[n.output] = x
        elif n.kind == "add":
            if shapes[ins[1]] != x:
                raise GraphError(f"node {n.id}: add shape mismatch")
            shapes[n.output] = x
        elif n.kind == "concat":
            parts = [shapes[t] for t in ins]
            if len({p[1:] for p in parts}) != 1:
                raise GraphError(f"node {n.id}: concat spatial mismatch")
            shapes[n.output] = (sum(p[0] for p in parts),) + parts[0][1:]
        else:
            raise GraphError(f"node {n.id}: unknown kind {n.kind!r}")
    return shapes


def validate(g) -> None:
    ids = [n.id for n in g.nodes]
    outs = [n.output for n in g.nodes]
    if len(set(ids)) != len(ids) or len(set(outs)) != len(outs):
        raise GraphError("duplicate node ids or output tensors")
    for n in g.nodes:
        if n.kind not in NODE_KINDS:
            raise GraphError(f"node {n.id}: unknown kind {n.kind!r}")
        if n.kind in COMPUTE_KINDS:
            for t in n.inputs[1:]:
                if t not in g.weights:
                    raise GraphError(f"node {n.id}: {t!r} is not a weight tensor")
    for wid, w in g.weights.items():
        if np.asarray(w).dtype != np.float32:
            raise GraphError(f"weight {wid!r} must be float32")
    tensor_shapes(g)
    output_tensor(g)
