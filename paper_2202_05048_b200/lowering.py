"""Lower a (reference-compatible) Graph to the ptq_graph_desc POD of the C ABI.

Tensor ids: 0 = graph input, i+1 = output of node i -- the same order in
which the reference's calibration observer first sees tensors
(/root/reference/pkg/src/ptqtune/calibration.py:67-76, fp32.py:81-113), so
histogram index == tensor id on both sides.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .ir import INPUT_TENSOR, GraphError, data_inputs


class LoweredGraph:
    """Owns the numpy buffers the descriptor points into."""

    def __init__(self, g):
        self.graph = g
        self.tensor_ids = {INPUT_TENSOR: 0}
        for i, n in enumerate(g.nodes):
            if n.output in self.tensor_ids:
                raise GraphError(f"duplicate tensor {n.output!r}")
            self.tensor_ids[n.output] = i + 1
        self.tensor_names = [None] * (len(g.nodes) + 1)
        for k, v in self.tensor_ids.items():
            self.tensor_names[v] = k
        self._w_arrays: list[np.ndarray] = []
        w_index: dict[str, int] = {}

        def widx(name):
            if name is None:
                return -1
            if name not in w_index:
                arr = np.ascontiguousarray(np.asarray(g.weights[name], dtype=np.float32))
                w_index[name] = len(self._w_arrays)
                self._w_arrays.append(arr)
            return w_index[name]

        nodes = (_lib.NodeDesc * len(g.nodes))()
        for i, n in enumerate(g.nodes):
            if n.kind not in _lib.KINDS:
                raise GraphError(f"node {n.id}: unsupported kind {n.kind!r}")
            ins = data_inputs(n)
            if len(ins) > _lib.PTQ_MAX_INPUTS:
                raise GraphError(f"node {n.id}: too many inputs")
            d = nodes[i]
            d.kind = _lib.KINDS[n.kind]
            d.n_inputs = len(ins)
            for j, t in enumerate(ins):
                if t not in self.tensor_ids:
                    raise GraphError(f"node {n.id}: unknown input {t!r}")
                d.inputs[j] = self.tensor_ids[t]
            compute = n.kind in ("conv2d", "depthwise_conv2d", "pointwise_conv2d", "fully_connected")
            d.weight = widx(n.inputs[1]) if compute else -1
            d.bias = widx(n.inputs[2]) if compute and len(n.inputs) > 2 else -1
            if n.kind in ("maxpool", "avgpool"):
                k = int(n.attrs["kernel"])
                d.kernel, d.stride, d.pad = k, int(n.attrs.get("stride", k)), 0
            else:
                d.kernel = 0
                d.stride = int(n.attrs.get("stride", 1))
                d.pad = int(n.attrs.get("padding", 0))
        weights = (_lib.WeightDesc * max(1, len(self._w_arrays)))()
        for i, a in enumerate(self._w_arrays):
            weights[i].data = a.ctypes.data_as(C.POINTER(C.c_float))
            for j, s in enumerate(a.shape):
                weights[i].shape[j] = s
            weights[i].ndim = a.ndim
        self._nodes, self._weights = nodes, weights
        c, h, w = (int(v) for v in g.input_shape)
        self.desc = _lib.GraphDesc(len(g.nodes), nodes, len(self._w_arrays), weights, c, h, w,
                                   int(g.output_classes))

    @property
    def n_tensors(self) -> int:
        return len(self.tensor_names)
