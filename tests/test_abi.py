"""CPU checks of the C-ABI boundary: the library builds/loads and exports every
symbol include/ptq_b200.h declares (no compute without a GPU)."""
import ctypes
import os
import re

from paper_2202_05048_b200 import _lib
from paper_2202_05048_b200.lowering import LoweredGraph

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "ptq_b200.h")).read()
    return sorted(set(re.findall(r"\b(ptq_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_header_symbols():
    lib = _lib.load()
    syms = header_symbols()
    assert len(syms) >= 10
    for s in syms:
        assert hasattr(lib, s), s
    assert set(_lib.EXPORTS) == set(syms)
    assert lib.ptq_version() == 1


def test_no_device_fails_loudly():
    lib = _lib.load()
    import torch
    if torch.cuda.is_available():
        return
    ctx = ctypes.c_void_p()
    from paper_2202_05048_b200.fixtures import generate_fixture
    lg = LoweredGraph(generate_fixture("lenet-ish", 1))
    import numpy as np
    imgs = np.zeros((4, 3, 32, 32), np.float32)
    lab = np.zeros(2, np.int64)
    rc = lib.ptq_create(ctypes.byref(ctx), 0, ctypes.byref(lg.desc), _lib.ptr(imgs), _lib.ptr(lab), 4, 2)
    assert rc != 0 and lib.ptq_last_error()


def test_lowering_tensor_order(toys):
    g = toys["resnet-toy"]
    lg = LoweredGraph(g)
    assert lg.tensor_names[0] == "input"
    assert lg.tensor_names[1:] == [n.output for n in g.nodes]
    d = lg.desc
    assert d.n_nodes == len(g.nodes) and d.in_c == 3 and d.n_classes == 10
    add = [i for i, n in enumerate(g.nodes) if n.kind == "add"][0]
    assert d.nodes[add].n_inputs == 2
