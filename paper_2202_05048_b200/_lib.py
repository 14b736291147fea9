"""ctypes binding of include/ptq_b200.h (the reference-side FFI stub).

The reference is pure Python, so this module is exactly the binding a
ptqtune maintainer would add.  It loads the in-tree
``libptq_b200.so`` and fails loudly when it is missing: there is no CPU
fallback anywhere on the product path.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# PTQ_B200_LIB: an alternative build of the same library (kernel A/B experiments only)
LIB_PATH = os.environ.get("PTQ_B200_LIB") or os.path.join(HERE, "libptq_b200.so")

PTQ_NBINS = 2048
PTQ_NWINDOWS = 1921
PTQ_MAX_INPUTS = 8
KINDS = {"conv2d": 0, "depthwise_conv2d": 1, "pointwise_conv2d": 2, "fully_connected": 3,
         "relu": 4, "maxpool": 5, "avgpool": 6, "add": 7, "concat": 8, "softmax": 9}

EXPORTS = ("ptq_last_error", "ptq_version", "ptq_create", "ptq_destroy", "ptq_num_tensors",
           "ptq_calibrate", "ptq_kl_sweep", "ptq_set_clip_ranges", "ptq_prepare",
           "ptq_eval_configs", "ptq_probe_codes", "ptq_probe_act_params", "ptq_histogram_host",
           "ptq_export_layer", "ptq_percentile_ranges",
           "ptq_set_option", "ptq_last_stats", "ptq_calib_forward", "ptq_calib_histogram",
           "ptq_stream", "ptq_conv_timings", "ptq_probe_tensors", "ptq_probe_acc",
           "ptq_probe_output", "ptq_probe_f32", "ptq_minmax_host")


class NodeDesc(C.Structure):
    _fields_ = [("kind", C.c_int32), ("n_inputs", C.c_int32), ("inputs", C.c_int32 * PTQ_MAX_INPUTS),
                ("weight", C.c_int32), ("bias", C.c_int32), ("kernel", C.c_int32),
                ("stride", C.c_int32), ("pad", C.c_int32)]


class WeightDesc(C.Structure):
    _fields_ = [("data", C.POINTER(C.c_float)), ("shape", C.c_int64 * 4), ("ndim", C.c_int32)]


class GraphDesc(C.Structure):
    _fields_ = [("n_nodes", C.c_int32), ("nodes", C.POINTER(NodeDesc)), ("n_weights", C.c_int32),
                ("weights", C.POINTER(WeightDesc)), ("in_c", C.c_int32), ("in_h", C.c_int32),
                ("in_w", C.c_int32), ("n_classes", C.c_int32)]


class ConfigDesc(C.Structure):
    _fields_ = [("cache", C.c_int32), ("scheme", C.c_int32), ("clipping", C.c_int32),
                ("granularity", C.c_int32), ("mixed", C.c_int32), ("fusion", C.c_int32)]


class PtqError(RuntimeError):
    """Non-zero status from the C ABI (the evaluator's failure signal)."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"ptq_b200 error {code}: {msg}")
        self.code = code


_lib = None


def load() -> C.CDLL:
    """Load the CUDA library (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} missing: run `python -m paper_2202_05048_b200.build` "
                           "(the evaluator has no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    P, i32, i64 = C.c_void_p, C.c_int32, C.c_int64
    lib.ptq_last_error.restype = C.c_char_p
    lib.ptq_version.restype = C.c_int
    sig = {
        "ptq_create": [C.POINTER(P), C.c_int, C.POINTER(GraphDesc), P, P, i64, i64],
        "ptq_destroy": [P],
        "ptq_num_tensors": [P, C.POINTER(i32)],
        "ptq_calibrate": [P, i32, P, P, P, P, P],
        "ptq_kl_sweep": [P, i32, P, P, P],
        "ptq_set_clip_ranges": [P, i32, i32, P],
        "ptq_percentile_ranges": [P, i32, P, P, C.c_double, P],
        "ptq_prepare": [P],
        "ptq_eval_configs": [P, C.POINTER(ConfigDesc), i32, P],
        "ptq_probe_codes": [P, C.POINTER(ConfigDesc), i32, P, C.POINTER(i64)],
        "ptq_probe_act_params": [P, i32, i32, i32, P, P],
        "ptq_histogram_host": [P, P, i64, C.c_float, C.c_float, P],
        "ptq_export_layer": [P, C.POINTER(ConfigDesc), i32, P, P, P, P],
        "ptq_set_option": [P, C.c_char_p, i64],
        "ptq_last_stats": [P, C.POINTER(i64), C.POINTER(C.c_double), C.POINTER(C.c_double),
                           C.POINTER(i64), C.POINTER(i64)],
        "ptq_calib_forward": [P, i32, P, P, P],
        "ptq_calib_histogram": [P, P, P],
        "ptq_stream": [P, C.POINTER(P)],
        "ptq_conv_timings": [P, P, i64, C.POINTER(i64)],
        "ptq_probe_tensors": [P, C.POINTER(ConfigDesc), i32, P, i32, P, P, P],
        "ptq_probe_acc": [P, C.POINTER(ConfigDesc), i32, i32, P, P],
        "ptq_probe_output": [P, C.POINTER(ConfigDesc), i32, P, P],
        "ptq_probe_f32": [P, C.POINTER(ConfigDesc), i32, i32, P, P],
        "ptq_minmax_host": [P, P, i32, i64, P],
    }
    for name, args in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = C.c_int
    _lib = lib
    return lib


def check(rc: int) -> None:
    if rc != 0:
        raise PtqError(rc, load().ptq_last_error().decode(errors="replace"))


def ptr(a: np.ndarray):
    return C.c_void_p(a.ctypes.data) if a is not None else None
