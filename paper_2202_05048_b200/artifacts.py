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
