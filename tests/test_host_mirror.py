"""Host mirror (dataset / fixtures / config) vs the reference's own outputs."""
import hashlib

import numpy as np

from paper_2202_05048_b200 import config as C


def sha(a):
    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.tobytes() + str(a.dtype).encode() + str(a.shape).encode()).hexdigest()[:16]


def test_dataset_bit_identical(ds, golden):
    _, meta = golden
    assert sha(ds.images) == meta["dataset_seed0"]["images"]
    assert sha(ds.labels) == meta["dataset_seed0"]["labels"]


def test_fixtures_bit_identical(toys, golden):
    _, meta = golden
    for rec, g in toys.items():
        assert {k: sha(v) for k, v in g.weights.items()} == meta["fixtures"][rec]


def test_space_and_select_images(golden):
    _, meta = golden
    space = C.enumerate_space(C.GENERIC)
    assert len(space) == 96 and len(set(space)) == 96
    assert space[2] == C.QuantConfig("S1", C.Scheme.Asymmetric, "Max", "Channel", "Off")
    for sc in C.CACHE_SIZES:
        assert C.select_images(300, sc, 0).tolist() == meta["cache_ids"][f"lenet-ish/{sc}"]
    assert len(C.enumerate_space(C.INTEGER_ONLY)) == 12


def test_config_validation():
    import pytest
    with pytest.raises(ValueError):
        C.QuantConfig(clipping="percentile")
    with pytest.raises(ValueError):
        C.QuantConfig(cache="S4")
