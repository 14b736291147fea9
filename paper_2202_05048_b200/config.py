"""Configuration-space types at the evaluator boundary.

Mirrors the reference's config vocabulary so host callers (search
strategies, CLI) keep working unchanged:

* ``Scheme`` — schemes.py:34-38 (four schemes);
* ``QuantConfig`` — quantize.py:54-84 (frozen, validated, hashable);
* ``TargetProfile`` / ``enumerate_space`` — tuner.py:49-81 (96 Generic
  configs in cache x scheme x clipping x granularity x mixed order);
* ``select_images`` — calibration.py:44-54 (numpy ``default_rng(seed)``
  draw without replacement, sorted), kept on the host for RNG parity.

The host packs a ``QuantConfig`` into the ``ptq_config`` POD of
include/ptq_b200.h with :func:`pack_config`.
"""

from __future__ import annotations

from dataclasses import dataclass
from enum import Enum
from itertools import product

import numpy as np

N_BINS = 2048
SIZE_CLASSES = {"S1": 1, "S2": 32, "S3": 256}
CACHE_SIZES = ("S1", "S2", "S3")
CLIPPINGS = ("Max", "KL")
GRANULARITIES = ("Tensor", "Channel")
MIXED_MODES = ("Off", "FirstLastFp32")
QMIN, QMAX = -128, 127
INT32_MIN, INT32_MAX = -(2 ** 31), 2 ** 31 - 1


class Scheme(str, Enum):
    Asymmetric = "Asymmetric"
    Symmetric = "Symmetric"
    SymmetricUint8 = "SymmetricUint8"
    SymmetricPower2 = "SymmetricPower2"


SCHEME_IDS = {Scheme.Asymmetric: 0, Scheme.Symmetric: 1,
              Scheme.SymmetricUint8: 2, Scheme.SymmetricPower2: 3}


@dataclass(frozen=True)
class QuantConfig:
    cache: str = "S3"
    scheme: Scheme = Scheme.Asymmetric
    clipping: str = "Max"
    granularity: str = "Tensor"
    mixed: str = "Off"
    fusion: bool = False

    def __post_init__(self):
        if self.cache not in CACHE_SIZES:
            raise ValueError(f"bad cache size class {self.cache!r}")
        if not isinstance(self.scheme, Scheme):
            object.__setattr__(self, "scheme", Scheme(self.scheme))
        if self.clipping not in CLIPPINGS:
            raise ValueError(f"bad clipping {self.clipping!r}")
        if self.granularity not in GRANULARITIES:
            raise ValueError(f"bad granularity {self.granularity!r}")
        if self.mixed not in MIXED_MODES:
            raise ValueError(f"bad mixed mode {self.mixed!r}")

    def to_dict(self) -> dict:
        return {"cache": self.cache, "scheme": self.scheme.value, "clipping": self.clipping,
                "granularity": self.granularity, "mixed": self.mixed, "fusion": self.fusion}

    @classmethod
    def from_dict(cls, d: dict) -> "QuantConfig":
        return cls(cache=d["cache"], scheme=Scheme(d["scheme"]), clipping=d["clipping"],
                   granularity=d["granularity"], mixed=d["mixed"],
                   fusion=bool(d.get("fusion", False)))


@dataclass(frozen=True)
class TargetProfile:
    name: str

    def contains(self, cfg) -> bool:
        if self.name == "Generic":
            return not cfg.fusion
        if self.name == "IntegerOnly":
            return (_scheme_of(cfg) == Scheme.SymmetricPower2 and cfg.granularity == "Tensor"
                    and cfg.mixed == "Off")
        raise ValueError(f"unknown profile {self.name!r}")


GENERIC = TargetProfile("Generic")
INTEGER_ONLY = TargetProfile("IntegerOnly")


def _scheme_of(cfg) -> Scheme:
    s = cfg.scheme
    return s if isinstance(s, Scheme) else Scheme(getattr(s, "value", s))


def enumerate_space(profile: TargetProfile = GENERIC) -> list[QuantConfig]:
    if profile.name == "Generic":
        return [QuantConfig(c, s, cl, g, m)
                for c, s, cl, g, m in product(CACHE_SIZES, tuple(Scheme), CLIPPINGS,
                                              GRANULARITIES, MIXED_MODES)]
    if profile.name == "IntegerOnly":
        return [QuantConfig(c, Scheme.SymmetricPower2, cl, "Tensor", "Off", f)
                for c, cl, f in product(CACHE_SIZES, CLIPPINGS, (False, True))]
    raise ValueError(f"unknown profile {profile.name!r}")


def select_images(n_pool: int, size_class: str, seed: int) -> np.ndarray:
    if size_class not in SIZE_CLASSES:
        raise ValueError(f"unknown size class {size_class!r}")
    n = SIZE_CLASSES[size_class]
    if n_pool < n:
        raise ValueError(f"pool of {n_pool} images cannot supply {size_class} ({n})")
    return np.sort(np.random.default_rng(seed).choice(n_pool, size=n, replace=False))


def config_key(cfg) -> tuple[int, int, int, int, int, int]:
    """(cache, scheme, clipping, granularity, mixed, fusion) as small ints."""
    return (CACHE_SIZES.index(cfg.cache), SCHEME_IDS[_scheme_of(cfg)],
            CLIPPINGS.index(cfg.clipping), GRANULARITIES.index(cfg.granularity),
            MIXED_MODES.index(cfg.mixed), int(bool(cfg.fusion)))
