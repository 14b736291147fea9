"""B200-native evaluator for Quantune-style PTQ configuration search.

The public entry point is :func:`make_accuracy_evaluator`, a drop-in for the
reference's ``ptqtune.tuner.make_accuracy_evaluator``
(/root/reference/pkg/src/ptqtune/tuner.py:434-444).
"""

from .config import (CACHE_SIZES, CLIPPINGS, GENERIC, GRANULARITIES, INTEGER_ONLY,
                     MIXED_MODES, QuantConfig, Scheme, TargetProfile, enumerate_space,
                     select_images)
from .dataset import Dataset, make_dataset
from .fixtures import build_model, generate_fixture
from .ir import Graph, GraphError, Node


def make_accuracy_evaluator(*args, **kwargs):
    from .evaluator import make_accuracy_evaluator as _impl
    return _impl(*args, **kwargs)
