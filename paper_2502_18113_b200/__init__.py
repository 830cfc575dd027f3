"""B200-native Flash HNSW construction (arXiv 2502.18113 hot path).

The compute core (`sm100`) is a drop-in for the reference package's core-module
contract (flashann/core.py:16-26); the host modules mirror the reference API
(flashann/__init__.py:11-78) for training the coder, encoding, building and
searching.  All compute runs in hand-written sm_100a kernels behind the C-ABI
of include/flashann_b200.h; there is no CPU fallback.
"""

__version__ = "0.1.0"

from . import errors, layout  # noqa: F401
from .builder import BuildResult, StrategyParams, build  # noqa: F401
from .dataset import GroundTruth, VectorDataset, baseline_config, brute_force_knn  # noqa: F401
from .errors import ConfigError, DeviceError, FlashAnnError, FormatError  # noqa: F401
from .evaluation import SearchParams, recall_at_k, search, search_batch  # noqa: F401
from .flash import (FlashModel, FlashProvider, encode_and_adt, flash_train,  # noqa: F401
                    sdt_distance)
from .graph import BuildParams, GraphIndex, assign_layers, check_invariants  # noqa: F401
from .pca import PCAModel, pca_train  # noqa: F401
from .serialize import load_index, save_index  # noqa: F401

HAVE_EXT = True


def core_name() -> str:
    return "sm100"
