"""B200-native Flash HNSW construction (arXiv 2502.18113 hot path).

The compute core (`sm100`) is a drop-in for the reference package's core-module
contract (flashann/core.py:16-26); the host modules mirror the reference API
for training the coder, encoding, building and searching.  All compute runs
in hand-written sm_100a kernels behind the C-ABI of include/flashann_b200.h.
"""

__version__ = "0.1.0"

from . import errors, layout  # noqa: F401
from .errors import ConfigError, DeviceError, FlashAnnError, FormatError  # noqa: F401
