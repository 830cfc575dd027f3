"""pytest plugin (TEST INFRASTRUCTURE): serve the reference's core-module
contract with the sm100 core.

Loaded with ``-p sm100_inject`` before any reference module is imported: the
sm100 module is registered as ``flashann._kernels._core``, which is where the
reference looks for its compiled core (flashann/core.py:19-25).  From then on
``core.HAVE_EXT`` is True, ``core.active_core()`` is sm100, and every
reference test that parametrises over ``CORES`` (tests/test_hnsw.py:13-15) or
uses ``EXT`` (tests/test_flash.py:23) exercises the GPU core.
"""

import os
import sys

_repo = os.environ.get("FLASHANN_B200_REPO")
if _repo and _repo not in sys.path:
    sys.path.insert(0, _repo)

from paper_2502_18113_b200 import sm100  # noqa: E402

sys.modules["flashann._kernels._core"] = sm100
