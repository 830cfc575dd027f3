"""Access to the reference implementation (TEST/BASELINE INFRASTRUCTURE ONLY).

* ``load_ref_core()`` loads the reference's own compiled core from
  oracle/_ref/ (built by ``make -C oracle ref`` from the read-only sources;
  the .so travels to the GPU box, the sources do not).
* ``import_reference()`` makes the full reference package importable in THIS
  container (``/root/reference/pkg/src``) with that compiled core injected as
  ``flashann._kernels._core``; it returns None where /root/reference is absent
  (the GPU box), so nothing on the box depends on it.
"""

from __future__ import annotations

import importlib.machinery
import importlib.util
import sys
import sysconfig
from pathlib import Path

HERE = Path(__file__).resolve().parent
REF_SRC = Path("/root/reference/pkg/src")
REF_SO = HERE / "_ref" / ("_core" + sysconfig.get_config_var("EXT_SUFFIX"))
SCAN_SO = HERE / "_ref" / "libscanbench.so"

_core = None


def load_ref_core():
    """The reference compiled core module, or None when it was not built."""
    global _core
    if _core is None:
        if not REF_SO.exists():
            return None
        loader = importlib.machinery.ExtensionFileLoader("_core", str(REF_SO))
        spec = importlib.util.spec_from_file_location("_core", str(REF_SO), loader=loader)
        mod = importlib.util.module_from_spec(spec)
        loader.exec_module(mod)
        _core = mod
    return _core


def import_reference():
    """The reference `flashann` package backed by its compiled core, or None."""
    if not REF_SRC.exists():
        return None
    core = load_ref_core()
    if core is None:
        return None
    if str(REF_SRC) not in sys.path:
        sys.path.insert(0, str(REF_SRC))
    sys.modules.setdefault("flashann._kernels._core", core)
    import flashann  # noqa: F401
    import flashann.core

    assert flashann.core.HAVE_EXT, "reference compiled core not injected"
    return flashann
