"""CPU: the C-ABI library and the core-module contract (no compute calls)."""

import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


@pytest.fixture(scope="module")
def lib():
    from paper_2502_18113_b200 import _build

    path = _build.build()
    return ctypes.CDLL(str(path))


def declared_symbols():
    names = set()
    for h in (ROOT / "include").glob("*.h"):
        text = h.read_text()
        names |= set(re.findall(r"^\s*(?:const\s+)?[\w\s\*]+?\b(fa_\w+)\s*\(", text, re.M))
    return sorted(names)


def test_header_declares_entry_points():
    names = declared_symbols()
    assert "fa_build_graph_host" in names and "fa_scan_select_dev" in names
    assert len(names) >= 20


def test_library_exports_every_declared_symbol(lib):
    missing = [n for n in declared_symbols() if not hasattr(lib, n)]
    assert missing == []


def test_ctypes_binding_covers_header():
    from paper_2502_18113_b200 import _lib

    assert sorted(_lib.EXPORTED) == declared_symbols()


def test_error_string_and_version(lib):
    lib.fa_last_error.restype = ctypes.c_char_p
    assert lib.fa_version() == 1
    assert isinstance(lib.fa_last_error(), bytes)


def test_core_module_contract():
    from paper_2502_18113_b200 import sm100

    for name in ("CORE_NAME", "available_kernels", "build_graph", "search_batch",
                 "greedy_search_layer", "select_neighbors", "flash_batch_distance",
                 "flash_batch_distance_many", "flash_batch_blocks", "flash_sdt_distance",
                 "flash_encode_adt", "quantize_distance", "l2sq_f32"):
        assert hasattr(sm100, name), name
    # the reference's kernel registry names (core.py:28), in id order, so
    # core.resolve_kernel needs no patch
    assert sm100.available_kernels() == ("scalar", "vector128", "vector256", "vector512")
    assert sm100.CORE_NAME == "sm100"


def test_no_cpu_fallback_without_device():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a device is present")
    import numpy as np

    from paper_2502_18113_b200 import errors, sm100

    with pytest.raises(errors.DeviceError):
        sm100.quantize_distance(np.zeros(3), 0.0, 1.0)
    with pytest.raises(ValueError):  # PQ (kind 1) is not served by this core
        sm100.build_graph(1, {}, np.zeros(1, np.int32), None, None, None, 8, 2)
    with pytest.raises(errors.DeviceError):  # the exact kind is, on a device only
        sm100.build_graph(0, {"vecs": np.zeros((1, 4), np.float32), "dim": 4},
                          np.zeros(1, np.int32), np.zeros((1, 36), np.uint8),
                          np.zeros(1, np.int64), np.zeros((0, 36), np.uint8), 8, 2)


def test_product_never_imports_oracle():
    pkg = ROOT / "paper_2502_18113_b200"
    for f in pkg.rglob("*.py"):
        text = f.read_text()
        assert not re.search(r"^\s*(from|import)\s+oracle", text, re.M), f


def test_device_limits_named_up_front():
    """Capacities of the sm_100a build raise ConfigError naming the limit
    before any device work (R <= 63, C <= 2048)."""
    from paper_2502_18113_b200 import errors, sm100

    sm100.check_limits(1000, 2048, 63, 128)
    for args in ((1000, 200, 64, 16), (1000, 4096, 32, 16), (1000, 200, 32, 129),
                 (1 << 31, 200, 32, 16)):
        with pytest.raises(errors.ConfigError):
            sm100.check_limits(*args)
