"""ctypes binding of the C-ABI in include/flashann_b200.h.

The CUDA core is the only compute path: if the shared library is missing or
no CUDA device is visible, every entry point raises DeviceError.  There is
no CPU fallback.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

from .errors import DeviceError

# FLASHANN_B200_LIB: an alternative build of the core (A/B experiments)
LIB_PATH = Path(os.environ.get("FLASHANN_B200_LIB") or
                Path(__file__).resolve().parent / "lib" / "libflashann_b200.so")

FA_OK, FA_EINVAL, FA_ENOMEM, FA_ECUDA, FA_EOVERFLOW, FA_EEMPTY = 0, -1, -2, -3, -4, -5
FA_DTYPE_F32, FA_DTYPE_BF16 = 0, 1

vp = C.c_void_p
i32 = C.c_int32
i64 = C.c_int64
f64 = C.c_double


class IndexDesc(C.Structure):
    _fields_ = [
        ("n", i64), ("m", C.c_int), ("R", C.c_int), ("dim", C.c_int), ("dproj", C.c_int),
        ("dmax", C.c_int), ("dist_min", f64), ("delta", f64),
        ("vecs", vp), ("proj", vp), ("cent", vp), ("dims", vp), ("offs", vp), ("sdt", vp),
        ("levels", vp), ("uoff", vp), ("n_upper_rows", i64),
    ]


class BuildOpts(C.Structure):
    _fields_ = [("C", C.c_int), ("batch_max", C.c_int), ("batch_frac", f64),
                ("seq_prefix", C.c_int), ("hash_log2", C.c_int), ("profile", C.c_int),
                ("tie", C.c_int), ("expand", C.c_int), ("point_stats", vp),
                ("batch_min", C.c_int), ("start", i64), ("end", i64)]


class BuildResult(C.Structure):
    _fields_ = [("entry_point", i64), ("max_layer", i32), ("n_batches", i32),
                ("dist_comps", i64), ("sym_comps", i64), ("kernel_calls", i64),
                ("visited", i64), ("reverse_prunes", i64), ("reverse_appends", i64),
                ("reverse_full_prunes", i64), ("launches", i64), ("ms_encode", f64), ("ms_search", f64), ("ms_sort", f64),
                ("ms_reverse", f64)]

    def counters(self) -> dict:
        return {"dist_comps": int(self.dist_comps), "sym_comps": int(self.sym_comps),
                "kernel_calls": int(self.kernel_calls), "visited": int(self.visited)}


_SIGS = {
    "fa_last_error": (C.c_char_p, []),
    "fa_version": (C.c_int, []),
    "fa_scan_cases_dev": (C.c_int, [vp, vp, C.c_int, i64, vp, vp]),
    "fa_scan_blocks_dev": (C.c_int, [vp, vp, C.c_int, C.c_int, vp, vp]),
    "fa_scan_select_dev": (C.c_int, [vp, C.c_int, vp, i64, i64, i64, C.c_int, C.c_int, vp,
                                     C.c_int, vp, vp]),
    "fa_scan_select_tma_dev": (C.c_int, [vp, C.c_int, vp, i64, i64, i64, C.c_int, C.c_int, vp,
                                         C.c_int, vp, vp]),
    "fa_quantize_dev": (C.c_int, [vp, i64, f64, f64, vp, vp]),
    "fa_l2sq_rows_dev": (C.c_int, [vp, i64, vp, i64, i64, C.c_int, vp, vp]),
    "fa_encode_adt_dev": (C.c_int, [vp, i64, i64, vp, vp, vp, C.c_int, C.c_int, f64, f64, vp,
                                    C.c_int, vp, C.c_int, vp]),
    "fa_sdt_sum_dev": (C.c_int, [vp, C.c_int, vp, i64, vp, i64, i64, vp, vp]),
    "fa_select_dev": (C.c_int, [vp, C.c_int, vp, C.c_int, vp, vp, C.c_int, C.c_int, vp, vp, vp]),
    "fa_select_exact_dev": (C.c_int, [vp, C.c_int, vp, vp, C.c_int, C.c_int, vp, vp, vp]),
    "fa_kmeans_scratch_bytes": (C.c_size_t, [C.c_int, C.c_int]),
    "fa_kmeans_subsample": (C.c_int, [i64, C.c_int, C.c_int, vp, vp]),
    "fa_assemble_blocks": (C.c_int, [vp, i64, i64, C.c_int, C.c_int, vp, vp, i64]),
    "fa_index_export_rows": (C.c_int, [vp, vp, vp, vp]),
    "fa_kmeans_subspaces_dev": (C.c_int, [vp, i64, C.c_int, vp, vp, C.c_int, vp, C.c_int, vp,
                                          C.c_int, vp, C.c_int, vp, vp, vp]),
    "fa_flash_range_dev": (C.c_int, [vp, i64, C.c_int, vp, vp, C.c_int, vp, C.c_int, vp, vp,
                                     vp, vp]),
    "fa_pca_cov_dev": (C.c_int, [vp, C.c_int, i64, C.c_int, vp, vp, vp]),
    "fa_pca_project_dev": (C.c_int, [vp, C.c_int, i64, C.c_int, vp, vp, C.c_int, C.c_int, vp,
                                     i64, vp]),
    "fa_pca_project_f64_dev": (C.c_int, [vp, i64, C.c_int, vp, vp, C.c_int, C.c_int, vp, vp]),
    "fa_index_create": (C.c_int, [C.POINTER(IndexDesc), C.POINTER(vp)]),
    "fa_index_destroy": (C.c_int, [vp]),
    "fa_index_encode": (C.c_int, [vp, vp]),
    "fa_index_set_codes": (C.c_int, [vp, vp, C.c_int, vp]),
    "fa_index_build": (C.c_int, [vp, C.POINTER(BuildOpts), C.POINTER(BuildResult), vp]),
    "fa_index_search": (C.c_int, [vp, vp, vp, C.c_int, C.c_int, C.c_int, C.c_int, i64, C.c_int,
                                  vp, vp, vp, vp]),
    "fa_index_search_layer": (C.c_int, [vp, vp, C.c_int, vp, C.c_int, C.c_int, vp, vp, vp, vp,
                                        vp]),
    "fa_index_set_search_tie": (C.c_int, [vp, C.c_int]),
    "fa_index_export_blocks": (C.c_int, [vp, vp, i64, vp, i64, vp]),
    "fa_index_import_blocks": (C.c_int, [vp, vp, i64, vp, i64, vp]),
    "fa_index_codes": (vp, [vp, C.POINTER(C.c_int)]),
    "fa_index_adjacency": (C.c_int, [vp, C.c_int, C.POINTER(vp), C.POINTER(vp),
                                     C.POINTER(C.c_int), C.POINTER(i64)]),
    "fa_build_graph_host": (C.c_int, [i64, C.c_int, vp, C.c_int, vp, vp, C.c_int, vp, C.c_int,
                                      vp, vp, vp, f64, f64, vp, vp, i64, vp, vp, i64, i64,
                                      C.c_int, C.c_int, C.POINTER(BuildOpts),
                                      C.POINTER(BuildResult)]),
    "fa_search_batch_host": (C.c_int, [i64, C.c_int, vp, C.c_int, vp, C.c_int, vp, C.c_int, vp,
                                       vp, vp, f64, f64, vp, vp, i64, vp, vp, i64, i64, C.c_int,
                                       i64, C.c_int, vp, vp, C.c_int, C.c_int, C.c_int,
                                       C.c_int, vp, vp, vp]),
    "fa_build_graph_exact_host": (C.c_int, [i64, C.c_int, vp, vp, vp, i64, vp, vp, i64, i64,
                                            C.c_int, C.c_int, vp, vp]),
    "fa_search_batch_exact_host": (C.c_int, [i64, C.c_int, vp, vp, vp, i64, vp, vp, i64, i64,
                                             C.c_int, i64, C.c_int, vp, C.c_int, C.c_int,
                                             C.c_int, C.c_int, vp, vp, vp]),
}

EXPORTED = tuple(_SIGS)

_lib = None


def load(require_device: bool = True):
    """Load the CUDA core; raise DeviceError when it cannot serve requests."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise DeviceError(
                f"CUDA core not built ({LIB_PATH} missing); run "
                "`python -m paper_2502_18113_b200._build`")
        try:
            lib = C.CDLL(str(LIB_PATH))
        except OSError as e:  # pragma: no cover - loader environment
            raise DeviceError(f"cannot load {LIB_PATH}: {e}") from e
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    if require_device:
        _require_device()
    return _lib


_device_ok = None


def _require_device() -> None:
    global _device_ok
    if _device_ok is None:
        import torch

        _device_ok = bool(torch.cuda.is_available())
    if not _device_ok:
        raise DeviceError("no CUDA device visible: the sm_100a core has no CPU fallback")


def check(rc: int) -> None:
    if rc == FA_OK:
        return
    msg = (_lib.fa_last_error() or b"").decode(errors="replace")
    if rc == FA_EINVAL:
        raise ValueError(msg)
    if rc == FA_ENOMEM:
        raise MemoryError(msg)
    if rc == FA_EEMPTY:
        raise ValueError(msg)
    if rc == FA_EOVERFLOW:
        raise DeviceError(f"capacity overflow: {msg}")
    raise DeviceError(f"CUDA error: {msg}")


def stream_handle():
    import torch

    return vp(torch.cuda.current_stream().cuda_stream)


def ptr(x) -> vp:
    """Address of a numpy array or torch tensor buffer (None -> NULL)."""
    if x is None:
        return vp(0)
    if hasattr(x, "data_ptr"):
        return vp(x.data_ptr())
    return vp(x.ctypes.data)
