"""sm_100a compute core: a drop-in for the reference's core-module contract.

The reference selects a compute core in flashann/core.py:16-26 and passes it
as ``core_impl=`` to ``builder.build`` (flashann/builder.py:88-111) and
``evaluation.search_batch`` (flashann/evaluation.py:72-89).  This module
exposes the same names and signatures as the compiled core
(flashann/_kernels/_core.pyx:711-1053):

    CORE_NAME, available_kernels(), build_graph(...), search_batch(...),
    greedy_search_layer(...), select_neighbors(...), flash_batch_distance(...),
    flash_batch_distance_many(...), flash_batch_blocks(...),
    flash_sdt_distance(...), flash_encode_adt(...), quantize_distance(...),
    l2sq_f32(...)

Every call runs on the GPU through the C-ABI (include/flashann_b200.h); array
arguments are host numpy buffers exactly as in the reference, blocks and
codes are mutated in place.  The Flash strategy (kind 4) and the exact
strategy (kind 0) are served — the PQ / SQ / PCA strategies are outside this
core's scope and raise ValueError.

Batched insertion replaces OpenMP threads: ``threads`` is accepted and
ignored; the batch schedule is set by BUILD_OPTIONS.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import _lib
from ._lib import check, ptr

CORE_NAME = "sm100"
KIND_FLASH = 4

# Lookup-kernel names; index = kernel id.  The reference resolves a kernel
# name through its own registry (core.py:28 KERNEL_IDS, :40-57 resolve_kernel)
# and evaluate() indexes this tuple by id (evaluation.py:142-143), so the core
# answers with the registry's names.  Every id selects the same sm_100a code
# path: the reference requires its kernels to be bit-identical to each other
# (tests/test_flash.py:207-217), which a single implementation is by
# construction.  Serving all four ids makes the core a drop-in without a patch
# to the reference's registry.
KERNEL_NAMES = ("scalar", "vector128", "vector256", "vector512")

BUILD_OPTIONS = {
    "batch_max": int(os.environ.get("FLASHANN_B200_BATCH_MAX", "65536")),
    "batch_frac": float(os.environ.get("FLASHANN_B200_BATCH_FRAC", "0.2")),
    "seq_prefix": int(os.environ.get("FLASHANN_B200_SEQ_PREFIX", "0")),
    # batches of at least min(inserted, batch_min) while batch_frac * inserted
    # is smaller: the GPU fills sooner (-1 = clamp(n / 256, 1, 4096))
    "batch_min": int(os.environ.get("FLASHANN_B200_BATCH_MIN", "-1")),
    "hash_log2": int(os.environ.get("FLASHANN_B200_HASH_LOG2", "0")),
    # tie order among equal distances during insertion searches: 2 = id
    # scramble salted per inserted vertex; 0 reproduces
    # the reference's semantic core (_pycore) exactly
    "tie": int(os.environ.get("FLASHANN_B200_TIE", "2")),
    # frontier entries expanded together per search step during insertion
    # (1 = the semantic core)
    "expand": int(os.environ.get("FLASHANN_B200_EXPAND", "1")),
    "profile": 0,
}


def available_kernels() -> tuple[str, ...]:
    return KERNEL_NAMES


def _lib_():
    return _lib.load()


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


def _torch():
    import torch

    return torch


def _dev(a):
    torch = _torch()
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


KIND_EXACT = 0  # providers/base.py:23-29 KIND_IDS["exact"]


def _require_flash(kind: int) -> None:
    if kind not in (KIND_FLASH, KIND_EXACT):
        raise ValueError("the sm100 core serves the Flash (4) and exact (0) strategies, "
                         f"got kind {kind}")


# Capacities of the sm_100a build (checked up front with the limit named,
# before any device work): layer-0 rows of 2R <= 127 slots (id rows of up to
# four 32-slot chunks held in registers), candidate width C <= 2048, m <= 128
# subspaces, and int32 vertex ids (n >= 2^24 - 1 selects the wide-id kernels:
# 64-bit search keys with 32-bit tie ids).
DEVICE_LIMITS = {"R_max": 63, "C_max": 2048, "m_max": 128, "n_max": (1 << 31) - 2}


def check_limits(n: int, C_: int, R: int, m: int = 0) -> None:
    from .errors import ConfigError

    lim = DEVICE_LIMITS
    if R > lim["R_max"]:
        raise ConfigError(f"R={R}: the sm100 core supports R <= {lim['R_max']} "
                          f"(layer-0 rows of 2R <= 127 slots)")
    if C_ > lim["C_max"]:
        raise ConfigError(f"C={C_}: the sm100 core supports C <= {lim['C_max']}")
    if m > lim["m_max"]:
        raise ConfigError(f"m={m}: the sm100 core supports m <= {lim['m_max']} subspaces")
    if n > lim["n_max"]:
        raise ConfigError(f"n={n}: the sm100 core addresses n <= {lim['n_max']} vertices "
                          "(int32 ids)")


def build_options(C_: int) -> _lib.BuildOpts:
    o = BUILD_OPTIONS
    return _lib.BuildOpts(C=C_, batch_max=o["batch_max"], batch_frac=o["batch_frac"],
                          seq_prefix=o["seq_prefix"], hash_log2=o["hash_log2"],
                          profile=o.get("profile", 0), tie=o.get("tie", 2),
                          expand=o.get("expand", 1), batch_min=o.get("batch_min", -1))


def _prov_arrays(prov: dict):
    cent = _c(prov["cent"], np.float32)
    dims = _c(prov["dims"], np.int32)
    offs = _c(prov["offs"], np.int32)
    sdt = _c(prov["sdt"], np.uint8)
    proj = _c(prov["proj"], np.float32)
    return cent, dims, offs, sdt, proj


# ---------------------------------------------------------------------------
# build / search (host-array drop-ins)


def build_graph(kind, prov, levels, base_blocks, upper_offsets, upper_blocks, C, R,
                threads=1, kernel=0):
    """Insert every vector; returns entry point, top layer and counters
    (reference build_graph, _core.pyx:711-764)."""
    _require_flash(kind)
    lib = _lib_()
    lv = _c(levels, np.int32)
    bb = np.ascontiguousarray(base_blocks)
    uo = _c(upper_offsets, np.int64)
    ub = np.ascontiguousarray(upper_blocks)
    n = lv.shape[0]
    codes = None
    if kind != KIND_EXACT:
        codes = np.ascontiguousarray(prov["codes"])
        if codes.dtype != np.uint8:
            raise TypeError("codes must be uint8")
    if n == 0:
        return {"entry_point": -1, "max_layer": -1,
                "counters": {"dist_comps": 0, "sym_comps": 0, "kernel_calls": 0, "visited": 0}}
    check_limits(n, int(C), int(R), 0 if kind == KIND_EXACT else int(np.shape(prov["cent"])[0]))
    res = _lib.BuildResult()
    opts = build_options(int(C))
    if kind == KIND_EXACT:
        # exact strategy: fp32 L2 of the vectors, no codes (_core.pyx:167-191)
        vecs = _c(prov["vecs"], np.float32)
        check(lib.fa_build_graph_exact_host(
            n, vecs.shape[1], ptr(vecs), ptr(lv), ptr(bb), bb.shape[1], ptr(uo), ptr(ub),
            ub.shape[0], ub.shape[1] if ub.ndim == 2 else 0, int(C), int(R), C_byref(opts),
            C_byref(res)))
        if bb is not base_blocks:
            base_blocks[...] = bb
        if ub is not upper_blocks:
            upper_blocks[...] = ub
        return {"entry_point": int(res.entry_point), "max_layer": int(res.max_layer),
                "counters": res.counters()}
    cent, dims, offs, sdt, proj = _prov_arrays(prov)
    m = cent.shape[0]
    check(lib.fa_build_graph_host(
        n, 0, None, proj.shape[1], ptr(proj), ptr(codes), m, ptr(cent), cent.shape[2], ptr(dims),
        ptr(offs), ptr(sdt), float(prov["dist_min"]), float(prov["delta"]), ptr(lv), ptr(bb),
        bb.shape[1], ptr(uo), ptr(ub), ub.shape[0], ub.shape[1] if ub.ndim == 2 else 0,
        int(C), int(R), C_byref(opts), C_byref(res)))
    if codes is not prov["codes"]:
        prov["codes"][...] = codes
    if bb is not base_blocks:
        base_blocks[...] = bb
    if ub is not upper_blocks:
        upper_blocks[...] = ub
    return {"entry_point": int(res.entry_point), "max_layer": int(res.max_layer),
            "counters": res.counters()}


def C_byref(x):
    return C.byref(x)


def search_batch(kind, prov, levels, base_blocks, upper_offsets, upper_blocks, C, R, entry,
                 max_layer, queries, qaux, ef, k, rerank_depth, threads=1, kernel=0):
    """Search many queries over a frozen graph (reference search_batch,
    _core.pyx:817-888): (ids int64 (nq,k) -1 padded, dists f64 +inf padded,
    counters)."""
    if entry < 0:
        raise ValueError("cannot search an empty graph")
    _require_flash(kind)
    lib = _lib_()
    lv = _c(levels, np.int32)
    bb = np.ascontiguousarray(base_blocks)
    uo = _c(upper_offsets, np.int64)
    ub = np.ascontiguousarray(upper_blocks)
    qs = _c(queries, np.float32)
    if kind == KIND_EXACT:
        vecs = _c(prov["vecs"], np.float32)
        nq = qs.shape[0]
        out_ids = np.full((nq, k), -1, dtype=np.int64)
        out_d = np.full((nq, k), np.inf, dtype=np.float64)
        ctr = np.zeros(4, dtype=np.int64)
        if nq:
            check(lib.fa_search_batch_exact_host(
                lv.shape[0], vecs.shape[1], ptr(vecs), ptr(lv), ptr(bb), bb.shape[1], ptr(uo),
                ptr(ub), ub.shape[0], ub.shape[1] if ub.ndim == 2 else 0, int(R), int(entry),
                int(max_layer), ptr(qs), nq, int(ef), int(k), int(rerank_depth), ptr(out_ids),
                ptr(out_d), ptr(ctr)))
        return out_ids, out_d, {"dist_comps": int(ctr[0]), "sym_comps": int(ctr[1]),
                                "kernel_calls": int(ctr[2]), "visited": int(ctr[3])}
    if qaux is None:
        raise ValueError("this strategy requires a prepared query payload (qaux)")
    qp = _c(qaux, np.float32)
    codes = _c(prov["codes"], np.uint8)
    vecs = _c(prov["vecs"], np.float32)
    cent, dims, offs, sdt, _ = _prov_arrays(prov)
    nq = qs.shape[0]
    out_ids = np.full((nq, k), -1, dtype=np.int64)
    out_d = np.full((nq, k), np.inf, dtype=np.float64)
    ctr = np.zeros(4, dtype=np.int64)
    if nq:
        check(lib.fa_search_batch_host(
            lv.shape[0], vecs.shape[1], ptr(vecs), qp.shape[1], ptr(codes), codes.shape[1],
            ptr(cent), cent.shape[2], ptr(dims), ptr(offs), ptr(sdt), float(prov["dist_min"]),
            float(prov["delta"]), ptr(lv), ptr(bb), bb.shape[1], ptr(uo), ptr(ub), ub.shape[0],
            ub.shape[1] if ub.ndim == 2 else 0, int(R), int(entry), int(max_layer), ptr(qs),
            ptr(qp), nq, int(ef), int(k), int(rerank_depth), ptr(out_ids), ptr(out_d), ptr(ctr)))
    counters = {"dist_comps": int(ctr[0]), "sym_comps": int(ctr[1]),
                "kernel_calls": int(ctr[2]), "visited": int(ctr[3])}
    return out_ids, out_d, counters


class DeviceIndex:
    """A device graph built from reference-layout host arrays (test hooks).

    kind 4 (Flash): codes, tables and the SDT from ``prov``; kind 0 (exact):
    the vectors only (a device index with m = 0)."""

    def __init__(self, prov, levels, base_blocks, upper_offsets, upper_blocks, R, vecs=None,
                 kind=KIND_FLASH):
        torch = _torch()
        self.lib = _lib_()
        self.keep = []
        lv = _c(levels, np.int32)
        uo = _c(upper_offsets, np.int64)
        self.n = lv.shape[0]
        self.kind = kind
        d = _lib.IndexDesc()
        d.n = self.n
        d.R = int(R)
        if kind == KIND_EXACT:
            vecs = prov["vecs"]
            d.m = 0
            for name, arr in (("levels", lv), ("uoff", uo)):
                t = _dev(arr)
                self.keep.append(t)
                setattr(d, name, t.data_ptr())
        else:
            cent, dims, offs, sdt, proj = _prov_arrays(prov)
            d.m = cent.shape[0]
            d.dproj = proj.shape[1]
            d.dmax = cent.shape[2]
            d.dist_min = float(prov["dist_min"])
            d.delta = float(prov["delta"])
            for name, arr in (("cent", cent), ("dims", dims), ("offs", offs), ("sdt", sdt),
                              ("levels", lv), ("uoff", uo), ("proj", proj)):
                t = _dev(arr)
                self.keep.append(t)
                setattr(d, name, t.data_ptr())
        if vecs is not None:
            t = _dev(_c(vecs, np.float32))
            self.keep.append(t)
            d.vecs = t.data_ptr()
            d.dim = t.shape[1]
            if kind == KIND_EXACT:
                d.dproj = d.dim
        ub = np.ascontiguousarray(upper_blocks)
        d.n_upper_rows = ub.shape[0]
        self.desc = d
        h = _lib.vp()
        check(self.lib.fa_index_create(C.byref(d), C.byref(h)))
        self.h = h
        if kind != KIND_EXACT:
            codes = _dev(_c(prov["codes"], np.uint8))
            check(self.lib.fa_index_set_codes(h, codes.data_ptr(), codes.shape[1], None))
        bb = _dev(np.ascontiguousarray(base_blocks))
        ubd = _dev(ub) if ub.size else torch.zeros(1, dtype=torch.uint8, device="cuda")
        check(self.lib.fa_index_import_blocks(h, bb.data_ptr(), bb.shape[1], ubd.data_ptr(),
                                              ub.shape[1] if ub.ndim == 2 else 0, None))
        torch.cuda.synchronize()

    def search_layer(self, qproj, entries, width, layer):
        """Batched single-layer search: (ids (nq,width) -1 padded, d, n, counters)."""
        torch = _torch()
        qp = _dev(_c(np.atleast_2d(qproj), np.float32))
        nq = qp.shape[0]
        ent = _dev(_c(entries, np.int64))
        oid = torch.empty((nq, width), dtype=torch.int32, device="cuda")
        od = torch.empty((nq, width), dtype=torch.float64, device="cuda")
        on = torch.empty(nq, dtype=torch.int32, device="cuda")
        ctr = np.zeros(4, dtype=np.int64)
        check(self.lib.fa_index_search_layer(self.h, qp.data_ptr(), nq, ent.data_ptr(),
                                             int(width), int(layer), oid.data_ptr(),
                                             od.data_ptr(), on.data_ptr(), ptr(ctr), None))
        return oid.cpu().numpy(), od.cpu().numpy(), on.cpu().numpy(), ctr

    def close(self):
        if getattr(self, "h", None):
            self.lib.fa_index_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def greedy_search_layer(kind, prov, levels, base_blocks, upper_offsets, upper_blocks, C, R,
                        entry, width, layer, query, qaux=None, kernel=0):
    """Single-layer candidate search: ([(id, dist)], counters)
    (reference hook _core.pyx:891-939; (d, id) ordering)."""
    _require_flash(kind)
    if kind == KIND_FLASH and qaux is None:
        raise ValueError("this strategy requires a prepared query payload (qaux)")
    torch = _torch()
    ix = DeviceIndex(prov, levels, base_blocks, upper_offsets, upper_blocks, R, kind=kind)
    try:
        # Flash: the reduced query (its table is built on the device); exact:
        # the query vector itself
        qsrc = query if kind == KIND_EXACT else qaux
        qp = _dev(_c(np.atleast_2d(qsrc), np.float32))
        ent = _dev(np.array([entry], dtype=np.int64))
        oid = torch.empty((1, width), dtype=torch.int32, device="cuda")
        od = torch.empty((1, width), dtype=torch.float64, device="cuda")
        on = torch.empty(1, dtype=torch.int32, device="cuda")
        ctr = np.zeros(4, dtype=np.int64)
        check(ix.lib.fa_index_search_layer(ix.h, qp.data_ptr(), 1, ent.data_ptr(), int(width),
                                           int(layer), oid.data_ptr(), od.data_ptr(),
                                           on.data_ptr(), ptr(ctr), None))
        nres = int(on.cpu()[0])
        ids = oid.cpu().numpy()[0, :nres]
        ds = od.cpu().numpy()[0, :nres]
    finally:
        ix.close()
    out = [(int(i), float(d)) for i, d in zip(ids, ds)]
    return out, {"dist_comps": int(ctr[0]), "sym_comps": int(ctr[1]),
                 "kernel_calls": int(ctr[2]), "visited": int(ctr[3])}


def _padded_codes(codes: np.ndarray) -> np.ndarray:
    codes = _c(codes, np.uint8)
    m = codes.shape[1]
    mp = -(-m // 16) * 16
    if mp == m:
        return codes
    out = np.zeros((codes.shape[0], mp), dtype=np.uint8)
    out[:, :m] = codes
    return out


def select_neighbors(kind, prov, cand_ids, cand_dists, cap):
    """Diversity pruning over ordered candidates (reference hook
    _core.pyx:942-959)."""
    _require_flash(kind)
    torch = _torch()
    lib = _lib_()
    ci = _c(cand_ids, np.int32)
    cd = _c(cand_dists, np.float64)
    n = ci.shape[0]
    if n == 0 or cap <= 0:
        return []
    if kind == KIND_EXACT:
        vecs = _dev(_c(prov["vecs"], np.float32))
        dci, dcd = _dev(ci), _dev(cd)
        out = torch.empty(n, dtype=torch.int32, device="cuda")
        nout = torch.zeros(1, dtype=torch.int32, device="cuda")
        check(lib.fa_select_exact_dev(vecs.data_ptr(), vecs.shape[1], dci.data_ptr(),
                                      dcd.data_ptr(), n, int(cap), out.data_ptr(),
                                      nout.data_ptr(), None))
        nk = int(nout.cpu()[0])
        return [int(x) for x in out.cpu().numpy()[:nk]]
    sdt = _dev(_c(prov["sdt"], np.uint8))
    codes = _dev(_padded_codes(prov["codes"]))
    m = int(prov["sdt"].shape[0])
    dci, dcd = _dev(ci), _dev(cd)
    out = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")
    nout = torch.zeros(1, dtype=torch.int32, device="cuda")
    check(lib.fa_select_dev(sdt.data_ptr(), m, codes.data_ptr(), codes.shape[1], dci.data_ptr(),
                            dcd.data_ptr(), n, int(cap), out.data_ptr(), nout.data_ptr(), None))
    nk = int(nout.cpu()[0])
    return [int(x) for x in out.cpu().numpy()[:nk]]


# ---------------------------------------------------------------------------
# kernel-level hooks (_core.pyx:965-1053)


def flash_batch_distance(adt, codes, kernel=0):
    """One 16-slot batch: adt (M,16) u8, codes (M,16) u8 -> u8[16]."""
    a = _c(adt, np.uint8)
    return flash_batch_distance_many(a[None], _c(codes, np.uint8)[None], kernel)[0]


def flash_batch_distance_many(adts, codes, kernel=0):
    """adts (N,M,16), codes (N,M,16) -> (N,16) u8."""
    torch = _torch()
    lib = _lib_()
    a = _c(adts, np.uint8)
    c = _c(codes, np.uint8)
    n, m = a.shape[0], a.shape[1]
    out = torch.empty((n, 16), dtype=torch.uint8, device="cuda")
    if n:
        da, dc = _dev(a), _dev(c)
        check(lib.fa_scan_cases_dev(da.data_ptr(), dc.data_ptr(), m, n, out.data_ptr(), None))
    return out.cpu().numpy()


def flash_batch_blocks(adt, codes_flat, nb, kernel=0):
    """Consecutive batches of a vertex block: codes_flat (nb*M*16,) -> (nb*16,)."""
    torch = _torch()
    lib = _lib_()
    a = _c(adt, np.uint8)
    c = _c(codes_flat, np.uint8)
    m = a.shape[0]
    out = torch.empty(max(nb, 0) * 16, dtype=torch.uint8, device="cuda")
    if nb:
        da, dc = _dev(a), _dev(c)
        check(lib.fa_scan_blocks_dev(da.data_ptr(), dc.data_ptr(), m, int(nb), out.data_ptr(),
                                     None))
    return out.cpu().numpy()


def flash_sdt_distance(sdt, code_a, code_b):
    torch = _torch()
    lib = _lib_()
    s = _c(sdt, np.uint8)
    a = _c(code_a, np.uint8)
    b = _c(code_b, np.uint8)
    m = s.shape[0]
    out = torch.empty(1, dtype=torch.int32, device="cuda")
    ds, da, db = _dev(s), _dev(a), _dev(b)
    check(lib.fa_sdt_sum_dev(ds.data_ptr(), m, da.data_ptr(), m, db.data_ptr(), m, 1,
                             out.data_ptr(), None))
    return int(out.cpu()[0])


def flash_encode_adt(cent, dims, offs, dist_min, delta, reduced):
    """(code u8 (M,), adt u8 (M,16)) of one reduced vector (_core.pyx:1017-1031)."""
    codes, adts = flash_encode_adt_many(cent, dims, offs, dist_min, delta,
                                        _c(reduced, np.float32)[None])
    return codes[0], adts[0]


def flash_encode_adt_many(cent, dims, offs, dist_min, delta, reduced):
    """Batched encode + table for rows of the reduced matrix."""
    torch = _torch()
    lib = _lib_()
    ct = _c(cent, np.float32)
    dm = _c(dims, np.int32)
    of = _c(offs, np.int32)
    rd = _c(np.atleast_2d(reduced), np.float32)
    m = ct.shape[0]
    n = rd.shape[0]
    codes = torch.empty((n, m), dtype=torch.uint8, device="cuda")
    adt = torch.empty((n, m, 16), dtype=torch.uint8, device="cuda")
    if n:
        dct, ddm, dof, drd = _dev(ct), _dev(dm), _dev(of), _dev(rd)
        check(lib.fa_encode_adt_dev(drd.data_ptr(), n, rd.shape[1], dct.data_ptr(),
                                    ddm.data_ptr(), dof.data_ptr(), m, ct.shape[2],
                                    float(dist_min), float(delta), codes.data_ptr(), m,
                                    adt.data_ptr(), m, None))
    return codes.cpu().numpy(), adt.cpu().numpy()


def quantize_distance(dist, dist_min, delta):
    torch = _torch()
    lib = _lib_()
    d = np.ascontiguousarray(np.atleast_1d(np.asarray(dist, dtype=np.float64)))
    out = torch.empty(d.shape[0], dtype=torch.uint8, device="cuda")
    if d.shape[0]:
        dd = _dev(d)
        check(lib.fa_quantize_dev(dd.data_ptr(), d.shape[0], float(dist_min), float(delta),
                                  out.data_ptr(), None))
    res = out.cpu().numpy()
    return res if np.ndim(dist) else res[0]


def l2sq_f32(a, b):
    """Squared distance with the reference core's fp32 operation tree."""
    torch = _torch()
    lib = _lib_()
    x = _c(a, np.float32)
    y = _c(b, np.float32)
    out = torch.empty(1, dtype=torch.float64, device="cuda")
    dx, dy = _dev(x), _dev(y)
    check(lib.fa_l2sq_rows_dev(dx.data_ptr(), 0, dy.data_ptr(), 0, 1, x.shape[0],
                               out.data_ptr(), None))
    return float(out.cpu()[0])
