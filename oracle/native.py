"""ctypes wrapper of oracle/build/liboracle.so (TEST INFRASTRUCTURE ONLY).

See oracle/oracle.c for what each function restates and the reference
file:line it follows.
"""

from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "build" / "liboracle.so"

vp, i32, i64, f64 = C.c_void_p, C.c_int32, C.c_int64, C.c_double


class Counters(C.Structure):
    _fields_ = [("dist_comps", i64), ("sym_comps", i64), ("kernel_calls", i64),
                ("visited", i64), ("reverse_prunes", i64), ("reverse_appends", i64)]

    def as_dict(self):
        return {k: int(getattr(self, k)) for k, _ in self._fields_}


class Graph(C.Structure):
    _fields_ = [("n", i64), ("nU", i64), ("m", C.c_int), ("cs", C.c_int), ("cap0", C.c_int),
                ("capU", C.c_int), ("adj0", vp), ("cnt0", vp), ("adjU", vp), ("cntU", vp),
                ("codes", vp), ("levels", vp), ("uoff", vp), ("upper_owner", vp),
                ("tie", C.c_int), ("expand", C.c_int), ("kind", C.c_int), ("vecs", vp),
                ("dim", C.c_int)]


class BuildResult(C.Structure):
    _fields_ = [("entry_point", i64), ("max_layer", i32), ("n_batches", i32),
                ("counters", Counters)]


_lib = None


def build_lib() -> Path:
    subprocess.run(["make", "-s", "-C", str(HERE), "all"], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            build_lib()
        L = C.CDLL(str(LIB_PATH))
        L.or_l2sq_f32.restype = f64
        L.or_l2sq_f32.argtypes = [vp, vp, C.c_int]
        L.or_quantize.restype = C.c_uint8
        L.or_quantize.argtypes = [f64, f64, f64]
        L.or_encode_adt.restype = None
        L.or_encode_adt.argtypes = [vp, vp, vp, vp, C.c_int, C.c_int, f64, f64, vp, vp]
        L.or_batch_lanes.restype = None
        L.or_batch_lanes.argtypes = [vp, vp, C.c_int, C.c_int, vp]
        L.or_sdt_sum.restype = C.c_int
        L.or_sdt_sum.argtypes = [vp, vp, vp, C.c_int]
        L.or_select.restype = C.c_int
        L.or_select.argtypes = [vp, C.c_int, vp, C.c_int, vp, vp, C.c_int, C.c_int, vp, vp]
        L.or_layer_search.restype = C.c_int
        L.or_layer_search.argtypes = [C.POINTER(Graph), vp, C.c_int, C.c_int, C.c_int, vp, vp,
                                      C.POINTER(Counters)]
        L.or_layer_search_exact.restype = C.c_int
        L.or_layer_search_exact.argtypes = [C.POINTER(Graph), vp, C.c_int, C.c_int, C.c_int, vp,
                                            vp, C.POINTER(Counters)]
        L.or_hill_climb.restype = C.c_int
        L.or_hill_climb.argtypes = [C.POINTER(Graph), vp, C.c_int, C.c_int, vp,
                                    C.POINTER(Counters)]
        L.or_schedule.restype = C.c_int
        L.or_schedule.argtypes = [vp, i64, C.c_int, f64, C.c_int, C.c_int, vp, vp]
        L.or_build.restype = C.c_int
        L.or_build.argtypes = [C.POINTER(Graph), vp, C.c_int, vp, vp, vp, C.c_int, f64, f64, vp,
                               C.c_int, C.c_int, C.c_int, f64, C.c_int, C.c_int,
                               C.POINTER(BuildResult)]
        L.or_search.restype = C.c_int
        L.or_search.argtypes = [C.POINTER(Graph), vp, C.c_int, vp, vp, vp, C.c_int, f64, f64,
                                C.c_int, C.c_int, C.c_int, vp, vp, C.c_int, C.c_int, C.c_int,
                                C.c_int, vp, vp, C.POINTER(Counters)]
        _lib = L
    return _lib


def _p(a):
    return vp(a.ctypes.data) if a is not None else vp(0)


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


# ---- kernels --------------------------------------------------------------

def l2sq_f32(a, b) -> float:
    a, b = _c(a, np.float32), _c(b, np.float32)
    return lib().or_l2sq_f32(_p(a), _p(b), a.shape[0])


def quantize(d, dmin, delta) -> np.ndarray:
    d = np.atleast_1d(np.asarray(d, dtype=np.float64))
    L = lib()
    return np.array([L.or_quantize(float(x), float(dmin), float(delta)) for x in d], np.uint8)


def encode_adt(red, cent, dims, offs, dmin, delta):
    red = _c(np.atleast_2d(red), np.float32)
    cent, dims, offs = _c(cent, np.float32), _c(dims, np.int32), _c(offs, np.int32)
    m, dmax = cent.shape[0], cent.shape[2]
    codes = np.empty((red.shape[0], m), np.uint8)
    adts = np.empty((red.shape[0], m, 16), np.uint8)
    L = lib()
    for r in range(red.shape[0]):
        L.or_encode_adt(_p(red[r]), _p(cent), _p(dims), _p(offs), m, dmax, float(dmin),
                        float(delta), _p(codes[r]), _p(adts[r]))
    return codes, adts


def batch_lanes(adt, codes_flat, nb):
    adt, codes = _c(adt, np.uint8), _c(codes_flat, np.uint8)
    out = np.empty(nb * 16, np.uint8)
    lib().or_batch_lanes(_p(adt), _p(codes), adt.shape[0], nb, _p(out))
    return out


def batch_many(adts, codes):
    adts, codes = _c(adts, np.uint8), _c(codes, np.uint8)
    out = np.empty((adts.shape[0], 16), np.uint8)
    L = lib()
    m = adts.shape[1]
    for i in range(adts.shape[0]):
        L.or_batch_lanes(_p(adts[i]), _p(codes[i]), m, 1, _p(out[i]))
    return out


def sdt_sum(sdt, a, b) -> int:
    sdt, a, b = _c(sdt, np.uint8), _c(a, np.uint8), _c(b, np.uint8)
    return lib().or_sdt_sum(_p(sdt), _p(a), _p(b), sdt.shape[0])


def select(sdt, codes, cand_ids, cand_d, cap):
    sdt, codes = _c(sdt, np.uint8), _c(codes, np.uint8)
    ids, d = _c(cand_ids, np.int32), _c(cand_d, np.float64)
    out = np.empty(max(len(ids), 1), np.int32)
    nk = lib().or_select(_p(sdt), sdt.shape[0], _p(codes), codes.shape[1], _p(ids), _p(d),
                         len(ids), int(cap), _p(out), vp(0))
    return [int(x) for x in out[:nk]]


def schedule(levels, batch_max, batch_frac, seq_prefix, batch_min=-1):
    levels = _c(levels, np.int32)
    n = levels.shape[0]
    st = np.zeros(max(n, 1), np.int32)
    sz = np.zeros(max(n, 1), np.int32)
    nb = lib().or_schedule(_p(levels), n, batch_max, batch_frac, seq_prefix, batch_min, _p(st),
                           _p(sz))
    return st[:nb].copy(), sz[:nb].copy()


# ---- graphs -----------------------------------------------------------------

class HostGraph:
    """Host graph in the device's logical layout (exact-cap id rows + counts)."""

    def __init__(self, levels, upper_offsets, R, m, codes=None, tie=0, expand=1, kind=4,
                 vecs=None):
        """kind 4 = Flash (u8 tables over `codes`), kind 0 = exact (fp32 L2 over
        `vecs`; m = 0)."""
        self.levels = _c(levels, np.int32)
        self.uoff = _c(upper_offsets, np.int64)
        self.n = self.levels.shape[0]
        self.nU = int(self.levels.astype(np.int64).sum())
        self.R, self.m = int(R), int(m)
        self.cap0, self.capU = 2 * self.R, self.R
        self.adj0 = np.full((self.n, self.cap0), -1, np.int32)
        self.cnt0 = np.zeros(self.n, np.int32)
        self.adjU = np.full((max(self.nU, 1), self.capU), -1, np.int32)
        self.cntU = np.zeros(max(self.nU, 1), np.int32)
        self.codes = np.zeros((self.n, self.m), np.uint8) if codes is None else _c(codes, np.uint8)
        owner = np.full(max(self.nU, 1), -1, np.int32)
        for v in np.flatnonzero(self.levels > 0):
            o = self.uoff[v]
            owner[o : o + self.levels[v]] = v
        self.owner = owner
        self.kind = int(kind)
        self.vecs = None if vecs is None else _c(vecs, np.float32)
        dim = 0 if self.vecs is None else self.vecs.shape[1]
        if self.kind == 0 and self.vecs is None:
            raise ValueError("the exact kind needs the vectors")
        self.s = Graph(self.n, self.nU, self.m, self.m, self.cap0, self.capU, _p(self.adj0),
                       _p(self.cnt0), _p(self.adjU), _p(self.cntU), _p(self.codes),
                       _p(self.levels), _p(self.uoff), _p(self.owner), int(tie),
                       int(expand), self.kind, _p(self.vecs), dim)

    @classmethod
    def from_blocks(cls, levels, upper_offsets, base_blocks, upper_blocks, R, codes, kind=4,
                    vecs=None):
        """Import reference-layout rows (live ids compacted to a prefix)."""
        if kind == 0:
            g = cls(levels, upper_offsets, R, 0, None, kind=0, vecs=vecs)
        else:
            g = cls(levels, upper_offsets, R, codes.shape[1], codes)

        def load(blocks, adj, cnt, cap):
            for r in range(blocks.shape[0]):
                c = int(blocks[r, :4].view(np.int32)[0])
                c = max(0, min(c, cap))
                ids = blocks[r, 4 : 4 + 4 * cap].view(np.int32)[:c]
                ids = ids[ids >= 0]
                adj[r, : len(ids)] = ids
                cnt[r] = len(ids)

        load(base_blocks, g.adj0, g.cnt0, g.cap0)
        if g.nU:
            load(upper_blocks, g.adjU, g.cntU, g.capU)
        return g

    def layer_search(self, adt, layer, entry, width):
        ids = np.empty(width + 1, np.int32)
        ds = np.empty(width + 1, np.int32)
        c = Counters()
        ts = lib().or_layer_search(C.byref(self.s), _p(_c(adt, np.uint8)), layer, entry, width,
                                   _p(ids), _p(ds), C.byref(c))
        return ids[:ts].copy(), ds[:ts].copy(), c.as_dict()

    def layer_search_exact(self, qvec, layer, entry, width):
        """Exact kind: distances are returned as float32 values."""
        ids = np.empty(width + 1, np.int32)
        ds = np.empty(width + 1, np.int32)
        c = Counters()
        ts = lib().or_layer_search_exact(C.byref(self.s), _p(_c(qvec, np.float32)), layer, entry,
                                         width, _p(ids), _p(ds), C.byref(c))
        return ids[:ts].copy(), ds[:ts].view(np.float32).astype(np.float64), c.as_dict()

    def hill_climb(self, adt, layer, entry):
        d = C.c_int(0)
        c = Counters()
        cur = lib().or_hill_climb(C.byref(self.s), _p(_c(adt, np.uint8)), layer, entry,
                                  C.byref(d), C.byref(c))
        return cur, d.value, c.as_dict()

    def build(self, proj, cent, dims, offs, dmin, delta, sdt, C_, batch_max=4096,
              batch_frac=0.02, seq_prefix=256, batch_min=-1):
        proj = _c(proj, np.float32)
        cent, dims, offs = _c(cent, np.float32), _c(dims, np.int32), _c(offs, np.int32)
        sdt = _c(sdt, np.uint8)
        res = BuildResult()
        rc = lib().or_build(C.byref(self.s), _p(proj), proj.shape[1], _p(cent), _p(dims),
                            _p(offs), cent.shape[2], float(dmin), float(delta), _p(sdt), int(C_),
                            self.R, int(batch_max), float(batch_frac), int(seq_prefix),
                            int(batch_min), C.byref(res))
        if rc:
            raise MemoryError("oracle build failed")
        return {"entry_point": int(res.entry_point), "max_layer": int(res.max_layer),
                "n_batches": int(res.n_batches), "counters": res.counters.as_dict()}

    def build_exact(self, C_, batch_max=4096, batch_frac=0.02, seq_prefix=256, batch_min=-1):
        """Exact kind: every distance is the fp32 L2 of the vectors."""
        z = np.zeros((1, 16, 1), np.float32)
        zi = np.zeros(1, np.int32)
        return self.build(self.vecs, z, zi, zi, 0.0, 1.0, np.zeros((1, 16, 16), np.uint8), C_,
                          batch_max, batch_frac, seq_prefix, batch_min)

    def search_exact(self, entry, max_layer, queries, ef, k):
        z = np.zeros((1, 16, 1), np.float32)
        zi = np.zeros(1, np.int32)
        q = _c(queries, np.float32)
        return self.search(self.vecs, z, zi, zi, 0.0, 1.0, entry, max_layer, q, q, ef, k, 0)

    def search(self, vecs, cent, dims, offs, dmin, delta, entry, max_layer, queries, qproj, ef,
               k, rerank_depth):
        vecs = _c(vecs, np.float32) if vecs is not None else np.zeros((1, 1), np.float32)
        queries = _c(queries, np.float32)
        qproj = _c(qproj, np.float32)
        cent, dims, offs = _c(cent, np.float32), _c(dims, np.int32), _c(offs, np.int32)
        nq = qproj.shape[0]
        oid = np.empty((nq, k), np.int64)
        od = np.empty((nq, k), np.float64)
        c = Counters()
        lib().or_search(C.byref(self.s), _p(vecs), vecs.shape[1], _p(cent), _p(dims), _p(offs),
                        cent.shape[2], float(dmin), float(delta), qproj.shape[1], int(entry),
                        int(max_layer), _p(queries), _p(qproj), nq, int(ef), int(k),
                        int(rerank_depth), _p(oid), _p(od), C.byref(c))
        return oid, od, c.as_dict()

    def neighbors(self, v, layer=0):
        if layer == 0:
            return self.adj0[v, : self.cnt0[v]].copy()
        r = self.uoff[v] + layer - 1
        return self.adjU[r, : self.cntU[r]].copy()
