"""Index files in the reference's FANNIDX1 container.

The byte format is the one the reference documents at
flashann/serialize.py:1-16 (magic "FANNIDX1", uint32 version, uint32-length
JSON meta, uint32 section count, then named arrays: uint32-length name,
uint32-length numpy dtype string, uint32 ndim + int64 shape, uint64 byte
length + raw bytes, all little-endian).  The section names and meta keys are
the reference's (save_index, flashann/serialize.py:74-113), so a file written
here loads in the reference package and vice versa: the graph sections are the
reference vertex-block layout (exported from / imported into the device
index), the provider sections are FlashProvider.state_dict().

The Flash and exact strategies are served; files of other strategies are
rejected with FormatError.
"""

from __future__ import annotations

import json
import struct

import numpy as np

from . import _lib
from .dataset import VectorDataset
from .errors import FormatError
from .flash import FlashProvider
from .graph import BuildParams, GraphIndex

MAGIC = b"FANNIDX1"
VERSION = 1


def _put_array(f, name: str, arr: np.ndarray) -> None:
    a = np.ascontiguousarray(arr)
    if a.dtype.byteorder == ">":
        a = a.astype(a.dtype.newbyteorder("<"))
    for blob in (name.encode(), a.dtype.str.encode()):
        f.write(struct.pack("<I", len(blob)))
        f.write(blob)
    f.write(struct.pack("<I", a.ndim))
    f.write(struct.pack(f"<{a.ndim}q", *a.shape))
    f.write(struct.pack("<Q", a.nbytes))
    f.write(memoryview(a).cast("B"))


def _get(f, fmt: str):
    size = struct.calcsize(fmt)
    raw = f.read(size)
    if len(raw) != size:
        raise FormatError("truncated index file")
    return struct.unpack(fmt, raw)


def _get_array(f) -> tuple[str, np.ndarray]:
    (nlen,) = _get(f, "<I")
    name = f.read(nlen).decode()
    (dlen,) = _get(f, "<I")
    dtype = np.dtype(f.read(dlen).decode())
    (ndim,) = _get(f, "<I")
    shape = _get(f, f"<{ndim}q") if ndim else ()
    (nbytes,) = _get(f, "<Q")
    raw = f.read(nbytes)
    if len(raw) != nbytes:
        raise FormatError("truncated index file")
    return name, np.frombuffer(raw, dtype=dtype).reshape(shape).copy()


def save_index(path, g: GraphIndex, provider: FlashProvider, dataset) -> None:
    """Write graph (reference block layout), trained model and vectors."""
    state = provider.state_dict()
    scalars = {k: (v.item() if isinstance(v, np.generic) else v)
               for k, v in state.items() if not isinstance(v, np.ndarray)}
    arrays = {k: v for k, v in state.items() if isinstance(v, np.ndarray)}
    meta = {
        "version": VERSION, "strategy": g.strategy, "n": g.n, "dim": g.dim,
        "C": g.params.C, "R": g.params.R, "seed": g.params.seed, "threads": g.params.threads,
        "entry_point": int(g.entry_point), "max_layer": int(g.max_layer),
        "code_subspaces": g.code_subspaces, "provider_scalars": scalars,
    }
    data = dataset.data if isinstance(dataset, VectorDataset) else dataset
    data = data.cpu().numpy() if hasattr(data, "cpu") else np.asarray(data)
    sections = {"levels": g.levels, "base_blocks": g.base_blocks,
                "upper_offsets": g.upper_offsets, "upper_blocks": g.upper_blocks,
                "vectors": data}
    for k, v in arrays.items():
        sections[f"prov.{k}"] = v
    if provider.kind in ("pq", "sq", "flash"):
        sections["codes"] = provider.core_arrays()["codes"]
    write_sections(path, meta, sections)


def write_sections(path, meta: dict, sections: dict) -> None:
    """The container itself: meta (JSON, sorted keys) + named arrays in order."""
    mb = json.dumps(meta, sort_keys=True).encode()
    with open(path, "wb") as f:
        f.write(MAGIC)
        f.write(struct.pack("<I", VERSION))
        f.write(struct.pack("<I", len(mb)))
        f.write(mb)
        f.write(struct.pack("<I", len(sections)))
        for name, arr in sections.items():
            _put_array(f, name, arr)


def read_sections(path) -> tuple[dict, dict]:
    """(meta, sections) of an index file, without touching the device."""
    with open(path, "rb") as f:
        if f.read(8) != MAGIC:
            raise FormatError(f"{path}: not an index file")
        (version,) = _get(f, "<I")
        if version != VERSION:
            raise FormatError(f"{path}: unsupported index version {version} (expected {VERSION})")
        (mlen,) = _get(f, "<I")
        meta = json.loads(f.read(mlen).decode())
        (count,) = _get(f, "<I")
        sections = dict(_get_array(f) for _ in range(count))
    return meta, sections


def load_index(path):
    """(graph, provider, dataset) with the graph resident on the device: the
    provider is re-attached (GPU projection + encode), the stored codes and
    blocks are imported into a device index."""
    import torch

    meta, sec = read_sections(path)
    if meta["strategy"] not in ("flash", "exact"):
        raise FormatError(f"{path}: strategy {meta['strategy']!r} is not served by this package")
    state = dict(meta["provider_scalars"])
    state.update({k[5:]: v for k, v in sec.items() if k.startswith("prov.")})
    dataset = VectorDataset(sec["vectors"])
    if meta["strategy"] == "exact":
        from .exact import ExactProvider

        provider = ExactProvider.from_state(state)
        provider.attach(dataset)
    else:
        provider = FlashProvider.from_state(state)
        provider.attach(dataset)
        codes = np.ascontiguousarray(sec["codes"], dtype=np.uint8)
        provider.dev["codes"][:, : codes.shape[1]].copy_(torch.from_numpy(codes).cuda())
    params = BuildParams(C=meta["C"], R=meta["R"], seed=meta["seed"], threads=meta["threads"])
    g = GraphIndex(meta["n"], meta["dim"], params, meta["strategy"], meta["code_subspaces"],
                   sec["levels"])
    g.create_device(provider)
    base = np.ascontiguousarray(sec["base_blocks"])
    upper = np.ascontiguousarray(sec["upper_blocks"])
    bd = torch.from_numpy(base).cuda()
    ud = torch.from_numpy(upper).cuda() if upper.size else torch.zeros(1, dtype=torch.uint8,
                                                                      device="cuda")
    _lib.check(_lib.load().fa_index_import_blocks(
        g.handle, bd.data_ptr(), base.shape[1], ud.data_ptr(),
        upper.shape[1] if upper.ndim == 2 else 0, None))
    torch.cuda.synchronize()
    g.entry_point, g.max_layer = int(meta["entry_point"]), int(meta["max_layer"])
    g._blocks = (base, upper)
    return g, provider, dataset
