"""Segment model host logic on CPU: world_size 2 over gloo.

Each rank plays one GPU: the coder is broadcast from rank 0, per-segment top-k
lists (local ids, u8 distances with ties, -1/+inf padding) are all-gathered
and merged by (distance, global id); the merge must equal a single-process
merge of the concatenated lists and a brute-force (d, id) sort."""

import os
import socket

import numpy as np
import pytest

from paper_2502_18113_b200 import segments


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _local_results(rank, nq=7, k=5, n_local=40):
    rng = np.random.default_rng(100 + rank)
    ids = np.stack([rng.choice(n_local, size=k, replace=False) for _ in range(nq)]).astype(np.int64)
    d = rng.integers(0, 4, size=(nq, k)).astype(np.float64)  # many ties
    ids[0, 3:] = -1
    d[0, 3:] = np.inf
    return ids, d


def _model():
    from paper_2502_18113_b200.flash import FlashModel
    from paper_2502_18113_b200.pca import PCAModel

    rng = np.random.default_rng(1)
    pca = PCAModel(mean=rng.normal(size=8), basis=np.linalg.qr(rng.normal(size=(8, 8)))[0],
                   eigvals=np.sort(rng.random(8))[::-1].copy(), d=8)
    return FlashModel(pca=pca, m=4, dims=np.full(4, 2, np.int32),
                      offs=np.arange(0, 8, 2, dtype=np.int32),
                      cent=rng.normal(size=(4, 16, 2)).astype(np.float32),
                      sdt=rng.integers(0, 255, size=(4, 16, 16)).astype(np.uint8),
                      dist_min=0.0, dist_max=7.5)


def _worker(rank, world, port, out):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        model = segments.broadcast_model(_model() if rank == 0 else None)
        ref = _model()
        ok_model = (np.array_equal(model.cent, ref.cent) and np.array_equal(model.sdt, ref.sdt)
                    and np.array_equal(model.pca.basis, ref.pca.basis)
                    and model.dist_max == ref.dist_max and model.m == ref.m)
        n_seg = 40
        lo, _ = segments.segment_range(world * n_seg, world, rank)
        ids, d = _local_results(rank)
        gi, gd = segments.merge_topk(torch.from_numpy(ids), torch.from_numpy(d), lo, 5)
        out[rank] = (ok_model, gi.numpy(), gd.numpy())
    finally:
        dist.destroy_process_group()


def test_segment_range_partitions():
    for n, w in ((10, 3), (7, 7), (5, 8), (1000, 4)):
        spans = [segments.segment_range(n, w, r) for r in range(w)]
        assert spans[0][0] == 0 and spans[-1][1] == n
        assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
        assert max(h - lo for lo, h in spans) - min(h - lo for lo, h in spans) <= 1


def test_two_rank_broadcast_and_merge():
    import torch.multiprocessing as mp

    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    # single-process reference: concatenate the global-id lists and sort by (d, id)
    ids = []
    ds = []
    for r in range(world):
        i, d = _local_results(r)
        lo, _ = segments.segment_range(world * 40, world, r)
        ids.append(np.where(i >= 0, i + lo, -1))
        ds.append(d)
    ids, ds = np.concatenate(ids, 1), np.concatenate(ds, 1)
    ei, ed = segments.merge_lists_np(ids, ds, 5)
    for r in range(world):
        ok_model, gi, gd = out[r]
        assert ok_model
        assert np.array_equal(gi, ei) and np.array_equal(gd, ed)
    # brute force: every returned pair is among the k smallest (d, id)
    for row in range(ids.shape[0]):
        pairs = sorted((d, i if i >= 0 else 1 << 62) for d, i in zip(ds[row], ids[row]))[:5]
        assert [p[1] if p[1] != 1 << 62 else -1 for p in pairs] == ei[row].tolist()


@pytest.mark.gpu
def test_segment_indexes_on_one_gpu(cuda):
    """Two segment indexes built and searched on one device, merged; equal to
    the oracle's segment builds + searches merged the same way."""
    import torch

    from oracle import native
    from paper_2502_18113_b200 import flash, graph, layout, sm100

    rng = np.random.default_rng(7)
    data = (rng.normal(size=(16, 16))[rng.integers(0, 16, 1200)]
            + 0.3 * rng.normal(size=(1200, 16))).astype(np.float32)
    q = rng.normal(size=(30, 16)).astype(np.float32)
    model = flash.flash_train(data, 16, 8, seed=0, kmeans_iters=3)
    R, C, k, world = 8, 32, 10, 2
    gids, gds, oids, ods = [], [], [], []
    for r in range(world):
        lo, hi = segments.segment_range(len(data), world, r)
        p = flash.FlashProvider(model)
        p.attach(data[lo:hi])
        prov = p.core_arrays()
        n, m = hi - lo, model.m
        levels = graph.assign_layers(n, r, R)
        uoff = graph.upper_offsets_of(levels)
        base = layout.empty_rows(n, 2 * R, m)
        upper = layout.empty_rows(int(levels.sum()), R, m)
        res = sm100.build_graph(4, prov, levels, base, uoff, upper, C, R)
        qaux = p.query_aux(q)
        ids, ds, _ = sm100.search_batch(4, prov, levels, base, uoff, upper, C, R,
                                        res["entry_point"], res["max_layer"], q, qaux, 32, k, 0)
        gids.append(np.where(ids >= 0, ids + lo, -1))
        gds.append(ds)
        hg = native.HostGraph(levels, uoff, R, m, tie=sm100.BUILD_OPTIONS["tie"])
        o = hg.build(prov["proj"], prov["cent"], prov["dims"], prov["offs"], prov["dist_min"],
                     prov["delta"], prov["sdt"], C, batch_max=sm100.BUILD_OPTIONS["batch_max"],
                     batch_frac=sm100.BUILD_OPTIONS["batch_frac"],
                     seq_prefix=sm100.BUILD_OPTIONS["seq_prefix"])
        hq = native.HostGraph.from_blocks(levels, uoff, base, upper, R, prov["codes"])
        oi, od, _ = hq.search(prov["vecs"], prov["cent"], prov["dims"], prov["offs"],
                              prov["dist_min"], prov["delta"], o["entry_point"], o["max_layer"],
                              q, qaux, 32, k, 0)
        oids.append(np.where(oi >= 0, oi + lo, -1))
        ods.append(od)
    mi, md = segments.merge_lists(torch.from_numpy(np.concatenate(gids, 1)),
                                  torch.from_numpy(np.concatenate(gds, 1)), k)
    ei, ed = segments.merge_lists_np(np.concatenate(oids, 1), np.concatenate(ods, 1), k)
    assert np.array_equal(mi.numpy(), ei) and np.array_equal(md.numpy(), ed)
