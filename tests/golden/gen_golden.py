"""Generate the golden fixtures from the REFERENCE implementation.

Run in the build container (needs /root/reference and `make -C oracle ref`):

    python tests/golden/gen_golden.py

Inputs are regenerated from seeds by the tests (numpy's PCG64 streams are
identical in every container of this image); the files hold the reference's
outputs plus the small models/graphs those outputs depend on.  Everything is
produced by the reference's own code path: its compiled core
(flashann/_kernels/_core.pyx hooks) and its numpy trainer (flashann/flash.py).
"""

from __future__ import annotations

import hashlib
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from oracle import refpkg  # noqa: E402
import golden_inputs as gi  # noqa: E402

OUT = Path(__file__).resolve().parent


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main() -> None:
    fa = refpkg.import_reference()
    if fa is None:
        raise SystemExit("reference not available (needs /root/reference and oracle/_ref)")
    EXT = fa.core.impl
    out = {}

    # fp32 L2 operation tree (_simd.h:44-51 as compiled)
    for d in gi.L2_DIMS:
        a, b = gi.l2_inputs(d)
        out[f"l2_{d}"] = np.array([EXT.l2sq_f32(x, y) for x, y in zip(a, b)])

    # uint8 quantiser (_simd.h:99-107)
    d, dmin, delta = gi.quantize_inputs()
    out["quant"] = EXT.quantize_distance(d, dmin, delta)

    # batch scan (_simd.h:111-197), scalar kernel = semantic definition
    for m in gi.SCAN_MS:
        adts, codes = gi.scan_cases(m)
        ref = EXT.flash_batch_distance_many(adts, codes, 0)
        out[f"scan_{m}_sha"] = np.array(sha(ref))
        out[f"scan_{m}_head"] = ref[:256]
    adt, flat = gi.block_case()
    out["blocks"] = EXT.flash_batch_blocks(adt, flat, 4, 0)

    # trained models (flash.py:63-107) + encoder (_simd.h:211-228)
    for name, spec in gi.MODELS.items():
        data = gi.model_data(spec)
        model = fa.flash_train(fa.VectorDataset(data), d_f=spec["d_f"], m_f=spec["m_f"],
                               seed=spec["seed"], kmeans_iters=spec["iters"])
        pfx = f"model_{name}_"
        out[pfx + "cent"] = model.cent
        out[pfx + "dims"] = model.dims
        out[pfx + "offs"] = model.offs
        out[pfx + "sdt"] = model.sdt
        out[pfx + "range"] = np.array([model.dist_min, model.dist_max])
        out[pfx + "mean"] = model.pca.mean
        out[pfx + "basis"] = model.pca.basis[:, : model.d]
        red = gi.encode_inputs(model.cent, model.dims, spec)
        codes = np.empty((red.shape[0], model.m), np.uint8)
        adts = np.empty((red.shape[0], model.m, 16), np.uint8)
        for r in range(red.shape[0]):
            codes[r], adts[r] = EXT.flash_encode_adt(model.cent, model.dims, model.offs,
                                                     model.dist_min, model.delta, red[r])
        out[pfx + "enc_codes"] = codes
        out[pfx + "enc_adt"] = adts
        # 1-ulp quantisation grid: one level ~ 1 ulp of the distance
        red_u, dmins, deltas = gi.ulp_inputs(model.cent, model.dims, model.offs, spec)
        cu = np.empty((red_u.shape[0], model.m), np.uint8)
        au = np.empty((red_u.shape[0], model.m, 16), np.uint8)
        for r in range(red_u.shape[0]):
            cu[r], au[r] = EXT.flash_encode_adt(model.cent, model.dims, model.offs, dmins[r],
                                                deltas[r], red_u[r])
        out[pfx + "ulp_codes"] = cu
        out[pfx + "ulp_adt"] = au

    # SDT sums (_simd.h:87-95) and selection (_core.pyx:388-408) on model c1s
    spec = gi.MODELS["c1s"]
    prov_codes = gi.select_codes(out["model_c1s_sdt"].shape[0])
    a, b = gi.sdt_pairs(prov_codes)
    out["sdt_sums"] = np.array([EXT.flash_sdt_distance(out["model_c1s_sdt"], x, y)
                                for x, y in zip(a, b)], np.int32)
    prov = {"vecs": np.zeros((prov_codes.shape[0], 1), np.float32), "codes": prov_codes,
            "cent": out["model_c1s_cent"], "dims": out["model_c1s_dims"],
            "offs": out["model_c1s_offs"], "sdt": out["model_c1s_sdt"],
            "proj": np.zeros((prov_codes.shape[0], 1), np.float32), "dist_min": 0.0,
            "delta": 1.0}
    sels = []
    for ids, dists, cap in gi.select_cases(prov_codes, out["model_c1s_sdt"]):
        sels.append(np.array(EXT.select_neighbors(4, prov, ids, dists, cap) + [-2], np.int32))
    out["select_out"] = np.concatenate(sels)

    # a small reference-built graph (threads=1, deterministic) to search on
    g = gi.GRAPH
    data, queries = gi.graph_data()
    res = fa.build(fa.VectorDataset(data), "flash",
                   fa.BuildParams(C=g["C"], R=g["R"], seed=g["seed"], threads=1),
                   fa.StrategyParams(m_f=g["m_f"], d_f=g["d_f"], kmeans_iters=g["iters"]))
    pv = res.provider.core_arrays()
    out["g_proj"] = pv["proj"]
    out["g_qproj"] = res.provider.query_aux(queries)
    out["g_codes"] = pv["codes"]
    out["g_cent"] = pv["cent"]
    out["g_dims"] = pv["dims"]
    out["g_offs"] = pv["offs"]
    out["g_sdt"] = pv["sdt"]
    out["g_range"] = np.array([pv["dist_min"], pv["delta"]])
    out["g_levels"] = res.graph.levels
    out["g_uoff"] = res.graph.upper_offsets
    out["g_base"] = res.graph.base_blocks
    out["g_upper"] = res.graph.upper_blocks
    out["g_state"] = np.array([res.graph.entry_point, res.graph.max_layer])
    gt = fa.brute_force_knn(fa.VectorDataset(data), fa.VectorDataset(queries), 10)
    out["g_gt"] = gt.ids
    recalls = []
    for rr in (0, g["ef"]):
        ids, _, _ = fa.search_batch(res.graph, res.provider, queries,
                                    fa.SearchParams(ef=g["ef"], k=10, rerank_depth=rr))
        recalls.append(fa.evaluation.recall_at_k(ids, gt))
    out["g_ref_recall"] = np.array(recalls)

    # the reference's semantic core (_pycore, ties by vertex id) on that graph:
    # greedy_search_layer results, with the compiled core's fp32 query tables
    hb, hu = out["g_base"], out["g_upper"]
    w = fa._pycore.GraphWriter(4, pv, out["g_levels"], hb, out["g_uoff"], hu, g["C"], g["R"])
    rng = np.random.default_rng(77)
    ents = rng.integers(0, hb.shape[0], size=out["g_qproj"].shape[0])
    rows = []
    for width in gi.PY_WIDTHS:
        for q in range(out["g_qproj"].shape[0]):
            _, adt = EXT.flash_encode_adt(pv["cent"], pv["dims"], pv["offs"], pv["dist_min"],
                                          pv["delta"], out["g_qproj"][q])
            res_q = w.greedy_search_layer({"adt": adt}, int(ents[q]), width, 0)
            rows.append(np.array([u for u, _ in res_q] + [-1] * (width - len(res_q)), np.int32))
    out["py_entries"] = ents
    out["py_search_ids"] = np.concatenate(rows)

    # a full sequential build by the semantic core (fp32 encoder patched in)
    real_enc = fa._pycore.flash_encode_adt
    fa._pycore.flash_encode_adt = lambda c, d, o, a, b, r: EXT.flash_encode_adt(
        c, d, o, a, b, np.asarray(r, np.float32))
    try:
        pb = gi.PY_BUILD
        data = gi.mixture(pb["n"], pb["dim"], pb["clusters"], 900, sigma=0.4, spread=1.0)
        model = fa.flash_train(fa.VectorDataset(data), d_f=pb["d_f"], m_f=pb["m_f"], seed=0,
                               kmeans_iters=5)
        prov = fa.FlashProvider(model)
        prov.attach(fa.VectorDataset(data))
        p2 = prov.core_arrays()
        levels = fa.assign_layers(pb["n"], pb["seed"], pb["R"])
        gi_ = fa.GraphIndex(pb["n"], pb["dim"], fa.BuildParams(C=pb["C"], R=pb["R"]), "flash",
                            model.m, levels)
        o2 = fa._pycore.build_graph(4, p2, levels, gi_.base_blocks, gi_.upper_offsets,
                                    gi_.upper_blocks, pb["C"], pb["R"])
    finally:
        fa._pycore.flash_encode_adt = real_enc
    for k in ("proj", "codes", "cent", "dims", "offs", "sdt"):
        out["pb_" + k] = p2[k]
    out["pb_range"] = np.array([p2["dist_min"], p2["delta"]])
    out["pb_levels"] = levels
    out["pb_uoff"] = gi_.upper_offsets
    out["pb_base"] = gi_.base_blocks
    out["pb_upper"] = gi_.upper_blocks
    out["pb_state"] = np.array([o2["entry_point"], o2["max_layer"]])

    np.savez_compressed(OUT / "reference_golden.npz", **out)
    print("wrote", OUT / "reference_golden.npz", "recall", recalls)


if __name__ == "__main__":
    main()
