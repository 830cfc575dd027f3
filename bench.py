#!/usr/bin/env python
"""Benchmark: Flash HNSW build throughput on one B200 (BASELINE configs).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Headline workload (BASELINE.json configs[1]): 1,000,000 x 128 float32
(256-component mixture, rounded and clipped to 0..255; seeded synthetic),
m = 64 subspaces x 4-bit, uint8 tables, M = 32 (R), efConstruction = 200 (C).

A "step" is one pass of the hot path over the whole input: project + encode
every vector and insert all of them with the batched GPU build (the
reference's graph_seconds: attach + build_graph).  The coder is trained once
on the GPU before the timed region (reported as coding_seconds, k-means at the
reference's default 25 iterations).  Inputs are resident in HBM when the
timed region starts; the working set (vectors 0.5 GB, adjacency 0.3 GB, codes
64 MB, visits spread over all of it) exceeds the 126 MB L2, so no flush is
needed between steps.

value  = vectors inserted per second (all ranks) — device time, CUDA events.
e2e    = the same metric through the reference-facing host-array drop-in
         (sm100.build_graph: numpy in, reference-layout blocks out), H2D/D2H
         inside the timed region.
roofline (dominant kernel = the build's search kernel) and a standalone block
scan (K1) at the config's block shape, each against MEASURED_PEAKS.json, with
the reference's own fa_batch_lanes (OpenMP, all host cores) timed beside it.
cpu_baseline: the reference's own compiled core (oracle/_ref, OpenMP on all
host cores) building a bounded prefix of the same data.
configs: the other BASELINE workloads at full size, device-timed (config 5 =
the dynamic rebuild: 4M bf16 vectors inserted in 65,536-vertex batches onto
an existing 1M-vector graph), each with its roofline; pca_gemm: the K9
tensor-core contractions (covariance, projection) at configs 4 and 5.

N > 1 (torchrun): "replicas only" — each rank builds its own full index; no
collective on the data path; value = total vectors / max time.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CFG = 2
KMEANS_ITERS = 25  # the reference's default (builder.py StrategyParams.kmeans_iters)
METRIC = "HNSW build vectors/sec and code-distance evals/sec (% HBM roofline), 1 B200"


def load_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.path = Path(f"/tmp/fa_clocks_{os.getpid()}.csv")

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        if not self.path.exists():
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        rows = [r.split(", ") for r in self.path.read_text().strip().splitlines() if r]
        sm = [float(r[1]) for r in rows if len(r) > 8 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if len(r) > 8 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows if len(r) > 8 for i in range(4)
                          if r[5 + i].strip().lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(rows)}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def ref_cpu_build(prov_full, levels_fn, n_sub, C, R, threads):
    """The reference's compiled build_graph on the first n_sub vectors.
    Returns (seconds, vec/s)."""
    from oracle import refpkg
    from paper_2502_18113_b200 import layout

    core = refpkg.load_ref_core()
    if core is None:
        return None
    m = prov_full["cent"].shape[0]
    prov = dict(prov_full)
    prov["proj"] = np.ascontiguousarray(prov_full["proj"][:n_sub])
    prov["vecs"] = np.ascontiguousarray(prov_full["vecs"][:n_sub])
    prov["codes"] = np.ascontiguousarray(prov_full["codes"][:n_sub]).copy()
    levels = levels_fn(n_sub)
    lv64 = levels.astype(np.int64)
    uoff = np.where(lv64 > 0, np.cumsum(lv64) - lv64, -1)
    base = layout.empty_rows(n_sub, 2 * R, m)
    upper = layout.empty_rows(int(lv64.sum()), R, m)
    t0 = time.perf_counter()
    core.build_graph(4, prov, levels, base, uoff, upper, C, R, threads=threads,
                     kernel=len(core.available_kernels()) - 1)
    dt = time.perf_counter() - t0
    return dt, n_sub / dt


def size_cpu_sample(build, n_max, target_s, n0=20_000):
    """Grow a prefix by doubling until one reference build takes at least
    target_s / 2 (the CPU rate falls steeply with n once the graph leaves the
    caches, so a small calibration cannot be extrapolated).  Returns
    (n, seconds, vec/s) of the last build, or None."""
    n = min(n_max, n0)
    r = build(n)
    if r is None:
        return None
    while r[0] < target_s / 2.0 and n < n_max:
        n = min(n_max, 2 * n)
        r = build(n)
    return n, r[0], r[1]


def cpu_prov(data, model):
    """Reference-shaped prov dict from a trained model (host arrays)."""
    proj = model["proj_fn"](data)
    return {"vecs": data, "dim": data.shape[1], "proj": proj,
            "codes": np.zeros((data.shape[0], model["cent"].shape[0]), np.uint8),
            "cent": model["cent"], "dims": model["dims"], "offs": model["offs"],
            "sdt": model["sdt"], "dist_min": model["dist_min"],
            "delta": model["dist_max"] - model["dist_min"]}


def run_reference(args):
    """--impl reference: the reference's CPU build on bounded samples."""
    world, rank, _ = dist_setup()
    if rank != 0:
        return
    from oracle import refpkg, train_np
    from paper_2502_18113_b200 import dataset, graph

    c = dataset.CONFIGS[CFG]
    threads = os.cpu_count() or 1
    if refpkg.load_ref_core() is None:
        print(json.dumps({"impl": "reference", "unavailable":
                          "oracle/_ref not built (make -C oracle ref needs /root/reference)"}))
        return
    # prefix-stable generator: these are exactly the first ref_max rows of the
    # GPU arm's workload
    data, _ = dataset.baseline_config(CFG, n=args.ref_max, nq=0)
    model = train_np.train(train_np.training_sample(data, 100_000, 0), c["d_f"], c["m_f"], 0, 25)
    prov = cpu_prov(data, model)
    lvf = lambda k: graph.assign_layers(k, 0, c["M"])  # noqa: E731
    # size each step so the whole run stays within ~3 minutes
    steps = args.steps + args.warmup
    n_sub = size_cpu_sample(lambda k: ref_cpu_build(prov, lvf, k, c["efC"], c["M"], threads),
                            args.ref_max, 150.0 / steps)[0]
    for _ in range(args.warmup):
        ref_cpu_build(prov, lvf, n_sub, c["efC"], c["M"], threads)
    times = [ref_cpu_build(prov, lvf, n_sub, c["efC"], c["M"], threads)[0]
             for _ in range(args.steps)]
    ms = 1000.0 * float(np.mean(times))
    value = n_sub / (ms / 1000.0)
    sample = (f"first {n_sub} of {c['n']} config-2 vectors (the same rows as the GPU arm's "
              f"prefix; CPU throughput falls with n, so this favours the CPU), "
              f"reference compiled build_graph threads={threads}")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": "vectors/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8",
        "data": "synthetic (seeded config-2 mixture, no dataset download)",
        # the same workload as our arm; each step times the first n rows of it
        # (n_workload = the full workload's size; cpu_baseline.sample)
        "config": {"workload": f"config{CFG}", "n": n_sub, "n_workload": c["n"],
                   "dim": c["dim"], "M": c["M"], "efConstruction": c["efC"], "m": c["m_f"],
                   "subspace_bits": 4, "prefix": True},
        "cpu_baseline": {"value": value, "unit": "vectors/s", "cores": threads,
                         "kind": "reference", "sample": sample},
        "e2e": {"value": value, "unit": "vectors/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }))


def load_traffic():
    """Per-launch DRAM bytes of the roofline kernels from the newest committed
    ncu capture summary (profiles/*_traffic.json), or {}."""
    files = sorted((ROOT / "profiles").glob("*_traffic.json"))
    return json.loads(files[-1].read_text()) if files else {}


def load_k4_issue():
    """Issue-slot roofline of K4 from the newest committed ncu capture summary
    (profiles/*_k4_roofline.json), or None."""
    files = sorted((ROOT / "profiles").glob("*_k4_roofline.json"))
    if not files:
        return None
    d = json.loads(files[-1].read_text())
    return {"bound": "issue", "issue_active_frac": d["issue_active_frac"],
            "warp_inst_per_expansion": d["warp_inst_per_expansion"],
            "lts_bytes_per_s": d["lts_bytes_per_s"],
            "lts_sector_frac_of_peak": d["lts_sector_frac_of_peak"],
            "l2_hit_rate": d["l2_hit_rate"], "warps_active": d["warps_active"],
            "source": files[-1].name}


def query_benchmark(torch, g, provider, data, queries, reps=3):
    """§8(f) row 1: search_batch over the built graph (K2 query tables + K8),
    device-resident queries, ef 64, k 10; recall@10 against GPU brute force."""
    from paper_2502_18113_b200 import dataset, evaluation

    gt = dataset.brute_force_knn(data, queries, 10)
    q_dev = torch.from_numpy(queries).cuda()
    res = {"queries": int(queries.shape[0]), "ef": 64, "k": 10}
    for tag, rr in (("flash", 0), ("rerank64", 64)):
        sp = evaluation.SearchParams(ef=64, k=10, rerank_depth=rr)
        for _ in range(2):
            evaluation.search_batch_dev(g, provider, q_dev, sp)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            ids, _, _ = evaluation.search_batch_dev(g, provider, q_dev, sp)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        res[tag] = {"qps": queries.shape[0] / (ms * 1e-3), "ms": ms,
                    "recall@10": evaluation.recall_at_k(ids.cpu().numpy(), gt)}
    return res


def scan_benchmark(lib, torch, m, cap, peak, reps=5):
    """Standalone K1 block scan over a > L2 padded block array."""
    from paper_2502_18113_b200._lib import check

    nb = (cap + 15) // 16
    codes_off = 16 + 4 * cap
    codes_off = (codes_off + 15) // 16 * 16
    stride = (codes_off + nb * m * 16 + 127) // 128 * 128
    nblocks = 1_000_000
    g = torch.Generator(device="cuda").manual_seed(1)
    blocks = torch.randint(0, 16, (nblocks, stride), dtype=torch.uint8, device="cuda",
                           generator=g)
    v = blocks[:, :16].view(torch.int32)
    v[:, 0] = cap  # full blocks
    ids = blocks[:, 16: 16 + 4 * cap].view(torch.int32)
    ids.copy_(torch.randint(0, nblocks, ids.shape, dtype=torch.int32, device="cuda",
                            generator=g))
    nq, ns = 4096, 256
    adt = torch.randint(0, 8, (nq, m, 16), dtype=torch.uint8, device="cuda", generator=g)
    sel = torch.randint(0, nblocks, (nq, ns), dtype=torch.int32, device="cuda", generator=g)
    out = torch.empty(nq, dtype=torch.int64, device="cuda")
    lanes = nq * ns * nb * 16
    alg_bytes = nq * ns * (4 + nb * 16 * (m + 4))  # count + per batch: ids + codes
    res = {}
    for name, fn in (("scan_select_kernel (K1, direct loads)", lib.fa_scan_select_dev),
                     ("scan_select_tma_kernel (K1, TMA bulk-staged)", lib.fa_scan_select_tma_dev)):
        call = lambda: check(fn(  # noqa: E731
            adt.data_ptr(), nq, blocks.data_ptr(), nblocks, stride, codes_off, cap, m,
            sel.data_ptr(), ns, out.data_ptr(), None))
        for _ in range(3):
            call()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            call()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        gbs = alg_bytes / (ms * 1e-3) / 1e9
        res[name] = {"kernel": name, "evals_per_s": lanes / (ms * 1e-3), "ms_per_launch": ms,
                     "bytes_per_launch": alg_bytes, "achieved": gbs, "peak": peak,
                     "unit": "GB/s", "frac": gbs / peak}
    cpu = scan_cpu_baseline(torch, blocks, stride, codes_off, cap, m, adt, nb)
    del blocks
    best = max(res.values(), key=lambda r: r["achieved"])
    # ncu DRAM bytes of one launch of the TMA variant at the config-2 shape
    tr = load_traffic().get("scan_select_tma_kernel")
    traffic = None
    if tr and tr.get("algorithmic_bytes") == alg_bytes and "tma" in best["kernel"]:
        traffic = tr["dram_bytes"]
    return dict(best, bound="hbm", traffic=traffic,
                shape=f"m={m} cap={cap}, {nq} queries x {ns} random blocks of {nblocks} "
                      f"(working set {nblocks * stride / 1e9:.2f} GB > L2)",
                variants={k: {"achieved": v["achieved"], "frac": v["frac"],
                              "ms_per_launch": v["ms_per_launch"]} for k, v in res.items()},
                cpu_baseline=cpu)

def scan_cpu_baseline(torch, blocks, stride, codes_off, cap, m, adt, nb, target_s=6.0):
    """The reference's own fa_batch_lanes (its widest ISA kernel, OpenMP on all
    host cores; oracle/scan_bench.c against _simd.h:180-197) over the same
    block layout and tables: a host copy of the first 262,144 blocks (> the
    host's L3), random selections, sized to ~target_s seconds."""
    import ctypes as C

    from oracle import refpkg

    if not refpkg.SCAN_SO.exists():
        return None
    lib = C.CDLL(str(refpkg.SCAN_SO))
    lib.scan_bench.restype = C.c_int64
    lib.scan_bench.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int64, C.c_int64, C.c_int,
                               C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_int]
    lib.scan_bench_widest_kernel.restype = C.c_int
    kern = lib.scan_bench_widest_kernel()
    nblk = min(262_144, blocks.shape[0])
    hb = blocks[:nblk].cpu().numpy()
    ha = adt.cpu().numpy()
    threads = os.cpu_count() or 1
    rng = np.random.default_rng(7)
    ns = 256

    def run(nq):
        sel = rng.integers(0, nblk, size=(nq, ns), dtype=np.int32)
        out = np.empty(nq, np.uint64)
        t0 = time.perf_counter()
        lanes = lib.scan_bench(ha.ctypes.data, nq, hb.ctypes.data, stride, codes_off, cap, m,
                               sel.ctypes.data, ns, out.ctypes.data, threads, kern)
        return lanes, time.perf_counter() - t0

    nq = ha.shape[0]
    lanes, dt = run(nq)  # warm-up and calibration
    reps = max(1, int(target_s / max(dt, 1e-6)))
    lanes, dt = 0, 0.0
    for _ in range(reps):
        lr, tr = run(nq)
        lanes += lr
        dt += tr
    evals = lanes / dt
    bytes_s = reps * nq * ns * (4 + nb * 16 * (m + 4)) / dt
    return {"evals_per_s": evals, "gbs": bytes_s / 1e9, "cores": threads, "kind": "reference",
            "kernel": ["scalar", "vector128", "vector256", "vector512"][kern],
            "sample": f"{reps} x {nq} queries x {ns} random blocks of {nblk} (host copy, "
                      f"{nblk * stride / 1e9:.2f} GB), {dt:.1f} s"}


def _device_sample(torch, x, size, seed=0):
    """training_sample (builder.py:60-65 semantics) of device rows: `size` rows
    in ascending order, chosen without replacement by a seeded device RNG."""
    n = x.shape[0]
    if n <= size:
        return x
    g = torch.Generator(device="cuda").manual_seed(seed)
    sel = torch.randperm(n, generator=g, device="cuda")[:size].sort().values
    return x[sel].contiguous()


def config_leg(cfg, torch, peak, tf32_peak, steps=2, warmup=3, cpu_seconds=0.0):
    """One BASELINE workload at full size, device-timed.  Configs 1/3/4: full
    builds (project + encode + insert every vector) as the headline.  Config
    5 (dynamic rebuild): each step first rebuilds the existing 1M-vector graph
    (untimed), then times projecting + encoding the 4M arriving bf16 vectors
    and inserting them in 65,536-vertex batches onto it."""
    from paper_2502_18113_b200 import _lib, builder, dataset, flash, graph, pca

    lib = _lib.load()
    c = dataset.CONFIGS[cfg]
    n = c["n"]
    t0 = time.perf_counter()
    x = dataset.baseline_config_dev(cfg, n)
    torch.cuda.synchronize()
    gen_s = time.perf_counter() - t0
    sample = _device_sample(torch, x, builder.DEFAULT_SAMPLE)
    model = flash.flash_train(sample, c["d_f"], c["m_f"], seed=0, kmeans_iters=KMEANS_ITERS)
    params = graph.BuildParams(C=c["efC"], R=c["M"], seed=0)
    levels = graph.assign_layers(n, 0, c["M"])
    provider = flash.FlashProvider(model)
    provider.attach(x, vecs_dev=x)
    g = graph.GraphIndex(n, c["dim"], params, "flash", model.m, levels)
    g.create_device(provider)
    split = 1_000_000 if cfg == 5 else 0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def step(profile=0):
        if split:
            provider.reproject(0, split)
            _lib.check(lib.fa_index_set_codes(g.handle, provider.dev["codes"].data_ptr(),
                                              provider.dev["codes"].shape[1], None))
            builder.build_device(g, provider, params, end=split)
            torch.cuda.synchronize()
            e0.record()
            provider.reproject(split, n)
            _lib.check(lib.fa_index_set_codes(g.handle, provider.dev["codes"].data_ptr(),
                                              provider.dev["codes"].shape[1], None))
            r = builder.build_device(g, provider, params, start=split, profile=profile)
            e1.record()
        else:
            torch.cuda.synchronize()
            e0.record()
            provider.reproject()
            _lib.check(lib.fa_index_set_codes(g.handle, provider.dev["codes"].data_ptr(),
                                              provider.dev["codes"].shape[1], None))
            r = builder.build_device(g, provider, params, profile=profile)
            e1.record()
        torch.cuda.synchronize()
        return r, e0.elapsed_time(e1)

    for _ in range(warmup):
        step()
    times, ctr = [], None
    for _ in range(steps):
        ctr, ms = step()
        times.append(ms)
    ms = float(np.mean(times))
    ninsert = n - split
    prof, _ = step(profile=1)
    mp = c["m_f"]
    evals = 16 * prof["kernel_calls"]
    sbytes = evals * (mp + 4) + prof["visited"] * 4
    gbs = sbytes / (prof["ms_search"] * 1e-3) / 1e9
    kernel_ms = {"encode": prof["ms_encode"], "search": prof["ms_search"],
                 "sort": prof["ms_sort"], "reverse": prof["ms_reverse"]}
    leg = {"workload": f"config{cfg}", "n": n, "dim": c["dim"], "M": c["M"],
           "efConstruction": c["efC"], "m": mp, "d_f": c["d_f"],
           "dtype_in": "bf16" if cfg == 5 else "f32",
           "data": "synthetic, generated on the device (dataset.baseline_config_dev: the "
                   "config's law, seeded)",
           "value": ninsert / (ms * 1e-3), "unit": "vectors/s", "ms_per_step": ms,
           "steps": steps, "warmup": warmup, "generated_s": gen_s,
           "kernel_ms_per_step": kernel_ms,
           "counters": {k: ctr[k] for k in ("dist_comps", "visited", "kernel_calls",
                                            "reverse_prunes", "n_batches")},
           "gpu_launches": int(ctr["launches"]),
           "roofline": {"bound": "hbm", "kernel": "build_search_kernel (K4+K5)",
                        "achieved": gbs, "peak": peak, "unit": "GB/s", "frac": gbs / peak,
                        "traffic": None, "evals_per_s": evals / (prof["ms_search"] * 1e-3),
                        "bytes_basis": "SURVEY 8(d): 16 x kernel_calls x (m + 4) B + 4 B "
                                       "per block",
                        "kernel_share": prof["ms_search"] / max(sum(kernel_ms.values()), 1e-9),
                # what actually bounds K4: issue slots and L2
                # latency, not HBM — from the committed ncu capture
                "issue_roofline": load_k4_issue()}}
    if split:
        leg["timed"] = (f"project + encode + insert vectors {split}..{n} in batches of "
                        f"{builder.build_options(params).batch_max} onto the existing "
                        f"{split}-vector graph (rebuilt untimed before each step)")
    if cfg in (4, 5):
        # K9 at this config's shapes: the training covariance and the full
        # projection (the timed steps above include the projection)
        mean = torch.from_numpy(model.pca.mean.astype(np.float32)).cuda()

        def ktime(fn, reps=3):
            fn()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(reps):
                fn()
            b.record()
            torch.cuda.synchronize()
            return a.elapsed_time(b) / reps

        ms_cov = ktime(lambda: pca.covariance_dev(sample, mean))
        ms_proj = ktime(lambda: pca.pca_project_all_dev(model.pca, x))
        D, d = c["dim"], c["d_f"]
        ns = sample.shape[0]
        # flops of the tiles the kernel computes (covariance: the upper
        # triangle of 128 x 128 tiles incl. the diagonal); the tensor core
        # issues 3x that (3xTF32)
        nbk = -(-D // 128)
        fl_cov = 2.0 * 128 * 128 * ns * nbk * (nbk + 1) / 2
        fl_proj = 2.0 * n * D * d
        leg["pca_gemm"] = {
            "kernel": "pca_gemm_kernel (K9, 3xTF32 tcgen05, TMA)", "bound": "tensor",
            "unit": "TFLOP/s", "peak": tf32_peak,
            "peak_basis": "MEASURED_PEAKS bf16_tflops / 2 (dense tf32 rate)",
            "covariance": {"rows": ns, "D": D, "ms": ms_cov,
                           "achieved": 3 * fl_cov / (ms_cov * 1e9),
                           "frac": 3 * fl_cov / (ms_cov * 1e9) / tf32_peak},
            "projection": {"rows": n, "D": D, "d": d, "ms": ms_proj,
                           "achieved": 3 * fl_proj / (ms_proj * 1e9),
                           "frac": 3 * fl_proj / (ms_proj * 1e9) / tf32_peak,
                           "hbm_gbs": x.element_size() * n * D / (ms_proj * 1e6)},
            "flops_basis": "tensor-core flops issued = 3 x useful (hi*hi, lo*hi, hi*lo)"}
    if cpu_seconds > 0:
        lvf = lambda k: graph.assign_layers(k, 0, c["M"])  # noqa: E731
        ncap = 400_000
        pv = {"vecs": x[:ncap].float().cpu().numpy(), "dim": c["dim"],
              "proj": provider.dev["proj"][:ncap].cpu().numpy(),
              "codes": np.ascontiguousarray(provider.dev["codes"][:ncap, :mp].cpu().numpy()),
              "cent": model.cent, "dims": model.dims, "offs": model.offs, "sdt": model.sdt,
              "dist_min": model.dist_min, "delta": model.delta}
        threads = os.cpu_count() or 1
        r = size_cpu_sample(lambda k: ref_cpu_build(pv, lvf, k, c["efC"], c["M"], threads),
                            ncap, cpu_seconds)
        if r is not None:
            n_cpu, dt, rate = r
            leg["cpu_baseline"] = {
                "value": rate, "unit": "vectors/s", "cores": threads, "kind": "reference",
                "sample": f"first {n_cpu} vectors built from scratch (the CPU cannot build the "
                          f"1M base in-run), same coder, reference compiled build_graph, "
                          f"OpenMP threads={threads}, {dt:.1f} s"}
    g.close()
    del provider, g, x, sample
    torch.cuda.empty_cache()
    return leg


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=None, help="override vector count")
    ap.add_argument("--ref-max", type=int, default=200_000)
    ap.add_argument("--cpu-seconds", type=float, default=20.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-search", action="store_true", help="skip the query-search leg")
    ap.add_argument("--configs", default="1,3,4,5",
                    help="other BASELINE configs to time at full size ('' = none)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)

    import torch

    world, rank, local = dist_setup()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2502_18113_b200 import _lib, builder, dataset, flash, graph, layout, sm100

    lib = _lib.load()
    c = dataset.CONFIGS[CFG]
    n = args.n or c["n"]
    peak, peak_kind = load_peaks()
    data, queries = dataset.baseline_config(CFG, n=n, nq=0 if args.no_search else c["nq"])
    x_dev = torch.from_numpy(data).cuda()

    # coder training on the GPU (coding_seconds).  The first call in a process
    # also pays the cuBLAS / cuSOLVER handle set-up (coding_seconds_cold); the
    # reported figure is the second, identical call.
    coding = []
    for _ in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        sample = builder.training_sample(data, builder.DEFAULT_SAMPLE, 0)
        model = flash.flash_train(sample, c["d_f"], c["m_f"], seed=0, kmeans_iters=KMEANS_ITERS)
        torch.cuda.synchronize()
        coding.append(time.perf_counter() - t0)
    coding_s = coding[-1]

    params = graph.BuildParams(C=c["efC"], R=c["M"], seed=0)
    levels = graph.assign_layers(n, 0, c["M"])
    provider = flash.FlashProvider(model)
    provider.attach(data, vecs_dev=x_dev)
    g = graph.GraphIndex(n, data.shape[1], params, "flash", model.m, levels)
    g.create_device(provider)

    def step(profile=0):
        provider.reproject()  # project + encode every vector (device, in place)
        _lib.check(lib.fa_index_set_codes(g.handle, provider.dev["codes"].data_ptr(),
                                          provider.dev["codes"].shape[1], None))
        return builder.build_device(g, provider, params, profile=profile)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        e0.record()
        ctrs = [step() for _ in range(args.steps)]
        e1.record()
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()
    value = n * world / (ms / 1000.0)

    # per-kernel device times (one extra profiled step, outside the timed region)
    prof = step(profile=1)
    kernel_ms = {"encode": prof["ms_encode"], "search": prof["ms_search"],
                 "sort": prof["ms_sort"], "reverse": prof["ms_reverse"]}
    cap0, mpad = 2 * c["M"], (c["m_f"] + 15) // 16 * 16
    # algorithmic bytes per SURVEY §8(d): one unit = one 16-lane batch
    # evaluation of a neighbour block = 16 (m + 4) B, plus 4 B of count per
    # block; units = 16 x the reference's kernel_calls counter (the build
    # counts it exactly as the reference does, ceil(live / 16) per expansion)
    evals = 16 * prof["kernel_calls"]
    search_bytes = evals * (c["m_f"] + 4) + prof["visited"] * 4
    search_gbs = search_bytes / (prof["ms_search"] * 1e-3) / 1e9
    # what this kernel actually has to read: an id row per expansion and the
    # code row of each fresh (unvisited) neighbour only
    touched = prof["visited"] * cap0 * 4 + prof["dist_comps"] * c["m_f"]
    # DRAM bytes per build at the captured launch's bytes per inserted vector
    tr = load_traffic().get("build_search_kernel")
    search_traffic = int(tr["dram_bytes"] / tr["vectors"] * n) if tr else None
    roofline = {"bound": "hbm", "kernel": "build_search_kernel (K4+K5)",
                "achieved": search_gbs, "peak": peak, "unit": "GB/s",
                "frac": search_gbs / peak, "traffic": search_traffic, "peak_kind": peak_kind,
                "bytes_per_build": search_bytes,
                "evals_per_s": evals / (prof["ms_search"] * 1e-3),
                "bytes_basis": "SURVEY 8(d): 16 x kernel_calls x (m + 4) B + 4 B per block",
                "touched_bytes_per_build": touched,
                "touched_frac": touched / (prof["ms_search"] * 1e-3) / 1e9 / peak,
                "traffic_basis": "per build: ncu DRAM bytes per inserted vector of one captured "
                                 "launch x n (profiles/*_traffic.json)",
                "kernel_share": prof["ms_search"] / max(sum(kernel_ms.values()), 1e-9),
                # what actually bounds K4: issue slots and L2
                # latency, not HBM — from the committed ncu capture
                "issue_roofline": load_k4_issue()}

    out = {"metric": METRIC, "value": value, "unit": "vectors/s", "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8",
           "data": "synthetic (seeded config-2 mixture, no dataset download)",
           "config": {"workload": f"config{CFG}", "n": n, "dim": c["dim"], "M": c["M"],
                      "efConstruction": c["efC"], "m": c["m_f"], "subspace_bits": 4,
                      "parallelism": f"replicas x{world}",
                      "l2": "inputs larger than L2 (no flush)",
                      "batch": {k: v for k, v in sm100.BUILD_OPTIONS.items() if k != "profile"}},
           "coding_seconds": coding_s, "coding_seconds_cold": coding[0],
           "coding_kmeans_iters": KMEANS_ITERS,
           "kernel_ms_per_build": kernel_ms,
           "counters": {k: ctrs[-1][k] for k in ("dist_comps", "sym_comps", "visited",
                                                  "kernel_calls", "reverse_prunes",
                                                  "reverse_appends", "n_batches")},
           "gpu_launches": int(ctrs[-1]["launches"] + 1) * args.steps,
           "roofline": roofline, "clocks": clk.summary()}

    if rank == 0:
        out["scan"] = scan_benchmark(lib, torch, c["m_f"], cap0, peak)
        # the same K1 scan at the other configs' block shapes (c1, c3, c5)
        out["scan_other_shapes"] = {}
        for cfg_o in (1, 3, 5):
            co = dataset.CONFIGS[cfg_o]
            r = scan_benchmark(lib, torch, co["m_f"], 2 * co["M"], peak, reps=3)
            out["scan_other_shapes"][f"config{cfg_o}"] = {
                "m": co["m_f"], "cap": 2 * co["M"], "kernel": r["kernel"],
                "achieved": r["achieved"], "frac": r["frac"], "evals_per_s": r["evals_per_s"]}
        if not args.no_search:
            out["search"] = query_benchmark(torch, g, provider, data, queries)
        if not args.no_e2e:
            prov = provider.core_arrays()
            prov = dict(prov, codes=prov["codes"].copy())
            base = layout.empty_rows(n, cap0, model.m)
            upper = layout.empty_rows(g.n_upper_rows, c["M"], model.m)
            h2d = prov["proj"].nbytes + prov["codes"].nbytes + levels.nbytes + \
                g.upper_offsets.nbytes + model.cent.nbytes + model.sdt.nbytes
            d2h = prov["codes"].nbytes + base.nbytes + upper.nbytes
            # one untimed call (pinned staging pool, allocator warm-up), then
            # the timed calls: each uploads its inputs and reads back all rows
            e2e_steps = max(1, min(args.steps, 3))
            for it in range(1 + e2e_steps):
                if it == 1:
                    torch.cuda.synchronize()
                    t1 = time.perf_counter()
                sm100.build_graph(4, prov, levels, base, g.upper_offsets, upper, c["efC"],
                                  c["M"])
            torch.cuda.synchronize()
            e2e_s = (time.perf_counter() - t1) / e2e_steps
            out["e2e"] = {"value": n / e2e_s, "unit": "vectors/s", "h2d_bytes_per_step": h2d,
                          "d2h_bytes_per_step": d2h, "seconds": e2e_s, "steps": e2e_steps,
                          "api": "sm100.build_graph (host numpy arrays, reference layout)"}
        if not args.no_cpu_baseline:
            from oracle import train_np

            threads = os.cpu_count() or 1
            pm = {"proj_fn": None, "cent": model.cent, "dims": model.dims, "offs": model.offs,
                  "sdt": model.sdt, "dist_min": model.dist_min, "dist_max": model.dist_max}
            cprov = provider.core_arrays()
            lvf = lambda k: graph.assign_layers(k, 0, c["M"])  # noqa: E731
            # bounded sample: the largest doubling of a 20K prefix whose build
            # stays near cpu_seconds
            r = size_cpu_sample(
                lambda k: ref_cpu_build(cprov, lvf, k, c["efC"], c["M"], threads), n,
                args.cpu_seconds)
            if r is None:
                out["cpu_baseline"] = None
            else:
                n_cpu, dt, rate = r
                out["cpu_baseline"] = {
                    "value": rate, "unit": "vectors/s", "cores": threads, "kind": "reference",
                    "sample": f"first {n_cpu} of {n} vectors (prefix, same model), reference "
                              f"compiled build_graph, OpenMP threads={threads}, {dt:.1f} s"}
            del pm, train_np
        # the other BASELINE workloads at full size (after the headline, so
        # its timed region and clock samples are untouched)
        peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) \
            if (ROOT / "MEASURED_PEAKS.json").exists() else {}
        tf32_peak = float(peaks.get("bf16_tflops", 2250.0)) / 2.0
        legs = {}
        for cf in [int(v) for v in args.configs.split(",") if v.strip()]:
            legs[f"config{cf}"] = config_leg(
                cf, torch, peak, tf32_peak,
                cpu_seconds=args.cpu_seconds if (cf == 5 and not args.no_cpu_baseline) else 0.0)
        if legs:
            out["configs"] = legs
        print(json.dumps(out))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
