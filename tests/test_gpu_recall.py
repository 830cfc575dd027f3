"""North-star recall bar at config 1, driver-visible.

The reference's compiled build_graph at threads = 1 (oracle/_ref, the
deterministic reference graph) and the default batched GPU build run on the
same config-1 data with the same coder, for seeds 0 .. 5; the reference's
compiled search_batch searches both graphs (oracle/recall.py).  The GPU graph
must not lose more than 0.5 recall@10 points (mean over the seeds) on Flash
search (ef 64), Flash + rerank 64, or exact-distance search over the graph.
Six seeds, not three: one HNSW build's exact-search recall varies by several
points from seed to seed for either builder (0.52 .. 0.63 at this config), so
a 3-seed mean cannot resolve a 0.5-point bar.
Queries: 2,000 fresh draws from config 1's mixture (the config names 200;
more queries make the 0.5-point bar resolvable: ~0.3 points of sampling error
per seed instead of ~0.9).
"""

import json

import numpy as np
import pytest

from oracle import recall, refpkg

pytestmark = pytest.mark.gpu

BAR = 0.005  # 0.5 recall@10 points


def test_config1_recall_parity(cuda):
    if refpkg.load_ref_core() is None:
        pytest.fail("oracle/_ref reference core missing (make -C oracle ref)")
    per_seed = [recall.build_pair(1, 20_000, 2000, s, threads=1, search_threads=16)
                for s in range(6)]
    summ = recall.summarize(per_seed)
    print(json.dumps(summ))
    ref, gpu = summ["reference"], summ["gpu"]
    for tag in ("flash", "rerank64", "exact"):
        assert gpu[tag]["mean"] >= ref[tag]["mean"] - BAR, (tag, ref[tag], gpu[tag])
    # Flash-only recall is ~3 %: there the bar is two-sided
    assert abs(gpu["flash"]["mean"] - ref["flash"]["mean"]) <= BAR
