"""graph.check_invariants (the reference's structural sweep, graph.py:137-187)
on the reference-built golden graph, then on deliberately broken copies."""

from types import SimpleNamespace

import numpy as np

import golden_inputs as gi
from paper_2502_18113_b200 import graph


def _graph(golden):
    R = gi.GRAPH["R"]
    lv = golden["g_levels"]
    e, ml = (int(x) for x in golden["g_state"])
    return SimpleNamespace(n=len(lv), entry_point=e, max_layer=ml, levels=lv,
                           params=graph.BuildParams(C=gi.GRAPH["C"], R=R),
                           base_blocks=golden["g_base"].copy(),
                           upper_offsets=golden["g_uoff"], upper_blocks=golden["g_upper"].copy())


def _set(blocks, row, slot, value):
    blocks[row, 4 + 4 * slot: 8 + 4 * slot] = np.array([value], np.int32).view(np.uint8)


def test_reference_graph_is_clean(golden):
    assert graph.check_invariants(_graph(golden)) == []


def test_each_violation_is_reported(golden):
    g = _graph(golden)
    R = g.params.R
    _set(g.base_blocks, 3, 0, 3)                                  # self loop
    _set(g.base_blocks, 4, 0, g.n + 7)                            # id out of range
    g.base_blocks[5, :4] = np.array([2 * R + 1], np.int32).view(np.uint8)  # above cap
    top = np.flatnonzero(g.levels >= 1)
    low = int(np.flatnonzero(g.levels == 0)[0])
    row = int(g.upper_offsets[top[0]])
    _set(g.upper_blocks, row, 0, low)                             # neighbor below its layer
    bad = " | ".join(graph.check_invariants(g))
    for what in ("self loop", "out of range", "above cap", "below its layer"):
        assert what in bad, what
    g2 = _graph(golden)
    g2.entry_point = int(np.flatnonzero(g2.levels < g2.max_layer)[0])
    assert "not on the top layer" in " | ".join(graph.check_invariants(g2))

