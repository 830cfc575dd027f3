"""k-means subsamples drawn by the core library on the host cores
(fa_kmeans_subsample) against numpy itself: the rows of
np.sort(default_rng(seed + i).permutation(ns)[:4096]) (flashann/kmeans.py:50-54)
and the generator state numpy leaves behind, bit for bit.  No device needed."""

import numpy as np
import pytest

from paper_2502_18113_b200 import flash


@pytest.mark.parametrize("ns,m,seed", [(4097, 3, 0), (20000, 32, 5), (100000, 4, 1)])
def test_subsample_matches_numpy(ns, m, seed):
    sel, states = flash._rng_streams(ns, m, seed)
    assert sel.shape == (m, 4096)
    for i in range(m):
        g = np.random.default_rng(seed + i)
        ref = np.sort(g.permutation(ns)[:4096])
        np.testing.assert_array_equal(sel[i], ref)
        st = g.bit_generator.state
        s, inc = st["state"]["state"], st["state"]["inc"]
        assert (int(states[i]["s_hi"]) << 64) | int(states[i]["s_lo"]) == s
        assert (int(states[i]["inc_hi"]) << 64) | int(states[i]["inc_lo"]) == inc
        assert int(states[i]["has"]) == st["has_uint32"]
        assert int(states[i]["u"]) == st["uinteger"]


def test_small_sample_uses_every_row():
    sel, states = flash._rng_streams(4096, 2, 0)
    assert sel is None
    st = np.random.default_rng(1).bit_generator.state
    assert (int(states[1]["s_hi"]) << 64) | int(states[1]["s_lo"]) == st["state"]["state"]
