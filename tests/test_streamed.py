"""Group slabs (paper_2412_03594_b200/streamed.py) on the host: slabs are runs of whole
groups whose row ranges tile the packed batch exactly once, with rebased offsets."""

import numpy as np

from paper_2412_03594_b200 import streamed as ST
from paper_2412_03594_b200 import workloads as W


def _check_tiling(spec, slabs):
    off = W.offsets(spec)
    assert slabs[0].g0 == 0 and slabs[-1].g1 == spec.G
    for a, b in zip(slabs, slabs[1:]):
        assert a.g1 == b.g0 and a.t1 == b.t0 and a.p1 == b.p0 and a.d1 == b.d0
    assert slabs[-1].t1 == off["cu_q"][-1] and slabs[-1].p1 == off["cu_prefix"][-1]
    assert slabs[-1].d1 == off["cu_distinct"][-1]
    for s in slabs:
        r0, r1 = off["cu_req"][s.g0], off["cu_req"][s.g1]
        assert np.array_equal(np.array(s.cu_req), off["cu_req"][s.g0:s.g1 + 1] - r0)
        assert np.array_equal(np.array(s.cu_q), off["cu_q"][r0:r1 + 1] - off["cu_q"][r0])
        assert np.array_equal(np.array(s.cu_prefix), off["cu_prefix"][s.g0:s.g1 + 1] - s.p0)
        assert np.array_equal(np.array(s.cu_distinct), off["cu_distinct"][r0:r1 + 1] - s.d0)
        assert s.cu_q[-1] == s.t1 - s.t0 and s.cu_prefix[-1] == s.p1 - s.p0
        assert s.cu_distinct[-1] == s.d1 - s.d0


def test_slabs_tile_the_batch():
    rb = {"q": 32 * 128 * 2, "kv_prefix": 8 * 256 * 2, "kv_distinct": 8 * 256 * 2}
    for name, cap in (("c4", 256 << 20), ("c5", 2 << 30), ("c2", 1 << 40), ("c4", 1)):
        spec = W.config(name)
        off = W.offsets(spec)
        slabs = ST.cut_slabs(off["cu_req"], off["cu_q"], off["cu_prefix"], off["cu_distinct"],
                             rb, cap)
        _check_tiling(spec, slabs)
        if cap == 1:
            assert len(slabs) == spec.G  # a group bigger than the cap is a slab of its own
        if name == "c2" and cap > 1 << 39:
            assert len(slabs) == 1
        if name == "c5":  # uniform groups: one structure, so one plan serves all full slabs
            assert len({s.structure for s in slabs}) <= 2
