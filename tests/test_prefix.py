"""Native prompt grouping (csrc/psa_prefix.cpp) against the reference's
prefix_tree.py: identical groups (prefixes, members, member order) on the
reference's synthetic workloads and on random prompt sets, the first-level
saving, and acceptance criterion 7 (8001 requests grouped in < 10 s,
test_acceptance.py:228-239)."""

import os
import sys
import time

import numpy as np
import pytest

from paper_2412_03594_b200 import prefix as PX
from paper_2412_03594_b200.errors import ValidationError

REF = "/root/reference/pkg/src"
needs_ref = pytest.mark.skipif(not os.path.isdir(REF), reason="reference not present")


def ref_modules():
    if REF not in sys.path:
        sys.path.insert(0, REF)
    from prefixbatch import prefix_tree as PT
    from prefixbatch import workload as WL
    return PT, WL


def ref_groups(PT, w, maximize=True):
    tree = PT.build_tree(w)
    if maximize:
        tree = PT.maximize_reuse(tree)
    return [(g.prefix, [(m.id, m.suffix) for m in g.members]) for g in PT.extract_groups(tree)]


class Req:
    def __init__(self, rid, tokens):
        self.id, self.tokens = rid, tuple(tokens)


class W:
    def __init__(self, reqs):
        self.requests = reqs


def random_workload(rng, n, vocab, shared):
    """Prompts built from a few shared stems, so the tree has real structure."""
    stems = [tuple(rng.integers(0, vocab, rng.integers(1, 40))) for _ in range(shared)]
    reqs = []
    for i in range(n):
        t = ()
        for _ in range(rng.integers(1, 4)):
            t += stems[rng.integers(0, shared)] if rng.random() < 0.7 else \
                tuple(rng.integers(0, vocab, rng.integers(1, 10)))
        reqs.append(Req(f"r{rng.integers(0, 10**6)}_{i}", t))
    if n > 3:  # identical prompts share one node: ordered by id
        reqs.append(Req("zz_dup", reqs[1].tokens))
        reqs.append(Req("aa_dup", reqs[1].tokens))
    return W(reqs)


@needs_ref
@pytest.mark.parametrize("seed", range(12))
@pytest.mark.parametrize("maximize", [True, False])
def test_random_workloads_match_reference(seed, maximize):
    PT, _ = ref_modules()
    rng = np.random.default_rng(seed)
    w = random_workload(rng, int(rng.integers(1, 200)), int(rng.choice([3, 50, 30000])),
                        int(rng.integers(1, 12)))
    assert PX.group_workload(w, maximize) == ref_groups(PT, w, maximize)


@needs_ref
def test_reference_synthetic_workloads_match():
    PT, WL = ref_modules()
    for spec in (WL.SyntheticSpec(prefix_len=64, distinct_len=16, sharing_degree=16,
                                  num_groups=8, output_len=4, seed=3),
                 WL.SyntheticSpec(prefix_len=500, distinct_len=30, sharing_degree=50,
                                  num_groups=3, output_len=2, seed=11)):
        w = WL.generate_microbenchmark(spec)
        assert PX.group_workload(w) == ref_groups(PT, w)
        groups, saved = PX.group_prompts([r.id for r in w.requests],
                                         [r.tokens for r in w.requests])
        assert saved == PT.first_level_saved_tokens(PT.maximize_reuse(PT.build_tree(w)))


@needs_ref
def test_criterion_7_industry_analogue_fast_and_identical():
    PT, WL = ref_modules()
    # test_acceptance.py:46-52: moment-matched stand-in for the profiled industry traffic
    w = WL.generate_microbenchmark(WL.SyntheticSpec(1570, 30, 3, 2667, 100, 13))
    assert len(w) == 8001
    t0 = time.perf_counter()
    native = PX.group_workload(w)
    native_s = time.perf_counter() - t0
    assert native_s < 10.0
    assert native == ref_groups(PT, w)
    print(f"criterion 7: {len(native)} groups from {len(w)} requests in {native_s:.3f} s native")


def test_small_known_answer_without_reference():
    # a:[1,2,3,4] b:[1,2,3,5] c:[1,2,9] d:[7]  -> radix: [1,2] -> {[3] -> {4, 5}, [9]}, [7]
    w = W([Req("a", [1, 2, 3, 4]), Req("b", [1, 2, 3, 5]), Req("c", [1, 2, 9]), Req("d", [7])])
    plain = PX.group_workload(w, maximize=False)
    assert plain == [((1, 2), [("a", (3, 4)), ("b", (3, 5)), ("c", (9,))]), ((), [("d", (7,))])]
    # forking [3] (2 leaves x 1 token) does not beat its parent span (2): unchanged
    assert PX.group_workload(w) == plain


def test_rejections():
    with pytest.raises(ValidationError):
        PX.group_prompts(["a", "b"], [[1], []])
    with pytest.raises(ValidationError):
        PX.group_prompts(["a", "a"], [[1], [2]])
