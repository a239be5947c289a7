"""Token batch -> paged kernel metadata (paper_2412_03594_b200/batching.py),
checked on batches recorded from the reference scheduler
(tests/golden/make_token_batches.py) and, where /root/reference exists, against a
fresh run of that scheduler."""

import os
import sys

import numpy as np
import pytest

from paper_2412_03594_b200 import batching as B
from paper_2412_03594_b200 import paged as PG

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
FIX = np.load(os.path.join(GOLDEN, "token_batches.npz"))
REF = "/root/reference/pkg/src"


def batches():
    return [{k: FIX[f"b{i}_{k}"] for k in B_KEYS} for i in range(int(FIX["num_batches"]))]


B_KEYS = ("cu_req", "cu_q", "cu_prefix", "cu_distinct", "prefix_pages", "distinct_pages",
          "token_entry", "token_offset", "request_entry", "entry_kind", "entry_tokens")


@pytest.mark.parametrize("i", range(int(FIX["num_batches"])))
def test_recorded_batch_invariants(i):
    b = batches()[i]
    bs, nblk = int(FIX["block_size"]), int(FIX["total_blocks"])
    for k in ("cu_req", "cu_q", "cu_prefix", "cu_distinct"):
        assert b[k][0] == 0 and np.all(np.diff(b[k]) >= 0)
    G, R = len(b["cu_req"]) - 1, len(b["cu_q"]) - 1
    assert len(b["cu_prefix"]) == G + 1 and len(b["cu_distinct"]) == R + 1
    assert np.all(np.diff(b["cu_req"]) >= 1) and np.all(np.diff(b["cu_q"]) >= 1)
    # page tables: ceil(len / block_size) pages per segment, valid block ids
    assert len(b["prefix_pages"]) == PG.pages_needed(np.diff(b["cu_prefix"]), bs).sum()
    assert len(b["distinct_pages"]) == PG.pages_needed(np.diff(b["cu_distinct"]), bs).sum()
    for t in (b["prefix_pages"], b["distinct_pages"]):
        assert np.all((t >= 0) & (t < nblk))
    # distinct pages of different requests never alias; prefix and distinct pools are disjoint
    assert len(set(b["distinct_pages"].tolist())) == len(b["distinct_pages"])
    assert not set(b["distinct_pages"].tolist()) & set(b["prefix_pages"].tolist())
    # every batch token appears exactly once; tokens per request = entry tokens
    n_entries = len(b["entry_kind"])
    assert sorted(set(b["request_entry"].tolist())) == list(range(n_entries))
    counts = np.bincount(b["token_entry"], minlength=n_entries)
    assert np.array_equal(counts, b["entry_tokens"])
    assert np.array_equal(np.diff(b["cu_q"]), b["entry_tokens"][b["request_entry"]])
    # decode entries: one token, KV >= 1; prefix chunks: a group of their own, no distinct KV
    D = np.diff(b["cu_distinct"])
    kind_r = b["entry_kind"][b["request_entry"]]
    assert np.all(np.diff(b["cu_q"])[kind_r == 0] == 1) and np.all(D[kind_r == 0] >= 1)
    assert np.all(D[kind_r == 2] == 0)
    grp_of_req = np.repeat(np.arange(G), np.diff(b["cu_req"]))
    for r in np.where(kind_r == 2)[0]:
        g = grp_of_req[r]
        assert b["cu_req"][g + 1] - b["cu_req"][g] == 1 and b["cu_prefix"][g + 1] > b["cu_prefix"][g]


def test_entry_token_rows_is_a_permutation():
    for b in batches():
        class E:
            def __init__(self, n):
                self.tokens = int(n)
        batch = type("Batch", (), {"entries": [E(n) for n in b["entry_tokens"]]})()
        kb = B.KernelBatch(16, b["cu_req"], b["cu_q"], b["cu_prefix"], b["cu_distinct"],
                           b["prefix_pages"], b["distinct_pages"], b["token_entry"],
                           b["token_offset"], b["request_entry"])
        rows = B.entry_token_rows(kb, batch)
        assert sorted(rows.tolist()) == list(range(kb.num_tokens))


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference scheduler not present")
def test_fixture_reproduces_from_the_reference_scheduler():
    sys.path.insert(0, GOLDEN)
    import make_token_batches as M
    sys.path.insert(0, REF)
    plain, _ = M.simulate(REF, hook=False)
    hooked, records = M.simulate(REF, hook=True)
    assert [r.__dict__ for r in plain.rows] == [r.__dict__ for r in hooked.rows]
    assert len(records) == int(FIX["num_batches"])
    for i, (_batch, kb, _state) in enumerate(records):
        for k in M.KEYS:
            assert np.array_equal(getattr(kb, k), FIX[f"b{i}_{k}"]), (i, k)


def test_prepare_rejects_non_batchllm_states_and_short_block_lists():
    """prepare() guards: fcfs_cap states and cache-hit tokens are not
    expressible; a block list shorter than the segment would shift page bases."""
    from types import SimpleNamespace as NS
    cfg = NS(block_size=16, policy="fcfs_cap")
    st = NS(config=cfg, allocator=None, groups=[], requests={})
    with pytest.raises(ValueError, match="batchllm"):
        B.prepare(st, NS(entries=[]))

    class Alloc:
        def grow(self, owner, n):
            pass

        def blocks_of(self, owner):
            return [0]  # one block, fewer than the 3 a 40-token segment needs

    req = NS(id="r0", group=None, suffix_done=0, decode_done=0, reused_tokens=0)
    st = NS(config=NS(block_size=16, policy="batchllm"), allocator=Alloc(), groups=[],
            requests={"r0": req})
    entry = NS(kind=B.DISTINCT_CHUNK, owner="r0", tokens=40)
    with pytest.raises(ValueError, match="blocks"):
        B.prepare(st, NS(entries=[entry]))
    req.reused_tokens = 16
    with pytest.raises(ValueError, match="reused"):
        B.prepare(st, NS(entries=[entry]))
