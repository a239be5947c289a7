"""Paged KV mode (include/psa.h page_size > 0): the kernel reads K/V through page
tables from caches whose unused rows hold large finite garbage. The output must be
bit-identical to the packed layout on the same data (same work items, same
arithmetic; packed with full forward boxes for partial last blocks, conftest
no_tail_shift), for every page size, with decode + prefill-chunk requests and
segment lengths that are not page multiples — and equal within bf16 rounding to
the default packed launch (back-shifted partial blocks)."""

import numpy as np
import pytest
import torch

from paper_2412_03594_b200 import packed as P
from paper_2412_03594_b200 import paged as PG
from paper_2412_03594_b200 import workloads as W
from paper_2412_03594_b200.errors import ValidationError
from conftest import no_tail_shift

pytestmark = pytest.mark.gpu

SPEC = W.Spec("paged", 16, 4, 128, 128, "bf16", "normal", [700, 33, 0, 2049],
              [[(1, 40), (37, 51), (1, 3), (1, 0)], [(1, 64), (20, 1)], [(3, 17)],
               [(1, 300)] * 40 + [(130, 77)]], seed=21)


def _paged_inputs(b, off, ps, rng):
    out = {}
    for seg, cu in (("prefix", off["cu_prefix"]), ("distinct", off["cu_distinct"])):
        lens = np.diff(cu)
        need = int(PG.pages_needed(lens, ps).sum())
        npages = need * 2 + 3
        pages = PG.random_page_tables(lens, ps, npages, rng)
        for kv in ("k", "v"):
            src = b[f"{kv}_{seg}"]
            cache = (torch.randn((npages * ps,) + tuple(src.shape[1:]), device=src.device) * 300.0
                     ).to(src.dtype)
            PG.scatter_to_cache(src, lens, pages, ps, cache)
            out[f"{kv}_{seg}"] = cache
        out[f"{seg}_pages"] = torch.as_tensor(pages, device=src.device)
    return out


@pytest.mark.parametrize("ps", [16, 32, 64])
def test_paged_matches_packed_bitwise(ps):
    spec = SPEC
    b = W.make_batch(spec, "cuda")
    off = W.offsets(spec)
    args = (off["cu_req"], off["cu_q"], off["cu_prefix"], off["cu_distinct"], spec.Hq, spec.Hkv,
            spec.d, spec.dv, torch.bfloat16, "cuda")
    shifted = P.PrefixSharedAttention(*args)(b["q"], b["k_prefix"], b["v_prefix"], b["k_distinct"],
                                             b["v_distinct"])
    with no_tail_shift():
        ref = P.PrefixSharedAttention(*args)(b["q"], b["k_prefix"], b["v_prefix"],
                                             b["k_distinct"], b["v_distinct"])
    torch.cuda.synchronize()
    assert float((shifted.float() - ref.float()).abs().max()) <= 1e-2
    rng = np.random.default_rng(ps)
    pg = _paged_inputs(b, off, ps, rng)
    op = P.PrefixSharedAttention(*args, page_size=ps)
    for _ in range(3):
        got = op(b["q"], pg["k_prefix"], pg["v_prefix"], pg["k_distinct"], pg["v_distinct"],
                 prefix_pages=pg["prefix_pages"], distinct_pages=pg["distinct_pages"])
        torch.cuda.synchronize()
        assert op.device_error() == 0
        assert torch.equal(got, ref)


def test_paged_skewed_batch_matches_packed():
    """c4's skewed groups (prefix tiles + decode pipeline + merges) through 16-token pages."""
    spec = W.config("c4").subset(range(0, 64, 4))
    b = W.make_batch(spec, "cuda")
    off = W.offsets(spec)
    args = (off["cu_req"], off["cu_q"], off["cu_prefix"], off["cu_distinct"], spec.Hq, spec.Hkv,
            spec.d, spec.dv, torch.bfloat16, "cuda")
    with no_tail_shift():
        ref = P.PrefixSharedAttention(*args)(b["q"], b["k_prefix"], b["v_prefix"],
                                             b["k_distinct"], b["v_distinct"])
    pg = _paged_inputs(b, off, 16, np.random.default_rng(7))
    got = P.PrefixSharedAttention(*args, page_size=16)(
        b["q"], pg["k_prefix"], pg["v_prefix"], pg["k_distinct"], pg["v_distinct"],
        prefix_pages=pg["prefix_pages"], distinct_pages=pg["distinct_pages"])
    torch.cuda.synchronize()
    assert torch.equal(got, ref)


def test_paged_rejections():
    spec = SPEC
    off = W.offsets(spec)
    with pytest.raises(ValidationError, match="page_size"):
        P.PrefixSharedAttention(off["cu_req"], off["cu_q"], off["cu_prefix"], off["cu_distinct"],
                                spec.Hq, spec.Hkv, 128, 128, torch.bfloat16, "cuda", page_size=24)
    with pytest.raises(ValidationError, match="paged KV needs the v2 kernel"):
        P.PrefixSharedAttention(off["cu_req"], off["cu_q"], off["cu_prefix"], off["cu_distinct"],
                                spec.Hq, spec.Hkv, 64, 64, torch.bfloat16, "cuda", page_size=16)
    op = P.PrefixSharedAttention(off["cu_req"], off["cu_q"], off["cu_prefix"], off["cu_distinct"],
                                 spec.Hq, spec.Hkv, 128, 128, torch.bfloat16, "cuda", page_size=16)
    b = W.make_batch(spec, "cuda")
    with pytest.raises(ValidationError, match="prefix_pages"):
        op(b["q"], b["k_prefix"][:16], b["v_prefix"][:16], b["k_distinct"][:16],
           b["v_distinct"][:16])
