"""Paged launches built from REFERENCE scheduler token batches
(tests/golden/token_batches.npz, recorded by tests/golden/make_token_batches.py):
for every batch — decode, distinct-chunk and prefix-chunk entries, 16-token
blocks from the reference's KVAllocator — the paged kernel output must match
the float64 oracle on K/V gathered through the same page tables, and be
bit-identical to the packed kernel on the gathered tensors (packed with full forward
boxes for partial last blocks, conftest no_tail_shift)."""

import os

import numpy as np
import pytest
import torch

from oracle import segmented as S
from paper_2412_03594_b200 import batching as B
from paper_2412_03594_b200 import packed as P
from paper_2412_03594_b200 import paged as PG
from conftest import no_tail_shift

pytestmark = pytest.mark.gpu
FIX = np.load(os.path.join(os.path.dirname(__file__), "golden", "token_batches.npz"))
HQ, HKV, D = 8, 2, 128


@pytest.mark.parametrize("i", range(int(FIX["num_batches"])))
def test_token_batch_paged_launch(i):
    bs, nblk = int(FIX["block_size"]), int(FIX["total_blocks"])
    kb = B.KernelBatch(bs, *(FIX[f"b{i}_{k}"] for k in (
        "cu_req", "cu_q", "cu_prefix", "cu_distinct", "prefix_pages", "distinct_pages",
        "token_entry", "token_offset", "request_entry")))
    gen = torch.Generator(device="cuda").manual_seed(100 + i)
    k_cache = torch.randn((nblk * bs, HKV, D), generator=gen, device="cuda").to(torch.bfloat16)
    v_cache = torch.randn((nblk * bs, HKV, D), generator=gen, device="cuda").to(torch.bfloat16)
    q = torch.randn((kb.num_tokens, HQ, D), generator=gen, device="cuda").to(torch.bfloat16)
    out = B.run(kb, q, k_cache, v_cache, HKV)
    torch.cuda.synchronize()
    # gather the same K/V through the page tables -> packed segments
    pr = torch.as_tensor(PG.physical_rows(np.diff(kb.cu_prefix), kb.prefix_pages, bs), device="cuda")
    dr = torch.as_tensor(PG.physical_rows(np.diff(kb.cu_distinct), kb.distinct_pages, bs),
                         device="cuda")
    kp, vp, kd, vd = k_cache[pr], v_cache[pr], k_cache[dr], v_cache[dr]
    with no_tail_shift():
        packed = P.prefix_shared_attention_packed(q, kp, vp, kd, vd, kb.cu_req, kb.cu_q,
                                                  kb.cu_prefix, kb.cu_distinct, HKV)
    torch.cuda.synchronize()
    assert torch.equal(out, packed)
    h = {k: t.double().cpu().numpy() for k, t in dict(q=q, kp=kp, vp=vp, kd=kd, vd=vd).items()}
    ref = S.packed_attention(h["q"], h["kp"], h["vp"], h["kd"], h["vd"], kb.cu_req, kb.cu_q,
                             kb.cu_prefix, kb.cu_distinct, HQ, HKV)
    assert float(np.abs(out.double().cpu().numpy() - ref).max()) <= 2e-2


@pytest.mark.parametrize("i", [2, 5, 9])
def test_token_batch_paged_causal_launch(i):
    """The same recorded scheduler batches with causal prefill (an extension): paged +
    causal kernel against the causal float64 oracle on the gathered KV."""
    bs, nblk = int(FIX["block_size"]), int(FIX["total_blocks"])
    kb = B.KernelBatch(bs, *(FIX[f"b{i}_{k}"] for k in (
        "cu_req", "cu_q", "cu_prefix", "cu_distinct", "prefix_pages", "distinct_pages",
        "token_entry", "token_offset", "request_entry")))
    gen = torch.Generator(device="cuda").manual_seed(300 + i)
    k_cache = torch.randn((nblk * bs, HKV, D), generator=gen, device="cuda").to(torch.bfloat16)
    v_cache = torch.randn((nblk * bs, HKV, D), generator=gen, device="cuda").to(torch.bfloat16)
    q = torch.randn((kb.num_tokens, HQ, D), generator=gen, device="cuda").to(torch.bfloat16)
    out = B.run(kb, q, k_cache, v_cache, HKV, causal=True)
    torch.cuda.synchronize()
    pr = torch.as_tensor(PG.physical_rows(np.diff(kb.cu_prefix), kb.prefix_pages, bs), device="cuda")
    dr = torch.as_tensor(PG.physical_rows(np.diff(kb.cu_distinct), kb.distinct_pages, bs),
                         device="cuda")
    h = {k: t.double().cpu().numpy() for k, t in dict(
        q=q, kp=k_cache[pr], vp=v_cache[pr], kd=k_cache[dr], vd=v_cache[dr]).items()}
    ref = S.packed_attention_causal(h["q"], h["kp"], h["vp"], h["kd"], h["vd"], kb.cu_req,
                                    kb.cu_q, kb.cu_prefix, kb.cu_distinct, HQ, HKV)
    assert float(np.abs(out.double().cpu().numpy() - ref).max()) <= 2e-2
