"""Causal prefill chunks (PSA_FLAG_CAUSAL, an extension: the reference attends every
key, attention.py:12-13): against the causal float64 oracle
(oracle/segmented.packed_attention_causal) on batches mixing decode tokens, prefill
chunks with own KV (fused tiles and separate distinct items), prefix-only chunk
requests and skewed lengths; decode-only batches are unchanged bit for bit."""

import numpy as np
import pytest
import torch

from oracle import segmented as S
from paper_2412_03594_b200 import packed as P
from paper_2412_03594_b200 import workloads as W
from paper_2412_03594_b200.errors import ValidationError

pytestmark = pytest.mark.gpu

SPECS = [
    W.Spec("causal_mixed", 16, 4, 128, 128, "bf16", "normal", [700, 33, 300, 2049],
           [[(1, 40), (37, 51), (1, 3)], [(1, 64), (20, 20)], [(64, 0)],
            [(1, 300)] * 10 + [(130, 200), (300, 300)]], seed=41),
    W.Spec("causal_chunks", 32, 8, 128, 128, "bf16", "normal", [2048, 0],
           [[(512, 512), (512, 700), (1, 256)], [(256, 256), (77, 1000)]], seed=42),
]


def _run(spec, causal, **opts):
    b = W.make_batch(spec, "cuda")
    op = P.PrefixSharedAttention(b["cu_req"], b["cu_q"], b["cu_prefix"], b["cu_distinct"],
                                 spec.Hq, spec.Hkv, spec.d, spec.dv, spec.torch_dtype, "cuda",
                                 options=P.PlanOptions(**opts))
    out = op(b["q"], b["k_prefix"], b["v_prefix"], b["k_distinct"], b["v_distinct"],
             causal=causal)
    torch.cuda.synchronize()
    assert op.device_error() == 0
    return b, out


@pytest.mark.parametrize("spec", SPECS, ids=lambda s: s.name)
@pytest.mark.parametrize("opts", [dict(), dict(min_chunk_keys=64), dict(disable_tiles=1)],
                         ids=["default", "small_chunks", "decode_pipeline_only"])
def test_causal_matches_oracle(spec, opts):
    b, out = _run(spec, True, **opts)
    h = {k: b[k].double().cpu().numpy() for k in ("q", "k_prefix", "v_prefix", "k_distinct",
                                                    "v_distinct")}
    ref = S.packed_attention_causal(h["q"], h["k_prefix"], h["v_prefix"], h["k_distinct"],
                                    h["v_distinct"], b["cu_req"], b["cu_q"], b["cu_prefix"],
                                    b["cu_distinct"], spec.Hq, spec.Hkv)
    assert float(np.abs(out.double().cpu().numpy() - ref).max()) <= 2e-2


def test_causal_is_a_no_op_for_decode_batches():
    spec = W.config("c2").subset(range(4))
    _, a = _run(spec, False)
    _, c = _run(spec, True)
    assert torch.equal(a, c)


def test_causal_needs_the_v2_kernel():
    spec = W.Spec("c64", 4, 4, 64, 64, "bf16", "normal", [64], [[(8, 8)]], seed=1)
    with pytest.raises(ValidationError, match="causal"):
        _run(spec, True)


@pytest.mark.parametrize("reqs,P", [([(40, 20)], 64), ([(80, 0)], 64)],
                         ids=["nq_gt_D", "prefix_only_nq_gt_P"])
def test_causal_rejects_chunks_longer_than_their_keys(reqs, P):
    """n_q > D (or n_q > P without distinct KV) cannot be expressed by the per-token key
    limits: it would leak later prefix keys to the first tokens — rejected."""
    spec = W.Spec("bad_causal", 8, 2, 128, 128, "bf16", "normal", [P], [reqs], seed=3)
    with pytest.raises(ValidationError, match="n_q <= D"):
        _run(spec, True)


def test_zero_scale_is_a_uniform_average_on_tiles():
    """scale == 0 (naive_attention allows it): every key weighs the same, also on the
    tile path with a partial last key block (the mask must not produce NaN)."""
    spec = W.Spec("scale0", 16, 4, 128, 128, "bf16", "normal", [200],
                  [[(1, 37)] * 40], seed=5)
    b = W.make_batch(spec, "cuda")
    op = P.PrefixSharedAttention(b["cu_req"], b["cu_q"], b["cu_prefix"], b["cu_distinct"],
                                 spec.Hq, spec.Hkv, spec.d, spec.dv, spec.torch_dtype, "cuda",
                                 scale=0.0)
    out = op(b["q"], b["k_prefix"], b["v_prefix"], b["k_distinct"], b["v_distinct"])
    torch.cuda.synchronize()
    assert not torch.isnan(out).any()
    kp, vp = b["k_prefix"].double(), b["v_prefix"].double()
    vd = b["v_distinct"].double()
    gqa = spec.Hq // spec.Hkv
    for r in (0, 17, 39):
        for h in range(spec.Hkv):
            keys = torch.cat([vp[:, h], vd[r * 37:(r + 1) * 37, h]])
            want = keys.mean(0)
            got = out[r, h * gqa:(h + 1) * gqa].double()
            assert float((got - want).abs().max()) <= 2e-2
