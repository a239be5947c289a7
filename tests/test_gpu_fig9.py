"""The 26 kernel-comparison shapes in the style of the paper's Fig. 9 (
workloads.fig9_specs): single groups with long prefixes and few requests (large merge
fan-in), many small groups, chunked prefill mixed with decode. Each shape runs through
the C ABI and is checked against the float64 oracle (oracle/segmented.py, the
restatement of attention.py:156-201) on sampled (group, kv head) pairs; every output
row must be written. Tolerance: bf16 max |out - ref| <= 2e-2."""

import pytest
import torch

from paper_2412_03594_b200 import packed as P
from paper_2412_03594_b200 import workloads as W
from test_gpu_parity import check_sampled_groups

pytestmark = pytest.mark.gpu

SHAPES = [name for name, _ in W.fig9_specs()]


@pytest.mark.parametrize("name", SHAPES)
def test_fig9_shape_matches_oracle(name):
    spec = W.config("fig9:" + name)
    b = W.make_batch(spec, "cuda")
    op = P.PrefixSharedAttention(b["cu_req"], b["cu_q"], b["cu_prefix"], b["cu_distinct"],
                                 spec.Hq, spec.Hkv, spec.d, spec.dv, spec.torch_dtype, "cuda")
    out = torch.full((b["q"].shape[0], spec.Hq, spec.dv), float("nan"), dtype=spec.torch_dtype,
                     device="cuda")
    for _ in range(2):  # the second launch reuses the self-resetting counters
        op(b["q"], b["k_prefix"], b["v_prefix"], b["k_distinct"], b["v_distinct"], out=out)
    torch.cuda.synchronize()
    assert op.device_error() == 0
    assert not torch.isnan(out).any()
    check_sampled_groups(spec, b, out, n_groups=2, n_heads=2, seed=1)
