"""Host-streamed execution (paper_2412_03594_b200/streamed.py, the bench's e2e path):
inputs in pinned host memory, group slabs copied in / computed / copied out on three
streams. Every row must come back, and it must match the oracle and the device launch."""

import numpy as np
import pytest
import torch

from paper_2412_03594_b200 import packed as P
from paper_2412_03594_b200 import streamed as ST
from paper_2412_03594_b200 import workloads as W
from test_gpu_parity import check_sampled_groups

pytestmark = pytest.mark.gpu
KEYS = ("q", "k_prefix", "v_prefix", "k_distinct", "v_distinct")


@pytest.mark.parametrize("name,slab_mb", [("c4", 300), ("c2", 64), ("c2", 1 << 20)])
def test_host_streamed_matches_device_launch(name, slab_mb):
    spec = W.config(name)
    b = W.make_batch(spec, "cuda")
    host = {k: b[k].cpu().pin_memory() for k in KEYS}
    out_h = torch.full((b["q"].shape[0], spec.Hq, spec.dv), float("nan"),
                       dtype=spec.torch_dtype).pin_memory()
    run = ST.HostStreamedAttention(b["cu_req"], b["cu_q"], b["cu_prefix"], b["cu_distinct"],
                                   spec.Hq, spec.Hkv, spec.d, spec.dv, spec.torch_dtype, "cuda",
                                   slab_bytes=slab_mb << 20)
    for _ in range(2):  # the second call reuses both slab buffers (stream ordering)
        out_h.fill_(float("nan"))
        run(*(host[k] for k in KEYS), out_h)
        torch.cuda.synchronize()
        assert not torch.isnan(out_h).any()
    if slab_mb < 1000:
        assert len(run.slabs) > 1
    ref = P.prefix_shared_attention_packed(*(b[k] for k in KEYS), b["cu_req"], b["cu_q"],
                                           b["cu_prefix"], b["cu_distinct"], spec.Hkv)
    assert float((out_h.float() - ref.float().cpu()).abs().max()) <= 1e-2
    check_sampled_groups(spec, b, out_h.cuda(), n_groups=3, n_heads=2)
    h2d, d2h = run.bytes_per_call()
    assert h2d == sum(host[k].numel() * host[k].element_size() for k in KEYS)
    assert d2h == out_h.numel() * out_h.element_size()
