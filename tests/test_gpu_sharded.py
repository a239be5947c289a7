"""Group-sharded execution (paper_2412_03594_b200/distributed.py) on one GPU: the
batch split into 4 LPT shards, one launch per shard, outputs reassembled in global
token order — equal to the single launch up to bf16 rounding of differently chunked
partials (the multi-process gather itself is tested with gloo in test_multiproc.py)."""

import pytest
import torch

from paper_2412_03594_b200 import distributed as D
from paper_2412_03594_b200 import packed as P
from paper_2412_03594_b200 import workloads as W

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,world", [("c4", 4), ("c5", 8)])
def test_shards_reassemble_to_the_single_launch(name, world):
    spec = W.config(name)
    if name == "c5":
        spec = spec.subset(range(32))
    b = W.make_batch(spec, "cuda")
    full = P.prefix_shared_attention_packed(b["q"], b["k_prefix"], b["v_prefix"], b["k_distinct"],
                                            b["v_distinct"], b["cu_req"], b["cu_q"],
                                            b["cu_prefix"], b["cu_distinct"], spec.Hkv)
    shards = D.shard(b["cu_req"], b["cu_q"], b["cu_prefix"], b["cu_distinct"], spec.Hq, spec.Hkv,
                     spec.d, spec.dv, spec.torch_dtype, world)
    assert sorted(g for s in shards for g in s.groups.tolist()) == list(range(spec.G))
    out = torch.full_like(full, float("nan"))
    for s in shards:
        if s.num_tokens:
            local = D.run_local(s, *D.select_shard(s, b["q"], b["k_prefix"], b["v_prefix"],
                                                   b["k_distinct"], b["v_distinct"]), spec.Hkv)
            out.index_copy_(0, torch.as_tensor(s.token_rows, device="cuda"), local)
    torch.cuda.synchronize()
    assert not torch.isnan(out).any()
    assert float((out.float() - full.float()).abs().max()) <= 1e-2
