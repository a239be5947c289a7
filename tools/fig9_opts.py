#!/usr/bin/env python
"""Our kernel on the Fig. 9-style shapes under several plan options (diagnostics)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from paper_2412_03594_b200 import packed as P  # noqa: E402
from paper_2412_03594_b200 import workloads as W  # noqa: E402
from cascade_compare import fig9_specs, timeit  # noqa: E402

variants = [dict(), dict(min_chunk_keys=1024), dict(min_chunk_keys=2048)]
for name, spec in fig9_specs():
    b = W.make_batch(spec, "cuda")
    ins = (b["q"], b["k_prefix"], b["v_prefix"], b["k_distinct"], b["v_distinct"])
    res = []
    for v in variants:
        op = P.PrefixSharedAttention(b["cu_req"], b["cu_q"], b["cu_prefix"], b["cu_distinct"],
                                     spec.Hq, spec.Hkv, spec.d, spec.dv, spec.torch_dtype, "cuda",
                                     options=P.PlanOptions(**v))
        out = torch.empty((b["q"].shape[0], spec.Hq, spec.dv), dtype=spec.torch_dtype, device="cuda")
        res.append(timeit(lambda: op(*ins, out=out)))
    print(f"{name:28s} " + "  ".join(f"{r:7.1f}" for r in res), flush=True)
    del b
