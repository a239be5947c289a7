#!/usr/bin/env python
"""Time one config under several PlanOptions (diagnostics): python tools/opt_sweep.py c4 tile_min_rows=16,8"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_03594_b200 import packed as P  # noqa: E402
from paper_2412_03594_b200 import workloads as W  # noqa: E402

cfg = sys.argv[1]
variants = [dict()]
for arg in sys.argv[2:]:
    k, vals = arg.split("=")
    variants += [{k: int(v)} for v in vals.split(",")]
spec = W.config(cfg)
b = W.make_batch(spec, "cuda")
ins = (b["q"], b["k_prefix"], b["v_prefix"], b["k_distinct"], b["v_distinct"])
ref = None
for v in variants + [dict()]:
    op = P.PrefixSharedAttention(b["cu_req"], b["cu_q"], b["cu_prefix"], b["cu_distinct"],
                                 spec.Hq, spec.Hkv, spec.d, spec.dv, spec.torch_dtype, "cuda",
                                 options=P.PlanOptions(**v))
    out = torch.empty((b["q"].shape[0], spec.Hq, spec.dv), dtype=spec.torch_dtype, device="cuda")
    for _ in range(5):
        op(*ins, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(40):
        op(*ins, out=out)
    e1.record()
    torch.cuda.synchronize()
    if ref is None:
        ref = out.clone()
    err = float((out.float() - ref.float()).abs().max())
    print(f"{cfg} {v}: {e0.elapsed_time(e1) / 40 * 1e3:.1f} us  items {op.num_items}  "
          f"max|diff| vs default {err:.1e}", flush=True)
