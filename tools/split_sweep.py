#!/usr/bin/env python
"""Time configs under several tile/decode CTA splits (diagnostics; PSA_TILE_CTAS = CTAs
that start on the TILE queue, the rest start on the decode queue):
    python tools/split_sweep.py c2,c4 148,128,96,64"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_03594_b200 import packed as P  # noqa: E402
from paper_2412_03594_b200 import workloads as W  # noqa: E402

cfgs = sys.argv[1].split(",")
splits = [None] + [int(v) for v in sys.argv[2].split(",")]
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 20
for cfg in cfgs:
    spec = W.config(cfg)
    b = W.make_batch(spec, "cuda")
    ins = (b["q"], b["k_prefix"], b["v_prefix"], b["k_distinct"], b["v_distinct"])
    op = P.PrefixSharedAttention(b["cu_req"], b["cu_q"], b["cu_prefix"], b["cu_distinct"],
                                 spec.Hq, spec.Hkv, spec.d, spec.dv, spec.torch_dtype, "cuda")
    out = torch.empty((b["q"].shape[0], spec.Hq, spec.dv), dtype=spec.torch_dtype, device="cuda")
    ref = None
    for sp in splits:
        if sp is None:
            os.environ.pop("PSA_TILE_CTAS", None)
        else:
            os.environ["PSA_TILE_CTAS"] = str(sp)
        for _ in range(3):
            op(*ins, out=out)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(iters):
            op(*ins, out=out)
        e1.record()
        torch.cuda.synchronize()
        if ref is None:
            ref = out.clone()
        err = float((out.float() - ref.float()).abs().max())
        print(f"{cfg} tile_ctas={sp if sp is not None else 'plan'}: "
              f"{e0.elapsed_time(e1) / iters * 1e3:.1f} us  err {op.device_error()} "
              f"max|diff| vs plan {err:.1e}", flush=True)
    os.environ.pop("PSA_TILE_CTAS", None)
    del b, ins, op, out, ref
    torch.cuda.empty_cache()
