#!/usr/bin/env python
"""Relaunch one config's planned op many times, synchronising after each launch;
reports the first failing launch and any output that differs bitwise from the
first launch (the kernel is deterministic by construction)."""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_03594_b200 import packed as P  # noqa: E402
from paper_2412_03594_b200 import workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c4")
ap.add_argument("--iters", type=int, default=100)
ap.add_argument("--variant", type=int, default=0)
ap.add_argument("--disable-tiles", type=int, default=0)
ap.add_argument("--num-sms", type=int, default=0)
args = ap.parse_args()
dev = torch.device("cuda", 0)
spec = W.config(args.config)
b = W.make_batch(spec, dev)
op = P.PrefixSharedAttention(b["cu_req"], b["cu_q"], b["cu_prefix"], b["cu_distinct"], spec.Hq,
                             spec.Hkv, spec.d, spec.dv, spec.torch_dtype, dev,
                             options=P.PlanOptions(kernel_variant=args.variant, disable_tiles=args.disable_tiles,
                                                   num_sms=args.num_sms))
ins = (b["q"], b["k_prefix"], b["v_prefix"], b["k_distinct"], b["v_distinct"])
ref = None
bad = 0
for i in range(args.iters):
    try:
        out = op(*ins)
        torch.cuda.synchronize()
    except Exception as e:  # noqa: BLE001
        print(f"launch {i} FAILED: {e}", flush=True)
        sys.exit(1)
    if ref is None:
        ref = out.clone()
    elif not torch.equal(out, ref):
        bad += 1
        diff = (out.float() - ref.float()).abs()
        rows = (diff.amax(dim=(1, 2)) > 0).nonzero().flatten()
        print(f"launch {i}: differs from launch 0 on {rows.numel()} tokens, first {rows[:8].tolist()}"
              f" max {diff.max().item():.3e}", flush=True)
print(f"{args.config}: {args.iters} launches ok, {bad} nondeterministic, items {op.num_items}, "
      f"err bits {op.device_error()}")
