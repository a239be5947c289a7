#!/usr/bin/env python
"""Run one config's planned op `--iters` times after `--warmup` (for ncu -s/-c)."""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_03594_b200 import packed as P  # noqa: E402
from paper_2412_03594_b200 import workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--ctas-per-sm", type=int, default=0)
ap.add_argument("--num-sms", type=int, default=0)
ap.add_argument("--warmup", type=int, default=3)
ap.add_argument("--iters", type=int, default=1)
args = ap.parse_args()
dev = torch.device("cuda", 0)
spec = W.config(args.config)
b = W.make_batch(spec, dev)
op = P.PrefixSharedAttention(b["cu_req"], b["cu_q"], b["cu_prefix"], b["cu_distinct"], spec.Hq,
                             spec.Hkv, spec.d, spec.dv, spec.torch_dtype, dev,
                                 options=P.PlanOptions(ctas_per_sm=args.ctas_per_sm, num_sms=args.num_sms))
ins = (b["q"], b["k_prefix"], b["v_prefix"], b["k_distinct"], b["v_distinct"])
for _ in range(args.warmup + args.iters):
    op(*ins)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    op(*ins)
e1.record()
torch.cuda.synchronize()
print(f"{args.config}: {e0.elapsed_time(e1) / 20 * 1e3:.1f} us/launch, items {op.num_items}")
