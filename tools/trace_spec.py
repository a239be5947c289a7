#!/usr/bin/env python
"""trace_report for an ad-hoc decode shape: python tools/trace_spec.py P D R k"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from paper_2412_03594_b200 import packed as P  # noqa: E402
from paper_2412_03594_b200 import workloads as W  # noqa: E402
import trace_report as TR  # noqa: E402

Pn, D, R, k = (int(x) for x in sys.argv[1:5])
G = R // k
spec = W.Spec("adhoc", 32, 8, 128, 128, "bf16", "normal", [Pn] * G, [[(1, D)] * k for _ in range(G)], seed=9)
b = W.make_batch(spec, "cuda")
op = P.PrefixSharedAttention(b["cu_req"], b["cu_q"], b["cu_prefix"], b["cu_distinct"], spec.Hq,
                             spec.Hkv, spec.d, spec.dv, spec.torch_dtype, "cuda")
ins = (b["q"], b["k_prefix"], b["v_prefix"], b["k_distinct"], b["v_distinct"])
for _ in range(3):
    op(*ins)
torch.cuda.synchronize()
tr, ctas = op.trace(*ins)
rep = TR.report(tr, op.plan_tables())
t = op.plan_tables()
items = t["items"]
rep["n_tile"] = int(t["num_tile_items"])
rep["vec_keys_hist"] = np.unique((items[:, 7] - items[:, 6]) + (items[:, 9] - items[:, 8]), return_counts=True)[1].tolist()[:10]
st = tr[:, 2].min()
rep["kernel_end_pct"] = [float(x) for x in np.percentile((ctas[:, 3] - st) / 1e3, [0, 50, 100])]
print(json.dumps(rep, indent=1))
