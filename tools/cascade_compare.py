#!/usr/bin/env python
"""External context: FlashInfer's two-level cascade attention
(shared-prefix level + per-request level, paged KV, merged by LSE) — the library
counterpart of this path — on the same synthetic batch as our kernel.

    python tools/cascade_compare.py [--config c2] [--page 16]

Prints one JSON line: both times (CUDA events, inputs resident, 50 launches after
warm-up) and the max |difference| of the outputs. FlashInfer is library code; it is
never on our product path.
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_03594_b200 import packed as P  # noqa: E402
from paper_2412_03594_b200 import paged as PG  # noqa: E402
from paper_2412_03594_b200 import workloads as W  # noqa: E402


def timeit(fn, iters=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters * 1e3


fig9_specs = W.fig9_specs


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--page", type=int, default=16)
    ap.add_argument("--fig9", action="store_true", help="sweep the Fig. 9-style shapes")
    args = ap.parse_args()
    if args.fig9:
        for name, spec in fig9_specs():
            compare(spec, name, args.page)
        return
    compare(W.config(args.config), args.config, args.page)


def compare(spec, name, ps):
    import flashinfer
    b = W.make_batch(spec, "cuda")
    off = W.offsets(spec)
    # ours (packed layout)
    op = P.PrefixSharedAttention(off["cu_req"], off["cu_q"], off["cu_prefix"], off["cu_distinct"],
                                 spec.Hq, spec.Hkv, spec.d, spec.dv, spec.torch_dtype, "cuda")
    ins = (b["q"], b["k_prefix"], b["v_prefix"], b["k_distinct"], b["v_distinct"])
    out = torch.empty((b["q"].shape[0], spec.Hq, spec.dv), dtype=spec.torch_dtype, device="cuda")
    ours_us = timeit(lambda: op(*ins, out=out))
    # FlashInfer: one page pool holding every prefix page and every request's pages
    plen, dlen = np.diff(off["cu_prefix"]), np.diff(off["cu_distinct"])
    npp, ndp = PG.pages_needed(plen, ps), PG.pages_needed(dlen, ps)
    total = int(npp.sum() + ndp.sum())
    pages = np.arange(total, dtype=np.int32)
    ppages, dpages = pages[:int(npp.sum())], pages[int(npp.sum()):]
    k_cache = torch.zeros((total * ps, spec.Hkv, spec.d), dtype=spec.torch_dtype, device="cuda")
    v_cache = torch.zeros_like(k_cache)
    PG.scatter_to_cache(b["k_prefix"], plen, ppages, ps, k_cache)
    PG.scatter_to_cache(b["v_prefix"], plen, ppages, ps, v_cache)
    PG.scatter_to_cache(b["k_distinct"], dlen, dpages, ps, k_cache)
    PG.scatter_to_cache(b["v_distinct"], dlen, dpages, ps, v_cache)
    cache = (k_cache.view(total, ps, spec.Hkv, spec.d), v_cache.view(total, ps, spec.Hkv, spec.d))
    dev = torch.device("cuda")
    i32 = lambda x: torch.as_tensor(np.asarray(x, dtype=np.int32), device=dev)  # noqa: E731
    tok_per_group = off["cu_q"][off["cu_req"]]
    last = lambda lens: np.where(lens % ps == 0, ps, lens % ps).astype(np.int32)  # noqa: E731
    qo = [i32(tok_per_group), i32(off["cu_q"])]
    kv_indptr = [i32(np.concatenate([[0], np.cumsum(npp)])), i32(np.concatenate([[0], np.cumsum(ndp)]))]
    kv_idx = [i32(ppages), i32(dpages)]
    kv_last = [i32(last(plen)), i32(last(dlen))]
    ws = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    wrapper = flashinfer.MultiLevelCascadeAttentionWrapper(2, ws, "NHD")
    wrapper.plan(qo, kv_indptr, kv_idx, kv_last, spec.Hq, spec.Hkv, spec.d, ps,
                 q_data_type=spec.torch_dtype, kv_data_type=spec.torch_dtype)
    fi_out = wrapper.run(b["q"], cache)
    fi_us = timeit(lambda: wrapper.run(b["q"], cache))
    diff = float((fi_out.float() - out.float()).abs().max())
    print(json.dumps({"config": name, "page_size": ps, "ours_us": round(ours_us, 1),
                      "flashinfer_cascade_us": round(fi_us, 1),
                      "speedup": round(fi_us / ours_us, 2), "max_abs_diff": diff,
                      "flashinfer": flashinfer.__version__}), flush=True)


if __name__ == "__main__":
    main()
