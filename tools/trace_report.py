#!/usr/bin/env python
"""Per-work-item timeline of one persistent launch (diagnostics).

    python tools/trace_report.py --config c2 [--warmup 3] [--json out.json]

Uses psa_debug_set_trace (include/psa.h): every item records its CTA, SM,
kind and %globaltimer start/end. Reports per-kind counts and durations, CTA
busy fraction, launch span and the tail after the first CTA ran dry.
"""

from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2412_03594_b200 import packed as P  # noqa: E402
from paper_2412_03594_b200 import workloads as W  # noqa: E402


def report(tr: np.ndarray, tables: dict) -> dict:
    cta = (tr[:, 0] & 0xFFFFFFFF).astype(np.int64)
    kind = tr[:, 1]
    t0, t1 = tr[:, 2], tr[:, 3]
    start = t0.min()
    span = (t1.max() - start) / 1e3
    dur = (t1 - t0) / 1e3
    out = {"items": int(len(tr)), "span_us": float(span)}
    items = tables["items"]
    keys = (items[:, 7] - items[:, 6]) + (items[:, 9] - items[:, 8])
    for k, name in ((0, "vec"), (1, "tile")):
        sel = kind == k
        if sel.any():
            out[name] = {"n": int(sel.sum()), "sum_us": float(dur[sel].sum()),
                         "mean_us": float(dur[sel].mean()), "p50_us": float(np.median(dur[sel])),
                         "max_us": float(dur[sel].max()),
                         "keys_mean": float(keys[sel].mean()),
                         "us_per_1k_keys": float(dur[sel].sum() / keys[sel].sum() * 1e3)}
    busy = np.bincount(cta, weights=dur)
    last_end = np.zeros(cta.max() + 1)
    np.maximum.at(last_end, cta, (t1 - start) / 1e3)
    out["cta_busy_frac_mean"] = float(busy.mean() / span)
    out["first_cta_idle_us"] = float(last_end.min())
    out["tail_us"] = float(span - last_end.min())
    gaps = []
    order = np.lexsort((t0, cta))
    c_s, t0_s, t1_s = cta[order], t0[order], t1[order]
    same = c_s[1:] == c_s[:-1]
    gaps = (t0_s[1:] - t1_s[:-1])[same] / 1e3
    out["gap_between_items_us_mean"] = float(gaps.mean()) if len(gaps) else 0.0
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--ctas-per-sm", type=int, default=0)
    ap.add_argument("--num-sms", type=int, default=0)
    ap.add_argument("--min-chunk", type=int, default=0)
    ap.add_argument("--waves", type=int, default=0)
    ap.add_argument("--groups", type=int, default=0)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--json")
    ap.add_argument("--tile2", type=int, default=1)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    spec = W.config(args.config)
    if args.groups:
        spec = spec.subset([g % spec.G for g in range(args.groups)])
        spec.group_ids = list(range(args.groups))
    b = W.make_batch(spec, dev)
    op = P.PrefixSharedAttention(b["cu_req"], b["cu_q"], b["cu_prefix"], b["cu_distinct"],
                                 spec.Hq, spec.Hkv, spec.d, spec.dv, spec.torch_dtype, dev,
                                 options=P.PlanOptions(ctas_per_sm=args.ctas_per_sm, num_sms=args.num_sms,
                                                       min_chunk_keys=args.min_chunk,
                                                       target_waves=args.waves))
    inputs = (b["q"], b["k_prefix"], b["v_prefix"], b["k_distinct"], b["v_distinct"])
    for _ in range(args.warmup):
        op(*inputs)
    torch.cuda.synchronize()
    tr, ctas = op.trace(*inputs)
    rep = report(tr, op.plan_tables())
    st = tr[:, 2].min()
    rep["cta_start_us_pct"] = [float(x) for x in np.percentile((ctas[:, 2] - st) / 1e3, [0, 50, 90, 100])]
    rep["ctas_per_sm"] = float(len(ctas) / max(1, len(np.unique(ctas[:, 0] >> 32))))
    rep["num_ctas"] = int(len(ctas))
    ev = getattr(op, "last_tile_events", None)
    if ev is not None and op.plan_tables()["num_tile_items"] > 0 and ev[0, 0] != 0 and args.tile2:
        # v2 tile events (CTA 0, slot 0): clock64 per block
        names = ["s_ready", "ld_done", "max_done", "exp_done", "p_arrive", "s_issue", "pv_issue",
                 "k_issue", "v_issue", "s1_ready", "s1_exp_done", "s1_p_arrive", "s1_s_issue",
                 "s1_pv_issue"]
        t0 = ev[7, 0]
        nb = int((ev[0] != 0).sum())
        rep["tile2_events_cycles"] = {nm: [int(x - t0) if x else 0 for x in ev[i, :min(nb, 24)]]
                                      for i, nm in enumerate(names)}
    elif ev is not None and ev[5, 2] != 0:
        t0 = ev[5, 2]
        names = ["prod_issue", "s_issue", "soft_s_ready", "p_arrive", "pv_issue", "misc",
                 "k_wait_start", "v_wait_start", "v_issue"]
        nb = int((ev[0] != 0).sum())
        rep["tile0_events_cycles"] = {nm: [int(x - t0) for x in ev[i, :nb]] for i, nm in enumerate(names) if nm != "misc"}
        rep["tile0_softmax_end"] = int(ev[5, 0] - t0)
        rep["tile0_item_end"] = int(ev[5, 1] - t0)
    dv = getattr(op, "last_dec_events", None)
    if dv is not None and dv[0, 0] != 0:
        t0 = dv[0, 0]
        nb = int((dv[2] != 0).sum())
        names = ["k_issue", "v_issue", "s_issue", "pv_issue", "soft_s_ready", "p_arrive", "item_end", "epi_ofull_wait", "epi_ofull_done", "epi_finish_done", "ld_done", "max_done", "bar1_done", "exp_done", "odone_done", "pstore_done", "fence_done"]
        rep["dec0_events_cycles"] = {nm: [int(x - t0) if x else 0 for x in dv[i, :min(nb, 16)]]
                                     for i, nm in enumerate(names)}
        d2 = getattr(op, "last_dec_events2", None)
        if d2 is not None:
            for i, nm in enumerate(["epi_tmem_ld_done", "item_full_done", "fetch_issued"]):
                rep["dec0_events_cycles"][nm] = [int(x - t0) if x else 0 for x in d2[i, :min(nb, 16)]]
    ph = getattr(op, "last_phase", None)
    if ph is not None and (ph[:, 3] != 0).any():
        st = tr[:, 2].min()
        sel = ph[:, 3] != 0
        rep["tile_phase_end_us_pct"] = {nm: [float(x) for x in np.percentile((ph[sel, i] - st) / 1e3, [0, 50, 90, 100])]
                                        for i, nm in enumerate(["softmax", "support", "merge", "barrier"])}
    dp = getattr(op, "last_dec_phase", None)
    if dp is not None and (dp[:, 0] != 0).any():
        st = tr[:, 2].min()
        sel = dp[:, 0] != 0
        rep["dec_phase_end_us_pct"] = {nm: [float(x) for x in np.percentile((dp[sel, i] - st) / 1e3, [0, 50, 90, 100])]
                                       for i, nm in enumerate(["softmax", "producer", "mma", "merge"])}
    mt = getattr(op, "last_merge_tasks", None)
    if mt is not None and (mt[0] != 0).any():
        sel = (mt[0] != 0) & (mt[3] != 0)
        rep["dec_arrival_cycles_p50"] = {
            "fence": 0, "atomic": float(np.median(mt[1, sel] - mt[0, sel])),
            "fence2": float(np.median(mt[2, sel] - mt[1, sel])),
            "merge": float(np.median(mt[3, sel] - mt[2, sel])), "n": int(sel.sum())}
    rep["config"] = args.config
    print(json.dumps(rep, indent=1))
    if args.json:
        with open(args.json, "w") as f:
            json.dump(rep, f, indent=1)
        np.save(args.json.replace(".json", ".npy"), tr)
        np.save(args.json.replace(".json", "_ctas.npy"), ctas)


if __name__ == "__main__":
    main()
