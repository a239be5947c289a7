"""Generate the golden fixtures by running the REFERENCE implementation.

Run in the build container (where ``/root/reference`` exists):

    python tests/golden/make_golden.py [--ref /root/reference/pkg/src]

For every case in ``cases.packed_cases()`` the packed inputs are regenerated,
split into single-head per-(group, kv head) calls exactly as SURVEY.md §8(a)
prescribes (rows of request r for kv head h = q[tokens of r, h*gqa:(h+1)*gqa]
flattened token-major), and passed to the reference's
``prefixbatch.attention.prefix_shared_attention`` (attention.py:156-201).
The float64 outputs are stored in ``packed.npz``; ``manifest.json`` records
each spec and the SHA-256 of its inputs. A handful of single-head group cases
(None prefix / None distinct / zero-length segments) exercise the list API.

This script is the only code in the repo that imports the reference; nothing
that runs on the GPU box does.
"""

from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import cases as C  # noqa: E402


def reference_packed(ref, arrays, Hq, Hkv):
    """Call the reference once per (group, kv head) and scatter into O."""
    q, kp, vp, kd, vd = (arrays[k].astype(np.float64) for k in ("q", "kp", "vp", "kd", "vd"))
    cu_req, cu_q = arrays["cu_req"], arrays["cu_q"]
    cu_p, cu_d = arrays["cu_prefix"], arrays["cu_distinct"]
    gqa = Hq // Hkv
    dv = vp.shape[-1]
    out = np.zeros((q.shape[0], Hq, dv))
    for g in range(len(cu_req) - 1):
        reqs = range(int(cu_req[g]), int(cu_req[g + 1]))
        for h in range(Hkv):
            queries, distinct = [], []
            for r in reqs:
                t0, t1 = int(cu_q[r]), int(cu_q[r + 1])
                queries.append(q[t0:t1, h * gqa:(h + 1) * gqa].reshape(-1, q.shape[-1]))
                d0, d1 = int(cu_d[r]), int(cu_d[r + 1])
                distinct.append((kd[d0:d1, h], vd[d0:d1, h]) if d1 > d0 else None)
            p0, p1 = int(cu_p[g]), int(cu_p[g + 1])
            prefix = (kp[p0:p1, h], vp[p0:p1, h]) if p1 > p0 else None
            res = ref.prefix_shared_attention(queries, ref.SegmentedKV(prefix, distinct))
            for i, r in enumerate(reqs):
                t0, t1 = int(cu_q[r]), int(cu_q[r + 1])
                out[t0:t1, h * gqa:(h + 1) * gqa] = res[i].reshape(t1 - t0, gqa, dv)
    return out


def single_head_cases(ref):
    """List-API groups with absent segments; inputs stored verbatim (small)."""
    rng = np.random.default_rng(77)
    out = {}
    specs = [
        # (prefix_len or None, [(n, D or None), ...], d)
        (48, [(2, 5), (1, None), (3, 0)], 16),
        (None, [(1, 7), (4, 12)], 8),
        (0, [(2, 3)], 4),
        (130, [(5, 64), (1, 1), (2, None)], 64),
    ]
    for ci, (P, reqs, d) in enumerate(specs):
        queries = [rng.uniform(-10, 10, (n, d)) for n, _ in reqs]
        distinct = []
        for _, D in reqs:
            distinct.append(None if D is None else
                            (rng.uniform(-10, 10, (D, d)), rng.uniform(-10, 10, (D, d))))
        prefix = None if P is None else (rng.uniform(-10, 10, (P, d)), rng.uniform(-10, 10, (P, d)))
        res = ref.prefix_shared_attention(queries, ref.SegmentedKV(prefix, distinct))
        key = f"sh{ci}"
        out[f"{key}_P"] = np.array(-1 if P is None else P)
        out[f"{key}_pk"] = prefix[0] if prefix is not None else np.zeros((0, d))
        out[f"{key}_pv"] = prefix[1] if prefix is not None else np.zeros((0, d))
        out[f"{key}_n"] = np.array(len(reqs))
        for i, qm in enumerate(queries):
            out[f"{key}_q{i}"] = qm
            pair = distinct[i]
            out[f"{key}_dnone{i}"] = np.array(pair is None)
            out[f"{key}_dk{i}"] = pair[0] if pair is not None else np.zeros((0, d))
            out[f"{key}_dv{i}"] = pair[1] if pair is not None else np.zeros((0, d))
            out[f"{key}_out{i}"] = res[i]
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default="/root/reference/pkg/src")
    args = ap.parse_args()
    sys.path.insert(0, args.ref)
    from prefixbatch import attention as ref  # the reference, imported read-only

    manifest = {"generator": "tests/golden/make_golden.py",
                "reference": "prefixbatch.attention.prefix_shared_attention "
                             "(pkg/src/prefixbatch/attention.py:156-201)",
                "cases": []}
    outs = {}
    for spec in C.packed_cases():
        arrays = C.make_packed(spec)
        outs[spec["name"]] = reference_packed(ref, arrays, spec["Hq"], spec["Hkv"])
        manifest["cases"].append({"spec": spec, "sha256": C.inputs_sha(arrays)})
    np.savez_compressed(os.path.join(HERE, "packed.npz"), **outs)
    np.savez_compressed(os.path.join(HERE, "single_head.npz"), **single_head_cases(ref))
    with open(os.path.join(HERE, "manifest.json"), "w") as f:
        json.dump(manifest, f, indent=1)
    print(f"wrote {len(outs)} packed cases")


if __name__ == "__main__":
    main()
