"""Float64 NumPy restatement of the reference's segmented-attention oracle.

TEST INFRASTRUCTURE (see ``oracle/__init__.py``). Restates
``/root/reference/pkg/src/prefixbatch/attention.py`` (cited below as
``attention.py:<line>``) so that the parity tests and the CPU baseline can run
where the reference is absent (the GPU box). Pinned against the reference's
own outputs by ``tests/golden/make_golden.py`` + ``tests/test_oracle.py``.

A partial result is the triple ``(o, m, l)``: unnormalised weighted-value
accumulator, running max logit, sum of exponentials shifted by ``m``
(attention.py:47-67). The empty triple ``(0, -inf, 0)`` is the merge identity.
"""

from __future__ import annotations

from typing import NamedTuple, Optional, Sequence

import numpy as np


class OracleValidationError(Exception):
    """Raised where the reference raises ``ValidationError`` (errors.py:18-19)."""


class Partial(NamedTuple):
    o: np.ndarray  # (rows, value_dim) float64
    m: np.ndarray  # (rows,)
    l: np.ndarray  # (rows,)


def to_matrix(x, what: str) -> np.ndarray:
    """attention.py:26-32 — float64 copy; 2-D, positive dims, all finite."""
    arr = np.array(x, dtype=np.float64, copy=True)
    if arr.ndim != 2 or min(arr.shape) < 1:
        raise OracleValidationError(f"{what} must be a 2-D matrix with positive dimensions")
    if not np.all(np.isfinite(arr)):
        raise OracleValidationError(f"{what} contains non-finite entries")
    return arr


def checked_segment(q: np.ndarray, keys, values, what: str):
    """attention.py:35-44 — keys share q's head dim; values share keys' length."""
    k = to_matrix(keys, f"{what} keys")
    v = to_matrix(values, f"{what} values")
    if k.shape[1] != q.shape[1]:
        raise OracleValidationError(
            f"{what} keys have head dim {k.shape[1]}, queries have {q.shape[1]}")
    if k.shape[0] != v.shape[0]:
        raise OracleValidationError(f"{what} keys and values disagree on sequence length")
    return k, v


def empty(rows: int, value_dim: int) -> Partial:
    """attention.py:70-75 — the merge identity."""
    return Partial(np.zeros((rows, value_dim)), np.full(rows, -np.inf), np.zeros(rows))


def segment_partial(q, keys, values, scale: Optional[float] = None,
                    logit_offset: float = 0.0) -> Partial:
    """attention.py:78-98 — unnormalised attention of q against one segment.

    A missing or zero-size key segment yields the empty partial whose value dim
    is taken from ``values`` when that is 2-D, else from q (attention.py:87-89).
    """
    q = to_matrix(q, "queries")
    if keys is None or values is None or np.size(keys) == 0:
        vals = None if values is None else np.asarray(values)
        dv = vals.shape[1] if (vals is not None and vals.ndim == 2) else q.shape[1]
        return empty(q.shape[0], dv)
    k, v = checked_segment(q, keys, values, "segment")
    s = (1.0 / np.sqrt(q.shape[1])) if scale is None else scale
    if s <= 0:
        raise OracleValidationError("scale must be positive")
    logits = s * (q @ k.T) + logit_offset
    row_max = np.max(logits, axis=1)
    w = np.exp(logits - row_max[:, None])
    return Partial(w @ v, row_max, np.sum(w, axis=1))


def combine(a: Partial, b: Partial) -> Partial:
    """attention.py:101-119 — online-softmax merge; rows with l == 0 contribute 0."""
    if a.o.shape != b.o.shape:
        raise OracleValidationError(f"partial result shapes differ: {a.o.shape} vs {b.o.shape}")
    m = np.maximum(a.m, b.m)
    with np.errstate(invalid="ignore"):
        wa = np.where(a.l > 0, np.exp(a.m - m), 0.0)
        wb = np.where(b.l > 0, np.exp(b.m - m), 0.0)
    return Partial(wa[:, None] * a.o + wb[:, None] * b.o, m, wa * a.l + wb * b.l)


def normalize(p: Partial) -> np.ndarray:
    """attention.py:122-126 — o / l; rows that saw no keys are an error."""
    if np.any(p.l <= 0):
        raise OracleValidationError(
            "cannot finalize: some rows attended to an empty segment set")
    return p.o / p.l[:, None]


def dense_attention(q, keys, values, scale: Optional[float] = None) -> np.ndarray:
    """attention.py:129-141 — dense softmax(scale Q K^T) V; scale 0 allowed."""
    q = to_matrix(q, "queries")
    k, v = checked_segment(q, keys, values, "full")
    s = (1.0 / np.sqrt(q.shape[1])) if scale is None else scale
    if s < 0:
        raise OracleValidationError("scale must be non-negative")
    z = s * (q @ k.T)
    z = z - z.max(axis=1, keepdims=True)
    w = np.exp(z)
    w = w / w.sum(axis=1, keepdims=True)
    return w @ v


def group_attention(queries: Sequence, prefix, distinct: Sequence,
                    scale: Optional[float] = None) -> list:
    """attention.py:156-201 — one prefix-sharing group.

    ``prefix`` is a (K, V) pair or None; ``distinct`` one (K, V) pair or None
    per request. The prefix partial is evaluated once on the vertically
    stacked queries (attention.py:174-179) and sliced back per request in list
    order with a running row cursor (attention.py:182-200).
    """
    if len(queries) != len(distinct):
        raise OracleValidationError("one distinct KV pair per request is required")
    qs = [to_matrix(q, f"queries[{i}]") for i, q in enumerate(queries)]
    d = qs[0].shape[1]  # IndexError on an empty list, like attention.py:167
    if any(q.shape[1] != d for q in qs):
        raise OracleValidationError("all query matrices must share the head dimension")
    s = (1.0 / np.sqrt(d)) if scale is None else scale

    shared = None
    if prefix is not None:
        shared = segment_partial(np.vstack(qs), prefix[0], prefix[1], s)

    out = []
    cursor = 0
    for q, pair in zip(qs, distinct):
        n = q.shape[0]
        if pair is None and shared is None:
            raise OracleValidationError("request has neither prefix nor distinct keys")
        own = (segment_partial(q, pair[0], pair[1], s) if pair is not None
               else empty(n, shared.o.shape[1]))
        if shared is not None:
            sl = slice(cursor, cursor + n)
            own = combine(Partial(shared.o[sl], shared.m[sl], shared.l[sl]), own)
        out.append(normalize(own))
        cursor += n
    return out


# --------------------------------------------------------------------------
# Multi-head / GQA adapter over the packed layout.
# The reference is single-head; for kv head h, request r contributes the rows
# q[tokens of r, h*gqa:(h+1)*gqa, :] flattened (token-major, head-minor). One
# group_attention call per (group, kv head).
# --------------------------------------------------------------------------

def packed_group_head(q, kp, vp, kd, vd, cu_req, cu_q, cu_prefix, cu_distinct,
                      g: int, h: int, num_q_heads: int, num_kv_heads: int,
                      scale: Optional[float] = None, prefix_present=True):
    """Run the oracle for one (group, kv head); returns a list of (n_r*gqa, dv)."""
    gqa = num_q_heads // num_kv_heads
    r0, r1 = int(cu_req[g]), int(cu_req[g + 1])
    queries, distinct = [], []
    for r in range(r0, r1):
        t0, t1 = int(cu_q[r]), int(cu_q[r + 1])
        queries.append(np.asarray(q[t0:t1, h * gqa:(h + 1) * gqa, :], dtype=np.float64)
                       .reshape((t1 - t0) * gqa, -1))
        d0, d1 = int(cu_distinct[r]), int(cu_distinct[r + 1])
        distinct.append((np.asarray(kd[d0:d1, h, :], dtype=np.float64),
                         np.asarray(vd[d0:d1, h, :], dtype=np.float64)) if d1 > d0 else None)
    p0, p1 = int(cu_prefix[g]), int(cu_prefix[g + 1])
    prefix = None
    if prefix_present and p1 > p0:
        prefix = (np.asarray(kp[p0:p1, h, :], dtype=np.float64),
                  np.asarray(vp[p0:p1, h, :], dtype=np.float64))
    return group_attention(queries, prefix, distinct, scale)


def packed_attention(q, kp, vp, kd, vd, cu_req, cu_q, cu_prefix, cu_distinct,
                     num_q_heads: int, num_kv_heads: int, scale=None,
                     groups: Optional[Sequence[int]] = None) -> np.ndarray:
    """Whole packed batch through the oracle: O[total_q, Hq, dv] float64.

    Layouts: q [T, Hq, d]; kp/vp [sum P_g, Hkv, d|dv];
    kd/vd [sum D_r, Hkv, d|dv]; requests of group g are cu_req[g]:cu_req[g+1].
    ``groups`` restricts evaluation to a subset (rows of other groups stay 0).
    """
    q = np.asarray(q)
    gqa = num_q_heads // num_kv_heads
    dv = np.asarray(vp).shape[-1] if np.asarray(vp).size else np.asarray(vd).shape[-1]
    out = np.zeros((q.shape[0], num_q_heads, dv))
    G = len(cu_req) - 1
    for g in (range(G) if groups is None else groups):
        for h in range(num_kv_heads):
            res = packed_group_head(q, kp, vp, kd, vd, cu_req, cu_q, cu_prefix,
                                    cu_distinct, g, h, num_q_heads, num_kv_heads, scale)
            for i, r in enumerate(range(int(cu_req[g]), int(cu_req[g + 1]))):
                t0, t1 = int(cu_q[r]), int(cu_q[r + 1])
                out[t0:t1, h * gqa:(h + 1) * gqa, :] = res[i].reshape(t1 - t0, gqa, dv)
    return out


# --------------------------------------------------------------------------
# Causal prefill (EXTENSION, no reference counterpart: the reference attends every
# key, attention.py:12-13). Used only to check PSA_FLAG_CAUSAL (include/psa.h):
# query token j of request r (n_q tokens) sees distinct keys 0 .. D_r - n_q + j and
# every prefix key; a request without distinct KV sees prefix keys 0 .. P - n_q + j.
# --------------------------------------------------------------------------

def packed_attention_causal(q, kp, vp, kd, vd, cu_req, cu_q, cu_prefix, cu_distinct,
                            num_q_heads: int, num_kv_heads: int, scale=None,
                            groups: Optional[Sequence[int]] = None) -> np.ndarray:
    q = np.asarray(q, dtype=np.float64)
    gqa = num_q_heads // num_kv_heads
    d = q.shape[-1]
    s = (1.0 / np.sqrt(d)) if scale is None else scale
    dv = np.asarray(vp).shape[-1] if np.asarray(vp).size else np.asarray(vd).shape[-1]
    out = np.zeros((q.shape[0], num_q_heads, dv))
    G = len(cu_req) - 1
    for g in (range(G) if groups is None else groups):
        p0, p1 = int(cu_prefix[g]), int(cu_prefix[g + 1])
        for r in range(int(cu_req[g]), int(cu_req[g + 1])):
            t0, t1 = int(cu_q[r]), int(cu_q[r + 1])
            d0, d1 = int(cu_distinct[r]), int(cu_distinct[r + 1])
            nq, P, D = t1 - t0, p1 - p0, d1 - d0
            for h in range(num_kv_heads):
                K = np.concatenate([np.asarray(kp[p0:p1, h], np.float64),
                                    np.asarray(kd[d0:d1, h], np.float64)])
                V = np.concatenate([np.asarray(vp[p0:p1, h], np.float64),
                                    np.asarray(vd[d0:d1, h], np.float64)])
                for j in range(nq):
                    vis = np.zeros(P + D, dtype=bool)
                    if D > 0:
                        vis[:P] = True
                        vis[P:P + D - nq + j + 1] = True
                    else:
                        vis[:P - nq + j + 1] = True
                    Qj = q[t0 + j, h * gqa:(h + 1) * gqa]          # [gqa, d]
                    z = s * (Qj @ K[vis].T)
                    z -= z.max(axis=1, keepdims=True)
                    w = np.exp(z)
                    out[t0 + j, h * gqa:(h + 1) * gqa] = (w @ V[vis]) / w.sum(axis=1, keepdims=True)
    return out
