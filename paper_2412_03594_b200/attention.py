"""Drop-in for ``prefixbatch.attention`` (pkg/src/prefixbatch/attention.py).

Same public names, argument meaning and error behaviour as the reference
module; every computation runs in libpsa.so on the GPU (there is no CPU
fallback — without a CUDA device or the native library these functions
raise).

Two modes, chosen by the inputs:
  * NumPy / nested lists (the reference's own calling convention): the strict
    drop-in. Inputs are evaluated in float64 on the GPU (DFMA path) and the
    results come back as float64 NumPy arrays, like the reference.
  * torch tensors: evaluated in the tensors' dtype (bf16/f16 on the tcgen05 +
    decode paths, f32 FFMA, f64 DFMA) on their CUDA device; results are
    tensors of that dtype.

Validation follows the reference's order exactly (the first error the
reference would raise is the one raised here); the finiteness checks of
``_as_matrix`` (attention.py:30-31) run on the device in one batched pass.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np
import torch

from . import packed as P
from .errors import ValidationError

__all__ = ["PartialResult", "SegmentedKV", "empty_partial", "partial_attention", "merge",
           "finalize", "naive_attention", "prefix_shared_attention", "run_selftest"]


# ---- data model (attention.py:47-75, :144-153) ------------------------------

@dataclass
class PartialResult:
    """Per-row running state (o, m, l); empty = (0, -inf, 0) (attention.py:47-67)."""

    o: object
    m: object
    l: object

    @property
    def rows(self) -> int:
        return self.o.shape[0]

    @property
    def value_dim(self) -> int:
        return self.o.shape[1]


def empty_partial(rows: int, value_dim: int) -> PartialResult:
    """attention.py:70-75."""
    return PartialResult(o=np.zeros((rows, value_dim)), m=np.full(rows, -np.inf),
                         l=np.zeros(rows))


@dataclass
class SegmentedKV:
    """Shared prefix (K, V) or None plus one (K, V) or None per request (attention.py:144-153)."""

    prefix: Optional[tuple]
    distinct: Sequence[Optional[tuple]]


# ---- input handling -----------------------------------------------------------

class _Ctx:
    """Execution mode: strict float64 (NumPy in/out) or torch dtype/device."""

    def __init__(self, *objs):
        ref = next((o for o in _flatten(objs) if isinstance(o, torch.Tensor)), None)
        if ref is None:
            self.torch_mode = False
            self.dtype = torch.float64
            self.device = torch.device("cuda", _cuda_device())
            self.out_device = None
        else:
            self.torch_mode = True
            self.dtype = ref.dtype if ref.dtype in (torch.float32, torch.float64, torch.bfloat16,
                                                     torch.float16) else torch.float32
            self.device = ref.device if ref.device.type == "cuda" else torch.device(
                "cuda", _cuda_device())
            self.out_device = ref.device

    def tensor(self, x) -> torch.Tensor:
        if isinstance(x, torch.Tensor):
            return x.detach().to(device=self.device, dtype=self.dtype)
        return torch.as_tensor(np.asarray(x, dtype=np.float64), device=self.device).to(self.dtype)

    def acc(self) -> torch.dtype:
        return P.acc_dtype(self.dtype)

    def result(self, t: torch.Tensor):
        if self.torch_mode:
            return t.to(self.out_device)
        return t.detach().to(torch.float64).cpu().numpy()


def _flatten(objs):
    for o in objs:
        if isinstance(o, (list, tuple)):
            yield from _flatten(o)
        elif isinstance(o, PartialResult):
            yield from (o.o, o.m, o.l)
        elif isinstance(o, SegmentedKV):
            yield from _flatten([o.prefix, list(o.distinct)])
        else:
            yield o


def _cuda_device() -> int:
    if not torch.cuda.is_available():
        raise RuntimeError("prefix-shared attention runs on a CUDA device only; none is visible "
                           "(this drop-in has no CPU fallback)")
    return torch.cuda.current_device()


def _shape(x):
    if isinstance(x, torch.Tensor):
        return tuple(x.shape)
    return np.shape(np.asarray(x, dtype=np.float64)) if x is not None else np.shape(
        np.asarray(None, dtype=np.float64))


def _size(x) -> int:
    return x.numel() if isinstance(x, torch.Tensor) else int(np.size(x))


class _Checks:
    """Records the reference's validation sequence; finiteness is resolved on device."""

    def __init__(self, ctx: _Ctx):
        self.ctx = ctx
        self.steps = []      # (kind, message, payload)
        self.tensors = []    # device tensors whose non-finite count decides a step
        self.stopped = False

    def matrix(self, x, name: str):
        """_as_matrix (attention.py:26-32). Returns the device tensor or None after a stop."""
        if self.stopped:
            return None
        shp = _shape(x)
        if len(shp) != 2 or shp[0] < 1 or shp[1] < 1:
            self.fail(f"{name} must be a 2-D matrix with positive dimensions")
            return None
        t = self.ctx.tensor(x)
        self.steps.append(("finite", f"{name} contains non-finite entries", len(self.tensors)))
        self.tensors.append(t)
        return t

    def fail(self, message: str):
        if not self.stopped:
            self.steps.append(("fail", message, None))
            self.stopped = True

    def resolve(self):
        """Raise the first error the reference would raise."""
        counts = None
        if self.tensors:
            counter = torch.zeros(len(self.tensors), dtype=torch.int32, device=self.ctx.device)
            for i, t in enumerate(self.tensors):
                P.count_nonfinite(t, counter[i:i + 1])
            counts = counter.cpu().tolist()
        for kind, message, idx in self.steps:
            if kind == "fail" or (kind == "finite" and counts[idx] > 0):
                raise ValidationError(message)


def _segment(chk: _Checks, q_dim: int, q_rows: int, k, v, name: str):
    """Validation half of partial_attention for one segment (attention.py:86-94).

    Returns (K, V, value_dim); K is None for an empty / absent segment.
    """
    if k is None or v is None or _size(k) == 0:
        vs = _shape(v) if v is not None else ()
        return None, None, (vs[1] if len(vs) == 2 else q_dim)
    kt = chk.matrix(k, f"{name} keys")
    vt = chk.matrix(v, f"{name} values")
    if chk.stopped:
        return None, None, 0
    if kt.shape[1] != q_dim:
        chk.fail(f"{name} keys have head dim {kt.shape[1]}, queries have {q_dim}")
    elif vt.shape[0] != kt.shape[0]:
        chk.fail(f"{name} keys and values disagree on sequence length")
    return kt, vt, (vt.shape[1] if vt is not None else 0)


def _run_group(ctx: _Ctx, qs, pk, pv, dks, dvs, dv: int, scale: float,
               partial_out: bool = False):
    """One single-head group through the persistent kernel (G=1, Hq=Hkv=1)."""
    n = [q.shape[0] for q in qs]
    d = qs[0].shape[1]
    Pn = pk.shape[0] if pk is not None else 0
    D = [k.shape[0] if k is not None else 0 for k in dks]
    cu_q = np.cumsum([0] + n)
    cu_d = np.cumsum([0] + D)
    op = P.PrefixSharedAttention([0, len(qs)], cu_q, [0, Pn], cu_d, 1, 1, d, dv, ctx.dtype,
                                 ctx.device, scale)
    q = torch.cat(qs).reshape(-1, 1, d).contiguous()
    kp = pk.reshape(Pn, 1, d).contiguous() if Pn else None
    vp = pv.reshape(Pn, 1, dv).contiguous() if Pn else None
    live = [i for i, x in enumerate(D) if x > 0]
    kd = torch.cat([dks[i] for i in live]).reshape(-1, 1, d).contiguous() if live else None
    vd = torch.cat([dvs[i] for i in live]).reshape(-1, 1, dv).contiguous() if live else None
    T = int(cu_q[-1])
    if partial_out:
        o = torch.empty((T, 1, dv), dtype=ctx.acc(), device=ctx.device)
        m = torch.empty((T, 1), dtype=ctx.acc(), device=ctx.device)
        l = torch.empty((T, 1), dtype=ctx.acc(), device=ctx.device)
        op(q, kp, vp, kd, vd, partial=(o, m, l))
        return o.reshape(T, dv), m.reshape(T), l.reshape(T)
    out = op(q, kp, vp, kd, vd)
    return out.reshape(T, dv)


# ---- public API -----------------------------------------------------------------

def partial_attention(q, k, v, scale: float | None = None,
                      logit_offset: float = 0.0) -> PartialResult:
    """attention.py:78-98 on the GPU. ``logit_offset`` shifts m only (o, l invariant)."""
    ctx = _Ctx(q, k, v)
    chk = _Checks(ctx)
    qt = chk.matrix(q, "queries")
    if chk.stopped:
        chk.resolve()
    kt, vt, dv = _segment(chk, qt.shape[1], qt.shape[0], k, v, "segment")
    if kt is not None and not chk.stopped:
        s = scale if scale is not None else 1.0 / math.sqrt(qt.shape[1])
        if s <= 0:
            chk.fail("scale must be positive")
    chk.resolve()
    if kt is None:
        e = empty_partial(qt.shape[0], dv)
        if ctx.torch_mode:
            return PartialResult(*(torch.as_tensor(a, dtype=ctx.acc(), device=ctx.out_device)
                                   for a in (e.o, e.m, e.l)))
        return e
    s = scale if scale is not None else 1.0 / math.sqrt(qt.shape[1])
    o, m, l = _run_group(ctx, [qt], None, None, [kt], [vt], dv, float(s), partial_out=True)
    m = m + logit_offset
    return PartialResult(ctx.result(o), ctx.result(m), ctx.result(l))


def merge(a: PartialResult, b: PartialResult) -> PartialResult:
    """attention.py:101-119 on the GPU (psa_merge)."""
    if tuple(_shape(a.o)) != tuple(_shape(b.o)):
        raise ValidationError(f"partial result shapes differ: {tuple(_shape(a.o))} vs "
                              f"{tuple(_shape(b.o))}")
    ctx = _Ctx(a, b)
    acc = ctx.acc()
    rows, dv = _shape(a.o)
    dev = ctx.device

    def t(x):
        return (x.detach() if isinstance(x, torch.Tensor) else torch.as_tensor(
            np.asarray(x, dtype=np.float64))).to(device=dev, dtype=acc).contiguous()

    ins = [t(x) for x in (a.o, a.m, a.l, b.o, b.m, b.l)]
    o = torch.empty((rows, dv), dtype=acc, device=dev)
    m = torch.empty((rows,), dtype=acc, device=dev)
    l = torch.empty((rows,), dtype=acc, device=dev)
    from . import _lib as L
    import ctypes as C
    with torch.cuda.device(dev):
        st = L.lib().psa_merge(rows, dv, P.psa_dtype(acc), *[P._ptr(x) for x in ins],
                               P._ptr(o), P._ptr(m), P._ptr(l),
                               C.c_void_p(torch.cuda.current_stream(dev).cuda_stream))
    if st != L.PSA_OK:
        P._raise_native(st, "psa_merge")
    return PartialResult(ctx.result(o), ctx.result(m), ctx.result(l))


def finalize(p: PartialResult):
    """attention.py:122-126 on the GPU (psa_finalize); rows with l <= 0 raise."""
    ctx = _Ctx(p)
    acc = ctx.acc()
    dev = ctx.device
    rows, dv = _shape(p.o)

    def t(x):
        return (x.detach() if isinstance(x, torch.Tensor) else torch.as_tensor(
            np.asarray(x, dtype=np.float64))).to(device=dev, dtype=acc).contiguous()

    o, l = t(p.o), t(p.l)
    out = torch.empty((rows, dv), dtype=acc, device=dev)
    bad = torch.zeros(1, dtype=torch.int32, device=dev)
    from . import _lib as L
    import ctypes as C
    with torch.cuda.device(dev):
        st = L.lib().psa_finalize(rows, dv, P.psa_dtype(acc), P._ptr(o), P._ptr(l), P._ptr(out),
                                  P._ptr(bad), C.c_void_p(torch.cuda.current_stream(dev).cuda_stream))
    if st != L.PSA_OK:
        P._raise_native(st, "psa_finalize")
    if int(bad.item()) > 0:
        raise ValidationError("cannot finalize: some rows attended to an empty segment set")
    return ctx.result(out)


def naive_attention(q, k, v, scale: float | None = None):
    """attention.py:129-141: dense softmax(scale Q K^T) V (scale 0 allowed) on the GPU."""
    ctx = _Ctx(q, k, v)
    chk = _Checks(ctx)
    qt = chk.matrix(q, "queries")
    kt = vt = None
    if not chk.stopped:
        kt = chk.matrix(k, "full keys")
        vt = chk.matrix(v, "full values")
        if not chk.stopped:
            if kt.shape[1] != qt.shape[1]:
                chk.fail(f"full keys have head dim {kt.shape[1]}, queries have {qt.shape[1]}")
            elif vt.shape[0] != kt.shape[0]:
                chk.fail("full keys and values disagree on sequence length")
    if not chk.stopped:
        s = scale if scale is not None else 1.0 / math.sqrt(qt.shape[1])
        if s < 0:
            chk.fail("scale must be non-negative")
    chk.resolve()
    s = scale if scale is not None else 1.0 / math.sqrt(qt.shape[1])
    return ctx.result(_run_group(ctx, [qt], None, None, [kt], [vt], vt.shape[1], float(s)))


def prefix_shared_attention(queries: Sequence, kv: SegmentedKV,
                            scale: float | None = None) -> list:
    """attention.py:156-201: attention of each request against [shared prefix; own distinct KV].

    The whole group is ONE persistent kernel launch: the shared prefix is
    evaluated once for all stacked query rows, the distinct segments per
    request, and the partials are merged in-kernel.
    """
    if len(queries) != len(kv.distinct):
        raise ValidationError("one distinct KV pair per request is required")
    ctx = _Ctx(list(queries), kv)
    chk = _Checks(ctx)
    qs = []
    for i, q in enumerate(queries):
        qs.append(chk.matrix(q, f"queries[{i}]"))
    if chk.stopped:
        chk.resolve()
    d = qs[0].shape[1]  # IndexError on an empty list, like attention.py:167
    if any(q.shape[1] != d for q in qs):
        chk.fail("all query matrices must share the head dimension")
        chk.resolve()
    s = scale if scale is not None else 1.0 / math.sqrt(d)
    total_rows = sum(q.shape[0] for q in qs)

    pk = pv = None
    prefix_dv = None
    if kv.prefix is not None:
        k0, v0 = kv.prefix
        pk, pv, prefix_dv = _segment(chk, d, total_rows, k0, v0, "segment")
        if pk is not None and not chk.stopped and s <= 0:
            chk.fail("scale must be positive")
    dks, dvs, vdims = [], [], []
    for i, (q, pair) in enumerate(zip(qs, kv.distinct)):
        if chk.stopped:
            break
        n = q.shape[0]
        if pair is None and kv.prefix is None:
            chk.fail("request has neither prefix nor distinct keys")
            break
        if pair is not None:
            k1, v1 = pair
            dk, dvv, part_dv = _segment(chk, d, n, k1, v1, "segment")
            if dk is not None and not chk.stopped and s <= 0:
                chk.fail("scale must be positive")
        else:
            dk = dvv = None
            part_dv = prefix_dv
        if chk.stopped:
            break
        if kv.prefix is not None and part_dv != prefix_dv:
            chk.fail(f"partial result shapes differ: {(n, prefix_dv)} vs {(n, part_dv)}")
            break
        if pk is None and dk is None:
            chk.fail("cannot finalize: some rows attended to an empty segment set")
            break
        vdims.append(int(part_dv))
        dks.append(dk)
        dvs.append(dvv)
    chk.resolve()
    res = [None] * len(qs)
    # Without a prefix each request is independent and may have its own value
    # dim (the reference never merges them); one launch per value dim then.
    for vdim in sorted(set(vdims)):
        idx = [i for i, x in enumerate(vdims) if x == vdim]
        out = _run_group(ctx, [qs[i] for i in idx], pk, pv, [dks[i] for i in idx],
                         [dvs[i] for i in idx], vdim, float(s))
        row = 0
        for i in idx:
            res[i] = ctx.result(out[row:row + qs[i].shape[0]])
            row += qs[i].shape[0]
    return res


def run_selftest(trials: int = 50, seed: int = 0) -> dict:
    """attention.py:204-274 run against this module's GPU implementations.

    Same generator, checks and tolerances as the reference self-test; the
    dense comparison (`naive_attention`) is the GPU one too, so this checks
    the GPU building blocks against each other in float64.
    """
    rng = np.random.default_rng(seed)
    err = dict(partial_vs_naive=0.0, two_way_merge_vs_naive=0.0, three_way_associativity=0.0,
               empty_segment_identity=0.0, prefix_shared_vs_naive=0.0)
    for _ in range(trials):
        n = int(rng.integers(1, 17))
        d = int(rng.integers(1, 33))
        total = int(rng.integers(3, 129))
        q = rng.uniform(-10, 10, (n, d))
        k = rng.uniform(-10, 10, (total, d))
        v = rng.uniform(-10, 10, (total, d))
        scale = 1.0 / np.sqrt(d)
        expect = naive_attention(q, k, v, scale)
        got = finalize(partial_attention(q, k, v, scale))
        err["partial_vs_naive"] = max(err["partial_vs_naive"], float(np.abs(got - expect).max()))
        cut = int(rng.integers(1, total))
        a = partial_attention(q, k[:cut], v[:cut], scale)
        b = partial_attention(q, k[cut:], v[cut:], scale)
        err["two_way_merge_vs_naive"] = max(err["two_way_merge_vs_naive"],
                                            float(np.abs(finalize(merge(a, b)) - expect).max()))
        c1, c2 = sorted(rng.choice(np.arange(1, total), size=2, replace=False).tolist())
        p1 = partial_attention(q, k[:c1], v[:c1], scale)
        p2 = partial_attention(q, k[c1:c2], v[c1:c2], scale)
        p3 = partial_attention(q, k[c2:], v[c2:], scale)
        left = finalize(merge(merge(p1, p2), p3))
        right = finalize(merge(p1, merge(p2, p3)))
        err["three_way_associativity"] = max(err["three_way_associativity"],
                                             float(np.abs(left - right).max()),
                                             float(np.abs(left - expect).max()))
        whole = partial_attention(q, k, v, scale)
        ident = finalize(merge(whole, empty_partial(n, d)))
        err["empty_segment_identity"] = max(err["empty_segment_identity"],
                                            float(np.abs(ident - finalize(whole)).max()))
        sizes = rng.integers(1, 5, size=3)
        group_q = [rng.uniform(-10, 10, (int(sz), d)) for sz in sizes]
        dl = [int(rng.integers(1, 33)) for _ in sizes]
        kvs = SegmentedKV(prefix=(k, v), distinct=[(rng.uniform(-10, 10, (m, d)),
                                                    rng.uniform(-10, 10, (m, d))) for m in dl])
        outs = prefix_shared_attention(group_q, kvs, scale)
        for gq, pair, out in zip(group_q, kvs.distinct, outs):
            ref = naive_attention(gq, np.vstack([k, pair[0]]), np.vstack([v, pair[1]]), scale)
            err["prefix_shared_vs_naive"] = max(err["prefix_shared_vs_naive"],
                                                float(np.abs(out - ref).max()))
    tol = dict(partial_vs_naive=1e-12, two_way_merge_vs_naive=1e-12,
               three_way_associativity=1e-10, empty_segment_identity=1e-12,
               prefix_shared_vs_naive=1e-10)
    return {"passed": all(err[k_] <= tol[k_] for k_ in err), "trials": trials,
            "max_abs_errors": err, "tolerances": tol}
