"""Group slabs: a packed batch cut into contiguous runs of whole groups.

Groups are independent (``prefix_shared_attention`` has no cross-group term,
attention.py:156-201), and in the packed layout (include/psa.h) the tokens,
prefix keys and distinct keys of consecutive groups are contiguous row ranges.
So a run of groups ``[g0, g1)`` is a batch of its own: row-range views of the
five packed tensors plus rebased offset tables — no gather, no copy.

Two users:

* :class:`HostStreamedAttention` — an offline batch resident in (pinned) host
  memory, larger than one wants to keep in HBM: slab ``i + 1`` is copied to the
  device on a copy stream while slab ``i`` runs (one persistent launch per
  slab), and each slab's output is copied back on a third stream. This is the
  end-to-end path ``bench.py`` times (host buffers in, host output out).
* ``distributed.SlabGather`` — the multi-GPU output gather overlapped with the
  compute of the next slab.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

from . import packed as P
from .errors import ValidationError


@dataclass(frozen=True)
class Slab:
    g0: int
    g1: int
    t0: int   # token rows [t0, t1)
    t1: int
    p0: int   # prefix key rows [p0, p1)
    p1: int
    d0: int   # distinct key rows [d0, d1)
    d1: int
    cu_req: tuple
    cu_q: tuple
    cu_prefix: tuple
    cu_distinct: tuple

    @property
    def structure(self) -> tuple:
        """Everything a plan depends on (slabs with equal structure share a plan)."""
        return (self.cu_req, self.cu_q, self.cu_prefix, self.cu_distinct)


def cut_slabs(cu_req, cu_q, cu_prefix, cu_distinct, row_bytes: dict,
              max_bytes: int) -> list[Slab]:
    """Greedy cut into runs of whole groups with at most ``max_bytes`` of inputs each
    (a group larger than ``max_bytes`` gets a slab of its own).

    ``row_bytes``: bytes per token row (``q``), prefix key row (``kv_prefix``: K + V)
    and distinct key row (``kv_distinct``)."""
    cu_req, cu_q, cu_prefix, cu_distinct = (np.asarray(x, dtype=np.int64)
                                            for x in (cu_req, cu_q, cu_prefix, cu_distinct))
    G = len(cu_req) - 1
    if G < 1:
        raise ValidationError("a batch needs at least one group")

    def group_bytes(g):
        r0, r1 = int(cu_req[g]), int(cu_req[g + 1])
        return (row_bytes["q"] * int(cu_q[r1] - cu_q[r0])
                + row_bytes["kv_prefix"] * int(cu_prefix[g + 1] - cu_prefix[g])
                + row_bytes["kv_distinct"] * int(cu_distinct[r1] - cu_distinct[r0]))

    bounds, g0, acc = [], 0, 0
    for g in range(G):
        b = group_bytes(g)
        if g > g0 and acc + b > max_bytes:
            bounds.append((g0, g))
            g0, acc = g, 0
        acc += b
    bounds.append((g0, G))
    slabs = []
    for a, b in bounds:
        r0, r1 = int(cu_req[a]), int(cu_req[b])
        slabs.append(Slab(
            a, b, int(cu_q[r0]), int(cu_q[r1]), int(cu_prefix[a]), int(cu_prefix[b]),
            int(cu_distinct[r0]), int(cu_distinct[r1]),
            tuple(int(x) for x in cu_req[a:b + 1] - cu_req[a]),
            tuple(int(x) for x in cu_q[r0:r1 + 1] - cu_q[r0]),
            tuple(int(x) for x in cu_prefix[a:b + 1] - cu_prefix[a]),
            tuple(int(x) for x in cu_distinct[r0:r1 + 1] - cu_distinct[r0])))
    return slabs


def slab_views(s: Slab, q, k_prefix, v_prefix, k_distinct, v_distinct):
    """Row-range views of the five packed tensors for slab ``s``."""
    return (q[s.t0:s.t1], k_prefix[s.p0:s.p1], v_prefix[s.p0:s.p1],
            k_distinct[s.d0:s.d1], v_distinct[s.d0:s.d1])


class SlabPlans:
    """One planned op per distinct slab structure (uniform batches share one plan)."""

    def __init__(self, num_q_heads, num_kv_heads, head_dim, value_dim, dtype, device,
                 scale=None, options: Optional[P.PlanOptions] = None):
        self.args = (num_q_heads, num_kv_heads, head_dim, value_dim, dtype, device, scale, options)
        self._ops: dict = {}

    def op(self, s: Slab) -> P.PrefixSharedAttention:
        key = s.structure
        if key not in self._ops:
            Hq, Hkv, d, dv, dt, dev, sc, opts = self.args
            self._ops[key] = P.PrefixSharedAttention(
                np.array(s.cu_req), np.array(s.cu_q), np.array(s.cu_prefix),
                np.array(s.cu_distinct), Hq, Hkv, d, dv, dt, dev, sc, opts)
        return self._ops[key]

    def __len__(self):
        return len(self._ops)


class HostStreamedAttention:
    """Prefix-shared attention over a packed batch held in host memory.

    Inputs and the output are host tensors (pinned for asynchronous copies). The
    batch is cut into group slabs of at most ``slab_bytes`` of inputs; two device
    slab buffers alternate: while slab i runs on the compute stream, slab i + 1 is
    copied in on the H2D stream and slab i - 1's output is copied out on the D2H
    stream. ``__call__`` enqueues the work behind the caller's current stream and
    makes the current stream wait for all of it (no host synchronisation)."""

    def __init__(self, cu_req, cu_q, cu_prefix, cu_distinct, num_q_heads: int,
                 num_kv_heads: int, head_dim: int, value_dim: Optional[int] = None,
                 dtype: torch.dtype = torch.bfloat16, device=None, scale=None,
                 options: Optional[P.PlanOptions] = None, slab_bytes: int = 2 << 30):
        dv = value_dim if value_dim is not None else head_dim
        elt = torch.finfo(dtype).bits // 8
        self.Hq, self.Hkv, self.d, self.dv, self.dtype = num_q_heads, num_kv_heads, head_dim, dv, dtype
        self.device = torch.device(device) if device is not None else torch.device("cuda")
        rb = {"q": num_q_heads * head_dim * elt,
              "kv_prefix": num_kv_heads * (head_dim + dv) * elt,
              "kv_distinct": num_kv_heads * (head_dim + dv) * elt}
        self.slabs = cut_slabs(cu_req, cu_q, cu_prefix, cu_distinct, rb, slab_bytes)
        self.plans = SlabPlans(num_q_heads, num_kv_heads, head_dim, dv, dtype, self.device,
                               scale, options)
        for s in self.slabs:
            self.plans.op(s)
        tmax = max(s.t1 - s.t0 for s in self.slabs)
        pmax = max(s.p1 - s.p0 for s in self.slabs)
        dmax = max(s.d1 - s.d0 for s in self.slabs)
        mk = lambda rows, heads, dim: torch.empty((rows, heads, dim), dtype=dtype,  # noqa: E731
                                                  device=self.device)
        self.bufs = [dict(q=mk(tmax, num_q_heads, head_dim),
                          kp=mk(pmax, num_kv_heads, head_dim), vp=mk(pmax, num_kv_heads, dv),
                          kd=mk(dmax, num_kv_heads, head_dim), vd=mk(dmax, num_kv_heads, dv),
                          out=mk(tmax, num_q_heads, dv)) for _ in range(2)]
        self.s_h2d = torch.cuda.Stream(self.device)
        self.s_run = torch.cuda.Stream(self.device)
        self.s_d2h = torch.cuda.Stream(self.device)
        self.launches_per_call = len(self.slabs)

    def bytes_per_call(self) -> tuple[int, int]:
        """(H2D bytes, D2H bytes) one call moves."""
        elt = torch.finfo(self.dtype).bits // 8
        h2d = d2h = 0
        for s in self.slabs:
            h2d += elt * ((s.t1 - s.t0) * self.Hq * self.d
                          + (s.p1 - s.p0 + s.d1 - s.d0) * self.Hkv * (self.d + self.dv))
            d2h += elt * (s.t1 - s.t0) * self.Hq * self.dv
        return h2d, d2h

    def __call__(self, q, k_prefix, v_prefix, k_distinct, v_distinct, out):
        for name, t in (("q", q), ("k_prefix", k_prefix), ("v_prefix", v_prefix),
                        ("k_distinct", k_distinct), ("v_distinct", v_distinct), ("out", out)):
            if t.device.type != "cpu" or t.dtype != self.dtype or not t.is_contiguous():
                raise ValidationError(f"{name} must be a contiguous {self.dtype} host tensor")
        cur = torch.cuda.current_stream(self.device)
        for s in (self.s_h2d, self.s_run, self.s_d2h):
            s.wait_stream(cur)
        ev_in = [torch.cuda.Event() for _ in range(2)]     # slab copied in
        ev_run = [torch.cuda.Event() for _ in range(2)]    # slab computed (inputs free)
        ev_out = [torch.cuda.Event() for _ in range(2)]    # slab output copied out
        used = [False, False]
        for i, s in enumerate(self.slabs):
            b = i & 1
            buf = self.bufs[b]
            src = slab_views(s, q, k_prefix, v_prefix, k_distinct, v_distinct)
            dst = slab_views(Slab(0, 0, 0, s.t1 - s.t0, 0, s.p1 - s.p0, 0, s.d1 - s.d0,
                                  (), (), (), ()),
                             buf["q"], buf["kp"], buf["vp"], buf["kd"], buf["vd"])
            with torch.cuda.stream(self.s_h2d):
                if used[b]:
                    self.s_h2d.wait_event(ev_run[b])
                for dt, st in zip(dst, src):
                    if st.numel():
                        dt.copy_(st, non_blocking=True)
                ev_in[b].record(self.s_h2d)
            with torch.cuda.stream(self.s_run):
                self.s_run.wait_event(ev_in[b])
                if used[b]:
                    self.s_run.wait_event(ev_out[b])
                o = buf["out"][:s.t1 - s.t0]
                self.plans.op(s)(*dst, out=o, stream=self.s_run)
                ev_run[b].record(self.s_run)
            with torch.cuda.stream(self.s_d2h):
                self.s_d2h.wait_event(ev_run[b])
                out[s.t0:s.t1].copy_(o, non_blocking=True)
                ev_out[b].record(self.s_d2h)
            used[b] = True
        for s in (self.s_h2d, self.s_run, self.s_d2h):
            cur.wait_stream(s)
        return out
