"""Group-sharded prefix-shared attention across the GPUs of one node.

Prefix groups are independent (``prefix_shared_attention`` has no cross-group term,
attention.py:156-201; "per-request partials may be computed in parallel and merged
in any order"), so a token batch is partitioned by whole groups
(greedy LPT over per-group costs, ``psa_shard_groups``). Every rank holds and
computes only its own groups — one persistent launch — and the only collective is
the output gather, skipped when the consumer is group-parallel too.

* :func:`shard` — per-rank offset tables + the global rows each rank's data comes from.
* :func:`select_shard` — cut a rank's rows out of full-batch tensors (tests, loaders).
* :func:`run_local` — one launch over a rank's SHARD-LOCAL tensors.
* :func:`gather_outputs` — one blocking all-gather, reassembled in global token order.
* :class:`SlabGather` — the gather overlapped with compute: the rank's groups run as
  a few group slabs (``streamed.cut_slabs``); slab i's output is all-gathered on a
  communication stream while slab i + 1 computes, so only the last slab's transfer
  is exposed. The persistent kernel leaves ``reserve_sms`` SMs free so the NCCL
  kernels of the overlapped collective can be scheduled next to it.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Optional

import numpy as np
import torch

from . import packed as P
from . import streamed as ST


@dataclass
class Shard:
    """One rank's part of a packed batch: its groups, local offset tables, and the
    global rows (tokens / prefix keys / distinct keys) they come from."""
    groups: np.ndarray
    cu_req: np.ndarray
    cu_q: np.ndarray
    cu_prefix: np.ndarray
    cu_distinct: np.ndarray
    token_rows: np.ndarray
    prefix_rows: np.ndarray
    distinct_rows: np.ndarray

    @property
    def num_tokens(self) -> int:
        return int(self.cu_q[-1])

    @property
    def num_groups(self) -> int:
        return len(self.groups)


def _ranges(cu: np.ndarray, idx) -> np.ndarray:
    parts = [np.arange(int(cu[i]), int(cu[i + 1]), dtype=np.int64) for i in idx]
    return np.concatenate(parts) if parts else np.zeros(0, dtype=np.int64)


def shard(cu_req, cu_q, cu_prefix, cu_distinct, num_q_heads: int, num_kv_heads: int,
          head_dim: int, value_dim: int, dtype: torch.dtype, world: int) -> list[Shard]:
    """Partition a batch by groups (LPT over psa_group_costs); one Shard per rank.
    A rank may get no group (world > number of groups)."""
    cu_req, cu_q, cu_prefix, cu_distinct = (np.asarray(x, dtype=np.int64)
                                            for x in (cu_req, cu_q, cu_prefix, cu_distinct))
    cost = P.group_costs(cu_req, cu_q, cu_prefix, cu_distinct, num_q_heads, num_kv_heads,
                         head_dim, value_dim, dtype)
    owner = P.shard_groups(cost, world)
    out = []
    for rank in range(world):
        gs = np.where(owner == rank)[0]
        reqs = [r for g in gs for r in range(int(cu_req[g]), int(cu_req[g + 1]))]
        cum = lambda lens: np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)  # noqa: E731
        out.append(Shard(
            groups=gs,
            cu_req=cum([int(cu_req[g + 1] - cu_req[g]) for g in gs]),
            cu_q=cum([int(cu_q[r + 1] - cu_q[r]) for r in reqs]),
            cu_prefix=cum([int(cu_prefix[g + 1] - cu_prefix[g]) for g in gs]),
            cu_distinct=cum([int(cu_distinct[r + 1] - cu_distinct[r]) for r in reqs]),
            token_rows=_ranges(cu_q, reqs),
            prefix_rows=_ranges(cu_prefix, gs),
            distinct_rows=_ranges(cu_distinct, reqs)))
    return out


def select_shard(shard_: Shard, q, k_prefix, v_prefix, k_distinct, v_distinct):
    """The shard's rows of full-batch tensors (what a loader would place on the rank)."""
    sel = lambda t, rows: t.index_select(0, torch.as_tensor(rows, device=t.device))  # noqa: E731
    return (sel(q, shard_.token_rows), sel(k_prefix, shard_.prefix_rows),
            sel(v_prefix, shard_.prefix_rows), sel(k_distinct, shard_.distinct_rows),
            sel(v_distinct, shard_.distinct_rows))


def run_local(shard_: Shard, q, k_prefix, v_prefix, k_distinct, v_distinct, num_kv_heads: int,
              scale=None, options=None, value_dim: Optional[int] = None):
    """This rank's launch over its SHARD-LOCAL tensors (``q`` [shard tokens, Hq, d],
    K/V [shard keys, Hkv, d]). An empty shard returns an empty [0, Hq, dv] output so
    the rank still joins the gather."""
    dv = value_dim if value_dim is not None else (
        v_prefix.shape[2] if v_prefix is not None and v_prefix.dim() == 3 else q.shape[2])
    if shard_.num_groups == 0:
        return torch.empty((0, q.shape[1], dv), dtype=q.dtype, device=q.device)
    if q.shape[0] != shard_.num_tokens:
        raise ValueError("run_local takes shard-local tensors (use select_shard)")
    op = P.PrefixSharedAttention(shard_.cu_req, shard_.cu_q, shard_.cu_prefix, shard_.cu_distinct,
                                 q.shape[1], num_kv_heads, q.shape[2], dv, q.dtype, q.device,
                                 scale, options)
    return op(q, k_prefix, v_prefix, k_distinct, v_distinct)


def _reassemble(slabs: list, rows_per_rank: list, token_rows: list, total: int, like):
    """Scatter per-rank slabs (each padded) to global token order."""
    out = torch.empty((total,) + tuple(like.shape[1:]), dtype=like.dtype, device=like.device)
    for r, (slab, n) in enumerate(zip(slabs, rows_per_rank)):
        if n:
            rows = torch.as_tensor(token_rows[r], device=like.device)
            out.index_copy_(0, rows, slab[:n])
    return out


def gather_outputs(local: torch.Tensor, shards: list[Shard], rank: int, group=None) -> torch.Tensor:
    """All ranks' outputs [T_rank, Hq, dv] -> the full batch output [T, Hq, dv] in global
    token order, on every rank: one all_gather of equal-size (padded) slabs."""
    import torch.distributed as dist
    world = len(shards)
    tmax = max(max(s.num_tokens for s in shards), 1)
    pad = torch.zeros((tmax,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[:local.shape[0]] = local
    slabs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(slabs, pad, group=group)
    return _reassemble(slabs, [s.num_tokens for s in shards], [s.token_rows for s in shards],
                       sum(s.num_tokens for s in shards), local)


class SlabGather:
    """Compute a rank's groups slab by slab and all-gather each slab's output while the
    next slab computes (overlapped output gather).

    ``shards``: every rank's Shard (all ranks build the same list). ``num_slabs``: slabs
    per rank (by groups; rank r's slab i holds groups [i*G_r/S, (i+1)*G_r/S)). The
    padded size of slab i is the max over ranks, so every rank issues the same
    collectives. ``compute(i, out_rows)``: writes slab i's output into ``out_rows``
    (a [rows_i, Hq, dv] view) on the current stream — the GPU launch, or the CPU oracle
    in the gloo tests. ``result()`` is the full output in global token order."""

    def __init__(self, shards: list[Shard], rank: int, num_slabs: int, out_shape_tail: tuple,
                 dtype: torch.dtype, device, group=None):
        self.shards, self.rank, self.group = shards, rank, group
        self.world = len(shards)
        self.device = torch.device(device)
        self.num_slabs = max(1, int(num_slabs))
        self.dtype, self.tail = dtype, tuple(out_shape_tail)
        # slab i of rank r: group range and token range (local to the rank)
        self.bounds = []
        for s in shards:
            G = s.num_groups
            cuts = [(G * i) // self.num_slabs for i in range(self.num_slabs + 1)]
            self.bounds.append([(cuts[i], cuts[i + 1], int(s.cu_q[s.cu_req[cuts[i]]]),
                                 int(s.cu_q[s.cu_req[cuts[i + 1]]])) for i in range(self.num_slabs)])
        self.pad_rows = [max(max(b[i][3] - b[i][2] for b in self.bounds), 1)
                         for i in range(self.num_slabs)]
        mk = lambda n: torch.empty((n,) + self.tail, dtype=dtype, device=self.device)  # noqa: E731
        self.send = [mk(n) for n in self.pad_rows]
        self.recv = [[mk(n) for _ in range(self.world)] for n in self.pad_rows]
        self.comm = torch.cuda.Stream(self.device) if self.device.type == "cuda" else None

    def slab_groups(self, i: int) -> tuple[int, int]:
        g0, g1, _, _ = self.bounds[self.rank][i]
        return g0, g1

    def run(self, compute: Callable[[int, torch.Tensor], None]) -> None:
        import torch.distributed as dist
        cuda = self.comm is not None
        cur = torch.cuda.current_stream(self.device) if cuda else None
        for i in range(self.num_slabs):
            g0, g1, t0, t1 = self.bounds[self.rank][i]
            if t1 > t0:
                compute(i, self.send[i][:t1 - t0])
            if cuda:
                ev = torch.cuda.Event()
                ev.record(cur)
                self.comm.wait_event(ev)
                with torch.cuda.stream(self.comm):
                    dist.all_gather(self.recv[i], self.send[i], group=self.group)
            else:
                dist.all_gather(self.recv[i], self.send[i], group=self.group)
        if cuda:
            cur.wait_stream(self.comm)

    def result(self) -> torch.Tensor:
        """Full output [T, Hq, dv] in global token order (after run())."""
        total = sum(s.num_tokens for s in self.shards)
        out = torch.empty((total,) + self.tail, dtype=self.dtype, device=self.device)
        for r, s in enumerate(self.shards):
            for i, (g0, g1, t0, t1) in enumerate(self.bounds[r]):
                if t1 > t0:
                    rows = torch.as_tensor(s.token_rows[t0:t1], device=self.device)
                    out.index_copy_(0, rows, self.recv[i][r][:t1 - t0])
        return out


def time_slab_gather(spec, b, dev, opts, world: int, steps: int, barrier, max_over_ranks,
                     num_slabs: int = 4, reserve_sms: int = 16) -> dict:
    """bench.py --gpus N: the rank's shard as ``num_slabs`` launches with the output
    all-gathered per slab on a side stream (kernel + overlapped gather, max over ranks).
    ``spec``/``b``: this rank's groups (already generated on the device)."""
    import torch.distributed as dist
    from . import workloads as W
    rank = dist.get_rank()
    # every rank's group counts/token counts, to agree on the padded slab sizes
    full = W.config(spec.name)
    gsz = torch.tensor([spec.G], device=dev)
    all_g = [torch.zeros_like(gsz) for _ in range(world)]
    dist.all_gather(all_g, gsz)
    # rebuild the shard list (same LPT owner table on every rank)
    off = W.offsets(full)
    shards = shard(off["cu_req"], off["cu_q"], off["cu_prefix"], off["cu_distinct"], full.Hq,
                   full.Hkv, full.d, full.dv, full.torch_dtype, world)
    sms = opts.num_sms or torch.cuda.get_device_properties(dev).multi_processor_count
    o2 = P.PlanOptions(**{**opts.__dict__, "num_sms": max(1, sms - reserve_sms)})
    sg = SlabGather(shards, rank, num_slabs, (spec.Hq, spec.dv), spec.torch_dtype, dev)
    me = shards[rank]
    elt = torch.finfo(spec.torch_dtype).bits // 8
    ops, views = [], []
    for i in range(num_slabs):
        g0, g1 = sg.slab_groups(i)
        if g1 <= g0:
            ops.append(None)
            views.append(None)
            continue
        r0, r1 = int(me.cu_req[g0]), int(me.cu_req[g1])
        t0, t1 = int(me.cu_q[r0]), int(me.cu_q[r1])
        p0, p1 = int(me.cu_prefix[g0]), int(me.cu_prefix[g1])
        d0, d1 = int(me.cu_distinct[r0]), int(me.cu_distinct[r1])
        ops.append(P.PrefixSharedAttention(
            me.cu_req[g0:g1 + 1] - me.cu_req[g0], me.cu_q[r0:r1 + 1] - t0,
            me.cu_prefix[g0:g1 + 1] - p0, me.cu_distinct[r0:r1 + 1] - d0,
            spec.Hq, spec.Hkv, spec.d, spec.dv, spec.torch_dtype, dev, options=o2))
        views.append((b["q"][t0:t1], b["k_prefix"][p0:p1], b["v_prefix"][p0:p1],
                      b["k_distinct"][d0:d1], b["v_distinct"][d0:d1]))

    def compute(i, out_rows):
        ops[i](*views[i], out=out_rows)

    sg.run(compute)
    torch.cuda.synchronize()
    barrier()
    stream = torch.cuda.current_stream(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        sg.run(compute)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = max_over_ranks(e0.elapsed_time(e1) / steps)
    out_bytes = sum(n * world for n in sg.pad_rows) * spec.Hq * spec.dv * elt
    return {"us_with_gather": round(ms * 1e3, 2), "slabs": num_slabs, "nccl_ranks": world,
            "reserve_sms": reserve_sms, "collective": "all_gather per slab on a side stream",
            "bytes_received_per_rank": int(out_bytes), "steps": steps,
            "groups_per_rank": [int(x.item()) for x in all_g]}
