"""Group-sharded prefix-shared attention across the GPUs of one node.

Prefix groups are independent (``prefix_shared_attention`` has no cross-group term,
attention.py:156-201), so a token batch is partitioned by whole groups (greedy LPT
over per-group costs, ``psa_shard_groups``), every rank runs ONE persistent launch
over its own groups, and the only collective is the output gather
(``all_gather_into_tensor`` over NCCL, or gloo for the CPU tests), skipped when the
consumer is group-parallel too.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import packed as P


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


def _ranges(cu: np.ndarray, idx) -> np.ndarray:
    parts = [np.arange(int(cu[i]), int(cu[i + 1]), dtype=np.int64) for i in idx]
    return np.concatenate(parts) if parts else np.zeros(0, dtype=np.int64)


def shard(cu_req, cu_q, cu_prefix, cu_distinct, num_q_heads: int, num_kv_heads: int,
          head_dim: int, value_dim: int, dtype: torch.dtype, world: int) -> list[Shard]:
    """Partition a batch by groups (LPT over psa_group_costs); one Shard per rank."""
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


def gather_outputs(local: torch.Tensor, shards: list[Shard], rank: int, group=None) -> torch.Tensor:
    """All ranks' outputs [T_rank, Hq, dv] -> the full batch output [T, Hq, dv] in global
    token order, on every rank: one all_gather of equal-size (padded) slabs."""
    import torch.distributed as dist
    world = len(shards)
    tmax = max(s.num_tokens for s in shards)
    pad = torch.zeros((tmax,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[:local.shape[0]] = local
    slabs = torch.empty((world * tmax,) + tuple(local.shape[1:]), dtype=local.dtype,
                        device=local.device)
    dist.all_gather_into_tensor(slabs, pad, group=group)
    total = sum(s.num_tokens for s in shards)
    out = torch.empty((total,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    for r, s in enumerate(shards):
        if s.num_tokens:
            rows = torch.as_tensor(s.token_rows, device=local.device)
            out.index_copy_(0, rows, slabs[r * tmax:r * tmax + s.num_tokens])
    return out


def run_local(shard_: Shard, q, k_prefix, v_prefix, k_distinct, v_distinct, num_kv_heads: int,
              scale=None, options=None):
    """This rank's launch on its groups (inputs given for the FULL batch; rows selected
    here — a real engine keeps only its shard's KV resident)."""
    dev = q.device
    sel = lambda t, rows: t.index_select(0, torch.as_tensor(rows, device=dev))  # noqa: E731
    op = P.PrefixSharedAttention(shard_.cu_req, shard_.cu_q, shard_.cu_prefix, shard_.cu_distinct,
                                 q.shape[1], num_kv_heads, q.shape[2], v_prefix.shape[2],
                                 q.dtype, dev, scale, options)
    return op(sel(q, shard_.token_rows), sel(k_prefix, shard_.prefix_rows),
              sel(v_prefix, shard_.prefix_rows), sel(k_distinct, shard_.distinct_rows),
              sel(v_distinct, shard_.distinct_rows))
