"""Token batch -> kernel metadata.

Turns one memory-centric token batch of the reference's scheduler
(``TokenBatch`` entries ``decode`` / ``distinct_chunk`` / ``prefix_chunk``,
scheduler.py:246-268, formed by ``form_token_batch`` :425-536) plus the block
lists of its ``KVAllocator`` (scheduler.py:140-187) into the offset tables and
page tables of ONE paged kernel launch (include/psa.h, ``page_size`` =
the scheduler's ``block_size``, scheduler.py:45).

Mapping (the caller-side mapping of SURVEY.md §8(a), applied by ``step``,
scheduler.py:634-696):

* ``decode`` (1 token) of request r: one query token; prefix = r's group prefix
  (complete: members decode only after the group prefix is done); distinct KV =
  suffix + decoded tokens including this one (``grow`` at :671).
* ``distinct_chunk`` (k tokens) of r: k query tokens; distinct KV = the suffix
  processed so far including the chunk (:663-664); fully visible (no mask, as
  the reference, attention.py:12-13).
* ``prefix_chunk`` (k tokens) of group g (owner ``prefix#g``): k query tokens
  against the prefix KV up to ``prefix_done`` after this chunk (:650-651), no
  distinct KV.

Kernel groups are (prefix owner, prefix length) pairs: decode and distinct
entries of one group share one kernel group (the shared-prefix tiles), each
prefix chunk is a group of its own, requests without a group prefix share the
empty-prefix group. Block ids come from the allocator *after* this batch's
``grow`` calls, which :func:`prepare` performs in ``step``'s entry order (so the
later ``step`` finds them done and assigns nothing new).

Works on duck-typed state: anything with ``requests[rid]`` (``group``,
``suffix_done``, ``decode_done``), ``groups[gi]`` (``owner``, ``prefix_len``,
``prefix_done``), ``allocator`` (``grow``, ``blocks_of``) and ``config.block_size``.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

PREFIX_CHUNK = "prefix_chunk"
DISTINCT_CHUNK = "distinct_chunk"
DECODE = "decode"


def _blocks_for(tokens: int, bs: int) -> int:
    return -(-tokens // bs)


@dataclass
class KernelBatch:
    page_size: int
    cu_req: np.ndarray
    cu_q: np.ndarray
    cu_prefix: np.ndarray
    cu_distinct: np.ndarray
    prefix_pages: np.ndarray     # int32, every kernel group's prefix pages in group order
    distinct_pages: np.ndarray   # int32, every kernel request's distinct pages
    # kernel token t <- (batch entry index, token offset within the entry)
    token_entry: np.ndarray
    token_offset: np.ndarray
    # per kernel request: the batch entry it came from
    request_entry: np.ndarray
    group_keys: list = field(default_factory=list)  # (prefix owner | None, prefix length)

    @property
    def num_tokens(self) -> int:
        return int(self.cu_q[-1])


def prepare(state, batch) -> KernelBatch:
    """Allocate this batch's KV blocks (``step``'s grows, in ``step``'s order) and
    build the paged kernel metadata. Call after ``form_token_batch`` and before
    ``step``."""
    bs = int(state.config.block_size)
    alloc = state.allocator
    policy = getattr(state.config, "policy", "batchllm")
    if policy != "batchllm":
        # fcfs-cap(-lru) states skip cache-hit prompt tokens (reused_tokens) whose KV
        # lives in another owner's blocks: D below would silently leave them out.
        raise ValueError(f"prepare() maps batchllm scheduler states only (got {policy!r})")
    # 1. post-step lengths + the grows step() will perform, in entry order
    groups = {}   # key -> dict(owner, P, reqs=[])
    order = []
    prefix_done = {}
    for ei, e in enumerate(batch.entries):
        if e.kind == PREFIX_CHUNK:
            gi = int(e.owner.split("#", 1)[1])
            g = state.groups[gi]
            done = prefix_done.get(gi, g.prefix_done) + e.tokens
            prefix_done[gi] = done
            alloc.grow(g.owner, _blocks_for(done, bs))
            key = (g.owner, done, ei)  # a chunk is a kernel group of its own
            groups[key] = dict(owner=g.owner, P=done, reqs=[(ei, e.tokens, None, 0)])
            order.append(key)
            continue
        r = state.requests[e.owner]
        if getattr(r, "reused_tokens", 0):
            raise ValueError(f"request {r.id} has {r.reused_tokens} reused (cache-hit) tokens; "
                             "their KV is not in its own blocks")
        if e.kind == DISTINCT_CHUNK:
            D = r.suffix_done + e.tokens
        elif e.kind == DECODE:
            D = r.suffix_done + r.decode_done + 1
        else:
            raise ValueError(f"unknown batch entry kind {e.kind!r}")
        alloc.grow(r.id, _blocks_for(D, bs))
        if r.group is not None:
            g = state.groups[r.group]
            key = (g.owner, g.prefix_len)
            owner, P = g.owner, g.prefix_len
        else:
            key, owner, P = (None, 0), None, 0
        if key not in groups:
            groups[key] = dict(owner=owner, P=P, reqs=[])
            order.append(key)
        groups[key]["reqs"].append((ei, e.tokens, r.id, D))
    # 2. tables in kernel order
    cu_req, cu_q, cu_prefix, cu_distinct = [0], [0], [0], [0]
    ppages, dpages, tok_e, tok_o, req_e = [], [], [], [], []
    for key in order:
        grp = groups[key]
        P = grp["P"]
        if P:
            blocks = alloc.blocks_of(grp["owner"])
            need = _blocks_for(P, bs)
            if len(blocks) < need:  # a short list would shift every later page-table base
                raise ValueError(f"{grp['owner']} holds {len(blocks)} blocks, {need} needed")
            ppages.extend(blocks[:need])
        cu_prefix.append(cu_prefix[-1] + P)
        for ei, n, rid, D in grp["reqs"]:
            cu_q.append(cu_q[-1] + n)
            cu_distinct.append(cu_distinct[-1] + D)
            if D:
                blocks = alloc.blocks_of(rid)
                need = _blocks_for(D, bs)
                if len(blocks) < need:
                    raise ValueError(f"request {rid} holds {len(blocks)} blocks, {need} needed")
                dpages.extend(blocks[:need])
            tok_e.extend([ei] * n)
            tok_o.extend(range(n))
            req_e.append(ei)
        cu_req.append(cu_req[-1] + len(grp["reqs"]))
    i64 = lambda x: np.asarray(x, dtype=np.int64)  # noqa: E731
    return KernelBatch(bs, i64(cu_req), i64(cu_q), i64(cu_prefix), i64(cu_distinct),
                       np.asarray(ppages, dtype=np.int32), np.asarray(dpages, dtype=np.int32),
                       i64(tok_e), i64(tok_o), i64(req_e), [k[:2] for k in order])


def entry_token_rows(kb: KernelBatch, batch) -> np.ndarray:
    """Kernel token index of every batch token, entries in batch order (to scatter
    the kernel output back into the engine's token order)."""
    starts = np.concatenate([[0], np.cumsum([e.tokens for e in batch.entries])]).astype(np.int64)
    rows = np.empty(int(starts[-1]), dtype=np.int64)
    rows[starts[kb.token_entry] + kb.token_offset] = np.arange(kb.num_tokens)
    return rows


def run(kb: KernelBatch, q, k_cache, v_cache, num_kv_heads: int, scale=None, options=None,
        causal: bool = False):
    """One paged launch for the batch: q [T, Hq, d] in kernel token order; the
    allocator's block pool as the page cache [num_blocks * block_size, Hkv, d]."""
    import torch

    from . import packed as P
    op = P.PrefixSharedAttention(kb.cu_req, kb.cu_q, kb.cu_prefix, kb.cu_distinct, q.shape[1],
                                 num_kv_heads, q.shape[2], v_cache.shape[2], q.dtype, q.device,
                                 scale, options, page_size=kb.page_size)
    dev = q.device
    pp = torch.as_tensor(kb.prefix_pages, device=dev)
    dp = torch.as_tensor(kb.distinct_pages, device=dev)
    return op(q, k_cache, v_cache, k_cache, v_cache, prefix_pages=pp, distinct_pages=dp,
              causal=causal)
