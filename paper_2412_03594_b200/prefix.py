"""Native prompt grouping: the reference's
``extract_groups(maximize_reuse(build_tree(workload)))`` (prefix_tree.py:107-301)
through ``psa_prefix_groups`` in libpsa.so (csrc/psa_prefix.cpp), plus the
mapping from groups to the kernel's packed offset tables.

The output equals the reference's groups exactly (order, prefixes, members and
member order; tests/test_prefix.py), so the scheduler (``order_groups``,
scheduler.py:304-312) and everything downstream see the same plan.
"""

from __future__ import annotations

import ctypes as C
import itertools
from dataclasses import dataclass
from typing import Sequence

import numpy as np

from . import _lib as L
from .errors import ValidationError


@dataclass(frozen=True)
class Group:
    """One shared prefix (the first ``prefix_len`` tokens of every member prompt)
    and its members in the reference's order (request indices into the input)."""
    prefix_len: int
    members: tuple


def group_prompts(ids: Sequence[str], prompts: Sequence[Sequence[int]],
                  maximize: bool = True) -> tuple[list[Group], int]:
    """Group prompts by shared first-level prefix. Returns (groups, saved tokens)."""
    R = len(prompts)
    if len(ids) != R:
        raise ValidationError("ids and prompts differ in length")
    if len(set(ids)) != R:
        raise ValidationError("duplicate request ids")
    lens = np.fromiter((len(p) for p in prompts), dtype=np.int64, count=R)
    if R and lens.min() <= 0:
        raise ValidationError("prompts must be non-empty")
    cu = np.zeros(R + 1, dtype=np.int64)
    np.cumsum(lens, out=cu[1:])
    flat = np.fromiter(itertools.chain.from_iterable(prompts), dtype=np.int64, count=int(cu[-1]))
    if flat.size and (flat.min() < -2**31 or flat.max() >= 2**31):
        raise ValidationError("token ids must fit in int32")
    tok = flat.astype(np.int32)
    rank = np.empty(R, dtype=np.int32)
    rank[sorted(range(R), key=lambda i: ids[i])] = np.arange(R, dtype=np.int32)
    ng = C.c_int32()
    plen = np.zeros(max(R, 1), dtype=np.int64)
    cum = np.zeros(R + 1, dtype=np.int32)
    mem = np.zeros(max(R, 1), dtype=np.int32)
    saved = C.c_int64()
    st = L.lib().psa_prefix_groups(R, cu.ctypes.data, tok.ctypes.data if tok.size else None,
                                   rank.ctypes.data, int(bool(maximize)), C.byref(ng),
                                   plen.ctypes.data, cum.ctypes.data, mem.ctypes.data,
                                   C.byref(saved))
    if st != L.PSA_OK:
        raise ValidationError("psa_prefix_groups rejected the prompts")
    groups = [Group(int(plen[g]), tuple(int(x) for x in mem[cum[g]:cum[g + 1]]))
              for g in range(ng.value)]
    return groups, int(saved.value)


def group_workload(workload, maximize: bool = True):
    """Reference-shaped groups for a workload with ``requests`` (``id``, ``tokens``):
    a list of (prefix tuple, [(member id, suffix tuple)]) exactly as the reference's
    ``PrefixSharingGroup(prefix, members)``."""
    reqs = list(workload.requests)
    groups, _ = group_prompts([r.id for r in reqs], [r.tokens for r in reqs], maximize)
    out = []
    for g in groups:
        first = tuple(reqs[g.members[0]].tokens)
        prefix = first[:g.prefix_len]
        out.append((prefix, [(reqs[i].id, tuple(reqs[i].tokens)[g.prefix_len:])
                             for i in g.members]))
    return out


def decode_batch_offsets(groups: Sequence[Group], prompt_lens: Sequence[int],
                         decoded: Sequence[int] | int = 0) -> dict:
    """Packed offset tables of one decode step over every member (one query token per
    request; distinct KV = suffix + tokens decoded so far), groups in the given order
    (e.g. the scheduler's ``order_groups``)."""
    R = sum(len(g.members) for g in groups)
    dec = np.broadcast_to(np.asarray(decoded, dtype=np.int64), (len(prompt_lens),))
    cu_req, cu_prefix, cu_distinct = [0], [0], [0]
    for g in groups:
        cu_req.append(cu_req[-1] + len(g.members))
        cu_prefix.append(cu_prefix[-1] + g.prefix_len)
        for r in g.members:
            cu_distinct.append(cu_distinct[-1] + int(prompt_lens[r]) - g.prefix_len + int(dec[r]))
    return dict(cu_req=np.asarray(cu_req, np.int64), cu_q=np.arange(R + 1, dtype=np.int64),
                cu_prefix=np.asarray(cu_prefix, np.int64),
                cu_distinct=np.asarray(cu_distinct, np.int64))
