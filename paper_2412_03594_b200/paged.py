"""Paged KV helpers: page tables for the paged kernel mode (include/psa.h).

The reference engine stores KV in fixed-size blocks owned per request / per
group prefix (``KVAllocator``, scheduler.py:140-187; block size 16 at
scheduler.py:45). The kernel addresses such a cache through two flattened
int32 page tables: every group's prefix pages in group order, and every
request's distinct pages in request order (``ceil(len / page_size)`` pages each).
These helpers build those tables and move packed segments into a page cache
(used by the token-batch adapter and the tests; the kernel itself never copies).
"""

from __future__ import annotations

from typing import Sequence

import numpy as np
import torch


def pages_needed(lengths: Sequence[int], page_size: int) -> np.ndarray:
    """Pages per segment, ceil(length / page_size)."""
    lengths = np.asarray(lengths, dtype=np.int64)
    return (lengths + page_size - 1) // page_size


def physical_rows(lengths: Sequence[int], pages: np.ndarray, page_size: int) -> np.ndarray:
    """Cache row of every logical key, segments concatenated in order (the packed row
    order): key j of segment s sits at pages[base(s) + j // page_size] * page_size +
    j % page_size."""
    lengths = np.asarray(lengths, dtype=np.int64)
    npg = pages_needed(lengths, page_size)
    base = np.concatenate([[0], np.cumsum(npg)[:-1]]).astype(np.int64)
    seg = np.repeat(np.arange(len(lengths)), lengths)
    start = np.concatenate([[0], np.cumsum(lengths)[:-1]]).astype(np.int64)
    j = np.arange(int(lengths.sum()), dtype=np.int64) - start[seg]
    return np.asarray(pages, dtype=np.int64)[base[seg] + j // page_size] * page_size + j % page_size


def scatter_to_cache(packed: torch.Tensor, lengths: Sequence[int], pages: np.ndarray,
                     page_size: int, cache: torch.Tensor) -> None:
    """Write packed segment rows [sum(lengths), H, d] into their cache pages."""
    if packed.shape[0] == 0:
        return
    rows = torch.as_tensor(physical_rows(lengths, pages, page_size), device=cache.device)
    cache.index_copy_(0, rows, packed)


def random_page_tables(lengths: Sequence[int], page_size: int, num_pages: int,
                       rng: np.random.Generator) -> np.ndarray:
    """Distinct random physical pages for every segment page (test/bench helper)."""
    need = int(pages_needed(lengths, page_size).sum())
    if need > num_pages:
        raise ValueError("page cache too small")
    return rng.permutation(num_pages)[:need].astype(np.int32)
