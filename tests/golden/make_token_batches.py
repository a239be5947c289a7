"""Record token batches of the REFERENCE scheduler and their paged kernel metadata.

Run in the build container (where ``/root/reference`` exists):

    python tests/golden/make_token_batches.py [--ref /root/reference/pkg/src]

Runs the reference's BatchLLM scheduler (``prefixbatch.scheduler.simulate``,
policy ``batchllm``, block_size 16) on a small grouped workload with
``form_token_batch`` hooked: every formed ``TokenBatch`` goes through
``paper_2412_03594_b200.batching.prepare`` (which performs ``step``'s block
grows in ``step``'s order) before the reference's ``step`` applies it. The
script checks that the hooked simulation reproduces the unhooked trace exactly
(per-iteration token counts and blocks in use, i.e. ``prepare`` allocates
exactly the blocks ``step`` would), then stores the per-iteration tables in
``token_batches.npz``
(consumed by tests/test_gpu_batching.py on the GPU box, where the reference
does not exist).
"""

from __future__ import annotations

import argparse
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from paper_2412_03594_b200 import batching as B  # noqa: E402

KEYS = ("cu_req", "cu_q", "cu_prefix", "cu_distinct", "prefix_pages", "distinct_pages",
        "token_entry", "token_offset", "request_entry")


def workload(ref):
    from prefixbatch.prefix_tree import GroupMember, PrefixSharingGroup

    def group(gid, prefix_len, suffix_lens, base):
        prefix = tuple(range(base, base + prefix_len))
        members = tuple(GroupMember(f"{gid}m{i}", tuple(range(base + 10_000 * (i + 1),
                                                               base + 10_000 * (i + 1) + n)))
                        for i, n in enumerate(suffix_lens))
        return PrefixSharingGroup(prefix, members)

    groups = [group("a", 100, [5, 0, 40, 3], 1000), group("b", 37, [3, 17], 2000),
              group("c", 0, [20, 9], 3000), group("d", 150, [1, 1, 1, 2, 70], 4000)]
    out = {}
    for gi, g in enumerate(groups):
        for mi, m in enumerate(g.members):
            out[m.id] = 2 + (gi + 3 * mi) % 5
    return groups, out


def simulate(ref, hook: bool):
    from prefixbatch import scheduler as S
    groups, output_lens = workload(ref)
    config = S.SchedulerConfig(policy="batchllm", chunk_size=64, block_size=16,
                               total_blocks=256)
    records = []
    orig = S.form_token_batch

    def hooked(state, cfg):
        batch = orig(state, cfg)
        kb = B.prepare(state, batch)
        records.append((batch, kb, state))
        return batch

    if hook:
        S.form_token_batch = hooked
    try:
        trace = S.simulate(groups, config, output_lens)
    finally:
        S.form_token_batch = orig
    return trace, records


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default="/root/reference/pkg/src")
    args = ap.parse_args()
    sys.path.insert(0, args.ref)
    plain, _ = simulate(args.ref, hook=False)
    hooked, records = simulate(args.ref, hook=True)
    assert [r.__dict__ for r in plain.rows] == [r.__dict__ for r in hooked.rows], \
        "prepare() changed the reference schedule"
    kinds = {"decode": 0, "distinct_chunk": 1, "prefix_chunk": 2}
    out = {"num_batches": np.array(len(records))}
    for i, (batch, kb, _state) in enumerate(records):
        for k in KEYS:
            out[f"b{i}_{k}"] = getattr(kb, k)
        out[f"b{i}_entry_kind"] = np.array([kinds[e.kind] for e in batch.entries], np.int32)
        out[f"b{i}_entry_tokens"] = np.array([e.tokens for e in batch.entries], np.int64)
    out["block_size"] = np.array(16)
    out["total_blocks"] = np.array(256)
    path = os.path.join(HERE, "token_batches.npz")
    np.savez_compressed(path, **out)
    n_kinds = np.bincount(np.concatenate([out[f"b{i}_entry_kind"] for i in range(len(records))]),
                          minlength=3)
    print(f"{len(records)} token batches ({n_kinds[0]} decode, {n_kinds[1]} distinct-chunk, "
          f"{n_kinds[2]} prefix-chunk entries) -> {path}")


if __name__ == "__main__":
    main()
