"""Multi-GPU host logic on CPU: world_size-2 gloo processes.

Each rank takes its groups from the LPT shard table (psa_shard_groups, C ABI, no
GPU needed), generates only those groups with the per-group counter seeds, and
the ranks check over gloo that (a) the shards are disjoint and cover every group,
(b) every rank's data for a group equals the single-process batch's data for
that group (sharding never changes inputs), (c) the oracle's per-group outputs
gathered from the ranks equal the single-process oracle output."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import segmented as S
from paper_2412_03594_b200 import packed as P
from paper_2412_03594_b200 import workloads as W


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _small_skewed():
    rng = np.random.default_rng(11)
    prefix = [int(x) for x in rng.integers(16, 200, 7)]
    reqs = [[(1, int(rng.integers(1, 40))) for _ in range(int(rng.integers(1, 5)))]
            for _ in range(7)]
    return W.Spec("mp", 4, 2, 16, 16, "f32", "normal", prefix, reqs, seed=9)


def _group_digest(b, g):
    r0, r1 = int(b["cu_req"][g]), int(b["cu_req"][g + 1])
    t0, t1 = int(b["cu_q"][r0]), int(b["cu_q"][r1])
    p0, p1 = int(b["cu_prefix"][g]), int(b["cu_prefix"][g + 1])
    d0, d1 = int(b["cu_distinct"][r0]), int(b["cu_distinct"][r1])
    parts = [b["q"][t0:t1], b["k_prefix"][p0:p1], b["v_prefix"][p0:p1],
             b["k_distinct"][d0:d1], b["v_distinct"][d0:d1]]
    return float(sum(float(x.double().sum()) + 1e-3 * float((x.double() ** 2).sum())
                     for x in parts))


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        spec = _small_skewed()
        off = W.offsets(spec)
        cost = P.group_costs(off["cu_req"], off["cu_q"], off["cu_prefix"], off["cu_distinct"],
                             spec.Hq, spec.Hkv, spec.d, spec.dv, spec.torch_dtype)
        owner = P.shard_groups(cost, world)
        mine = [g for g in range(spec.G) if owner[g] == rank]
        sub = spec.subset(mine)
        b = W.make_batch(sub, "cpu")
        digests = {sub.gid(i): _group_digest(b, i) for i in range(sub.G)}
        host = {k: b[k].double().numpy() for k in ("q", "k_prefix", "v_prefix", "k_distinct",
                                                     "v_distinct")}
        outs = {}
        for i in range(sub.G):
            res = S.packed_group_head(host["q"], host["k_prefix"], host["v_prefix"],
                                      host["k_distinct"], host["v_distinct"], b["cu_req"],
                                      b["cu_q"], b["cu_prefix"], b["cu_distinct"], i, 0,
                                      spec.Hq, spec.Hkv)
            outs[sub.gid(i)] = [r.tolist() for r in res]
        gathered = [None] * world
        dist.all_gather_object(gathered, {"mine": mine, "digests": digests, "outs": outs})
        if rank == 0:
            q.put(gathered)
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_gloo_world2_group_sharding():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    gathered = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    spec = _small_skewed()
    allg = sorted(g for part in gathered for g in part["mine"])
    assert allg == list(range(spec.G)), "shards must be disjoint and cover every group"
    full = W.make_batch(spec, "cpu")
    host = {k: full[k].double().numpy() for k in ("q", "k_prefix", "v_prefix", "k_distinct",
                                                    "v_distinct")}
    for part in gathered:
        for g, dig in part["digests"].items():
            assert dig == pytest.approx(_group_digest(full, g), rel=1e-12, abs=1e-9)
        for g, res in part["outs"].items():
            want = S.packed_group_head(host["q"], host["k_prefix"], host["v_prefix"],
                                       host["k_distinct"], host["v_distinct"], full["cu_req"],
                                       full["cu_q"], full["cu_prefix"], full["cu_distinct"], g, 0,
                                       spec.Hq, spec.Hkv)
            for a, w in zip(res, want):
                assert np.abs(np.array(a) - w).max() < 1e-12


def test_bench_rank_specs_weak_and_strong():
    import importlib.util
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    spec_ = importlib.util.spec_from_file_location("bench", os.path.join(root, "bench.py"))
    bench = importlib.util.module_from_spec(spec_)
    spec_.loader.exec_module(bench)
    # c2 weak scaling: each rank gets its own 16 groups with distinct global ids
    ids = set()
    for r in range(4):
        s, scaling = bench.rank_spec("c2", r, 4)
        assert scaling == "weak" and s.G == 16
        ids |= set(s.group_ids)
    assert len(ids) == 64
    # c5 strong scaling: LPT shards cover the 1024 groups exactly once
    seen = []
    for r in range(8):
        s, scaling = bench.rank_spec("c5", r, 8)
        assert scaling == "strong"
        seen += s.group_ids
    assert sorted(seen) == list(range(1024))


def _gather_worker(rank, world, port, q):
    """Each rank runs the float64 oracle on its shard (the kernel's stand-in on CPU) and
    the gather reassembles the full batch output in global token order."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2412_03594_b200 import distributed as D
        spec = _small_skewed()
        b = W.make_batch(spec, "cpu")
        shards = D.shard(b["cu_req"], b["cu_q"], b["cu_prefix"], b["cu_distinct"], spec.Hq,
                         spec.Hkv, spec.d, spec.dv, spec.torch_dtype, world)
        s = shards[rank]
        host = {k: b[k].double().numpy() for k in ("q", "k_prefix", "v_prefix", "k_distinct",
                                                     "v_distinct")}
        local = S.packed_attention(host["q"][s.token_rows], host["k_prefix"][s.prefix_rows],
                                   host["v_prefix"][s.prefix_rows],
                                   host["k_distinct"][s.distinct_rows],
                                   host["v_distinct"][s.distinct_rows], s.cu_req, s.cu_q,
                                   s.cu_prefix, s.cu_distinct, spec.Hq, spec.Hkv)
        full = D.gather_outputs(torch.as_tensor(local), shards, rank)
        if rank == 0:
            ref = S.packed_attention(host["q"], host["k_prefix"], host["v_prefix"],
                                     host["k_distinct"], host["v_distinct"], b["cu_req"],
                                     b["cu_q"], b["cu_prefix"], b["cu_distinct"], spec.Hq,
                                     spec.Hkv)
            q.put(float(np.abs(full.numpy() - ref).max()))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_gloo_world2_shard_run_and_output_gather():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gather_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    err = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert err == 0.0


def test_shard_edge_cases_on_host():
    """More ranks than groups (empty shards), one rank, and token/key row maps that
    tile the batch exactly once (no GPU: the planner's cost model is host code)."""
    from paper_2412_03594_b200 import distributed as D
    spec = _small_skewed()
    off = W.offsets(spec)
    for world in (1, 3, spec.G + 2):
        shards = D.shard(off["cu_req"], off["cu_q"], off["cu_prefix"], off["cu_distinct"],
                         spec.Hq, spec.Hkv, spec.d, spec.dv, spec.torch_dtype, world)
        assert len(shards) == world
        assert sorted(g for s in shards for g in s.groups.tolist()) == list(range(spec.G))
        for name, total in (("token_rows", off["cu_q"][-1]), ("prefix_rows", off["cu_prefix"][-1]),
                            ("distinct_rows", off["cu_distinct"][-1])):
            rows = np.concatenate([getattr(s, name) for s in shards])
            assert sorted(rows.tolist()) == list(range(int(total)))
        for s in shards:
            assert s.cu_q[-1] == len(s.token_rows) and s.cu_prefix[-1] == len(s.prefix_rows)
            assert s.cu_distinct[-1] == len(s.distinct_rows)
            assert len(s.cu_req) == len(s.groups) + 1
