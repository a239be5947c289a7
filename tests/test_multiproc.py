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


def test_bench_rank_groups_strong_sharding():
    import importlib.util
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    spec_ = importlib.util.spec_from_file_location("bench", os.path.join(root, "bench.py"))
    bench = importlib.util.module_from_spec(spec_)
    spec_.loader.exec_module(bench)
    assert bench.DEFAULT_CONFIG == "c5"
    # every config is strong-scaled: LPT shards cover the groups exactly once
    for name, world in (("c5", 8), ("c4", 4), ("c2", 2)):
        full = W.config(name)
        seen = []
        for r in range(world):
            seen += bench.rank_groups(full, r, world)
        assert sorted(seen) == list(range(full.G))
    # the config dict is the workload identity, identical for both arms
    c = bench.config_dict(W.config("c5"), 1)
    assert c["workload"] == "c5" and c["groups"] == 1024 and c["tokens"] == 65536


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
        if s.num_groups:
            local = S.packed_attention(host["q"][s.token_rows], host["k_prefix"][s.prefix_rows],
                                       host["v_prefix"][s.prefix_rows],
                                       host["k_distinct"][s.distinct_rows],
                                       host["v_distinct"][s.distinct_rows], s.cu_req, s.cu_q,
                                       s.cu_prefix, s.cu_distinct, spec.Hq, spec.Hkv)
        else:  # more ranks than groups: the empty shard still joins the gather
            local = np.zeros((0, spec.Hq, spec.dv))
        full = D.gather_outputs(torch.as_tensor(local), shards, rank)
        if rank == 0:
            ref = S.packed_attention(host["q"], host["k_prefix"], host["v_prefix"],
                                     host["k_distinct"], host["v_distinct"], b["cu_req"],
                                     b["cu_q"], b["cu_prefix"], b["cu_distinct"], spec.Hq,
                                     spec.Hkv)
            q.put(float(np.abs(full.numpy() - ref).max()))
    finally:
        dist.destroy_process_group()


def _spawn(target, world, *extra):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=target, args=(r, world, port, q) + extra) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


@pytest.mark.timeout(300)
def test_gloo_world2_shard_run_and_output_gather():
    assert _spawn(_gather_worker, 2) == 0.0


@pytest.mark.timeout(300)
def test_gloo_more_ranks_than_groups_gather():
    """world > G: empty shards still join the collective (no hang), output exact."""
    assert _spawn(_gather_worker, _small_skewed().G + 1) == 0.0


def _slab_worker(rank, world, port, q, num_slabs):
    """SlabGather: per-slab compute (oracle stand-in) + per-slab all_gather, then the
    reassembled output equals the single-process oracle."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2412_03594_b200 import distributed as D
        spec = _small_skewed()
        off = W.offsets(spec)
        shards = D.shard(off["cu_req"], off["cu_q"], off["cu_prefix"], off["cu_distinct"],
                         spec.Hq, spec.Hkv, spec.d, spec.dv, spec.torch_dtype, world)
        me = shards[rank]
        sub = spec.subset(me.groups.tolist())
        b = W.make_batch(sub, "cpu")   # only this rank's groups (per-group seeds)
        host = {k: b[k].double().numpy() for k in ("q", "k_prefix", "v_prefix", "k_distinct",
                                                     "v_distinct")}
        sg = D.SlabGather(shards, rank, num_slabs, (spec.Hq, spec.dv), torch.float64, "cpu")
        calls = []

        def compute(i, out_rows):
            g0, g1 = sg.slab_groups(i)
            calls.append((g0, g1))
            res = S.packed_attention(host["q"], host["k_prefix"], host["v_prefix"],
                                     host["k_distinct"], host["v_distinct"], b["cu_req"],
                                     b["cu_q"], b["cu_prefix"], b["cu_distinct"], spec.Hq,
                                     spec.Hkv, groups=range(g0, g1))
            t0, t1 = int(b["cu_q"][b["cu_req"][g0]]), int(b["cu_q"][b["cu_req"][g1]])
            out_rows.copy_(torch.as_tensor(res[t0:t1]))

        sg.run(compute)
        full = sg.result()
        assert sum(g1 - g0 for g0, g1 in calls) == me.num_groups
        if rank == 0:
            fb = W.make_batch(spec, "cpu")
            fh = {k: fb[k].double().numpy() for k in ("q", "k_prefix", "v_prefix", "k_distinct",
                                                        "v_distinct")}
            ref = S.packed_attention(fh["q"], fh["k_prefix"], fh["v_prefix"], fh["k_distinct"],
                                     fh["v_distinct"], fb["cu_req"], fb["cu_q"], fb["cu_prefix"],
                                     fb["cu_distinct"], spec.Hq, spec.Hkv)
            q.put(float(np.abs(full.numpy() - ref).max()))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
@pytest.mark.parametrize("world,num_slabs", [(2, 3), (3, 2)])
def test_gloo_slab_gather_overlapped_output(world, num_slabs):
    assert _spawn(_slab_worker, world, num_slabs) < 1e-12


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
