"""The C++ planner in libpsa.so (psa_plan) against its Python restatement
(oracle/plan.py): the int32 work-item / merge-unit / contribution tables and
the group->rank shard table must be byte-identical. CPU only (num_sms given,
so the library makes no CUDA call)."""

import json
import os

import numpy as np
import pytest
import torch

import cases as C
from oracle import plan as OP
from paper_2412_03594_b200 import packed as P
from paper_2412_03594_b200 import workloads as W
from paper_2412_03594_b200.errors import ValidationError

DT = {"f32": (torch.float32, 0), "bf16": (torch.bfloat16, 1), "f16": (torch.float16, 2),
      "f64": (torch.float64, 3)}
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _compare(off, Hq, Hkv, d, dv, dt, **opt):
    tdt, pdt = DT[dt]
    opts = P.PlanOptions(**{"num_sms": 148, **opt})
    got = P.plan_tables_host(off["cu_req"], off["cu_q"], off["cu_prefix"], off["cu_distinct"],
                             Hq, Hkv, d, dv, tdt, opts)
    v2 = OP.v2_selected(pdt, d, dv, opts.disable_vec_fast, opts.kernel_variant)
    want = OP.build_plan(len(off["cu_req"]) - 1, len(off["cu_q"]) - 1, Hq, Hkv, d, dv, pdt,
                         off["cu_req"], off["cu_q"], off["cu_prefix"], off["cu_distinct"],
                         num_sms=opts.num_sms, ctas_per_sm=1 if v2 else (opts.ctas_per_sm or 2),
                         tile_pair=int(v2), fuse_own=int(v2),
                         tile_min_rows=opts.tile_min_rows or (OP.V2_TILE_MIN_ROWS if v2 else 32),
                         disable_tiles=opts.disable_tiles,
                         min_chunk_keys=opts.min_chunk_keys or 512,
                         max_chunk_keys=opts.max_chunk_keys or 16384,
                         target_waves=opts.target_waves or 1)
    assert got["items"].tobytes() == want["items"].tobytes()
    assert got["units"].tobytes() == want["units"].tobytes()
    assert got["contribs"].tobytes() == want["contribs"].tobytes()
    assert got["workspace_rows"] == want["workspace_rows"]
    assert got["num_tile_items"] == want["num_tile_items"]
    return got


def _manifest():
    with open(os.path.join(GOLDEN, "manifest.json")) as f:
        return [e["spec"] for e in json.load(f)["cases"]]


@pytest.mark.parametrize("spec", _manifest(), ids=lambda s: s["name"])
@pytest.mark.parametrize("opt", [{}, {"disable_tiles": 1}, {"num_sms": 4, "min_chunk_keys": 64},
                                 {"kernel_variant": 1}])
def test_plan_bit_exact_golden_cases(spec, opt):
    a = C.make_packed(spec)
    _compare(a, spec["Hq"], spec["Hkv"], spec["d"], spec["dv"], spec["dtype"], **opt)


@pytest.mark.parametrize("variant", [0, 1])
@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4", "c5"])
def test_plan_bit_exact_bench_configs(name, variant):
    s = W.config(name)
    got = _compare(W.offsets(s), s.Hq, s.Hkv, s.d, s.dv, s.dtype, kernel_variant=variant)
    assert got["items"].shape[0] > 0


def test_plan_bit_exact_random_property():
    rng = np.random.default_rng(1234)
    for _ in range(60):
        G = int(rng.integers(1, 5))
        Hkv = int(rng.choice([1, 2, 4]))
        gqa = int(rng.choice([1, 2, 3, 4, 8]))
        groups = []
        for _g in range(G):
            Pn = int(rng.choice([0, int(rng.integers(1, 3000))]))
            reqs = []
            for _r in range(int(rng.integers(1, 12))):
                n = int(rng.choice([1, 1, 1, int(rng.integers(1, 300))]))
                D = int(rng.integers(0 if Pn else 1, 900))
                reqs.append((n, D))
            groups.append((Pn, reqs))
        flat = [r for _, rs in groups for r in rs]
        off = dict(cu_req=np.cumsum([0] + [len(rs) for _, rs in groups]),
                   cu_q=np.cumsum([0] + [n for n, _ in flat]),
                   cu_prefix=np.cumsum([0] + [p for p, _ in groups]),
                   cu_distinct=np.cumsum([0] + [D for _, D in flat]))
        dt = str(rng.choice(["bf16", "f16", "f32"]))
        d = int(rng.choice([64, 128]))
        _compare(off, gqa * Hkv, Hkv, d, d, dt, num_sms=int(rng.choice([8, 148])),
                 min_chunk_keys=int(rng.choice([64, 256])),
                 kernel_variant=int(rng.choice([0, 1])))


def test_plan_invariants_c3():
    """Every stacked row of every (group, kv head) is covered by exactly one merge
    unit; each unit's contributions cover all its KV exactly once."""
    s = W.config("c3")
    off = W.offsets(s)
    t = P.plan_tables_host(off["cu_req"], off["cu_q"], off["cu_prefix"], off["cu_distinct"],
                           s.Hq, s.Hkv, s.d, s.dv, torch.bfloat16, P.PlanOptions(num_sms=148))
    items, units = t["items"], t["units"]
    gqa = s.Hq // s.Hkv
    for g in (0, 17, 63):
        for h in (0, 7):
            us = units[(units[:, OP.UN_GROUP] == g) & (units[:, OP.UN_HEAD] == h)]
            rows = us[:, OP.UN_ROWS].sum()
            assert rows == gqa * (off["cu_q"][off["cu_req"][g + 1]] - off["cu_q"][off["cu_req"][g]])
    # each unit: sum of covering items' keys == prefix + the request's distinct length
    idx_of_unit = {}
    for it in items:
        for u in range(it[OP.IT_UNIT0], it[OP.IT_UNIT1]):
            idx_of_unit.setdefault(u, []).append(it)
    for u in range(0, len(units), 97):
        its = idx_of_unit[u]
        keys = sum((it[OP.IT_PK1] - it[OP.IT_PK0]) + (it[OP.IT_DK1] - it[OP.IT_DK0]) for it in its)
        assert len(its) == units[u, OP.UN_CCOUNT]
        g = units[u, OP.UN_GROUP]
        reqs = {it[OP.IT_REQUEST] for it in its if it[OP.IT_REQUEST] >= 0}
        assert len(reqs) <= 1
        D = sum(off["cu_distinct"][r + 1] - off["cu_distinct"][r] for r in reqs)
        assert keys == off["cu_prefix"][g + 1] - off["cu_prefix"][g] + D
    assert t["num_tile_items"] > 0


@pytest.mark.parametrize("bad, msg", [
    (dict(cu_q=[0, 1, 1]), "positive dimensions"),
    (dict(cu_prefix=[0, 0, 0], cu_distinct=[0, 5, 5]), "neither prefix nor distinct"),
    (dict(cu_req=[0, 2, 2]), "has no requests"),
    (dict(cu_req=[0, 1, 3]), "end at num_requests"),
])
def test_plan_rejects_invalid_offsets(bad, msg):
    off = dict(cu_req=[0, 1, 2], cu_q=[0, 1, 2], cu_prefix=[0, 4, 8], cu_distinct=[0, 5, 5])
    off.update(bad)
    with pytest.raises(ValidationError, match=msg):
        P.plan_tables_host(off["cu_req"], off["cu_q"], off["cu_prefix"], off["cu_distinct"],
                           2, 1, 64, 64, torch.bfloat16, P.PlanOptions(num_sms=148))


def test_shard_groups_bit_exact():
    rng = np.random.default_rng(7)
    for world in (1, 2, 4, 8):
        cost = rng.integers(1, 10**12, size=int(rng.integers(1, 300)))
        assert (P.shard_groups(cost, world) == OP.shard_groups(cost, world)).all()
    for name in ("c4", "c5"):
        s = W.config(name)
        off = W.offsets(s)
        got = P.group_costs(off["cu_req"], off["cu_q"], off["cu_prefix"], off["cu_distinct"],
                            s.Hq, s.Hkv, s.d, s.dv, s.torch_dtype)
        want = OP.group_costs(s.G, s.Hq, s.Hkv, s.d, s.dv, 1, off["cu_req"], off["cu_q"],
                              off["cu_prefix"], off["cu_distinct"])
        assert (got == want).all()
        for world in (2, 4, 8):
            owner = P.shard_groups(got, world)
            assert (owner == OP.shard_groups(want, world)).all()
            loads = np.bincount(owner, weights=got.astype(np.float64), minlength=world)
            assert loads.max() <= loads.min() + got.max()  # LPT bound
