"""Pure-Python restatement of the work-item planner in libpsa.so (psa_plan).

TEST INFRASTRUCTURE (see ``oracle/__init__.py``). The reference has no
work-item table; its only index table is the implicit stacked-row cursor of
``attention.py:174`` / ``:182-200`` (request r owns rows
[sum_{j<r} n_j, +n_r) of the group's stacked queries). The C++ planner
generalises that cursor to (group, kv head, row range, KV chunk) work items
and merge units; this module restates it line for line so that
``tests/test_plan.py`` can require byte-identical int32 tables.
"""

from __future__ import annotations

import numpy as np

ITEM_WORDS = 16
UNIT_WORDS = 8
(IT_KIND, IT_GROUP, IT_HEAD, IT_ROW0, IT_ROWS, IT_REQUEST, IT_PK0, IT_PK1, IT_DK0, IT_DK1,
 IT_UNIT0, IT_UNIT1, IT_WSROW, IT_CANON, IT_PAIR) = range(15)
(UN_GROUP, UN_HEAD, UN_ROW0, UN_ROWS, UN_CBEGIN, UN_CCOUNT) = range(6)
KIND_VEC, KIND_TILE = 0, 1
TILE_M = 128
VEC_ROWS = 8
CHUNK_ALIGN = 64
VEC_MAX_KEYS = 512
VEC_WARPS = 8
VEC_WAVES = 2
BYTE_WEIGHT = 356
VEC_FLOP_WEIGHT = 32
RIDGE = 257
DTYPE_BYTES = {0: 4, 1: 2, 2: 2, 3: 8}  # psa_dtype: F32, BF16, F16, F64


def _cdiv(a, b):
    return (a + b - 1) // b


def _rup(a, b):
    return _cdiv(a, b) * b


def tiles_supported(dtype, d, dv, Hq, Hkv, disable_tiles=0):
    if disable_tiles:
        return False
    if dtype not in (1, 2):
        return False
    if d not in (64, 128) or dv != d:
        return False
    return Hq // Hkv <= TILE_M


V2_TILE_MIN_ROWS = 16  # psa_plan_create's default tile threshold for the v2 kernel


def v2_selected(dtype, d, dv, disable_vec_fast=0, kernel_variant=0):
    """psa_plan_create's kernel choice: the v2 kernel (tile_pair, fuse_own, one CTA
    per SM) for bf16/f16 with d == dv == 128 unless a diagnostic option opts out."""
    return dtype in (1, 2) and d == 128 and dv == 128 and not disable_vec_fast \
        and not kernel_variant


def build_plan(G, R, Hq, Hkv, d, dv, dtype, cu_req, cu_q, cu_prefix, cu_distinct,
               num_sms=148, ctas_per_sm=2, tile_min_rows=32, disable_tiles=0,
               min_chunk_keys=512, max_chunk_keys=16384, target_waves=1, tile_pair=0,
               fuse_own=0):
    """Returns dict(items, units, contribs, workspace_rows, chunk_keys, num_tile_items)."""
    cu_req = [int(x) for x in cu_req]
    cu_q = [int(x) for x in cu_q]
    cu_prefix = [int(x) for x in cu_prefix]
    cu_distinct = [int(x) for x in cu_distinct]
    gqa = Hq // Hkv
    tiles = tiles_supported(dtype, d, dv, Hq, Hkv, disable_tiles)
    tile_rows = gqa * (TILE_M // gqa) if tiles else 0
    elt = DTYPE_BYTES[dtype]
    width = d + dv

    item_rows = 2 * tile_rows if tile_pair else tile_rows

    def kind_for(rows):
        return KIND_TILE if (tiles and rows >= tile_min_rows) else KIND_VEC

    def step_for(kind):
        return item_rows if kind == KIND_TILE else VEC_ROWS

    # Row segments per group (psa_plan.cpp `Segment`): (row0, rows, req, P, D).
    segs, sep = [], []
    for g in range(G):
        tok0 = cu_q[cu_req[g]]
        Ng = gqa * (cu_q[cu_req[g + 1]] - tok0)
        P = cu_prefix[g + 1] - cu_prefix[g]
        sg, sp = [], []
        if not fuse_own:
            if P > 0:
                sg.append((0, Ng, -1, P, 0))
            sp = [r for r in range(cu_req[g], cu_req[g + 1]) if cu_distinct[r + 1] > cu_distinct[r]]
        else:
            run0 = -1
            for r in range(cu_req[g], cu_req[g + 1]):
                rb = gqa * (cu_q[r] - tok0)
                nr = gqa * (cu_q[r + 1] - cu_q[r])
                D = cu_distinct[r + 1] - cu_distinct[r]
                if D > 0 and kind_for(nr) == KIND_TILE:
                    if run0 >= 0 and P > 0:
                        sg.append((run0, rb - run0, -1, P, 0))
                    run0 = -1
                    sg.append((rb, nr, r, P, D))
                else:
                    if run0 < 0:
                        run0 = rb
                    if D > 0:
                        sp.append(r)
            if run0 >= 0 and P > 0:
                sg.append((run0, Ng - run0, -1, P, 0))
        segs.append(sg)
        sep.append(sp)

    total_vec = 0
    tile_segs = []  # (row blocks x Hkv, keys)
    for g in range(G):
        for (_r0, rows, _req, P, D) in segs[g]:
            k = kind_for(rows)
            blocks = _cdiv(rows, step_for(k))
            if k == KIND_TILE:
                tile_segs.append((blocks * Hkv, P + D))
            else:
                total_vec += blocks * (P + D)
        for r in sep[g]:
            D = cu_distinct[r + 1] - cu_distinct[r]
            nr = gqa * (cu_q[r + 1] - cu_q[r])
            k = kind_for(nr)
            blocks = _cdiv(nr, step_for(k))
            if k == KIND_TILE:
                tile_segs.append((blocks * Hkv, D))
            else:
                total_vec += blocks * D
    ctas = max(1, num_sms) * max(1, ctas_per_sm)
    vec_ctas = max(1, num_sms) * 2 if tile_pair else ctas
    tile_target = ctas * max(1, target_waves)

    def tile_items(ck):
        return sum(m * _cdiv(L, ck) for m, L in tile_segs)

    lo = _rup(max(min_chunk_keys, 1), CHUNK_ALIGN)
    hi = max(lo, _rup(max(max_chunk_keys, 1), CHUNK_ALIGN))
    if tile_items(lo) > tile_target:
        while lo < hi:
            mid = _rup((lo + hi) // 2, CHUNK_ALIGN)
            if mid >= hi:
                break
            if tile_items(mid) <= tile_target:
                hi = mid
            else:
                lo = mid + CHUNK_ALIGN
        lo = lo if tile_items(lo) <= tile_target else hi
    chunk = lo
    vec_consumers = vec_ctas * VEC_WAVES if tile_pair else vec_ctas * VEC_WARPS * VEC_WAVES
    vchunk = _cdiv(total_vec * Hkv, vec_consumers)
    vchunk = _rup(min(max(vchunk, CHUNK_ALIGN), VEC_MAX_KEYS), CHUNK_ALIGN)

    def per(L, kind):
        ck = chunk if kind == KIND_TILE else vchunk
        n = _cdiv(L, ck)
        return _rup(_cdiv(L, n), CHUNK_ALIGN)

    items, units, unit_items = [], [], []
    for g in range(G):
        tok0 = cu_q[cu_req[g]]
        Ng = gqa * (cu_q[cu_req[g + 1]] - tok0)
        for h in range(Hkv):
            first = len(items)

            def push(kind, row0, rows, req, pk0, pk1, dk0, dk1):
                it = [0] * ITEM_WORDS
                it[IT_KIND], it[IT_GROUP], it[IT_HEAD] = kind, g, h
                it[IT_ROW0], it[IT_ROWS], it[IT_REQUEST] = row0, rows, req
                it[IT_PK0], it[IT_PK1], it[IT_DK0], it[IT_DK1] = pk0, pk1, dk0, dk1
                it[IT_WSROW] = -1
                it[IT_CANON] = len(items)
                items.append(it)

            for (r0, rows, req, P, D) in segs[g]:
                kind = kind_for(rows)
                L = P + D
                step, pp = step_for(kind), per(L, kind)
                for o in range(0, rows, step):
                    for k0 in range(0, L, pp):
                        k1 = min(L, k0 + pp)
                        push(kind, r0 + o, min(step, rows - o), req, min(k0, P), min(k1, P),
                             max(k0 - P, 0), max(k1 - P, 0))
            for r in sep[g]:
                D = cu_distinct[r + 1] - cu_distinct[r]
                rb = gqa * (cu_q[r] - tok0)
                nr = gqa * (cu_q[r + 1] - cu_q[r])
                kind = kind_for(nr)
                step, pp = step_for(kind), per(D, kind)
                for o in range(0, nr, step):
                    for k0 in range(0, D, pp):
                        push(kind, rb + o, min(step, nr - o), r, 0, 0, k0, min(D, k0 + pp))
            cuts = {0, Ng}
            for it in items[first:]:
                cuts.add(it[IT_ROW0])
                cuts.add(it[IT_ROW0] + it[IT_ROWS])
                if it[IT_KIND] == KIND_TILE and it[IT_ROWS] > tile_rows:
                    cuts.add(it[IT_ROW0] + tile_rows)
            for r in range(cu_req[g], cu_req[g + 1]):
                cuts.add(gqa * (cu_q[r] - tok0))
            cuts = sorted(cuts)
            ubase = len(units)
            for u in range(len(cuts) - 1):
                rec = [0] * UNIT_WORDS
                rec[UN_GROUP], rec[UN_HEAD] = g, h
                rec[UN_ROW0], rec[UN_ROWS] = cuts[u], cuts[u + 1] - cuts[u]
                units.append(rec)
                unit_items.append([])
            index = {c: i for i, c in enumerate(cuts)}
            for i in range(first, len(items)):
                it = items[i]
                u0 = index[it[IT_ROW0]]
                u1 = index[it[IT_ROW0] + it[IT_ROWS]]
                it[IT_UNIT0], it[IT_UNIT1] = ubase + u0, ubase + u1
                for u in range(u0, u1):
                    unit_items[ubase + u].append(i)
            for u in range(ubase, len(units)):
                if not unit_items[u]:
                    raise AssertionError("merge unit without contributions")

    ws = 0
    for it in items:
        direct = all(len(unit_items[u]) == 1 for u in range(it[IT_UNIT0], it[IT_UNIT1]))
        if not direct:
            it[IT_WSROW] = ws
            ws += it[IT_ROWS]
    contribs = []
    for u, rec in enumerate(units):
        rec[UN_CBEGIN] = len(contribs)
        rec[UN_CCOUNT] = len(unit_items[u])
        for i in unit_items[u]:
            it = items[i]
            contribs.append(-1 if it[IT_WSROW] < 0 else it[IT_WSROW] + (rec[UN_ROW0] - it[IT_ROW0]))

    # pair merges (psa_plan.cpp, before step 4): one of exactly two contributors of one
    # unit spanning the item's rows -> other contribution's ws row * 2 + (it comes first)
    for it in items:
        pair = -1
        if it[IT_WSROW] >= 0 and it[IT_UNIT1] - it[IT_UNIT0] == 1:
            u = units[it[IT_UNIT0]]
            if u[UN_ROW0] == it[IT_ROW0] and u[UN_ROWS] == it[IT_ROWS] and u[UN_CCOUNT] == 2:
                c0, c1 = contribs[u[UN_CBEGIN]], contribs[u[UN_CBEGIN] + 1]
                first = c0 != it[IT_WSROW]
                pair = (c0 if first else c1) * 2 + (1 if first else 0)
                if pair > 2**31 - 1:
                    pair = -1
        it[IT_PAIR] = pair
    cost = []
    for it in items:
        keys = (it[IT_PK1] - it[IT_PK0]) + (it[IT_DK1] - it[IT_DK0])
        nbytes = (keys + it[IT_ROWS]) * width * elt
        if it[IT_KIND] == KIND_TILE:
            slots = _cdiv(it[IT_ROWS], max(tile_rows, 1))
            cost.append(max(nbytes * BYTE_WEIGHT, 2 * TILE_M * slots * keys * width))
        else:
            cost.append(max(nbytes * BYTE_WEIGHT,
                            2 * _rup(it[IT_ROWS], 4) * keys * width * VEC_FLOP_WEIGHT))
    # TILE items first (CTA-level queue), then VEC items. TILE items by (group, kv head)
    # bundle: bundle cost descending, then bundle, then item cost descending; VEC items
    # by cost descending, equal-cost VEC items with the kv heads of one (request, key
    # chunk) side by side (psa_plan.cpp build_plan step 4).
    bundle = {}
    for i, it in enumerate(items):
        if it[IT_KIND] == KIND_TILE:
            k = it[IT_GROUP] * Hkv + it[IT_HEAD]
            bundle[k] = bundle.get(k, 0) + cost[i]

    def _key(i):
        it = items[i]
        if it[IT_KIND] == KIND_TILE:
            k = it[IT_GROUP] * Hkv + it[IT_HEAD]
            return (False, -bundle[k], (k, -cost[i]))
        return (True, -cost[i], (it[IT_GROUP], it[IT_REQUEST], it[IT_ROW0], it[IT_PK0],
                                 it[IT_DK0], it[IT_HEAD]))
    order = sorted(range(len(items)), key=_key)
    return dict(
        items=np.array([items[i] for i in order], dtype=np.int32).reshape(-1, ITEM_WORDS),
        units=np.array(units, dtype=np.int32).reshape(-1, UNIT_WORDS),
        contribs=np.array(contribs, dtype=np.int32),
        workspace_rows=ws, chunk_keys=chunk,
        num_tile_items=sum(1 for it in items if it[IT_KIND] == KIND_TILE))


def group_costs(G, Hq, Hkv, d, dv, dtype, cu_req, cu_q, cu_prefix, cu_distinct):
    elt = DTYPE_BYTES[dtype]
    width = d + dv
    out = []
    for g in range(G):
        P = int(cu_prefix[g + 1] - cu_prefix[g])
        keys, tokens, pairs = P, 0, 0
        for r in range(int(cu_req[g]), int(cu_req[g + 1])):
            n = int(cu_q[r + 1] - cu_q[r])
            D = int(cu_distinct[r + 1] - cu_distinct[r])
            keys += D
            tokens += n
            pairs += n * (P + D)
        nbytes = Hkv * keys * width * elt + tokens * Hq * width * elt
        flops = 2 * Hq * pairs * width
        out.append(max(nbytes * RIDGE, flops))
    return np.array(out, dtype=np.int64)


def shard_groups(cost, world):
    """Greedy LPT: largest cost first, to the least-loaded rank (lowest rank on ties)."""
    order = sorted(range(len(cost)), key=lambda g: -int(cost[g]))
    load = [0] * world
    owner = np.zeros(len(cost), dtype=np.int32)
    for g in order:
        best = min(range(world), key=lambda w: (load[w], w))
        owner[g] = best
        load[best] += int(cost[g])
    return owner
