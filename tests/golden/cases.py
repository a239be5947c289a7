"""Deterministic input generators for the golden parity cases (pure NumPy).

The golden fixtures (``tests/golden/*.npz`` + ``manifest.json``) store, per
case, the SHA-256 of the generated inputs and the reference's float64 outputs;
inputs are regenerated here from the seed so the fixtures stay small. The
manifest's SHA check fails loudly if this generator ever drifts.

Packed layout: q [T, Hq, d]; kp/vp [sum P_g, Hkv, d|dv];
kd/vd [sum D_r, Hkv, d|dv]; cu_req [G+1], cu_q [R+1], cu_prefix [G+1],
cu_distinct [R+1] (int64).
"""

from __future__ import annotations

import hashlib

import numpy as np


def round_to_bf16(x: np.ndarray) -> np.ndarray:
    """Round float32 to the nearest bf16 value (ties to even), kept as float32."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)


def _draw(rng, shape, dist: str, dtype: str) -> np.ndarray:
    if dist == "normal":
        x = rng.standard_normal(shape)
    elif dist == "uniform10":
        x = rng.uniform(-10.0, 10.0, shape)
    else:
        raise ValueError(dist)
    if dtype == "bf16":
        return round_to_bf16(x.astype(np.float32))
    if dtype == "f16":
        return x.astype(np.float16).astype(np.float32)
    if dtype == "f32":
        return x.astype(np.float32)
    return x.astype(np.float64)


def make_packed(spec: dict) -> dict:
    """Build a packed multi-group, multi-head problem from a case spec.

    spec keys: seed, Hq, Hkv, d, dv, dist, dtype, groups=[{"P": int,
    "reqs": [[n_q, D], ...]}, ...].
    """
    rng = np.random.default_rng(spec["seed"])
    Hq, Hkv, d, dv = spec["Hq"], spec["Hkv"], spec["d"], spec["dv"]
    groups = spec["groups"]
    P = [g["P"] for g in groups]
    reqs = [tuple(r) for g in groups for r in g["reqs"]]
    cu_req = np.cumsum([0] + [len(g["reqs"]) for g in groups]).astype(np.int64)
    cu_q = np.cumsum([0] + [r[0] for r in reqs]).astype(np.int64)
    cu_prefix = np.cumsum([0] + P).astype(np.int64)
    cu_distinct = np.cumsum([0] + [r[1] for r in reqs]).astype(np.int64)
    dist, dt = spec["dist"], spec["dtype"]
    q = _draw(rng, (int(cu_q[-1]), Hq, d), dist, dt)
    kp = _draw(rng, (int(cu_prefix[-1]), Hkv, d), dist, dt)
    vp = _draw(rng, (int(cu_prefix[-1]), Hkv, dv), dist, dt)
    kd = _draw(rng, (int(cu_distinct[-1]), Hkv, d), dist, dt)
    vd = _draw(rng, (int(cu_distinct[-1]), Hkv, dv), dist, dt)
    return dict(q=q, kp=kp, vp=vp, kd=kd, vd=vd, cu_req=cu_req, cu_q=cu_q,
                cu_prefix=cu_prefix, cu_distinct=cu_distinct)


def inputs_sha(arrays: dict) -> str:
    h = hashlib.sha256()
    for key in ("q", "kp", "vp", "kd", "vd", "cu_req", "cu_q", "cu_prefix", "cu_distinct"):
        a = np.ascontiguousarray(arrays[key])
        h.update(key.encode())
        h.update(str(a.dtype).encode())
        h.update(str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def _g(P, reqs):
    return {"P": P, "reqs": [list(r) for r in reqs]}


def packed_cases() -> list:
    """The packed golden cases (GPU parity tests run every one of them)."""
    rs = np.random.default_rng(20241203)
    cases = []
    # BASELINE.json configs[0] exactly: 1 group, P=512, 8 requests x 64 distinct,
    # one decode step, 8 heads (MHA), d=64, fp32, U(-10,10) like rand_case.
    cases.append(dict(name="c1_exact", seed=1, Hq=8, Hkv=8, d=64, dv=64,
                      dist="uniform10", dtype="f32",
                      groups=[_g(512, [(1, 64)] * 8)]))
    # GQA-4 decode, d=128, bf16, two groups of different shape.
    cases.append(dict(name="gqa4_decode_bf16", seed=2, Hq=8, Hkv=2, d=128, dv=128,
                      dist="normal", dtype="bf16",
                      groups=[_g(96, [(1, int(x)) for x in rs.integers(1, 81, 3)]),
                              _g(200, [(1, int(x)) for x in rs.integers(1, 81, 5)])]))
    # Mixed token batch: prefill chunks (rows straddle 128-row tiles) + decode.
    cases.append(dict(name="mixed_chunks_bf16", seed=3, Hq=8, Hkv=2, d=128, dv=128,
                      dist="normal", dtype="bf16",
                      groups=[_g(128, [(1, 40), (37, 50), (1, 3), (20, 20)]),
                              _g(64, [(45, 64), (1, 1)])]))
    # d=64 MHA with absent segments: group 1 has no prefix, request with no distinct.
    cases.append(dict(name="d64_absent_segments_bf16", seed=4, Hq=4, Hkv=4, d=64, dv=64,
                      dist="normal", dtype="bf16",
                      groups=[_g(70, [(2, 0), (1, 33)]),
                              _g(0, [(3, 17), (1, 5)]),
                              _g(257, [(1, 0)])]))
    # Llama-3-8B head shape, skewed groups (C4 in miniature).
    groups = []
    for P, R in ((16, 1), (300, 9), (1000, 2), (64, 20)):
        groups.append(_g(P, [(1, int(rs.integers(16, 200))) for _ in range(R)]))
    cases.append(dict(name="skewed_llama_bf16", seed=5, Hq=32, Hkv=8, d=128, dv=128,
                      dist="normal", dtype="bf16", groups=groups))
    # 40 decode requests x gqa 4 = 160 stacked rows -> two row tiles over one prefix.
    cases.append(dict(name="two_tiles_bf16", seed=6, Hq=8, Hkv=2, d=128, dv=128,
                      dist="normal", dtype="bf16",
                      groups=[_g(700, [(1, int(x)) for x in rs.integers(0, 40, 40)])]))
    # fp16 variant of a decode group.
    cases.append(dict(name="gqa2_decode_f16", seed=7, Hq=4, Hkv=2, d=64, dv=64,
                      dist="normal", dtype="f16",
                      groups=[_g(333, [(1, 10), (2, 0), (1, 129)])]))
    # fp32 with dv != d and odd head dim (generic CUDA-core path).
    cases.append(dict(name="f32_odd_dims", seed=8, Hq=3, Hkv=1, d=40, dv=24,
                      dist="uniform10", dtype="f32",
                      groups=[_g(50, [(2, 7), (1, 0)]), _g(9, [(4, 30)])]))
    # float64 strict drop-in path, single head, small arbitrary d.
    cases.append(dict(name="f64_single_head", seed=9, Hq=1, Hkv=1, d=32, dv=32,
                      dist="uniform10", dtype="f64",
                      groups=[_g(128, [(int(rs.integers(1, 6)), int(rs.integers(1, 65)))
                                       for _ in range(3)])]))
    # bf16 long prefix + long distinct for a single request (KV split into chunks).
    cases.append(dict(name="long_kv_bf16", seed=10, Hq=8, Hkv=2, d=128, dv=128,
                      dist="normal", dtype="bf16",
                      groups=[_g(3000, [(1, 2500), (2, 700)])]))
    return cases
