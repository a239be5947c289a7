"""Synthetic token batches for the BASELINE.json configs.

Each config is a list of prefix-sharing groups; each group has a shared prefix
of P tokens and requests (n_q query tokens, D distinct KV tokens). Inputs are
generated on the device with a counter-based per-group seed (the idea of the
reference's workload.py:82-102), so any subset of groups — e.g. one rank's
shard — sees exactly the data it would see in the full batch.

  c1  1 group, P=512, 8 requests x 64 distinct, 1 decode token, MHA 8 heads, d=64, fp32, U(-10,10)
  c2  16 groups x P=2048 x 32 requests x D=256, Llama-3-8B heads (32 q / 8 kv, d=128), bf16
  c3  64 groups x P=2048, per group 32 decode (D=256) + 2 prefill chunks (512 tokens, D=512), bf16
  c4  64 skewed groups: P 256-8k, 1-256 requests, D 16-512 (exact draw: SURVEY.md Appendix A), bf16
  c5  1024 groups x P=4096 x 64 requests x D=256, bf16 (sharded by group across GPUs)
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np
import torch

DTYPES = {"f32": torch.float32, "bf16": torch.bfloat16, "f16": torch.float16,
          "f64": torch.float64}


@dataclass
class Spec:
    name: str
    Hq: int
    Hkv: int
    d: int
    dv: int
    dtype: str
    dist: str                     # "normal" | "uniform10"
    prefix: list                  # P per group
    reqs: list                    # per group: list of (n_q, D)
    seed: int = 0
    group_ids: Optional[list] = None  # global ids (for per-group seeds) of these groups
    meta: dict = field(default_factory=dict)

    @property
    def G(self) -> int:
        return len(self.prefix)

    @property
    def torch_dtype(self) -> torch.dtype:
        return DTYPES[self.dtype]

    def gid(self, g: int) -> int:
        return self.group_ids[g] if self.group_ids is not None else g

    def subset(self, groups: Sequence[int]) -> "Spec":
        groups = list(groups)
        return Spec(self.name, self.Hq, self.Hkv, self.d, self.dv, self.dtype, self.dist,
                    [self.prefix[g] for g in groups], [self.reqs[g] for g in groups], self.seed,
                    [self.gid(g) for g in groups], dict(self.meta))


def config(name: str) -> Spec:
    name = name.lower()
    if name == "c1":
        return Spec("c1", 8, 8, 64, 64, "f32", "uniform10", [512], [[(1, 64)] * 8], seed=1)
    if name == "c2":
        return Spec("c2", 32, 8, 128, 128, "bf16", "normal", [2048] * 16,
                    [[(1, 256)] * 32 for _ in range(16)], seed=2)
    if name == "c3":
        reqs = [(1, 256)] * 16 + [(512, 512)] + [(1, 256)] * 16 + [(512, 512)]
        return Spec("c3", 32, 8, 128, 128, "bf16", "normal", [2048] * 64,
                    [list(reqs) for _ in range(64)], seed=3)
    if name == "c4":
        rng = np.random.default_rng(4)
        G = 64
        P = (16 * np.round(np.exp(rng.uniform(np.log(256), np.log(8192), G)) / 16)).astype(int)
        R = np.clip(np.round(np.exp(rng.uniform(0, np.log(256), G))), 1, 256).astype(int)
        reqs = [[(1, int(rng.integers(16, 513))) for _ in range(R[g])] for g in range(G)]
        return Spec("c4", 32, 8, 128, 128, "bf16", "normal", [int(p) for p in P], reqs, seed=4)
    if name == "c5":
        return Spec("c5", 32, 8, 128, 128, "bf16", "normal", [4096] * 1024,
                    [[(1, 256)] * 64 for _ in range(1024)], seed=5)
    # diagnostic halves of c2: the shared-prefix tiles alone / the decode part alone
    if name == "c2_prefix":
        return Spec("c2_prefix", 32, 8, 128, 128, "bf16", "normal", [2048] * 16,
                    [[(1, 0)] * 32 for _ in range(16)], seed=2)
    if name == "c2_decode":
        return Spec("c2_decode", 32, 8, 128, 128, "bf16", "normal", [0] * 16,
                    [[(1, 256)] * 32 for _ in range(16)], seed=2)
    # diagnostic halves of c5
    if name == "c5_prefix":
        return Spec("c5_prefix", 32, 8, 128, 128, "bf16", "normal", [4096] * 1024,
                    [[(1, 0)] * 64 for _ in range(1024)], seed=5)
    if name == "c5_decode":
        return Spec("c5_decode", 32, 8, 128, 128, "bf16", "normal", [0] * 1024,
                    [[(1, 256)] * 64 for _ in range(1024)], seed=5)
    # diagnostic parts of c3: the prefix tiles alone / the prefill chunks' own KV alone
    if name == "c3_prefix":
        reqs = [(1, 0)] * 16 + [(512, 0)] + [(1, 0)] * 16 + [(512, 0)]
        return Spec("c3_prefix", 32, 8, 128, 128, "bf16", "normal", [2048] * 64,
                    [list(reqs) for _ in range(64)], seed=3)
    if name == "c3_chunks":
        return Spec("c3_chunks", 32, 8, 128, 128, "bf16", "normal", [0] * 64,
                    [[(512, 512)] * 2 for _ in range(64)], seed=3)
    if name.startswith("fig9:"):
        for n, spec in fig9_specs():
            if n.lower() == name[5:]:
                return spec
    raise ValueError(f"unknown config {name!r} (c1..c5, c2_prefix, c2_decode, c3_prefix, "
                     "c3_chunks, fig9:<shape>)")


def fig9_specs() -> list:
    """Kernel-comparison shapes in the style of the paper's Fig. 9:
    P/D/k = shared-prefix length / distinct length / requests per prefix group;
    decoding with 32 and 256 requests, and chunked prefill (7 prefill chunks of 512
    tokens with 512 own keys, plus 256 decoding requests). Llama-3-8B heads, bf16.
    Names: dec{R}_{P}/{D}/{k|all}, chunked7+256_{P}/256/{k}."""
    out = []
    for R in (32, 256):
        for P, D in ((256, 2048), (2048, 256), (2048, 2048), (8192, 256)):
            for k in (R, 16, 4):
                G = R // k
                out.append((f"dec{R}_{P}/{D}/{'all' if k == R else k}",
                            Spec("fig9", 32, 8, 128, 128, "bf16", "normal", [P] * G,
                                 [[(1, D)] * k for _ in range(G)], seed=9)))
    for P, k in ((2048, 32), (2048, 263)):
        G = 263 // k if k < 263 else 1
        reqs = [[(1, 256)] * k for _ in range(G)]
        for i in range(7):  # prefill chunks spread over the groups
            reqs[i % G].append((512, 512))
        out.append((f"chunked7+256_{P}/256/{k}",
                    Spec("fig9", 32, 8, 128, 128, "bf16", "normal", [P] * G, reqs, seed=9)))
    return out


def offsets(spec: Spec) -> dict:
    flat = [r for g in spec.reqs for r in g]
    return dict(
        cu_req=np.cumsum([0] + [len(g) for g in spec.reqs]).astype(np.int64),
        cu_q=np.cumsum([0] + [n for n, _ in flat]).astype(np.int64),
        cu_prefix=np.cumsum([0] + list(spec.prefix)).astype(np.int64),
        cu_distinct=np.cumsum([0] + [D for _, D in flat]).astype(np.int64),
    )


def _seed(base: int, gid: int, stream: int) -> int:
    """splitmix64-style counter hash (reference workload.py:89-93 idea)."""
    z = (base * 0x9E3779B97F4A7C15 + gid * 0xBF58476D1CE4E5B9 + stream * 0x94D049BB133111EB
         + 0x2545F4914F6CDD1D) & 0xFFFFFFFFFFFFFFFF
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & 0xFFFFFFFFFFFFFFFF
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & 0xFFFFFFFFFFFFFFFF
    return (z ^ (z >> 31)) & 0x7FFFFFFFFFFFFFFF


def _fill(t: torch.Tensor, dist: str, gen: torch.Generator) -> None:
    if t.numel() == 0:
        return
    if dist == "normal":
        tmp = torch.randn(t.shape, generator=gen, device=t.device, dtype=torch.float32)
    else:
        tmp = torch.rand(t.shape, generator=gen, device=t.device, dtype=torch.float32)
        tmp.mul_(20.0).sub_(10.0)
    t.copy_(tmp)


def make_batch(spec: Spec, device) -> dict:
    """Allocate and fill the packed tensors of ``spec`` on ``device``."""
    off = offsets(spec)
    dt = spec.torch_dtype
    T, Pn, Dn = int(off["cu_q"][-1]), int(off["cu_prefix"][-1]), int(off["cu_distinct"][-1])
    out = dict(
        q=torch.empty((T, spec.Hq, spec.d), dtype=dt, device=device),
        k_prefix=torch.empty((Pn, spec.Hkv, spec.d), dtype=dt, device=device),
        v_prefix=torch.empty((Pn, spec.Hkv, spec.dv), dtype=dt, device=device),
        k_distinct=torch.empty((Dn, spec.Hkv, spec.d), dtype=dt, device=device),
        v_distinct=torch.empty((Dn, spec.Hkv, spec.dv), dtype=dt, device=device),
    )
    gen = torch.Generator(device=device)
    for g in range(spec.G):
        gid = spec.gid(g)
        r0, r1 = int(off["cu_req"][g]), int(off["cu_req"][g + 1])
        t0, t1 = int(off["cu_q"][r0]), int(off["cu_q"][r1])
        p0, p1 = int(off["cu_prefix"][g]), int(off["cu_prefix"][g + 1])
        d0, d1 = int(off["cu_distinct"][r0]), int(off["cu_distinct"][r1])
        for stream, (key, a, b) in enumerate((("q", t0, t1), ("k_prefix", p0, p1),
                                              ("v_prefix", p0, p1), ("k_distinct", d0, d1),
                                              ("v_distinct", d0, d1))):
            gen.manual_seed(_seed(spec.seed, gid, stream))
            _fill(out[key][a:b], spec.dist, gen)
    out.update(off)
    return out


def algorithmic_cost(spec: Spec) -> dict:
    """FLOP and HBM bytes the algorithm must spend.

    FLOP = 4*d per (query row, key) pair (QK^T and PV; d == dv here, else 2*(d+dv)).
    Bytes = prefix KV once per group + distinct KV once per request + Q read + O write.
    """
    elt = torch.finfo(spec.torch_dtype).bits // 8
    width = spec.d + spec.dv
    f_pre = f_dis = 0
    b_pre = b_dis = b_q = b_o = 0
    for g in range(spec.G):
        P = spec.prefix[g]
        b_pre += spec.Hkv * P * width * elt
        for n, D in spec.reqs[g]:
            f_pre += 2 * width * spec.Hq * n * P
            f_dis += 2 * width * spec.Hq * n * D
            b_dis += spec.Hkv * D * width * elt
            b_q += n * spec.Hq * spec.d * elt
            b_o += n * spec.Hq * spec.dv * elt
    return dict(flops=f_pre + f_dis, flops_prefix=f_pre, flops_distinct=f_dis,
                bytes=b_pre + b_dis + b_q + b_o, bytes_prefix=b_pre, bytes_distinct=b_dis,
                bytes_q=b_q, bytes_o=b_o)
