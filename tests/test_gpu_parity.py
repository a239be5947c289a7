"""GPU parity: libpsa.so (through the C ABI) against the reference's golden
outputs and the CPU oracle. Tolerances (BASELINE.json):
  bf16 / f16 : max |out - ref| <= 2e-2 (N(0,1) inputs)
  fp32       : normwise max|out - ref| / max|ref| <= 1e-4 (FFMA, no TF32)
  fp64       : max |out - ref| <= 1e-10 (strict drop-in mode)
"""

import json
import os

import numpy as np
import pytest
import torch

import cases as C
from oracle import segmented as S
from paper_2412_03594_b200 import packed as P
from paper_2412_03594_b200 import workloads as W

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
TDT = {"f32": torch.float32, "bf16": torch.bfloat16, "f16": torch.float16, "f64": torch.float64}


def assert_close(got: np.ndarray, want: np.ndarray, dtype: str):
    err = float(np.abs(got - want).max()) if want.size else 0.0
    if dtype in ("bf16", "f16"):
        assert err <= 2e-2, f"max abs err {err}"
    elif dtype == "f32":
        assert err <= 1e-4 * max(float(np.abs(want).max()), 1e-30), f"normwise err {err}"
    else:
        assert err <= 1e-10, f"max abs err {err}"
    return err


def _manifest():
    with open(os.path.join(GOLDEN, "manifest.json")) as f:
        return [e["spec"] for e in json.load(f)["cases"]]


def _device_batch(a, dtype):
    dev = torch.device("cuda")
    t = {k: torch.as_tensor(a[k]).to(dev, TDT[dtype]).contiguous()
         for k in ("q", "kp", "vp", "kd", "vd")}
    return t


@pytest.mark.parametrize("spec", _manifest(), ids=lambda s: s["name"])
@pytest.mark.parametrize("opts", [dict(), dict(disable_tiles=1), dict(min_chunk_keys=64),
                                  dict(disable_vec_fast=1), dict(disable_vec_fast=2)],
                         ids=["default", "no_tiles", "small_chunks", "generic_vec", "warp_vec"])
def test_packed_matches_reference_golden(spec, opts):
    a = C.make_packed(spec)
    want = np.load(os.path.join(GOLDEN, "packed.npz"))[spec["name"]]
    t = _device_batch(a, spec["dtype"])
    op = P.PrefixSharedAttention(a["cu_req"], a["cu_q"], a["cu_prefix"], a["cu_distinct"],
                                 spec["Hq"], spec["Hkv"], spec["d"], spec["dv"],
                                 TDT[spec["dtype"]], "cuda", options=P.PlanOptions(**opts))
    out = op(t["q"], t["kp"], t["vp"], t["kd"], t["vd"])
    torch.cuda.synchronize()
    assert op.device_error() == 0
    assert_close(out.double().cpu().numpy(), want, spec["dtype"])


def test_repeat_launches_are_bit_identical_and_reset_counters():
    spec = [s for s in _manifest() if s["name"] == "mixed_chunks_bf16"][0]
    a = C.make_packed(spec)
    t = _device_batch(a, "bf16")
    op = P.PrefixSharedAttention(a["cu_req"], a["cu_q"], a["cu_prefix"], a["cu_distinct"],
                                 spec["Hq"], spec["Hkv"], spec["d"], spec["dv"], torch.bfloat16,
                                 "cuda", options=P.PlanOptions(min_chunk_keys=64))
    outs = [op(t["q"], t["kp"], t["vp"], t["kd"], t["vd"]).clone() for _ in range(4)]
    torch.cuda.synchronize()
    for o in outs[1:]:
        assert torch.equal(o, outs[0])
    ctrl = op.workspace[:16].view(torch.int32).cpu()
    assert ctrl[0].item() == 0 and ctrl[1].item() == 0


@pytest.mark.parametrize("opts", [dict(), dict(disable_tiles=1), dict(kernel_variant=1),
                                  dict(kernel_variant=1, disable_tiles=1)],
                         ids=["v2", "v2_dec_only", "v1", "v1_dec_only"])
def test_skewed_batch_many_launches_bit_identical(opts):
    """c4 (skewed groups) relaunched many times: every launch must be bitwise equal.
    Catches pipeline phase races (e.g. a ring slot consumed one phase early), which
    show up as rare single-token differences or a faulting mbarrier."""
    spec = W.config("c4")
    b = W.make_batch(spec, "cuda")
    op = P.PrefixSharedAttention(b["cu_req"], b["cu_q"], b["cu_prefix"], b["cu_distinct"],
                                 spec.Hq, spec.Hkv, spec.d, spec.dv, spec.torch_dtype, "cuda",
                                 options=P.PlanOptions(**opts))
    keys = ("q", "k_prefix", "v_prefix", "k_distinct", "v_distinct")
    ref = op(*(b[k] for k in keys)).clone()
    out = torch.empty_like(ref)
    for i in range(60):
        op(*(b[k] for k in keys), out=out)
        torch.cuda.synchronize()
        assert torch.equal(out, ref), f"launch {i + 1} differs from launch 0"
    assert op.device_error() == 0
    check_sampled_groups(spec, b, ref, n_groups=2, n_heads=1)


@pytest.mark.parametrize("name", ["c2", "c4"])
def test_relaunch_with_new_inputs_recomputes_everything(name):
    """One planned op, several launches with different inputs (and a poisoned
    output buffer each time): every launch must redo every work item, i.e. the
    queue cursors and merge counters are reset by the kernel itself."""
    spec = W.config(name)
    b = W.make_batch(spec, "cuda")
    op = P.PrefixSharedAttention(b["cu_req"], b["cu_q"], b["cu_prefix"], b["cu_distinct"],
                                 spec.Hq, spec.Hkv, spec.d, spec.dv, spec.torch_dtype, "cuda")
    keys = ("q", "k_prefix", "v_prefix", "k_distinct", "v_distinct")
    for trial in range(3):
        if trial:
            for k in keys:
                b[k].mul_(-1.0 if k == "v_distinct" else 1.0).add_(0.0)
            b["q"].copy_(torch.randn_like(b["q"]))
        out = torch.full((b["q"].shape[0], spec.Hq, spec.dv), float("nan"),
                         dtype=spec.torch_dtype, device="cuda")
        op(*(b[k] for k in keys), out=out)
        torch.cuda.synchronize()
        assert not torch.isnan(out).any(), f"launch {trial} left rows unwritten"
        check_sampled_groups(spec, b, out, n_groups=2, n_heads=2, seed=trial)


def test_lse_output_matches_oracle():
    spec = [s for s in _manifest() if s["name"] == "gqa4_decode_bf16"][0]
    a = C.make_packed(spec)
    t = _device_batch(a, "bf16")
    op = P.PrefixSharedAttention(a["cu_req"], a["cu_q"], a["cu_prefix"], a["cu_distinct"],
                                 spec["Hq"], spec["Hkv"], spec["d"], spec["dv"], torch.bfloat16,
                                 "cuda")
    lse = torch.empty(t["q"].shape[:2], dtype=torch.float32, device="cuda")
    op(t["q"], t["kp"], t["vp"], t["kd"], t["vd"], lse=lse)
    # oracle LSE: log sum exp over [prefix; distinct] of scale * q.k
    gqa = spec["Hq"] // spec["Hkv"]
    scale = 1.0 / np.sqrt(spec["d"])
    q = a["q"].astype(np.float64)
    for g in range(len(a["cu_req"]) - 1):
        for r in range(a["cu_req"][g], a["cu_req"][g + 1]):
            for tok in range(a["cu_q"][r], a["cu_q"][r + 1]):
                for hq in range(spec["Hq"]):
                    h = hq // gqa
                    k = np.vstack([a["kp"][a["cu_prefix"][g]:a["cu_prefix"][g + 1], h],
                                   a["kd"][a["cu_distinct"][r]:a["cu_distinct"][r + 1], h]])
                    z = scale * (k.astype(np.float64) @ q[tok, hq])
                    ref = z.max() + np.log(np.exp(z - z.max()).sum())
                    assert abs(lse[tok, hq].item() - ref) < 2e-3


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4", "c5"])
def test_bench_config_parity_against_oracle(name):
    """Full-size bench batches (c5: all 1024 groups, 87 GB, one launch); the oracle
    checks a sample of (group, kv head) pairs and every row must be written."""
    spec = W.config(name)
    b = W.make_batch(spec, "cuda")
    op = P.PrefixSharedAttention(b["cu_req"], b["cu_q"], b["cu_prefix"], b["cu_distinct"],
                                 spec.Hq, spec.Hkv, spec.d, spec.dv, spec.torch_dtype, "cuda")
    out = torch.full((b["q"].shape[0], spec.Hq, spec.dv), float("nan"), dtype=spec.torch_dtype,
                     device="cuda")
    op(b["q"], b["k_prefix"], b["v_prefix"], b["k_distinct"], b["v_distinct"], out=out)
    torch.cuda.synchronize()
    assert op.device_error() == 0
    assert not torch.isnan(out).any()
    n = 5 if name == "c5" else 3
    check_sampled_groups(spec, b, out, n_groups=n, n_heads=2)
    if name == "c5":  # the first and the last group too (queue head / tail)
        check_sampled_groups(spec.subset([0, spec.G - 1]), _group_batch(b, [0, spec.G - 1]),
                             _group_rows(b, out, [0, spec.G - 1]), n_groups=2, n_heads=8)


def _group_rows(b, out, groups):
    return torch.cat([out[int(b["cu_q"][b["cu_req"][g]]):int(b["cu_q"][b["cu_req"][g + 1]])]
                      for g in groups])


def _group_batch(b, groups):
    """Sub-batch of whole groups (device tensor slices + rebased offsets)."""
    def cat(t, cu, idx):
        return torch.cat([t[int(cu[i]):int(cu[i + 1])] for i in idx])
    reqs = [r for g in groups for r in range(int(b["cu_req"][g]), int(b["cu_req"][g + 1]))]
    cum = lambda lens: np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)  # noqa: E731
    return dict(q=cat(b["q"], b["cu_q"], reqs), k_prefix=cat(b["k_prefix"], b["cu_prefix"], groups),
                v_prefix=cat(b["v_prefix"], b["cu_prefix"], groups),
                k_distinct=cat(b["k_distinct"], b["cu_distinct"], reqs),
                v_distinct=cat(b["v_distinct"], b["cu_distinct"], reqs),
                cu_req=cum([int(b["cu_req"][g + 1] - b["cu_req"][g]) for g in groups]),
                cu_q=cum([int(b["cu_q"][r + 1] - b["cu_q"][r]) for r in reqs]),
                cu_prefix=cum([int(b["cu_prefix"][g + 1] - b["cu_prefix"][g]) for g in groups]),
                cu_distinct=cum([int(b["cu_distinct"][r + 1] - b["cu_distinct"][r]) for r in reqs]))


def group_host_slice(b: dict, g: int) -> dict:
    """Float64 host copy of one group's slices with group-local offsets."""
    r0, r1 = int(b["cu_req"][g]), int(b["cu_req"][g + 1])
    t0, t1 = int(b["cu_q"][r0]), int(b["cu_q"][r1])
    p0, p1 = int(b["cu_prefix"][g]), int(b["cu_prefix"][g + 1])
    d0, d1 = int(b["cu_distinct"][r0]), int(b["cu_distinct"][r1])
    return dict(q=b["q"][t0:t1].double().cpu().numpy(),
                kp=b["k_prefix"][p0:p1].double().cpu().numpy(),
                vp=b["v_prefix"][p0:p1].double().cpu().numpy(),
                kd=b["k_distinct"][d0:d1].double().cpu().numpy(),
                vd=b["v_distinct"][d0:d1].double().cpu().numpy(),
                cu_req=np.array([0, r1 - r0]), cu_q=b["cu_q"][r0:r1 + 1] - t0,
                cu_prefix=np.array([0, p1 - p0]), cu_distinct=b["cu_distinct"][r0:r1 + 1] - d0,
                t0=t0)


def check_sampled_groups(spec, b, out, n_groups=3, n_heads=2, seed=0):
    gqa = spec.Hq // spec.Hkv
    rng = np.random.default_rng(seed)
    worst = 0.0
    for g in sorted(set(rng.integers(0, spec.G, n_groups).tolist())):
        hs = group_host_slice(b, g)
        for h in sorted(set(rng.integers(0, spec.Hkv, n_heads).tolist())):
            res = S.packed_group_head(hs["q"], hs["kp"], hs["vp"], hs["kd"], hs["vd"],
                                      hs["cu_req"], hs["cu_q"], hs["cu_prefix"],
                                      hs["cu_distinct"], 0, h, spec.Hq, spec.Hkv)
            for i in range(len(hs["cu_q"]) - 1):
                t0, t1 = hs["t0"] + hs["cu_q"][i], hs["t0"] + hs["cu_q"][i + 1]
                got = out[t0:t1, h * gqa:(h + 1) * gqa].double().cpu().numpy()
                worst = max(worst, assert_close(got.reshape(-1, spec.dv), res[i], spec.dtype))
    return worst


@pytest.mark.parametrize("dtype", ["f16", "bf16"])
def test_v2_kernel_half_precision_mixed_batch(dtype):
    """The v2 kernel in both 16-bit formats (golden cases cover f16 only at d=64):
    decode + prefill-chunk requests, two-slot and single-slot tiles, merges."""
    spec = W.Spec("mixed16", 16, 4, 128, 128, dtype, "normal", [700, 33, 0, 2049],
                  [[(1, 40), (37, 51), (1, 3), (1, 0)], [(1, 64), (20, 1)], [(3, 17)],
                   [(1, 300)] * 40 + [(130, 77)]], seed=31)
    b = W.make_batch(spec, "cuda")
    op = P.PrefixSharedAttention(b["cu_req"], b["cu_q"], b["cu_prefix"], b["cu_distinct"],
                                 spec.Hq, spec.Hkv, spec.d, spec.dv, spec.torch_dtype, "cuda")
    out = op(b["q"], b["k_prefix"], b["v_prefix"], b["k_distinct"], b["v_distinct"])
    torch.cuda.synchronize()
    assert op.device_error() == 0
    host = {k: b[k].double().cpu().numpy() for k in ("q", "k_prefix", "v_prefix", "k_distinct",
                                                       "v_distinct")}
    ref = S.packed_attention(host["q"], host["k_prefix"], host["v_prefix"], host["k_distinct"],
                             host["v_distinct"], b["cu_req"], b["cu_q"], b["cu_prefix"],
                             b["cu_distinct"], spec.Hq, spec.Hkv)
    assert_close(out.double().cpu().numpy(), ref, dtype)
