"""The drop-in module (paper_2412_03594_b200.attention) run through the
reference's own test cases: pkg/tests/test_attention.py restated with the
reference's inputs and tolerances, acceptance criterion 6
(pkg/tests/test_acceptance.py:178-225) and the golden single-head groups.
NumPy inputs select the strict float64 mode (GPU DFMA path)."""

import os

import numpy as np
import pytest
import torch

from paper_2412_03594_b200.attention import (SegmentedKV, empty_partial, finalize, merge,
                                             naive_attention, partial_attention,
                                             prefix_shared_attention, run_selftest)
from paper_2412_03594_b200.errors import PrefixBatchError, ValidationError
from oracle import segmented as S

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def rand_case(rng, n=None, total=None, d=None):  # test_attention.py:17-24
    n = n or int(rng.integers(1, 9))
    d = d or int(rng.integers(1, 17))
    total = total or int(rng.integers(2, 65))
    return (rng.uniform(-10, 10, (n, d)), rng.uniform(-10, 10, (total, d)),
            rng.uniform(-10, 10, (total, d)), 1.0 / np.sqrt(d))


def test_single_key_returns_value_row():  # :28-30
    out = naive_attention([[1.0]], [[1.0]], [[2.0]], 1.0)
    assert isinstance(out, np.ndarray) and out.dtype == np.float64
    assert np.abs(out - [[2.0]]).max() == 0.0


def test_zero_scale_uniform_weights():  # :32-36
    q, k, v, _ = rand_case(np.random.default_rng(0), n=4, total=12, d=8)
    assert np.abs(naive_attention(q, k, v, scale=0.0) - v.mean(axis=0)).max() < 1e-12


def test_naive_shape_validation():  # :48-54
    with pytest.raises(ValidationError):
        naive_attention([[1.0, 2.0]], [[1.0]], [[1.0]], 1.0)
    with pytest.raises(ValidationError):
        naive_attention([[1.0]], [[1.0], [2.0]], [[1.0]], 1.0)
    with pytest.raises(ValidationError):
        naive_attention([[np.inf]], [[1.0]], [[1.0]], 1.0)


def test_partial_single_key_and_identical_keys():  # :58-65
    assert np.abs(finalize(partial_attention([[1.0]], [[1.0]], [[2.0]], 1.0)) - [[2.0]]).max() < 1e-15
    part = partial_attention([[0.5, -0.25]], [[1.0, 2.0], [1.0, 2.0]], [[3.0, 0.0], [5.0, 4.0]], 1.0)
    assert np.abs(finalize(part) - [[4.0, 2.0]]).max() < 1e-12


def test_partial_matches_naive_random():  # :67-74
    rng = np.random.default_rng(2)
    worst = 0.0
    for _ in range(100):
        q, k, v, s = rand_case(rng)
        got = finalize(partial_attention(q, k, v, s))
        worst = max(worst, float(np.abs(got - S.dense_attention(q, k, v, s)).max()))
    assert worst < 1e-12


def test_stable_for_large_logits():  # :82-88
    out = finalize(partial_attention(np.array([[700.0]]), np.array([[1.0], [0.5]]),
                                     np.array([[1.0], [-1.0]]), 1.0))
    assert np.isfinite(out).all() and abs(out[0, 0] - 1.0) < 1e-12


def test_logit_offset_invariance():  # :90-96
    rng = np.random.default_rng(4)
    for c in (-500.0, -3.7, 250.0, 500.0):
        q, k, v, s = rand_case(rng)
        base = finalize(partial_attention(q, k, v, s))
        shifted = finalize(partial_attention(q, k, v, s, logit_offset=c))
        assert np.abs(base - shifted).max() < 1e-10


def test_empty_segment_and_invalid_scale():  # :98-107
    part = partial_attention(np.ones((3, 2)), np.zeros((0, 2)), np.zeros((0, 2)), 1.0)
    assert np.all(part.l == 0) and np.all(np.isneginf(part.m))
    with pytest.raises(ValidationError):
        finalize(part)
    with pytest.raises(ValidationError):
        partial_attention([[1.0]], [[1.0]], [[1.0]], scale=0.0)


def test_merge_properties():  # :111-160
    rng = np.random.default_rng(5)
    worst = 0.0
    for _ in range(50):
        q, k, v, s = rand_case(rng)
        cut = int(rng.integers(1, k.shape[0]))
        m = merge(partial_attention(q, k[:cut], v[:cut], s), partial_attention(q, k[cut:], v[cut:], s))
        worst = max(worst, float(np.abs(finalize(m) - S.dense_attention(q, k, v, s)).max()))
    assert worst < 1e-12
    q, k, v, s = rand_case(np.random.default_rng(6), n=5, total=20, d=4)
    whole = partial_attention(q, k, v, s)
    for m in (merge(whole, empty_partial(5, 4)), merge(empty_partial(5, 4), whole)):
        assert np.abs(finalize(m) - finalize(whole)).max() < 1e-12
    both = merge(empty_partial(2, 3), empty_partial(2, 3))
    assert np.all(both.l == 0) and np.all(both.o == 0)
    q, k, v, s = rand_case(np.random.default_rng(7))
    cut = k.shape[0] // 2
    a = partial_attention(q, k[:cut], v[:cut], s)
    b = partial_attention(q, k[cut:], v[cut:], s)
    assert np.abs(finalize(merge(a, b)) - finalize(merge(b, a))).max() < 1e-12
    with pytest.raises(ValidationError):
        merge(empty_partial(2, 3), empty_partial(2, 4))


def test_group_matches_per_request_naive():  # :164-179
    rng = np.random.default_rng(9)
    d = 32
    pk = rng.uniform(-10, 10, (128, d))
    pv = rng.uniform(-10, 10, (128, d))
    queries, distinct = [], []
    for _ in range(3):
        n = int(rng.integers(1, 6))
        m = int(rng.integers(1, 65))
        queries.append(rng.uniform(-10, 10, (n, d)))
        distinct.append((rng.uniform(-10, 10, (m, d)), rng.uniform(-10, 10, (m, d))))
    outs = prefix_shared_attention(queries, SegmentedKV((pk, pv), distinct))
    for q, (dk, dv), out in zip(queries, distinct, outs):
        ref = S.dense_attention(q, np.vstack([pk, dk]), np.vstack([pv, dv]))
        assert np.abs(out - ref).max() < 1e-10


def test_empty_distinct_and_sharing_degree_one():  # :181-200
    rng = np.random.default_rng(10)
    d = 8
    pk, pv = rng.uniform(-1, 1, (32, d)), rng.uniform(-1, 1, (32, d))
    queries = [rng.uniform(-1, 1, (2, d)), rng.uniform(-1, 1, (3, d))]
    outs = prefix_shared_attention(queries, SegmentedKV((pk, pv), [None, None]))
    for q, out in zip(queries, outs):
        assert np.abs(out - S.dense_attention(q, pk, pv)).max() < 1e-12
    rng = np.random.default_rng(11)
    d = 4
    q = rng.uniform(-1, 1, (3, d))
    pk, pv = rng.uniform(-1, 1, (16, d)), rng.uniform(-1, 1, (16, d))
    dk, dv = rng.uniform(-1, 1, (5, d)), rng.uniform(-1, 1, (5, d))
    (out,) = prefix_shared_attention([q], SegmentedKV((pk, pv), [(dk, dv)]))
    expected = S.normalize(S.combine(S.segment_partial(q, pk, pv), S.segment_partial(q, dk, dv)))
    assert np.abs(out - expected).max() < 1e-12


def test_rejections_and_error_types():  # :202-210 + errors.py hierarchy
    q = np.ones((1, 2))
    with pytest.raises(ValidationError, match="neither prefix nor distinct"):
        prefix_shared_attention([q], SegmentedKV(None, [None]))
    with pytest.raises(ValidationError, match="one distinct KV pair per request"):
        prefix_shared_attention([q, q], SegmentedKV(None, [None]))
    with pytest.raises(IndexError):  # attention.py:167 quirk
        prefix_shared_attention([], SegmentedKV(None, []))
    with pytest.raises(ValidationError, match="queries\\[1\\] contains non-finite"):
        prefix_shared_attention([q, [[np.nan, 0.0]]], SegmentedKV((q, q), [None, None]))
    with pytest.raises(ValidationError, match="segment keys have head dim 3, queries have 2"):
        prefix_shared_attention([q], SegmentedKV((np.ones((4, 3)), np.ones((4, 3))), [None]))
    with pytest.raises(ValidationError, match="cannot finalize"):
        prefix_shared_attention([q], SegmentedKV((np.zeros((0, 2)), np.zeros((0, 2))), [None]))
    with pytest.raises(ValidationError, match="partial result shapes differ"):
        prefix_shared_attention([q], SegmentedKV((q, np.ones((1, 3))), [(q, q)]))
    assert issubclass(ValidationError, PrefixBatchError) and not issubclass(ValidationError, ValueError)


def test_single_head_golden_from_reference():
    z = np.load(os.path.join(GOLDEN, "single_head.npz"))
    for ci in range(4):
        key = f"sh{ci}"
        Pn = int(z[f"{key}_P"])
        prefix = None if Pn < 0 else (z[f"{key}_pk"], z[f"{key}_pv"])
        n = int(z[f"{key}_n"])
        queries = [z[f"{key}_q{i}"] for i in range(n)]
        distinct = [None if bool(z[f"{key}_dnone{i}"]) else (z[f"{key}_dk{i}"], z[f"{key}_dv{i}"])
                    for i in range(n)]
        outs = prefix_shared_attention(queries, SegmentedKV(prefix, distinct))
        for i in range(n):
            assert outs[i].dtype == np.float64
            assert np.abs(outs[i] - z[f"{key}_out{i}"]).max() <= 1e-10


def test_criterion_6_on_gpu():  # test_acceptance.py:178-225 (generator + tolerances)
    rng = np.random.default_rng(123)
    worst = dict(merge=0.0, assoc=0.0, empty=0.0, group=0.0)
    for _ in range(100):
        n = int(rng.integers(1, 65))
        d = int(rng.integers(1, 65))
        total = int(rng.integers(3, 513))
        q = rng.uniform(-10, 10, (n, d))
        k = rng.uniform(-10, 10, (total, d))
        v = rng.uniform(-10, 10, (total, d))
        s = 1.0 / np.sqrt(d)
        expected = S.dense_attention(q, k, v, s)
        cut = int(rng.integers(1, total))
        merged = finalize(merge(partial_attention(q, k[:cut], v[:cut], s),
                                partial_attention(q, k[cut:], v[cut:], s)))
        worst["merge"] = max(worst["merge"], float(np.abs(merged - expected).max()))
        c1, c2 = sorted(rng.choice(np.arange(1, total), 2, replace=False).tolist())
        p1 = partial_attention(q, k[:c1], v[:c1], s)
        p2 = partial_attention(q, k[c1:c2], v[c1:c2], s)
        p3 = partial_attention(q, k[c2:], v[c2:], s)
        left = finalize(merge(merge(p1, p2), p3))
        right = finalize(merge(p1, merge(p2, p3)))
        worst["assoc"] = max(worst["assoc"], float(np.abs(left - right).max()),
                             float(np.abs(left - expected).max()))
        whole = partial_attention(q, k, v, s)
        ident = finalize(merge(whole, empty_partial(n, d)))
        worst["empty"] = max(worst["empty"], float(np.abs(ident - finalize(whole)).max()))
        dl = int(rng.integers(1, 65))
        dk = rng.uniform(-10, 10, (dl, d))
        dv = rng.uniform(-10, 10, (dl, d))
        (out,) = prefix_shared_attention([q], SegmentedKV((k, v), [(dk, dv)]), s)
        ref = S.dense_attention(q, np.vstack([k, dk]), np.vstack([v, dv]), s)
        worst["group"] = max(worst["group"], float(np.abs(out - ref).max()))
    assert worst["merge"] < 1e-10 and worst["assoc"] < 1e-10
    assert worst["empty"] < 1e-12 and worst["group"] < 1e-10


def test_selftest_passes():  # :213-219
    result = run_selftest(trials=10, seed=3)
    assert result["passed"] is True, result


def test_torch_mode_bf16_and_f32():
    rng = np.random.default_rng(21)
    d = 128
    pk = rng.standard_normal((300, d))
    pv = rng.standard_normal((300, d))
    qs = [rng.standard_normal((n, d)) for n in (1, 4, 40)]
    dist = [(rng.standard_normal((m, d)), rng.standard_normal((m, d))) for m in (10, 0, 77)]
    for dt, tol in ((torch.bfloat16, 2e-2), (torch.float32, 1e-4)):
        to = lambda x: torch.as_tensor(x).to("cuda", dt)  # noqa: E731
        outs = prefix_shared_attention([to(q) for q in qs],
                                       SegmentedKV((to(pk), to(pv)),
                                                   [(to(a), to(b)) for a, b in dist]))
        for q, (a, b), out in zip(qs, dist, outs):
            assert out.dtype == dt and out.is_cuda
            qq = to(q).double().cpu().numpy()
            k = np.vstack([to(pk).double().cpu().numpy(), to(a).double().cpu().numpy()])
            v = np.vstack([to(pv).double().cpu().numpy(), to(b).double().cpu().numpy()])
            ref = S.dense_attention(qq, k, v)
            assert np.abs(out.double().cpu().numpy() - ref).max() <= tol * max(1.0, np.abs(ref).max())
