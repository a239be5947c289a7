"""Pins the CPU oracle (oracle/segmented.py) before anything trusts it.

1. Against golden vectors produced by the reference itself
   (tests/golden/make_golden.py → packed.npz, single_head.npz).
2. Against every known-answer / property test the reference holds for this
   path: pkg/tests/test_attention.py (cited per test) and acceptance
   criterion 6 (pkg/tests/test_acceptance.py:178-225), restated here.
"""

import json
import os

import numpy as np
import pytest

import cases as C
from oracle import segmented as S

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _manifest():
    with open(os.path.join(GOLDEN, "manifest.json")) as f:
        return json.load(f)["cases"]


@pytest.mark.parametrize("entry", _manifest(), ids=lambda e: e["spec"]["name"])
def test_oracle_matches_reference_golden(entry):
    spec = entry["spec"]
    arrays = C.make_packed(spec)
    assert C.inputs_sha(arrays) == entry["sha256"], "input generator drifted"
    want = np.load(os.path.join(GOLDEN, "packed.npz"))[spec["name"]]
    got = S.packed_attention(arrays["q"], arrays["kp"], arrays["vp"], arrays["kd"],
                             arrays["vd"], arrays["cu_req"], arrays["cu_q"],
                             arrays["cu_prefix"], arrays["cu_distinct"],
                             spec["Hq"], spec["Hkv"])
    assert got.shape == want.shape
    assert np.abs(got - want).max() <= 1e-12 * max(1.0, np.abs(want).max())


def test_oracle_single_head_golden():
    z = np.load(os.path.join(GOLDEN, "single_head.npz"))
    ci = 0
    while f"sh{ci}_n" in z:
        key = f"sh{ci}"
        P = int(z[f"{key}_P"])
        prefix = None if P < 0 else (z[f"{key}_pk"], z[f"{key}_pv"])
        n = int(z[f"{key}_n"])
        queries = [z[f"{key}_q{i}"] for i in range(n)]
        distinct = [None if bool(z[f"{key}_dnone{i}"]) else (z[f"{key}_dk{i}"], z[f"{key}_dv{i}"])
                    for i in range(n)]
        outs = S.group_attention(queries, prefix, distinct)
        for i in range(n):
            assert np.abs(outs[i] - z[f"{key}_out{i}"]).max() <= 1e-12
        ci += 1
    assert ci == 4


# ---- restated known-answer tests (pkg/tests/test_attention.py) ----------

def rand_case(rng, n=None, total=None, d=None):
    """test_attention.py:17-24."""
    n = n or int(rng.integers(1, 9))
    d = d or int(rng.integers(1, 17))
    total = total or int(rng.integers(2, 65))
    q = rng.uniform(-10, 10, (n, d))
    k = rng.uniform(-10, 10, (total, d))
    v = rng.uniform(-10, 10, (total, d))
    return q, k, v, 1.0 / np.sqrt(d)


def test_single_key_returns_value_row():  # test_attention.py:28-30, :58-60
    assert np.abs(S.dense_attention([[1.0]], [[1.0]], [[2.0]], 1.0) - [[2.0]]).max() == 0.0
    part = S.segment_partial([[1.0]], [[1.0]], [[2.0]], 1.0)
    assert np.abs(S.normalize(part) - [[2.0]]).max() < 1e-15


def test_zero_scale_uniform_weights():  # :32-36
    q, k, v, _ = rand_case(np.random.default_rng(0), n=4, total=12, d=8)
    assert np.abs(S.dense_attention(q, k, v, scale=0.0) - v.mean(axis=0)).max() < 1e-12


def test_identical_keys_average_values():  # :62-65
    part = S.segment_partial([[0.5, -0.25]], [[1.0, 2.0], [1.0, 2.0]],
                             [[3.0, 0.0], [5.0, 4.0]], 1.0)
    assert np.abs(S.normalize(part) - [[4.0, 2.0]]).max() < 1e-12


def test_partial_matches_naive_random():  # :67-74
    rng = np.random.default_rng(2)
    worst = 0.0
    for _ in range(100):
        q, k, v, s = rand_case(rng)
        got = S.normalize(S.segment_partial(q, k, v, s))
        worst = max(worst, float(np.abs(got - S.dense_attention(q, k, v, s)).max()))
    assert worst < 1e-12


def test_large_logits_stable():  # :82-88
    out = S.normalize(S.segment_partial([[700.0]], [[1.0], [0.5]], [[1.0], [-1.0]], 1.0))
    assert np.isfinite(out).all() and abs(out[0, 0] - 1.0) < 1e-12


def test_logit_offset_invariance():  # :90-96
    rng = np.random.default_rng(4)
    for c in (-500.0, -3.7, 250.0, 500.0):
        q, k, v, s = rand_case(rng)
        base = S.normalize(S.segment_partial(q, k, v, s))
        shifted = S.normalize(S.segment_partial(q, k, v, s, logit_offset=c))
        assert np.abs(base - shifted).max() < 1e-10


def test_empty_segment_and_invalid_scale():  # :98-107
    part = S.segment_partial(np.ones((3, 2)), np.zeros((0, 2)), np.zeros((0, 2)), 1.0)
    assert np.all(part.l == 0) and np.all(np.isneginf(part.m))
    with pytest.raises(S.OracleValidationError):
        S.normalize(part)
    with pytest.raises(S.OracleValidationError):
        S.segment_partial([[1.0]], [[1.0]], [[1.0]], scale=0.0)


def test_merge_split_identity_commutative_assoc():  # :111-156
    rng = np.random.default_rng(5)
    worst = 0.0
    for _ in range(50):
        q, k, v, s = rand_case(rng)
        cut = int(rng.integers(1, k.shape[0]))
        m = S.combine(S.segment_partial(q, k[:cut], v[:cut], s),
                      S.segment_partial(q, k[cut:], v[cut:], s))
        worst = max(worst, float(np.abs(S.normalize(m) - S.dense_attention(q, k, v, s)).max()))
    assert worst < 1e-12
    q, k, v, s = rand_case(np.random.default_rng(6), n=5, total=20, d=4)
    whole = S.segment_partial(q, k, v, s)
    for m in (S.combine(whole, S.empty(5, 4)), S.combine(S.empty(5, 4), whole)):
        assert np.abs(S.normalize(m) - S.normalize(whole)).max() < 1e-12
    both = S.combine(S.empty(2, 3), S.empty(2, 3))
    assert np.all(both.l == 0) and np.all(both.o == 0)
    with pytest.raises(S.OracleValidationError):
        S.combine(S.empty(2, 3), S.empty(2, 4))


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
    outs = S.group_attention(queries, (pk, pv), distinct)
    for q, (dk, dv), out in zip(queries, distinct, outs):
        ref = S.dense_attention(q, np.vstack([pk, dk]), np.vstack([pv, dv]))
        assert np.abs(out - ref).max() < 1e-10


def test_group_rejections():  # :202-210
    q = np.ones((1, 2))
    with pytest.raises(S.OracleValidationError):
        S.group_attention([q], None, [None])
    with pytest.raises(S.OracleValidationError):
        S.group_attention([q, q], None, [None])


def test_criterion_6_attention_oracle_equivalence():
    """pkg/tests/test_acceptance.py:178-225, same generator and tolerances."""
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
        merged = S.normalize(S.combine(S.segment_partial(q, k[:cut], v[:cut], s),
                                       S.segment_partial(q, k[cut:], v[cut:], s)))
        worst["merge"] = max(worst["merge"], float(np.abs(merged - expected).max()))
        c1, c2 = sorted(rng.choice(np.arange(1, total), 2, replace=False).tolist())
        p1 = S.segment_partial(q, k[:c1], v[:c1], s)
        p2 = S.segment_partial(q, k[c1:c2], v[c1:c2], s)
        p3 = S.segment_partial(q, k[c2:], v[c2:], s)
        left = S.normalize(S.combine(S.combine(p1, p2), p3))
        right = S.normalize(S.combine(p1, S.combine(p2, p3)))
        worst["assoc"] = max(worst["assoc"], float(np.abs(left - right).max()),
                             float(np.abs(left - expected).max()))
        whole = S.segment_partial(q, k, v, s)
        ident = S.normalize(S.combine(whole, S.empty(n, d)))
        worst["empty"] = max(worst["empty"], float(np.abs(ident - S.normalize(whole)).max()))
        dl = int(rng.integers(1, 65))
        dk = rng.uniform(-10, 10, (dl, d))
        dv = rng.uniform(-10, 10, (dl, d))
        (out,) = S.group_attention([q], (k, v), [(dk, dv)], s)
        ref = S.dense_attention(q, np.vstack([k, dk]), np.vstack([v, dv]), s)
        worst["group"] = max(worst["group"], float(np.abs(out - ref).max()))
    assert worst["merge"] < 1e-10 and worst["assoc"] < 1e-10
    assert worst["empty"] < 1e-12 and worst["group"] < 1e-10


def test_gqa_adapter_equals_per_query_head():
    """stacking gqa heads as rows == one call per query head."""
    spec = dict(seed=31, Hq=8, Hkv=2, d=16, dv=16, dist="normal", dtype="f64",
                groups=[{"P": 20, "reqs": [[3, 5], [1, 9]]}])
    a = C.make_packed(spec)
    got = S.packed_attention(a["q"], a["kp"], a["vp"], a["kd"], a["vd"], a["cu_req"],
                             a["cu_q"], a["cu_prefix"], a["cu_distinct"], 8, 2)
    for hq in range(8):
        h = hq // 4
        for r in range(2):
            t0, t1 = a["cu_q"][r], a["cu_q"][r + 1]
            d0, d1 = a["cu_distinct"][r], a["cu_distinct"][r + 1]
            k = np.vstack([a["kp"][:, h], a["kd"][d0:d1, h]])
            v = np.vstack([a["vp"][:, h], a["vd"][d0:d1, h]])
            ref = S.dense_attention(a["q"][t0:t1, hq], k, v)
            assert np.abs(got[t0:t1, hq] - ref).max() < 1e-12
