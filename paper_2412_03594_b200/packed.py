"""Packed multi-group, multi-head API — the hot path the bench and engines call.

One call evaluates a whole token batch: every prefix-sharing group, every kv
head, decode and prefill-chunk requests alike, in ONE persistent kernel
launch (libpsa.so, include/psa.h). Semantics per (group, kv head) are exactly
the reference's ``prefix_shared_attention`` (attention.py:156-201) on the gqa
query heads stacked as rows.

Layout (see include/psa.h): q [T, Hq, d]; k_prefix/v_prefix [sum P_g, Hkv, d|dv];
k_distinct/v_distinct [sum D_r, Hkv, d|dv]; offsets cu_req [G+1], cu_q [R+1],
cu_prefix [G+1], cu_distinct [R+1] (host int64).
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

from . import _lib as L
from .errors import ValidationError

_TORCH_TO_PSA = {torch.float32: L.DTYPE_F32, torch.bfloat16: L.DTYPE_BF16,
                 torch.float16: L.DTYPE_F16, torch.float64: L.DTYPE_F64}


def psa_dtype(dt: torch.dtype) -> int:
    try:
        return _TORCH_TO_PSA[dt]
    except KeyError:
        raise ValidationError(f"unsupported dtype {dt}") from None


def acc_dtype(dt: torch.dtype) -> torch.dtype:
    return torch.float64 if dt == torch.float64 else torch.float32


def _i64(x) -> np.ndarray:
    if isinstance(x, torch.Tensor):
        x = x.detach().cpu().numpy()
    return np.ascontiguousarray(np.asarray(x, dtype=np.int64))


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else C.c_void_p(t.data_ptr())


def _raise_native(status: int, what: str):
    msg = L.last_error()
    if status in (L.PSA_INVALID_ARGUMENT, L.PSA_UNSUPPORTED):
        raise ValidationError(msg)
    raise RuntimeError(f"{what}: {msg}")


@dataclass
class PlanOptions:
    """Mirror of psa_plan_opts (0 = library default)."""
    num_sms: int = 0
    ctas_per_sm: int = 0
    tile_min_rows: int = 0
    disable_tiles: int = 0
    min_chunk_keys: int = 0
    max_chunk_keys: int = 0
    target_waves: int = 0
    disable_vec_fast: int = 0
    kernel_variant: int = 0  # 0 = auto (v2 for bf16/f16 d=dv=128), 1 = 2-CTA/SM kernel

    def to_c(self) -> L.PlanOpts:
        return L.PlanOpts(self.num_sms, self.ctas_per_sm, self.tile_min_rows, self.disable_tiles,
                          self.min_chunk_keys, self.max_chunk_keys, self.target_waves,
                          self.disable_vec_fast, self.kernel_variant)


class PrefixSharedAttention:
    """A planned prefix-shared attention op for one batch structure.

    The plan (work items, merge units) depends only on the offset tables and
    head shape; build it once per token batch and call it for every layer.
    The device workspace is owned by this object (allocated through torch).
    """

    def __init__(self, cu_req, cu_q, cu_prefix, cu_distinct, num_q_heads: int,
                 num_kv_heads: int, head_dim: int, value_dim: Optional[int] = None,
                 dtype: torch.dtype = torch.bfloat16, device=None,
                 scale: Optional[float] = None, options: Optional[PlanOptions] = None,
                 page_size: int = 0):
        """``page_size`` > 0 plans for a paged KV cache (see :meth:`__call__` and
        include/psa.h): K/V come from page caches through page tables instead of the
        packed segment layout; the plan (work items, merge units) is the same."""
        self.page_size = int(page_size)
        self.cu_req, self.cu_q = _i64(cu_req), _i64(cu_q)
        self.cu_prefix, self.cu_distinct = _i64(cu_prefix), _i64(cu_distinct)
        self.G = len(self.cu_req) - 1
        self.R = len(self.cu_q) - 1
        if self.G < 1 or self.R < 1:
            raise ValidationError("a batch needs at least one group and one request")
        if len(self.cu_prefix) != self.G + 1 or len(self.cu_distinct) != self.R + 1:
            raise ValidationError("offset tables disagree on the number of groups/requests")
        self.Hq, self.Hkv = int(num_q_heads), int(num_kv_heads)
        self.d = int(head_dim)
        self.dv = int(value_dim) if value_dim is not None else self.d
        self.dtype = dtype
        dev = torch.device(device) if device is not None else torch.device("cuda")
        if dev.type != "cuda":
            raise ValidationError("the op runs on a CUDA device only (no CPU fallback)")
        if dev.index is None:
            dev = torch.device("cuda", torch.cuda.current_device())
        self.device = dev
        self.scale = float(scale) if scale is not None else 1.0 / math.sqrt(self.d)
        self.options = options or PlanOptions()
        self.num_tokens = int(self.cu_q[-1])
        self.num_prefix_keys = int(self.cu_prefix[-1])
        self.num_distinct_keys = int(self.cu_distinct[-1])
        if self.page_size:
            ps = self.page_size
            self.num_prefix_pages = int(sum(-(-int(n) // ps) for n in np.diff(self.cu_prefix)))
            self.num_distinct_pages = int(sum(-(-int(n) // ps) for n in np.diff(self.cu_distinct)))
        prob = self._problem(flags=0)
        handle = C.c_void_p()
        with torch.cuda.device(self.device):
            st = L.lib().psa_plan_create(C.byref(prob), C.byref(self.options.to_c()),
                                         C.byref(handle))
        if st != L.PSA_OK:
            _raise_native(st, "psa_plan_create")
        self._plan = handle
        nbytes = C.c_size_t()
        L.check(L.lib().psa_plan_workspace_bytes(self._plan, C.byref(nbytes)))
        self.workspace = torch.empty(max(int(nbytes.value), 256), dtype=torch.uint8,
                                     device=self.device)
        with torch.cuda.device(self.device):
            st = L.lib().psa_plan_upload(self._plan, _ptr(self.workspace), self.workspace.numel(),
                                         C.c_void_p(torch.cuda.current_stream(self.device).cuda_stream))
        if st != L.PSA_OK:
            _raise_native(st, "psa_plan_upload")

    def __del__(self):
        plan = getattr(self, "_plan", None)
        if plan is not None and plan.value:
            try:
                L.lib().psa_plan_destroy(plan)
            except Exception:
                pass
            self._plan = None

    # -- helpers -------------------------------------------------------------
    def _problem(self, flags: int) -> L.Problem:
        p = L.Problem()
        p.num_groups, p.num_requests = self.G, self.R
        p.num_q_heads, p.num_kv_heads = self.Hq, self.Hkv
        p.head_dim, p.value_dim = self.d, self.dv
        p.dtype = psa_dtype(self.dtype)
        p.flags = flags
        p.scale = self.scale
        i64p = C.POINTER(C.c_int64)
        p.cu_req = self.cu_req.ctypes.data_as(i64p)
        p.cu_q = self.cu_q.ctypes.data_as(i64p)
        p.cu_prefix = self.cu_prefix.ctypes.data_as(i64p)
        p.cu_distinct = self.cu_distinct.ctypes.data_as(i64p)
        p.page_size = self.page_size
        return p

    def plan_tables(self) -> dict:
        """The plan's int32 tables as NumPy arrays (bit-exact with oracle/plan.py)."""
        v = L.PlanView()
        L.check(L.lib().psa_plan_view_get(self._plan, C.byref(v)))
        items = np.ctypeslib.as_array(v.items, shape=(v.num_items * v.item_words,)).copy()
        units = np.ctypeslib.as_array(v.units, shape=(v.num_units * v.unit_words,)).copy()
        contribs = (np.ctypeslib.as_array(v.contribs, shape=(v.num_contribs,)).copy()
                    if v.num_contribs else np.zeros(0, np.int32))
        return dict(items=items.reshape(-1, v.item_words), units=units.reshape(-1, v.unit_words),
                    contribs=contribs, workspace_rows=int(v.workspace_rows),
                    num_tile_items=int(v.num_tile_items))

    @property
    def num_items(self) -> int:
        v = L.PlanView()
        L.check(L.lib().psa_plan_view_get(self._plan, C.byref(v)))
        return int(v.num_items)

    def _check(self, name, t: Optional[torch.Tensor], rows: int, heads: int, dim: int):
        if rows == 0:
            return
        if t is None:
            raise ValidationError(f"{name} is required")
        if t.device != self.device or t.dtype != self.dtype:
            raise ValidationError(f"{name} must be {self.dtype} on {self.device}")
        if tuple(t.shape) != (rows, heads, dim) or not t.is_contiguous():
            raise ValidationError(f"{name} must be a contiguous [{rows}, {heads}, {dim}] tensor, "
                                  f"got {tuple(t.shape)}")

    def _check_out(self, name, t, shape: tuple, dtype: torch.dtype):
        """Caller-supplied output buffers: psa_run cannot check sizes, so a wrong shape,
        dtype, layout or device here would be an out-of-bounds device write."""
        if not isinstance(t, torch.Tensor):
            raise ValidationError(f"{name} must be a torch tensor")
        if t.device != self.device or t.dtype != dtype or tuple(t.shape) != shape \
                or not t.is_contiguous():
            raise ValidationError(f"{name} must be a contiguous {dtype} tensor of shape "
                                  f"{list(shape)} on {self.device}, got {t.dtype} "
                                  f"{list(t.shape)} on {t.device}")

    def _check_pages(self, name, t, n):
        if n == 0:
            return
        if t is None or t.device != self.device or t.dtype != torch.int32 or t.dim() != 1 \
                or t.numel() != n or not t.is_contiguous():
            raise ValidationError(f"{name} must be a contiguous int32 [{n}] tensor on {self.device}")

    def __call__(self, q, k_prefix, v_prefix, k_distinct, v_distinct, out=None, lse=None,
                 partial: Optional[tuple] = None, stream: Optional[torch.cuda.Stream] = None,
                 prefix_pages: Optional[torch.Tensor] = None,
                 distinct_pages: Optional[torch.Tensor] = None, causal: bool = False):
        """Run the planned op. Returns ``out`` [T, Hq, dv] (or the partial tuple).

        Paged plans (``page_size`` > 0): ``k_prefix``/``v_prefix`` and
        ``k_distinct``/``v_distinct`` are page caches [rows, Hkv, d|dv] (rows a multiple
        of page_size; one cache may back both), ``prefix_pages`` lists the cache pages
        of every group's prefix in group order (ceil(P_g / page_size) each) and
        ``distinct_pages`` those of every request's distinct KV (int32 on the device).

        ``causal``: prefill-chunk tokens see only keys up to their own position
        (include/psa.h PSA_FLAG_CAUSAL — an extension; the reference attends every key)."""
        T = self.num_tokens
        self._check("q", q, T, self.Hq, self.d)
        if self.page_size:
            ps = self.page_size
            for name, t, dim, n in (("k_prefix", k_prefix, self.d, self.num_prefix_keys),
                                    ("v_prefix", v_prefix, self.dv, self.num_prefix_keys),
                                    ("k_distinct", k_distinct, self.d, self.num_distinct_keys),
                                    ("v_distinct", v_distinct, self.dv, self.num_distinct_keys)):
                if n and (t is None or t.dim() != 3 or t.shape[0] % ps or t.shape[1] != self.Hkv
                          or t.shape[2] != dim or t.dtype != self.dtype or t.device != self.device
                          or not t.is_contiguous()):
                    raise ValidationError(f"{name} must be a contiguous [pages * {ps}, {self.Hkv}, "
                                          f"{dim}] {self.dtype} page cache on {self.device}")
            self._check_pages("prefix_pages", prefix_pages, self.num_prefix_pages)
            self._check_pages("distinct_pages", distinct_pages, self.num_distinct_pages)
        else:
            self._check("k_prefix", k_prefix, self.num_prefix_keys, self.Hkv, self.d)
            self._check("v_prefix", v_prefix, self.num_prefix_keys, self.Hkv, self.dv)
            self._check("k_distinct", k_distinct, self.num_distinct_keys, self.Hkv, self.d)
            self._check("v_distinct", v_distinct, self.num_distinct_keys, self.Hkv, self.dv)
        flags = 0
        m_out = l_out = None
        acc = acc_dtype(self.dtype)
        if partial is not None:
            flags = L.FLAG_PARTIAL_OUT
            if not isinstance(partial, (tuple, list)) or len(partial) != 3:
                raise ValidationError("partial must be a tuple (o, m, l)")
            out, m_out, l_out = partial
            # the kernel writes unnormalised rows in the accumulate type
            self._check_out("partial o", out, (T, self.Hq, self.dv), acc)
            self._check_out("partial m", m_out, (T, self.Hq), acc)
            self._check_out("partial l", l_out, (T, self.Hq), acc)
        elif out is None:
            out = torch.empty((T, self.Hq, self.dv), dtype=self.dtype, device=self.device)
        else:
            self._check_out("out", out, (T, self.Hq, self.dv), self.dtype)
        if lse is not None:
            self._check_out("lse", lse, (T, self.Hq), torch.float32)
        if causal:
            flags |= L.FLAG_CAUSAL
        prob = self._problem(flags)
        prob.q, prob.k_prefix, prob.v_prefix = _ptr(q), _ptr(k_prefix), _ptr(v_prefix)
        prob.k_distinct, prob.v_distinct = _ptr(k_distinct), _ptr(v_distinct)
        prob.out, prob.lse = _ptr(out), _ptr(lse)
        prob.m_out, prob.l_out = _ptr(m_out), _ptr(l_out)
        if self.page_size:
            prob.prefix_pages, prob.distinct_pages = _ptr(prefix_pages), _ptr(distinct_pages)
            prob.prefix_cache_rows = int(k_prefix.shape[0]) if k_prefix is not None else 0
            prob.distinct_cache_rows = int(k_distinct.shape[0]) if k_distinct is not None else 0
            if v_prefix is not None and k_prefix is not None and v_prefix.shape[0] != k_prefix.shape[0]:
                raise ValidationError("k_prefix and v_prefix caches must have the same rows")
            if v_distinct is not None and k_distinct is not None and \
                    v_distinct.shape[0] != k_distinct.shape[0]:
                raise ValidationError("k_distinct and v_distinct caches must have the same rows")
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        with torch.cuda.device(self.device):
            st = L.lib().psa_run(C.byref(prob), self._plan, _ptr(self.workspace),
                                 self.workspace.numel(), C.c_void_p(s.cuda_stream))
        if st != L.PSA_OK:
            _raise_native(st, "psa_run")
        return partial if partial is not None else out

    def trace(self, *inputs) -> np.ndarray:
        """Run once with per-item timing on (diagnostics). Returns int64 [items, 4]:
        (cta | smid << 32 | warp << 48, kind, t_start_ns, t_end_ns), rows in queue order;
        rows num_items + b hold CTA b's kernel start/end (kind -1)."""
        n = self.num_items + 4096  # items, then one residency record per CTA
        buf = torch.zeros((n + 2048, 4), dtype=torch.int64, device=self.device)  # + tile/dec events
        L.check(L.lib().psa_debug_set_trace(_ptr(buf), n), "psa_debug_set_trace")
        try:
            self(*inputs)
            torch.cuda.synchronize(self.device)
        finally:
            L.lib().psa_debug_set_trace(None, 0)
        out = buf.cpu().numpy()
        self.last_tile_events = out[n:].reshape(-1)[:14 * 64].reshape(14, 64)
        self.last_dec_events = out[n:].reshape(-1)[16 * 64:33 * 64].reshape(17, 64)
        self.last_merge_tasks = out[n:].reshape(-1)[36 * 64:40 * 64].reshape(4, 64)
        self.last_dec_events2 = out[n:].reshape(-1)[40 * 64:43 * 64].reshape(3, 64)
        self.last_phase = out[self.num_items + 2048:self.num_items + 3072]
        self.last_dec_phase = out[self.num_items + 3072:self.num_items + 4096]
        ctas = out[self.num_items:n]
        return out[:self.num_items], ctas[ctas[:, 1] == -1]

    def device_error(self) -> int:
        """Error bits of the last run (synchronises the current stream)."""
        bits = C.c_int32()
        L.check(L.lib().psa_workspace_error(
            _ptr(self.workspace), C.c_void_p(torch.cuda.current_stream(self.device).cuda_stream),
            C.byref(bits)))
        return int(bits.value)


def plan_tables_host(cu_req, cu_q, cu_prefix, cu_distinct, num_q_heads, num_kv_heads,
                     head_dim, value_dim, dtype: torch.dtype, options: PlanOptions) -> dict:
    """Build a plan on the host only (options.num_sms > 0: no CUDA call) and return
    its int32 tables — used by the CPU bit-exactness tests of the planner."""
    if options.num_sms <= 0:
        raise ValidationError("plan_tables_host needs options.num_sms > 0")
    cu_req, cu_q, cu_prefix, cu_distinct = map(_i64, (cu_req, cu_q, cu_prefix, cu_distinct))
    p = L.Problem()
    p.num_groups, p.num_requests = len(cu_req) - 1, len(cu_q) - 1
    p.num_q_heads, p.num_kv_heads, p.head_dim, p.value_dim = num_q_heads, num_kv_heads, head_dim, value_dim
    p.dtype = psa_dtype(dtype)
    p.scale = 1.0
    i64p = C.POINTER(C.c_int64)
    p.cu_req, p.cu_q = cu_req.ctypes.data_as(i64p), cu_q.ctypes.data_as(i64p)
    p.cu_prefix, p.cu_distinct = cu_prefix.ctypes.data_as(i64p), cu_distinct.ctypes.data_as(i64p)
    handle = C.c_void_p()
    st = L.lib().psa_plan_create(C.byref(p), C.byref(options.to_c()), C.byref(handle))
    if st != L.PSA_OK:
        _raise_native(st, "psa_plan_create")
    try:
        v = L.PlanView()
        L.check(L.lib().psa_plan_view_get(handle, C.byref(v)))
        items = np.ctypeslib.as_array(v.items, shape=(v.num_items * v.item_words,)).copy()
        units = np.ctypeslib.as_array(v.units, shape=(v.num_units * v.unit_words,)).copy()
        contribs = (np.ctypeslib.as_array(v.contribs, shape=(v.num_contribs,)).copy()
                    if v.num_contribs else np.zeros(0, np.int32))
        nbytes = C.c_size_t()
        L.check(L.lib().psa_plan_workspace_bytes(handle, C.byref(nbytes)))
        return dict(items=items.reshape(-1, v.item_words), units=units.reshape(-1, v.unit_words),
                    contribs=contribs, workspace_rows=int(v.workspace_rows),
                    num_tile_items=int(v.num_tile_items), workspace_bytes=int(nbytes.value))
    finally:
        L.lib().psa_plan_destroy(handle)


def prefix_shared_attention_packed(q, k_prefix, v_prefix, k_distinct, v_distinct, cu_req, cu_q,
                                   cu_prefix, cu_distinct, num_kv_heads: int,
                                   scale: Optional[float] = None, lse=None,
                                   options: Optional[PlanOptions] = None):
    """One-shot packed call: plan + one persistent launch. Returns O [T, Hq, dv]."""
    op = PrefixSharedAttention(cu_req, cu_q, cu_prefix, cu_distinct, q.shape[1], num_kv_heads,
                               q.shape[2], v_prefix.shape[2] if v_prefix is not None and
                               v_prefix.numel() else v_distinct.shape[2], q.dtype, q.device,
                               scale, options)
    return op(q, k_prefix, v_prefix, k_distinct, v_distinct, lse=lse)


def count_nonfinite(t: torch.Tensor, counter: torch.Tensor) -> None:
    """Accumulate the number of non-finite entries of ``t`` into device int32 ``counter``."""
    t = t.contiguous()
    with torch.cuda.device(t.device):
        st = L.lib().psa_count_nonfinite(_ptr(t), t.numel(), psa_dtype(t.dtype), _ptr(counter),
                                         C.c_void_p(torch.cuda.current_stream(t.device).cuda_stream))
    if st != L.PSA_OK:
        _raise_native(st, "psa_count_nonfinite")


def shard_groups(group_cost, world_size: int) -> np.ndarray:
    """Greedy LPT group -> rank owner table (psa_shard_groups)."""
    cost = _i64(group_cost)
    owner = np.zeros(len(cost), dtype=np.int32)
    L.check(L.lib().psa_shard_groups(len(cost), cost.ctypes.data_as(C.POINTER(C.c_int64)),
                                     int(world_size), owner.ctypes.data_as(C.POINTER(C.c_int32))),
            "psa_shard_groups")
    return owner


def group_costs(cu_req, cu_q, cu_prefix, cu_distinct, num_q_heads, num_kv_heads, head_dim,
                value_dim, dtype: torch.dtype) -> np.ndarray:
    cu_req, cu_q, cu_prefix, cu_distinct = map(_i64, (cu_req, cu_q, cu_prefix, cu_distinct))
    p = L.Problem()
    p.num_groups, p.num_requests = len(cu_req) - 1, len(cu_q) - 1
    p.num_q_heads, p.num_kv_heads, p.head_dim, p.value_dim = num_q_heads, num_kv_heads, head_dim, value_dim
    p.dtype = psa_dtype(dtype)
    p.scale = 1.0
    i64p = C.POINTER(C.c_int64)
    p.cu_req, p.cu_q = cu_req.ctypes.data_as(i64p), cu_q.ctypes.data_as(i64p)
    p.cu_prefix, p.cu_distinct = cu_prefix.ctypes.data_as(i64p), cu_distinct.ctypes.data_as(i64p)
    cost = np.zeros(p.num_groups, dtype=np.int64)
    st = L.lib().psa_group_costs(C.byref(p), cost.ctypes.data_as(i64p))
    if st != L.PSA_OK:
        _raise_native(st, "psa_group_costs")
    return cost
