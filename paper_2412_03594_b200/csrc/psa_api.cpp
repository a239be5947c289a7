// psa_api.cpp — the extern "C" boundary (include/psa.h): validation, plan
// objects, workspace layout and launch. No torch, no exceptions across the ABI.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "../../include/psa.h"
#include "psa_kernel.h"
#include "psa_plan.h"

struct psa_plan {
  psa::Plan plan;
  psa::PlanInput dims;  // pointers inside are NOT kept valid
  int32_t num_sms = 0, ctas_per_sm = 0;
  bool use_tiles = false;
  bool use_vec_fast = false;
  bool use_dec = false;
  bool use_v2 = false;
  std::vector<int64_t> group_tok0, group_pbase, req_dbase;
  std::vector<int32_t> tok_lim;  // causal key limits per token (PSA_FLAG_CAUSAL)
  bool causal_ok = true;         // every request satisfies n_q <= D (D > 0) or n_q <= P
  int32_t page_size = 0;
  int64_t prefix_pages = 0, distinct_pages = 0;  // paged: page-table lengths
  int64_t num_tokens = 0, prefix_keys = 0, distinct_keys = 0;
  // workspace layout (byte offsets)
  size_t off_ctrl = 0, off_cnt = 0, off_items = 0, off_units = 0, off_contribs = 0;
  size_t off_tok0 = 0, off_pbase = 0, off_dbase = 0, off_lim = 0, off_wso = 0, off_wsml = 0, total = 0;
};

namespace {

thread_local std::string g_error;
thread_local int64_t* g_trace = nullptr;
thread_local int64_t g_trace_cap = 0;

psa_status fail(psa_status s, const std::string& msg) {
  g_error = msg;
  return s;
}

psa_status cuda_fail(int e, const char* where) {
  return fail(PSA_CUDA_ERROR, std::string(where) + ": " +
                                  cudaGetErrorString(static_cast<cudaError_t>(e)));
}

std::mutex g_sm_mutex;
int32_t g_sms[64] = {0};

psa_status current_sms(int32_t* out) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  std::lock_guard<std::mutex> lock(g_sm_mutex);
  if (dev < 64 && g_sms[dev] > 0) {
    *out = g_sms[dev];
    return PSA_OK;
  }
  int n = 0;
  e = cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceGetAttribute");
  int major = 0;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  if (major != 10) return fail(PSA_UNSUPPORTED, "libpsa is built for sm_100a (B200) only");
  if (dev < 64) g_sms[dev] = n;
  *out = n;
  return PSA_OK;
}

psa::PlanInput dims_of(const psa_problem* p) {
  psa::PlanInput in;
  in.G = p->num_groups; in.R = p->num_requests; in.Hq = p->num_q_heads;
  in.Hkv = p->num_kv_heads; in.d = p->head_dim; in.dv = p->value_dim; in.dtype = p->dtype;
  in.cu_req = p->cu_req; in.cu_q = p->cu_q; in.cu_prefix = p->cu_prefix;
  in.cu_distinct = p->cu_distinct;
  return in;
}

psa_status check_problem_header(const psa_problem* p) {
  if (!p) return fail(PSA_INVALID_ARGUMENT, "problem is NULL");
  if (psa::dtype_bytes(p->dtype) == 0) return fail(PSA_UNSUPPORTED, "unsupported dtype");
  if (p->head_dim > 256 || p->value_dim > 256)
    return fail(PSA_UNSUPPORTED, "unsupported head dim (max 256)");
  if (!(std::isfinite(p->scale)) || p->scale < 0)
    return fail(PSA_INVALID_ARGUMENT, "scale must be non-negative and finite");
  return PSA_OK;
}

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

void layout(psa_plan* pl) {
  const size_t acc = pl->dims.dtype == PSA_DTYPE_F64 ? 8 : 4;
  size_t o = 0;
  auto take = [&](size_t bytes) { size_t at = o; o = align_up(o + bytes, 256); return at; };
  pl->off_ctrl = take(sizeof(psa::Ctrl));
  pl->off_cnt = take(sizeof(int32_t) * pl->plan.num_units);
  pl->off_items = take(sizeof(int32_t) * pl->plan.items.size());
  pl->off_units = take(sizeof(int32_t) * pl->plan.units.size());
  pl->off_contribs = take(sizeof(int32_t) * pl->plan.contribs.size());
  pl->off_tok0 = take(sizeof(int64_t) * pl->group_tok0.size());
  pl->off_pbase = take(sizeof(int64_t) * pl->group_pbase.size());
  pl->off_dbase = take(sizeof(int64_t) * pl->req_dbase.size());
  pl->off_lim = take(sizeof(int32_t) * pl->tok_lim.size());
  pl->off_wso = take(acc * size_t(pl->plan.workspace_rows) * pl->dims.dv);
  pl->off_wsml = take(acc * size_t(pl->plan.workspace_rows) * 2);
  pl->total = o;
}

}  // namespace

extern "C" {

const char* psa_last_error(void) { return g_error.c_str(); }
int32_t psa_abi_version(void) { return PSA_ABI_VERSION; }

psa_status psa_device_sms(int32_t* num_sms) {
  if (!num_sms) return fail(PSA_INVALID_ARGUMENT, "num_sms is NULL");
  return current_sms(num_sms);
}

psa_status psa_plan_create(const psa_problem* prob, const psa_plan_opts* opts, psa_plan** out) {
  if (!out) return fail(PSA_INVALID_ARGUMENT, "plan out-pointer is NULL");
  *out = nullptr;
  psa_status st = check_problem_header(prob);
  if (st != PSA_OK) return st;
  psa::PlanOptions o;
  if (opts) {
    if (opts->num_sms > 0) o.num_sms = opts->num_sms;
    if (opts->ctas_per_sm > 0) o.ctas_per_sm = opts->ctas_per_sm;
    if (opts->tile_min_rows > 0) o.tile_min_rows = opts->tile_min_rows;
    o.disable_tiles = opts->disable_tiles;
    if (opts->min_chunk_keys > 0) o.min_chunk_keys = opts->min_chunk_keys;
    if (opts->max_chunk_keys > 0) o.max_chunk_keys = opts->max_chunk_keys;
    if (opts->target_waves > 0) o.target_waves = opts->target_waves;
  }
  if (!opts || opts->num_sms <= 0) {
    st = current_sms(&o.num_sms);
    if (st != PSA_OK) return st;
  }
  const bool v2 = psa::v2_supported(prob->dtype, prob->head_dim, prob->value_dim) &&
                  !(opts && (opts->disable_vec_fast != 0 || opts->kernel_variant != 0));
  if (v2) {
    o.ctas_per_sm = 1;
    o.tile_pair = 1;
    o.fuse_own = 1;
    // ping-pong tiles beat the decode pipeline from 16 stacked rows on (c4: prefixes
    // of small groups are read once instead of once per 8-row VEC item)
    if (!opts || opts->tile_min_rows <= 0) o.tile_min_rows = 16;
  }
  const int32_t ps = prob->page_size;
  if (ps != 0) {
    if (ps != 16 && ps != 32 && ps != 64)
      return fail(PSA_INVALID_ARGUMENT, "page_size must be 0 (packed), 16, 32 or 64");
    if (!v2)
      return fail(PSA_UNSUPPORTED,
                  "paged KV needs the v2 kernel (bf16/f16, head_dim == value_dim == 128)");
  }
  psa_plan* pl = new (std::nothrow) psa_plan();
  if (!pl) return fail(PSA_INVALID_ARGUMENT, "out of host memory");
  pl->page_size = ps;
  pl->dims = dims_of(prob);
  std::string err = psa::build_plan(pl->dims, o, &pl->plan);
  if (!err.empty()) {
    delete pl;
    return fail(PSA_INVALID_ARGUMENT, err);
  }
  pl->num_sms = o.num_sms;
  pl->ctas_per_sm = o.ctas_per_sm;
  pl->use_tiles = pl->plan.num_tile_items > 0;
  pl->use_vec_fast = psa::vec_fast_supported(prob->dtype, prob->head_dim, prob->value_dim) &&
                     !(opts && opts->disable_vec_fast == 1);
  pl->use_dec = psa::dec_supported(prob->dtype, prob->head_dim, prob->value_dim) &&
                !(opts && opts->disable_vec_fast == 2);
  pl->use_v2 = v2;
  const auto& in = pl->dims;
  pl->group_tok0.resize(in.G);
  pl->group_pbase.resize(in.G);
  pl->req_dbase.resize(in.R);
  // segment bases: packed key offsets, or (paged) offsets into the page tables
  int64_t pages = 0;
  for (int32_t g = 0; g < in.G; ++g) {
    pl->group_tok0[g] = in.cu_q[in.cu_req[g]];
    const int64_t P = in.cu_prefix[g + 1] - in.cu_prefix[g];
    pl->group_pbase[g] = ps ? pages : in.cu_prefix[g];
    if (ps) pages += (P + ps - 1) / ps;
  }
  pl->prefix_pages = pages;
  pages = 0;
  for (int32_t r = 0; r < in.R; ++r) {
    const int64_t D = in.cu_distinct[r + 1] - in.cu_distinct[r];
    pl->req_dbase[r] = ps ? pages : in.cu_distinct[r];
    if (ps) pages += (D + ps - 1) / ps;
  }
  pl->distinct_pages = pages;
  // causal limits (include/psa.h PSA_FLAG_CAUSAL): last visible prefix / distinct key
  pl->tok_lim.resize(size_t(in.cu_q[in.R]) * 2);
  pl->causal_ok = true;
  for (int32_t g = 0; g < in.G; ++g) {
    const int64_t P = in.cu_prefix[g + 1] - in.cu_prefix[g];
    for (int64_t r = in.cu_req[g]; r < in.cu_req[g + 1]; ++r) {
      const int64_t nq = in.cu_q[r + 1] - in.cu_q[r];
      const int64_t D = in.cu_distinct[r + 1] - in.cu_distinct[r];
      // the limits below can only express chunks that end the keys they attend to
      if (nq > (D > 0 ? D : P)) pl->causal_ok = false;
      for (int64_t j = 0; j < nq; ++j) {
        const int64_t t = in.cu_q[r] + j;
        const int64_t lp = D > 0 ? P - 1 : P - nq + j;
        const int64_t ld = D - nq + j;
        pl->tok_lim[size_t(t) * 2] = int32_t(std::max<int64_t>(lp, -1));
        pl->tok_lim[size_t(t) * 2 + 1] = int32_t(std::max<int64_t>(ld, -1));
      }
    }
  }
  pl->num_tokens = in.cu_q[in.R];
  pl->prefix_keys = in.cu_prefix[in.G];
  pl->distinct_keys = in.cu_distinct[in.R];
  pl->dims.cu_req = pl->dims.cu_q = pl->dims.cu_prefix = pl->dims.cu_distinct = nullptr;
  layout(pl);
  *out = pl;
  return PSA_OK;
}

psa_status psa_plan_view_get(const psa_plan* pl, psa_plan_view* v) {
  if (!pl || !v) return fail(PSA_INVALID_ARGUMENT, "NULL argument");
  v->num_items = pl->plan.num_items;
  v->num_units = pl->plan.num_units;
  v->num_contribs = int32_t(pl->plan.contribs.size());
  v->item_words = psa::kItemWords;
  v->unit_words = psa::kUnitWords;
  v->num_tile_items = pl->plan.num_tile_items;
  v->workspace_rows = pl->plan.workspace_rows;
  v->items = pl->plan.items.data();
  v->units = pl->plan.units.data();
  v->contribs = pl->plan.contribs.data();
  return PSA_OK;
}

psa_status psa_plan_workspace_bytes(const psa_plan* pl, size_t* bytes) {
  if (!pl || !bytes) return fail(PSA_INVALID_ARGUMENT, "NULL argument");
  *bytes = pl->total;
  return PSA_OK;
}

psa_status psa_plan_upload(const psa_plan* pl, void* ws, size_t ws_bytes, void* stream) {
  if (!pl || !ws) return fail(PSA_INVALID_ARGUMENT, "NULL argument");
  if (ws_bytes < pl->total) return fail(PSA_INVALID_ARGUMENT, "workspace too small");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  char* base = static_cast<char*>(ws);
  cudaError_t e = cudaMemsetAsync(base, 0, pl->off_items, s);  // ctrl + unit counters
  if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync");
  struct Blob { size_t off; const void* src; size_t n; } blobs[] = {
      {pl->off_items, pl->plan.items.data(), pl->plan.items.size() * 4},
      {pl->off_units, pl->plan.units.data(), pl->plan.units.size() * 4},
      {pl->off_contribs, pl->plan.contribs.data(), pl->plan.contribs.size() * 4},
      {pl->off_tok0, pl->group_tok0.data(), pl->group_tok0.size() * 8},
      {pl->off_pbase, pl->group_pbase.data(), pl->group_pbase.size() * 8},
      {pl->off_dbase, pl->req_dbase.data(), pl->req_dbase.size() * 8},
      {pl->off_lim, pl->tok_lim.data(), pl->tok_lim.size() * 4},
  };
  for (const auto& b : blobs) {
    if (b.n == 0) continue;
    e = cudaMemcpyAsync(base + b.off, b.src, b.n, cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpyAsync");
  }
  return PSA_OK;
}

void psa_plan_destroy(psa_plan* pl) { delete pl; }

psa_status psa_run(const psa_problem* prob, const psa_plan* pl, void* ws, size_t ws_bytes,
                   void* stream) {
  psa_status st = check_problem_header(prob);
  if (st != PSA_OK) return st;
  if (!pl || !ws) return fail(PSA_INVALID_ARGUMENT, "NULL plan or workspace");
  if (ws_bytes < pl->total) return fail(PSA_INVALID_ARGUMENT, "workspace too small");
  const auto& in = pl->dims;
  if (prob->num_groups != in.G || prob->num_requests != in.R || prob->num_q_heads != in.Hq ||
      prob->num_kv_heads != in.Hkv || prob->head_dim != in.d || prob->value_dim != in.dv ||
      prob->dtype != in.dtype)
    return fail(PSA_INVALID_ARGUMENT, "problem does not match the plan");
  if (!prob->q || !prob->out) return fail(PSA_INVALID_ARGUMENT, "q/out must not be NULL");
  if ((prob->flags & PSA_FLAG_PARTIAL_OUT) && (!prob->m_out || !prob->l_out))
    return fail(PSA_INVALID_ARGUMENT, "partial output needs m_out and l_out");
  if (prob->page_size != pl->page_size)
    return fail(PSA_INVALID_ARGUMENT, "page_size does not match the plan");
  int64_t prefix_rows = pl->prefix_keys, distinct_rows = pl->distinct_keys;
  if (pl->page_size) {
    if ((pl->prefix_pages && !prob->prefix_pages) || (pl->distinct_pages && !prob->distinct_pages))
      return fail(PSA_INVALID_ARGUMENT, "paged KV needs prefix_pages / distinct_pages");
    prefix_rows = prob->prefix_cache_rows;
    distinct_rows = prob->distinct_cache_rows;
    if (prefix_rows < 0 || distinct_rows < 0 || prefix_rows % pl->page_size ||
        distinct_rows % pl->page_size || prefix_rows >= (int64_t(1) << 31) ||
        distinct_rows >= (int64_t(1) << 31))
      return fail(PSA_INVALID_ARGUMENT,
                  "cache rows must be non-negative multiples of page_size below 2^31");
    if ((pl->prefix_pages && prefix_rows == 0) || (pl->distinct_pages && distinct_rows == 0))
      return fail(PSA_INVALID_ARGUMENT, "empty page cache for a non-empty segment");
  }
  char* base = static_cast<char*>(ws);
  psa::KParams k{};
  k.page_size = pl->page_size;
  k.prefix_pages = prob->prefix_pages;
  k.distinct_pages = prob->distinct_pages;
  k.prefix_cache_rows = int32_t(prefix_rows);
  k.distinct_cache_rows = int32_t(distinct_rows);
  k.q = prob->q; k.kp = prob->k_prefix; k.vp = prob->v_prefix;
  k.kd = prob->k_distinct; k.vd = prob->v_distinct;
  k.out = prob->out; k.lse = prob->lse; k.m_out = prob->m_out; k.l_out = prob->l_out;
  k.items = reinterpret_cast<const int32_t*>(base + pl->off_items);
  k.units = reinterpret_cast<const int32_t*>(base + pl->off_units);
  k.contribs = reinterpret_cast<const int32_t*>(base + pl->off_contribs);
  k.group_tok0 = reinterpret_cast<const int64_t*>(base + pl->off_tok0);
  k.group_pbase = reinterpret_cast<const int64_t*>(base + pl->off_pbase);
  k.req_dbase = reinterpret_cast<const int64_t*>(base + pl->off_dbase);
  k.tok_lim = reinterpret_cast<const int32_t*>(base + pl->off_lim);
  if ((prob->flags & PSA_FLAG_CAUSAL) && !pl->use_v2)
    return fail(PSA_UNSUPPORTED,
                "causal masking needs the v2 kernel (bf16/f16, head_dim == value_dim == 128)");
  if ((prob->flags & PSA_FLAG_CAUSAL) && !pl->causal_ok)
    return fail(PSA_INVALID_ARGUMENT,
                "causal masking needs n_q <= D (requests with distinct KV) or n_q <= P "
                "(prefix-only chunks): the query tokens must be the last keys they attend to");
  k.ws_o = base + pl->off_wso;
  k.ws_ml = base + pl->off_wsml;
  k.unit_cnt = reinterpret_cast<int32_t*>(base + pl->off_cnt);
  k.ctrl = reinterpret_cast<psa::Ctrl*>(base + pl->off_ctrl);
  k.num_items = pl->plan.num_items;
  k.n_tile_items = pl->plan.num_tile_items;
  {
    // Every CTA starts on the tile queue: memory-bound tiles would otherwise be
    // starved of memory-level parallelism by the deep per-warp VEC rings, and
    // CTAs without a tile item move on to the VEC queue at once.
    const int grid = pl->num_sms * pl->ctas_per_sm;
    int nt = pl->plan.num_tile_items > 0 ? grid : 0;
    if (pl->use_v2 && pl->plan.num_tile_items > 0) nt = pl->plan.tile_ctas;
    if (const char* e = std::getenv("PSA_TILE_CTAS"))  // diagnostics: override the split
      nt = std::max(0, std::min(grid, std::atoi(e)));
    k.n_tile_ctas = nt;
  }
  {  // diagnostics (PSA_DEBUG bit 1024): full forward boxes for partial last blocks
    const char* dbg = std::getenv("PSA_DEBUG");
    k.tail_shift = (dbg && (std::atoi(dbg) & 1024)) ? 0 : 1;
  }
  k.Hq = in.Hq; k.Hkv = in.Hkv; k.gqa = in.Hq / in.Hkv; k.d = in.d; k.dv = in.dv;
  k.max_vec_rows = pl->plan.max_vec_rows;
  k.dec_help = pl->plan.vec_fan_in > 2 ? 1 : 0;  // two: the in-register pair merge covers it
#ifdef PSA_NO_DEC_HELP
  k.dec_help = 0;  // diagnostics build: decode merge queues drained by their merge warps only
#endif
  k.gqa_shift = -1;
  for (int sh = 0; sh < 31; ++sh)
    if ((1 << sh) == k.gqa) k.gqa_shift = sh;
  k.flags = prob->flags;
  // scale == 0 (uniform weights; allowed by naive_attention, attention.py:135-136): the
  // softmaxes mask a key by setting its raw score to -inf before scaling, and -inf * 0
  // is NaN. A scale of 1e-30 gives every finite logit |s| * 1e-30 < 2^-60 — exp of it
  // is exactly 1 in fp32 and fp64 — while masked keys stay at -inf.
  k.scale = prob->scale > 0 ? prob->scale : 1e-30;
  k.trace = g_trace;
  k.trace_cap = int32_t(g_trace_cap);
  k.use_tiles = pl->use_tiles ? 1 : 0;
  k.use_v2 = pl->use_v2 ? 1 : 0;
  if (pl->use_v2) {  // the v2 kernel handles PSA_FLAG_PARTIAL_OUT on both paths
    k.use_vec_fast = 0;
    k.use_dec = pl->plan.num_items > pl->plan.num_tile_items ? 1 : 0;
  } else {
    k.use_vec_fast = (pl->use_vec_fast && !(prob->flags & PSA_FLAG_PARTIAL_OUT)) ? 1 : 0;
    k.use_dec = (k.use_vec_fast && pl->use_dec) ? 1 : 0;
  }
  if (k.use_tiles || k.use_vec_fast || k.use_dec || k.use_v2) {
    const uintptr_t align = reinterpret_cast<uintptr_t>(prob->q) |
                            reinterpret_cast<uintptr_t>(prob->k_prefix) |
                            reinterpret_cast<uintptr_t>(prob->v_prefix) |
                            reinterpret_cast<uintptr_t>(prob->k_distinct) |
                            reinterpret_cast<uintptr_t>(prob->v_distinct);
    if (align & 15) return fail(PSA_INVALID_ARGUMENT, "TMA paths need 16-byte aligned buffers");
    int te = psa::encode_tile_maps(k, in.dtype, pl->num_tokens, prefix_rows, distinct_rows);
    if (te != 0) return cuda_fail(te, "cuTensorMapEncodeTiled");
  }
  int e = psa::launch_psa(k, in.dtype, pl->num_sms, pl->ctas_per_sm, pl->use_tiles, stream);
  if (e != 0) return cuda_fail(e, "psa kernel launch");
  return PSA_OK;
}

psa_status psa_workspace_bytes(const psa_problem* prob, const psa_plan_opts* opts, size_t* bytes) {
  if (!bytes) return fail(PSA_INVALID_ARGUMENT, "bytes is NULL");
  psa_plan* pl = nullptr;
  psa_status st = psa_plan_create(prob, opts, &pl);
  if (st != PSA_OK) return st;
  *bytes = pl->total;
  psa_plan_destroy(pl);
  return PSA_OK;
}

psa_status psa_prefix_shared_attention(const psa_problem* prob, const psa_plan_opts* opts,
                                       void* ws, size_t ws_bytes, void* stream) {
  psa_plan* pl = nullptr;
  psa_status st = psa_plan_create(prob, opts, &pl);
  if (st != PSA_OK) return st;
  st = psa_plan_upload(pl, ws, ws_bytes, stream);
  if (st == PSA_OK) st = psa_run(prob, pl, ws, ws_bytes, stream);
  // pageable-source cudaMemcpyAsync has been staged when it returns: safe to free
  psa_plan_destroy(pl);
  return st;
}

psa_status psa_workspace_error(const void* ws, void* stream, int32_t* bits) {
  if (!ws || !bits) return fail(PSA_INVALID_ARGUMENT, "NULL argument");
  psa::Ctrl c;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e = cudaMemcpyAsync(&c, ws, sizeof(c), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_fail(e, "psa_workspace_error");
  *bits = c.error;
  return PSA_OK;
}

psa_status psa_merge(int64_t rows, int32_t dv, int32_t dtype, const void* oa, const void* ma,
                     const void* la, const void* ob, const void* mb, const void* lb, void* o,
                     void* m, void* l, void* stream) {
  if (dtype != PSA_DTYPE_F32 && dtype != PSA_DTYPE_F64)
    return fail(PSA_UNSUPPORTED, "merge supports f32/f64 partials");
  if (rows < 0 || dv < 1 || dv > 1024) return fail(PSA_INVALID_ARGUMENT, "bad merge shape");
  int e = psa::launch_merge(rows, dv, dtype, oa, ma, la, ob, mb, lb, o, m, l, stream);
  return e ? cuda_fail(e, "psa_merge") : PSA_OK;
}

psa_status psa_finalize(int64_t rows, int32_t dv, int32_t dtype, const void* o, const void* l,
                        void* out, int32_t* bad, void* stream) {
  if (dtype != PSA_DTYPE_F32 && dtype != PSA_DTYPE_F64)
    return fail(PSA_UNSUPPORTED, "finalize supports f32/f64 partials");
  if (rows < 0 || dv < 1 || !bad) return fail(PSA_INVALID_ARGUMENT, "bad finalize arguments");
  int e = psa::launch_finalize(rows, dv, dtype, o, l, out, bad, stream);
  return e ? cuda_fail(e, "psa_finalize") : PSA_OK;
}

psa_status psa_count_nonfinite(const void* data, int64_t n, int32_t dtype, int32_t* count,
                               void* stream) {
  if (psa::dtype_bytes(dtype) == 0) return fail(PSA_UNSUPPORTED, "unsupported dtype");
  if (n < 0 || !count || (n > 0 && !data)) return fail(PSA_INVALID_ARGUMENT, "bad arguments");
  int e = psa::launch_count_nonfinite(data, n, dtype, count, stream);
  return e ? cuda_fail(e, "psa_count_nonfinite") : PSA_OK;
}

psa_status psa_debug_set_trace(void* buf, int64_t capacity_items) {
  if (capacity_items < 0 || (capacity_items > 0 && !buf))
    return fail(PSA_INVALID_ARGUMENT, "bad trace buffer");
  g_trace = static_cast<int64_t*>(buf);
  g_trace_cap = capacity_items > INT32_MAX ? INT32_MAX : capacity_items;
  return PSA_OK;
}

psa_status psa_shard_groups(int32_t G, const int64_t* cost, int32_t world, int32_t* owner) {
  if (G < 0 || world < 1 || (G > 0 && (!cost || !owner)))
    return fail(PSA_INVALID_ARGUMENT, "bad shard arguments");
  psa::shard_groups(G, cost, world, owner);
  return PSA_OK;
}

psa_status psa_group_costs(const psa_problem* prob, int64_t* cost) {
  psa_status st = check_problem_header(prob);
  if (st != PSA_OK) return st;
  if (!cost) return fail(PSA_INVALID_ARGUMENT, "cost is NULL");
  psa::PlanInput in = dims_of(prob);
  std::string err = psa::validate_offsets(in);
  if (!err.empty()) return fail(PSA_INVALID_ARGUMENT, err);
  psa::group_costs(in, cost);
  return PSA_OK;
}

}  // extern "C"
