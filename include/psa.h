/*
 * psa.h — C ABI of the B200-native prefix-shared attention op (libpsa.so).
 *
 * Drop-in boundary for the reference entry point
 *   prefixbatch.attention.prefix_shared_attention(queries, kv, scale)
 *   (/root/reference/pkg/src/prefixbatch/attention.py:156-201)
 * and its building blocks partial_attention / merge / finalize
 *   (attention.py:78-98, :101-119, :122-126).
 * The reference has no FFI (pure NumPy); every entry point below is what a
 * ctypes/cffi binding of that module would bind — see INTEGRATION.md.
 *
 * Conventions
 *  - extern "C", plain pointers and sizes only; no C++ or torch types.
 *  - Every function returns psa_status; on failure psa_last_error() returns a
 *    thread-local message. No exception crosses the ABI.
 *  - The caller owns every buffer (inputs, outputs, workspace). The library
 *    never allocates device memory; it allocates host memory only inside
 *    psa_plan objects.
 *  - Device work is stream-ordered on the caller's stream (a cudaStream_t
 *    passed as void*; NULL = legacy default stream).
 *  - Stateless and re-entrant; the only globals are cached device attributes
 *    and the cuTensorMapEncodeTiled entry point, initialised once.
 *
 * Packed layout (all row-major, contiguous):
 *   q           [T, Hq, d]             T = total query tokens of the batch
 *   k_prefix    [sum_g P_g, Hkv, d]    v_prefix   [sum_g P_g, Hkv, dv]
 *   k_distinct  [sum_r D_r, Hkv, d]    v_distinct [sum_r D_r, Hkv, dv]
 *   out         [T, Hq, dv]            lse (optional, fp32) [T, Hq]
 *   Requests of group g are cu_req[g] .. cu_req[g+1]-1; request r owns tokens
 *   cu_q[r] .. cu_q[r+1]-1 (tokens of one group are contiguous), prefix keys
 *   cu_prefix[g] .. cu_prefix[g+1]-1 and distinct keys cu_distinct[r] ..
 *   cu_distinct[r+1]-1. A zero-length segment is an absent segment.
 * Multi-head mapping: query head j attends kv head j / gqa,
 * gqa = Hq / Hkv. For kv head h the rows of request r are its tokens x the
 * gqa heads h*gqa .. h*gqa+gqa-1, token-major — exactly the reference called
 * once per (group, kv head) on those stacked rows.
 */
#ifndef PSA_H_
#define PSA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PSA_ABI_VERSION 3

typedef enum psa_status {
  PSA_OK = 0,
  PSA_INVALID_ARGUMENT = 1, /* shim maps to ValidationError (errors.py:18-19) */
  PSA_UNSUPPORTED = 2,      /* shape/dtype outside the kernel set; never a CPU fallback */
  PSA_CUDA_ERROR = 3        /* shim maps to RuntimeError */
} psa_status;

typedef enum psa_dtype {
  PSA_DTYPE_F32 = 0,  /* CUDA-core FFMA, fp32 accumulate (not TF32) */
  PSA_DTYPE_BF16 = 1, /* tcgen05 tiles + CUDA-core decode, fp32 accumulate */
  PSA_DTYPE_F16 = 2,  /* as bf16 */
  PSA_DTYPE_F64 = 3   /* CUDA-core DFMA: the strict float64 drop-in mode */
} psa_dtype;

/* psa_problem.flags */
#define PSA_FLAG_PARTIAL_OUT 1u /* write unnormalised (o, m, l) instead of out=o/l */
/* Causal prefill (extension: the reference has no mask, attention.py:12-13; SURVEY.md
 * §8(f) row 4). Query token j (0-based) of request r with n_q tokens attends distinct
 * keys 0 .. D_r - n_q + j (the chunk is the tail of its own KV) and every prefix key;
 * a request without distinct KV (a prefix chunk) attends prefix keys 0 .. P_g - n_q + j.
 * Decode tokens (n_q = 1) are unaffected. v2 kernel only (else PSA_UNSUPPORTED). */
#define PSA_FLAG_CAUSAL 2u

typedef struct psa_problem {
  int32_t num_groups;   /* G >= 1 */
  int32_t num_requests; /* R >= 1 */
  int32_t num_q_heads;  /* Hq, multiple of Hkv */
  int32_t num_kv_heads; /* Hkv >= 1 */
  int32_t head_dim;     /* d */
  int32_t value_dim;    /* dv */
  int32_t dtype;        /* psa_dtype of q/k/v/out */
  uint32_t flags;       /* PSA_FLAG_* */
  double scale;         /* softmax scale; > 0 unless every segment is empty */
  /* Host offset tables (int64), read by the planner. */
  const int64_t* cu_req;      /* [G+1] */
  const int64_t* cu_q;        /* [R+1] */
  const int64_t* cu_prefix;   /* [G+1] */
  const int64_t* cu_distinct; /* [R+1] */
  /* Device buffers. */
  const void* q;
  const void* k_prefix;
  const void* v_prefix;
  const void* k_distinct;
  const void* v_distinct;
  void* out;   /* [T,Hq,dv] in dtype; with PARTIAL_OUT: o in the accumulate type
                  (f32, or f64 for PSA_DTYPE_F64) */
  float* lse;  /* optional [T,Hq] natural-log LSE = m + log(l) (NULL = skip) */
  void* m_out; /* PARTIAL_OUT only: [T,Hq] running max logit (accumulate type) */
  void* l_out; /* PARTIAL_OUT only: [T,Hq] shifted exp-sum (accumulate type) */
  /* Paged KV cache (vLLM-style blocks; the reference's KVAllocator, scheduler.py:140-187,
   * block_size 16 at scheduler.py:45). page_size == 0: the packed layout above.
   * page_size in {16, 32, 64} (bf16/f16, d == dv == 128 only; else PSA_UNSUPPORTED):
   * k_prefix/v_prefix and k_distinct/v_distinct are page caches
   * [*_cache_rows, Hkv, d|dv] (the same cache may back both), and logical key j of
   * group g's prefix lives at cache row
   *   prefix_pages[pp(g) + j / page_size] * page_size + j % page_size,
   *   pp(g) = sum_{g' < g} ceil(P_g' / page_size),
   * likewise distinct key j of request r via distinct_pages and
   * dp(r) = sum_{r' < r} ceil(D_r' / page_size). Page tables are device int32. */
  int32_t page_size;
  int32_t reserved0;
  const int32_t* prefix_pages;
  const int32_t* distinct_pages;
  int64_t prefix_cache_rows;
  int64_t distinct_cache_rows;
} psa_problem;

typedef struct psa_plan_opts {
  int32_t num_sms;        /* 0 = query the current device */
  int32_t ctas_per_sm;    /* 0 = default (2) */
  int32_t tile_min_rows;  /* stacked rows at which a segment uses tcgen05 tiles (0 = default: 16 for
                             the v2 kernel, 32 otherwise) */
  int32_t disable_tiles;  /* 1 = every item on the CUDA-core path (diagnostics) */
  int32_t min_chunk_keys; /* tile items: minimum KV chunk, 0 = default (512) */
  int32_t max_chunk_keys; /* 0 = default (16384) */
  int32_t target_waves;   /* tile items per CTA the chunking aims at, 0 = default (1) */
  int32_t disable_vec_fast; /* 1 = VEC items on the generic CUDA-core path, 2 = on the warp-level
                               CUDA-core decode path instead of tcgen05 (diagnostics) */
  int32_t kernel_variant;   /* 0 = auto: bf16/f16 with d == dv == 128 run the v2 kernel (one CTA
                               per SM, 256-row paired tiles, prefill chunks fused with their own
                               KV, two decode pipelines); 1 = the 2-CTA/SM kernel (diagnostics) */
} psa_plan_opts;

/* Read-only view of a plan's int32 tables (bit-exact with oracle/plan.py). */
typedef struct psa_plan_view {
  int32_t num_items;
  int32_t num_units;
  int32_t num_contribs;
  int32_t item_words;      /* int32 words per item record */
  int32_t unit_words;      /* int32 words per unit record */
  int32_t num_tile_items;
  int64_t workspace_rows;  /* fp32/f64 partial rows in the workspace */
  const int32_t* items;    /* [num_items * item_words], queue (LPT) order */
  const int32_t* units;    /* [num_units * unit_words] */
  const int32_t* contribs; /* [num_contribs] workspace row of each contribution */
} psa_plan_view;

typedef struct psa_plan psa_plan; /* opaque */

const char* psa_last_error(void);
int32_t psa_abi_version(void);

/* Number of SMs of the current device (cached per device). */
psa_status psa_device_sms(int32_t* num_sms);

/* Build the deterministic work-item plan from the host offset tables. */
psa_status psa_plan_create(const psa_problem* prob, const psa_plan_opts* opts, psa_plan** plan);
psa_status psa_plan_view_get(const psa_plan* plan, psa_plan_view* view);
/* Device workspace the plan needs (tables + partials + counters). */
psa_status psa_plan_workspace_bytes(const psa_plan* plan, size_t* bytes);
/* Copy the plan tables into the workspace and zero its counters (stream-ordered).
 * Needed once per (plan, workspace); psa_run keeps the counters zero between calls. */
psa_status psa_plan_upload(const psa_plan* plan, void* workspace, size_t workspace_bytes,
                           void* stream);
void psa_plan_destroy(psa_plan* plan);

/* One persistent launch over every work item of the plan. */
psa_status psa_run(const psa_problem* prob, const psa_plan* plan, void* workspace,
                   size_t workspace_bytes, void* stream);

/* Convenience: plan + upload + run + destroy (the workspace must be large enough;
 * query with psa_workspace_bytes). */
psa_status psa_workspace_bytes(const psa_problem* prob, const psa_plan_opts* opts, size_t* bytes);
psa_status psa_prefix_shared_attention(const psa_problem* prob, const psa_plan_opts* opts,
                                       void* workspace, size_t workspace_bytes, void* stream);

/* Device error word written by the last psa_run on this workspace
 * (bit 0: a row finalised with l <= 0). Synchronises the stream. */
psa_status psa_workspace_error(const void* workspace, void* stream, int32_t* error_bits);

/* merge (attention.py:101-119) of two partials, elementwise on device.
 * o*: [rows, dv]; m*, l*: [rows]; dtype PSA_DTYPE_F32 or PSA_DTYPE_F64.
 * Output may alias either input. */
psa_status psa_merge(int64_t rows, int32_t value_dim, int32_t dtype,
                     const void* oa, const void* ma, const void* la,
                     const void* ob, const void* mb, const void* lb,
                     void* o, void* m, void* l, void* stream);
/* finalize (attention.py:122-126): out = o / l; counts rows with l <= 0 into
 * *bad_rows_dev (device int32, accumulated). */
psa_status psa_finalize(int64_t rows, int32_t value_dim, int32_t dtype, const void* o,
                        const void* l, void* out, int32_t* bad_rows_dev, void* stream);

/* Input validation for _as_matrix (attention.py:26-32): counts non-finite
 * elements of a device buffer into *count_dev (device int32, accumulated). */
psa_status psa_count_nonfinite(const void* data, int64_t n, int32_t dtype, int32_t* count_dev,
                               void* stream);

/* Diagnostics: subsequent psa_run calls on this host thread record, per work
 * item, {cta | smid << 32, kind, t_start_ns, t_end_ns} (int64, %globaltimer)
 * into the device buffer `buf` (capacity_items records). NULL/0 turns it off. */
psa_status psa_debug_set_trace(void* buf, int64_t capacity_items);

/* Group -> rank partition for multi-GPU sharding: greedy LPT
 * over per-group costs, deterministic ties (bit-exact with oracle/plan.py shard_groups). */
psa_status psa_shard_groups(int32_t num_groups, const int64_t* group_cost, int32_t world_size,
                            int32_t* owner);
/* Per-group cost used by psa_shard_groups (same model as the planner). */
psa_status psa_group_costs(const psa_problem* prob, int64_t* group_cost);

/* Host preprocessing: the reference's prompt grouping
 *   extract_groups(maximize_reuse(build_tree(workload)))   (prefix_tree.py:107-301)
 * natively. Prompts are tokens[cu_tokens[r] .. cu_tokens[r+1]) (non-empty, int32 ids);
 * id_rank[r] orders requests with identical prompts like the reference's sorted()
 * of their string ids. maximize = 0 skips the first-level enlargement. Outputs
 * (caller-allocated, R = num_requests): *num_groups = G <= R; group g shares the
 * first group_prefix_len[g] tokens of each member prompt (0 = singleton: the whole
 * prompt is the suffix) and its members, in the reference's order, are
 * members[cu_members[g] .. cu_members[g+1]) (request indices; cu_members has R+1
 * slots). *saved_tokens (nullable) = sum_g (members - 1) * prefix_len. */
psa_status psa_prefix_groups(int32_t num_requests, const int64_t* cu_tokens, const int32_t* tokens,
                             const int32_t* id_rank, int32_t maximize, int32_t* num_groups,
                             int64_t* group_prefix_len, int32_t* cu_members, int32_t* members,
                             int64_t* saved_tokens);

#ifdef __cplusplus
}
#endif

#endif /* PSA_H_ */
