// psa_kernel.h — host/device contract of the persistent prefix-shared attention kernel.
#pragma once

#include <cuda.h>

#include <cstddef>
#include <cstdint>

namespace psa {

// Control block at the start of every workspace. Zero between launches: the
// last CTA to leave resets next_item/done, the last arriver of a merge unit
// resets that unit's counter, so consecutive launches need no memset.
struct Ctrl {
  int32_t next_item;  // global work queue cursor
  int32_t done;       // CTAs that left the persistent loop
  int32_t error;      // bit 0: a row was finalised with l <= 0
  int32_t next_vec;   // warp-level VEC queue cursor (fast mode)
  int32_t pad[12];
};

struct KParams {
  // TMA descriptors (TILE items only): q as 4-D (d, gqa, Hkv, T); k/v as 3-D (d, Hkv, keys).
  alignas(64) CUtensorMap tm_q;
  alignas(64) CUtensorMap tm_kp;
  alignas(64) CUtensorMap tm_vp;
  alignas(64) CUtensorMap tm_kd;
  alignas(64) CUtensorMap tm_vd;
  // VEC fast path: k/v as 3-D (d, Hkv, keys), (d, 1, 8) boxes, no swizzle.
  alignas(64) CUtensorMap tmv_kp;
  alignas(64) CUtensorMap tmv_vp;
  alignas(64) CUtensorMap tmv_kd;
  alignas(64) CUtensorMap tmv_vd;
  // tcgen05 decode path: k/v as 3-D (d, Hkv, keys), (64, 1, 128) boxes, 128-byte swizzle.
  alignas(64) CUtensorMap tmd_kp;
  alignas(64) CUtensorMap tmd_vp;
  alignas(64) CUtensorMap tmd_kd;
  alignas(64) CUtensorMap tmd_vd;
  // decode Q rows: q as 4-D (d, gqa, Hkv, T), (64, gqa, 1, 16 / gqa) boxes, 128-byte
  // swizzle — one item's <= 16 stacked rows (whole tokens) per box pair
  alignas(64) CUtensorMap tmd_q;
  const void* q;
  const void* kp;
  const void* vp;
  const void* kd;
  const void* vd;
  void* out;
  float* lse;
  void* m_out;
  void* l_out;
  const int32_t* items;
  const int32_t* units;
  const int32_t* contribs;
  const int64_t* group_tok0;   // [G] first token of each group
  const int64_t* group_pbase;  // [G] cu_prefix[g]
  const int64_t* req_dbase;    // [R] cu_distinct[r]
  void* ws_o;                  // [ws_rows, dv] accumulate type
  void* ws_ml;                 // [ws_rows, 2]  (m, l) accumulate type
  int32_t* unit_cnt;           // [num_units]
  Ctrl* ctrl;
  int32_t num_items;
  int32_t n_tile_items;  // items [0, n_tile_items) are TILE items (planner order)
  int32_t n_tile_ctas;   // fast mode: CTAs that start on the tile queue
  int32_t Hq, Hkv, gqa, d, dv;
  int32_t gqa_shift;     // log2(gqa) when gqa is a power of two, else -1
  int32_t max_vec_rows;  // largest VEC item of the plan (rows)
  int32_t dec_help;      // decode merge queues get helper warps (plan has VEC units with > 2 contributions)
  uint32_t flags;
  int32_t use_tiles;     // the plan has TILE items: allocate TMEM, init barriers
  int32_t use_vec_fast;  // bf16/f16, d == dv in {64, 128}: TMA-staged decode path
  int32_t trace_cap;     // diagnostics: capacity (items) of `trace`, 0 = off
  int32_t use_dec;       // VEC items on the tcgen05 decode pipeline (d == dv == 128)
  int32_t tile_stages;   // TILE K/V ring depth (set by the launcher from the smem budget)
  int32_t dec_slots;     // decode K/V ring slots (ditto)
  int32_t use_v2;       // v2 kernel: 1 CTA/SM, paired tile slots + two decode pipelines
  int32_t dec_pipes;    // v2: decode pipelines per CTA (2; 1 under PSA_DEBUG bit 0)
  int32_t dec_q_tma;    // tmd_q is valid (gqa is a power of two <= 16)
  int32_t tile_pp;      // v2 single-slot tile items ping-pong S buffers (0 under PSA_DEBUG bit 5)
  int32_t tail_shift;   // packed partial last blocks read back-shifted boxes (0 under PSA_DEBUG bit 10)
  int32_t dec_fast;     // v2 decode items may merge a finished prefix partial in registers (0 under PSA_DEBUG bit 8)
  int32_t dbg_cta;      // diagnostics: CTA whose per-block events are traced (PSA_DBG_CTA, default 0)
  const int32_t* tok_lim;        // causal: per token {last prefix key, last distinct key}
  int32_t page_size;             // 0 = packed K/V; else paged caches (psa.h)
  const int32_t* prefix_pages;   // paged: page tables (group_pbase / req_dbase index them)
  const int32_t* distinct_pages;
  int32_t prefix_cache_rows, distinct_cache_rows;  // paged: TMA out-of-bounds row (zero fill)
  double scale;
  int64_t* trace;        // diagnostics: per item {cta | smid << 32, kind, t_start, t_end}
};

// Encodes the TMA descriptors of `p` (tokens T, prefix keys, distinct keys):
// the TILE maps when p.use_tiles, the VEC maps when p.use_vec_fast.
int encode_tile_maps(KParams& p, int32_t dtype, int64_t T, int64_t prefix_keys,
                     int64_t distinct_keys);
// True when the VEC fast path applies to this dtype / head shape.
bool vec_fast_supported(int32_t dtype, int32_t d, int32_t dv);
// True when VEC items can run on the tcgen05 decode pipeline.
bool dec_supported(int32_t dtype, int32_t d, int32_t dv);
// True when the v2 kernel (1 CTA/SM: paired tcgen05 tiles + two decode pipelines) applies.
bool v2_supported(int32_t dtype, int32_t d, int32_t dv);

// Launches one persistent grid on `stream`. Returns a cudaError_t value.
int launch_psa(const KParams& p, int32_t dtype, int32_t num_sms, int32_t ctas_per_sm,
               bool use_tiles, void* stream);
int launch_merge(int64_t rows, int32_t dv, int32_t dtype, const void* oa, const void* ma,
                 const void* la, const void* ob, const void* mb, const void* lb, void* o,
                 void* m, void* l, void* stream);
int launch_finalize(int64_t rows, int32_t dv, int32_t dtype, const void* o, const void* l,
                    void* out, int32_t* bad, void* stream);
int launch_count_nonfinite(const void* data, int64_t n, int32_t dtype, int32_t* count,
                           void* stream);
size_t kernel_smem_bytes(int32_t dtype, bool use_tiles);

}  // namespace psa
