// psa_dec.cuh — VEC work items (few query rows vs. a request's distinct KV) on the
// 5th-gen tensor cores, with the key dimension as the MMA's M.
//
// A decode item has <= 16 query rows (the gqa heads of one token, padded) and
// up to 512 keys — the reference's per-request partial_attention(q_r, dk_r,
// dv_r) (attention.py:187-189). On CUDA cores it costs ~50 instructions per key;
// here the dot products run as
//     S^T[128 keys x 16 rows] = K_blk[128 x d] . Q^T          (A = K, smem)
//     O^T[dv x 16 rows]      += V_blk^T[dv x 128] . P^T        (A = V^T, MN-major)
// so the CUDA cores only do the softmax: one thread per key, <= 16 values each.
//
// The CTA runs a decoupled, persistent pipeline over the VEC queue:
//   warp 4   producer: pulls items, stages Q rows, streams K/V blocks into a
//            3-slot ring of 32 KB slots (K_j, V_j, K_j+1, ...) with TMA,
//            running ahead into the next item;
//   warp 5   MMA issuer: polls its two streams (S for the next block, PV for
//            the oldest finished softmax) and issues whichever is ready;
//   warps 0-3 softmax + epilogue (thread t = key t of the block; at the end of
//            an item thread t = value column t).
// TMEM: S^T [0,16), O^T double buffer [32,48) / [48,64).
#pragma once

#include "psa_device.cuh"

namespace psa {

// One K or V block of `rows` keys (two 64-column chunks, SW128 K-major in `dst`) of
// a segment: the packed layout (one box per chunk at cache row base + key) or a
// paged cache (one box per page; page p of the segment is table[base + p]; pages at
// or past key_end load the all-out-of-bounds row, i.e. zeros). Issued by one lane.
// Packed partial last block: when the item's key range [key_begin, key_end) holds a
// full block before it, the box is shifted back by kv_shift() keys so it ends at
// key_end — the extra rows are the previous block's (just read: L2 hits) instead of
// the next segment's (DRAM reads that were ~0.6 GB per c4 launch). Consumers mask
// columns [0, shift) of such a block. Used by the decode pipelines (ragged per-request
// KV); the tile producer passes key_begin = key (forward boxes: prefix chunks are
// long, their partial blocks rare).
__device__ __forceinline__ int kv_shift(const KParams& p, int key, int key_end, int key_begin, int rows) {
  return (p.tail_shift && p.page_size == 0 && key_end - key < rows && key_end - key_begin >= rows)
             ? rows - (key_end - key) : 0;
}
__device__ __forceinline__ void load_kv_block(const KParams& p, uint8_t* dst, const CUtensorMap* m,
                                              uint64_t* bar, int h, bool prefix, int64_t base,
                                              int key, int key_end, int key_begin, int rows) {
  if (p.page_size == 0) {
    const int k0 = key - kv_shift(p, key, key_end, key_begin, rows);
    dev::tma_load_3d(dst, m, bar, 0, h, int(base + k0));
    dev::tma_load_3d(dst + rows * 128, m, bar, 64, h, int(base + k0));
    return;
  }
  const int ps = p.page_size;
  const int32_t* tab = prefix ? p.prefix_pages : p.distinct_pages;
  const int oob = prefix ? p.prefix_cache_rows : p.distinct_cache_rows;
  const int np = rows / ps;
  int prow[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int lk = key + i * ps;
    prow[i] = (i < np && lk < key_end) ? __ldg(tab + base + lk / ps) * ps : oob;
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    if (i < np) {
      dev::tma_load_3d(dst + i * ps * 128, m, bar, 0, h, prow[i]);
      dev::tma_load_3d(dst + (rows + i * ps) * 128, m, bar, 64, h, prow[i]);
    }
  }
}

// Output row (token * Hq + query head) of stacked row `row` of kv head h.
__device__ __forceinline__ int64_t out_index(const KParams& p, int64_t tok0, int h, int row) {
  const int tq = p.gqa_shift >= 0 ? row >> p.gqa_shift : row / p.gqa;
  return (tok0 + tq) * p.Hq + (int64_t)h * p.gqa + (row - tq * p.gqa);
}

// Decode MMA issuer: warp-wide (elect.sync) or lane 0 alone, independently of the
// tile issuer (PSA_DEC_WARP_WIDE, default PSA_MMA_WARP_WIDE).
#ifndef PSA_DEC_WARP_WIDE
#define PSA_DEC_WARP_WIDE PSA_MMA_WARP_WIDE
#endif
#if PSA_DEC_WARP_WIDE
#define PSA_DEC_MMA_SS ::psa::dev::mma_f16_ss_w
#define PSA_DEC_MMA_COMMIT ::psa::dev::mma_commit_w
#else
#define PSA_DEC_MMA_SS ::psa::dev::mma_f16_ss
#define PSA_DEC_MMA_COMMIT ::psa::dev::mma_commit
#endif

namespace dec {

constexpr int kBK = 128;               // keys per block (MMA M)
constexpr int kN = 16;                 // query rows per item (MMA N), padded
constexpr int kR = 8;                  // rows per VEC item (planner kVecRows)
constexpr int kMaxSlots = 6;           // K/V ring slots: p.dec_slots (3 with 2 CTAs/SM, 6 with 1)
constexpr int kSlotBytes = kBK * 128 * 2;  // one K or V block, d = 128 bf16 = 32 KB
constexpr int kQBytes = kN * 128 * 2;  // one item's Q rows = 4 KB
constexpr int kPBytes = kN * kBK * 2;  // P^T = 4 KB
constexpr uint32_t kTmemS = 0, kTmemO = 32;
constexpr float kRescaleThreshold = 8.0f;

__host__ __device__ constexpr size_t smem_bytes(int slots) {
  return size_t(slots) * kSlotBytes + 2 * kQBytes + kPBytes + 1024;
}
// Offset between the shared-memory regions of two pipelines of one CTA.
__host__ __device__ constexpr size_t pipe_stride(int slots) {
  return (smem_bytes(slots) + 1023) & ~size_t(1023);
}

struct alignas(16) Shared {
  uint64_t slot_full[kMaxSlots], slot_empty[kMaxSlots];
  uint64_t item_full[2], item_empty[2];
  uint64_t s_full, s_free, p_full[2], o_done, o_full[2], o_empty[2];
  int item_idx[2];
  float red[2][4][kR];  // per-warp partial row maxima (double-buffered by block parity) / sums
  int item_fast[2];     // producer's fast-merge decision per item slot (see NoFast)
  // Item metadata staged by the producer (it already holds the record one item ahead),
  // so the softmax warps start an item without dependent global round trips.
  alignas(16) int32_t item_rec[2][16];  // the ItemRec
  int64_t item_tok0[2];                 // first token of the item's group
  int item_other[2];                    // fast merge: workspace row of the other contribution
  int64_t item_oidx[2][kR];             // output row (token * Hq + query head) of each item row
  // merge queue: softmax thread 0 appends the units this CTA completes, warps 6-7 merge them
  dev::MergeQueue mq;
};

__device__ __forceinline__ void init_barriers(Shared* s) {
  for (int i = 0; i < kMaxSlots; ++i) {
    dev::mbar_init(&s->slot_full[i], 1);
    dev::mbar_init(&s->slot_empty[i], 1);
  }
  for (int i = 0; i < 2; ++i) {
    dev::mbar_init(&s->item_full[i], 1);
    dev::mbar_init(&s->item_empty[i], 2);  // MMA (after the item's last S) + softmax epilogue
    dev::mbar_init(&s->p_full[i], 4);
    dev::mbar_init(&s->o_full[i], 1);
    dev::mbar_init(&s->o_empty[i], 4);
  }
  dev::mbar_init(&s->s_full, 1);
  dev::mbar_init(&s->s_free, 4);
  dev::mbar_init(&s->o_done, 1);
  dev::mq_init(&s->mq);
  dev::fence_mbar_init();
}

// Softmax thread 0: hand an item whose partial rows are stored (and ordered before
// this by a named barrier) to the merge warps (warps 6-7 of the pipeline).
__device__ __forceinline__ void enqueue_merge(Shared* sh, int idx) { dev::mq_push(&sh->mq, idx); }

// Warps 6-7: arrive at / merge the queued items' units until the queue is closed and drained.
template <typename MergeUnit>
__device__ __forceinline__ void merge_loop(const KParams& p, Shared* sh, MergeUnit&& merge_unit) {
  int n = 0;
  dev::mq_drain(&sh->mq, 1, [&](int task) {
    // diagnostics: CTA 0, pipeline 0: start / end clock of the first 32 tasks per merge warp
    const bool rec = false;
    const int slot = ((threadIdx.x >> 5) & 1) * 32 + n;
    long long t0 = 0;
    if (rec) asm volatile("mov.u64 %0, %%clock64;" : "=l"(t0));
    merge_unit(task);
    if (rec) {
      long long t1;
      asm volatile("mov.u64 %0, %%clock64;" : "=l"(t1));
      p.trace[(int64_t(p.num_items) + 4096) * 4 + 34 * 64 + slot] = t0;
      p.trace[(int64_t(p.num_items) + 4096) * 4 + 35 * 64 + slot] = t1;
    }
    ++n;
  });
}

// Diagnostics: clock64 of per-block events of CTA 0's first 64 decode blocks, after
// the tile events (psa_debug_set_trace). Slot = (16 + event) * 64 + global block.
__device__ __forceinline__ void dbg(const KParams& p, int ev, uint32_t g) {
  if (kTraceEvents && p.trace_cap > 0 && int(blockIdx.x) == p.dbg_cta && g < 64) {
    long long t;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(t));
    p.trace[(int64_t(p.num_items) + 4096) * 4 + (16 + ev) * 64 + g] = t;
  }
}

// Softmax warps of decode pipeline `pi` (barrier ids 4, 5: ids 1-3 belong to other phases).
__device__ __forceinline__ void named_sync_softmax(int pi = 0) {
  asm volatile("bar.sync %0, 128;" ::"r"(4 + pi) : "memory");
}

struct Geo {
  uint8_t* base;  // 1024-aligned
  uint32_t slots;
  __device__ __forceinline__ uint8_t* slot(uint32_t i) const { return base + i * kSlotBytes; }
  __device__ __forceinline__ uint8_t* q(uint32_t i) const {
    return base + slots * kSlotBytes + i * kQBytes;
  }
  __device__ __forceinline__ uint8_t* pt() const { return base + slots * kSlotBytes + 2 * kQBytes; }
};

__device__ __forceinline__ Geo carve(uint8_t* smem_raw, int slots) {
  Geo g;
  g.slots = uint32_t(slots);
  g.base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                      ~uintptr_t(1023));
  return g;
}

// Byte offset of element (row r, col c) in a K-major SW128 tile with 64-element
// chunks of `rows` rows: chunk (c / 64), row r, 16-byte unit ((c % 64) / 8) ^ (r % 8).
__device__ __forceinline__ uint32_t sw128_off(int r, int c, int rows) {
  return uint32_t((c >> 6) * rows * 128 + r * 128 + ((((c & 63) >> 3) ^ (r & 7)) << 4) +
                  (c & 7) * 2);
}

// Warp sum of n (4 or 8) per-lane values by reduce-scatter: each butterfly level
// keeps half of the remaining rows and ships the other half (n/2 + n/4 + ... + the
// last log2(32/n) full levels: 9 shuffles for n = 8, 6 for n = 4, instead of 5n).
// Returns the full sum of row (lane >> (5 - log2 n)) in every lane.
template <int n>
__device__ __forceinline__ float warp_sum_scatter(const float (&v)[kR], int lane) {
  static_assert(n == 4 || n == 8, "rows per item");
  float w[n];
#pragma unroll
  for (int i = 0; i < n; ++i) w[i] = v[i];
  int width = n;
#pragma unroll
  for (int bit = 16; bit >= 1; bit >>= 1) {
    if (width > 1) {
      const bool hi = lane & bit;
      const int half = width / 2;
#pragma unroll
      for (int i = 0; i < n / 2; ++i) {
        if (i < half) {
          const float mine = hi ? w[half + i] : w[i];
          const float other = hi ? w[i] : w[half + i];
          w[i] = mine + __shfl_xor_sync(0xffffffffu, other, bit);
        }
      }
      width = half;
    } else {
      w[0] += __shfl_xor_sync(0xffffffffu, w[0], bit);
    }
  }
  return w[0];
}

template <typename ItemT>
__device__ __forceinline__ void item_blocks(const KParams& p, const ItemT& it, int& nbA, int& nb,
                                            int64_t& pbase, int64_t& dbase) {
  const int npA = it.pk1 - it.pk0, npB = it.dk1 - it.dk0;
  nbA = (npA + kBK - 1) / kBK;
  nb = nbA + (npB + kBK - 1) / kBK;
  pbase = npA ? __ldg(p.group_pbase + it.g) + it.pk0 : 0;
  dbase = (it.req >= 0) ? __ldg(p.req_dbase + it.req) + it.dk0 : 0;
}

template <typename ItemT>
__device__ __forceinline__ int block_nvalid(const ItemT& it, int nbA, int j) {
  return j < nbA ? min(kBK, it.pk1 - it.pk0 - j * kBK) : min(kBK, it.dk1 - it.dk0 - (j - nbA) * kBK);
}

// The decode pipeline. `load(idx)` returns the ItemRec of queue entry idx;
// `finish` / `merge_unit` are provided by the kernel (output + merges). Pipeline
// `pi` runs on warps 8*pi .. 8*pi+7 (the v2 kernel runs two per CTA).
// `fast` (see psa_kernel.cu, DecFast): an item whose only merge unit has one other
// contributor that already arrived (typically the group's prefix tile) merges that
// contributor's partial in registers and writes the final rows itself — no partial
// rows, no arrival task, no merge. fast.probe(it, other_row) (producer lane 0; sets the
// workspace row of the other contribution) / fast.fetch(other_row, t, R, Other&) (all
// threads, at the item start) / fast.finish(it, oidx, t, R, m, L, ov, o).
struct NoFast {
  struct Other {};
  template <typename I> __device__ int probe(const I&, int&) const { return 0; }
  __device__ void fetch(int, int, int, Other&) const {}
  template <typename I>
  __device__ void finish(const I&, const int64_t*, int, int, const float (&)[kR], const float (&)[kR],
                         const float (&)[kR], const Other&) const {}
};

template <typename T, bool kCausal = false, int kRows = kR, typename LoadItem, typename Finish,
          typename MergeUnit, typename Fast = NoFast>
__device__ void run(const KParams& p, uint8_t* smem_raw, Shared* sh, uint32_t tmem, int pi,
                    LoadItem&& load_item_at, Finish&& finish, MergeUnit&& merge_unit,
                    const Fast& fast = Fast()) {
  const int warp = (threadIdx.x >> 5) - 8 * pi, lane = threadIdx.x & 31;
  const Geo G = carve(smem_raw, p.dec_slots);
  const uint32_t NSL = uint32_t(p.dec_slots);
  const int n_items = p.num_items;

  if (warp == 4) {
    // ================= producer =================
    // Software-pipelined over items: the queue slot of item k+2 (global atomic) and
    // the record of item k+1 are in flight while item k's K/V loads are issued (and
    // wait for ring slots). Q rows come by TMA (whole tokens, SW128) on the item_full
    // barrier, so a 2-block decode item pays no dependent global round trips before
    // its first K/V load.
    const T* Q = static_cast<const T*>(p.q);
    int raw = 0;
    if (lane == 0) raw = p.n_tile_items + atomicAdd(&p.ctrl->next_vec, 1);
    int idx = __shfl_sync(0xffffffffu, raw, 0);
    if (lane == 0) raw = p.n_tile_items + atomicAdd(&p.ctrl->next_vec, 1);  // item k + 1
    decltype(load_item_at(0)) it{};
    int64_t tok0 = 0;
    if (idx < n_items) {
      it = load_item_at(idx);
      tok0 = __ldg(p.group_tok0 + it.g);
    }
    uint32_t c = 0;  // K/V slot loads issued
    for (uint32_t k = 0;; ++k) {
      const uint32_t q = k & 1;
      int fast_k = 0, other_k = -1;
      if (lane == 0 && idx < n_items) fast_k = fast.probe(it, other_k);  // latency overlaps the wait
      dev::mbar_wait(&sh->item_empty[q], ((k >> 1) & 1) ^ 1);
      if (idx >= n_items) {
        if (lane == 0) {
          sh->item_idx[q] = -1;
          dev::mbar_arrive(&sh->item_full[q]);
        }
        break;
      }
      uint8_t* qs = G.q(q);
      const bool q_tma = p.dec_q_tma && (it.row0 % p.gqa) == 0;
      if (!q_tma) {  // Q rows -> K-major SW128 [16 rows][128] (2 chunks of 64), lane-parallel
        for (int u = lane; u < kN * 16; u += 32) {  // 16-byte units: row u/16, unit u%16
          const int r = u >> 4, cu = u & 15;
          uint4 v = make_uint4(0u, 0u, 0u, 0u);
          if (r < it.nrows) {
            const int row = it.row0 + r;
            const T* qr = Q + ((tok0 + row / p.gqa) * p.Hq + (int64_t)it.h * p.gqa + row % p.gqa) * 128;
            v = __ldg(reinterpret_cast<const uint4*>(qr) + cu);
          }
          *reinterpret_cast<uint4*>(qs + sw128_off(r, cu * 8, kN)) = v;
        }
        dev::fence_proxy_async_smem();
        __syncwarp();
      }
      if (lane < kR && lane < it.nrows) sh->item_oidx[q][lane] = out_index(p, tok0, it.h, it.row0 + lane);
      __syncwarp();  // ordered before lane 0's item_full arrival
      // next item: its index (claimed one iteration ago) and its record
      const int next = __shfl_sync(0xffffffffu, raw, 0);
      if (lane == 0 && next < n_items) raw = p.n_tile_items + atomicAdd(&p.ctrl->next_vec, 1);
      decltype(load_item_at(0)) it_next{};
      int64_t tok_next = 0;
      if (next < n_items) {
        it_next = load_item_at(next);
        tok_next = __ldg(p.group_tok0 + it_next.g);
      }
      if (lane == 0) {
        sh->item_idx[q] = idx;
        sh->item_fast[q] = fast_k;
        sh->item_other[q] = other_k;
        sh->item_tok0[q] = tok0;
        static_assert(sizeof(it) <= sizeof(sh->item_rec[0]), "item record too large");
        *reinterpret_cast<decltype(load_item_at(0))*>(sh->item_rec[q]) = it;
        if (q_tma) {
          const int t0 = int(tok0 + it.row0 / p.gqa);
          dev::mbar_arrive_expect_tx(&sh->item_full[q], uint32_t(kQBytes));
          dev::tma_load_4d(qs, &p.tmd_q, &sh->item_full[q], 0, 0, it.h, t0);
          dev::tma_load_4d(qs + kN * 128, &p.tmd_q, &sh->item_full[q], 64, 0, it.h, t0);
        } else {
          dev::mbar_arrive(&sh->item_full[q]);
        }
        const int nbA = (it.pk1 - it.pk0 + kBK - 1) / kBK;
        const int nb = nbA + (it.dk1 - it.dk0 + kBK - 1) / kBK;
        const int64_t gbase = nbA ? __ldg(p.group_pbase + it.g) : 0;
        const int64_t rbase = (it.req >= 0 && it.dk1 > it.dk0) ? __ldg(p.req_dbase + it.req) : 0;
        for (int j = 0; j < nb; ++j) {
          const bool pre = j < nbA;
          const CUtensorMap* km = pre ? &p.tmd_kp : &p.tmd_kd;
          const CUtensorMap* vm = pre ? &p.tmd_vp : &p.tmd_vd;
          const int key = pre ? it.pk0 + j * kBK : it.dk0 + (j - nbA) * kBK;
          const int end = pre ? it.pk1 : it.dk1;
          for (int w = 0; w < 2; ++w, ++c) {  // K then V
            const uint32_t s = c % NSL;
            dev::mbar_wait(&sh->slot_empty[s], ((c / NSL) & 1) ^ 1);
            dbg(p, w, c >> 1);
            dev::mbar_arrive_expect_tx(&sh->slot_full[s], kSlotBytes);
            load_kv_block(p, G.slot(s), w == 0 ? km : vm, &sh->slot_full[s], it.h, pre,
                          pre ? gbase : rbase, key, end, pre ? it.pk0 : it.dk0, kBK);
          }
        }
      }
      __syncwarp();
      idx = next;
      it = it_next;
      tok0 = tok_next;
    }
  } else if (warp == 5) {
    // ================= MMA issuer =================
    if (PSA_DEC_WARP_WIDE || lane == 0) {
      // warp-wide issue (PSA_DEC_WARP_WIDE): every barrier test is lane 0's verdict,
      // so the branches stay warp-uniform around the elect.sync issue forms
      auto test = [&](uint64_t* bar, uint32_t par) {
        bool r = dev::mbar_test(bar, par);
        if (PSA_DEC_WARP_WIDE) r = __shfl_sync(0xffffffffu, int(r), 0) != 0;
        return r;
      };
      constexpr uint32_t fmt = tile::AbFormat<T>::v;
      const uint32_t idesc_s = dev::umma_idesc_f16(fmt, kBK, kN, 0, 0);
      const uint32_t idesc_o = dev::umma_idesc_f16(fmt, 128, kN, 1, 0);
      const uint32_t tS = tmem + kTmemS;
      const uint32_t pt = dev::smem_u32(G.pt());
      // S stream: (item k_s, block j_s, global block gS); PV stream lags behind.
      uint32_t k_s = 0, gS = 0;
      int j_s = 0, nb_s = -1, nbA_s = 0;
      uint32_t k_p = 0, gP = 0;
      int j_p = 0, nb_p = -1;
      bool s_done = false;
      int nbs_ring[2] = {0, 0};  // blocks per in-flight item (by k & 1)
      for (;;) {
        bool progress = false;
        // ---- S stream
        if (!s_done) {
          const uint32_t q = k_s & 1;
          if (nb_s < 0 && test(&sh->item_full[q], (k_s >> 1) & 1)) {
            const int idx = sh->item_idx[q];
            if (idx < 0) {
              s_done = true;
              nbs_ring[q] = -1;
            } else {
              const auto it = load_item_at(idx);
              int64_t pb, db;
              item_blocks(p, it, nbA_s, nb_s, pb, db);
              nbs_ring[q] = nb_s;
              j_s = 0;
            }
            progress = true;
          }
          if (nb_s > 0) {
            const uint32_t cK = 2 * gS, s = cK % NSL;
            const bool sfree = gS == 0 || test(&sh->s_free, (gS - 1) & 1);
            // A parity test tells phase o from phase o - 2 only once phase o - 1 has
            // completed. With an odd ring, K_g's slot previously held V_j (cK - NSL =
            // 2j + 1), which only the PV stream waits for: require PV_j issued (so V_j
            // landed), else K_g's test could pass on phase o - 2 while V_j is in flight.
            const int32_t prev = int32_t(cK) - int32_t(NSL);
            const bool prev_ok = prev < 0 || !(prev & 1) || gP > uint32_t((prev - 1) >> 1);
            if (sfree && prev_ok && test(&sh->slot_full[s], (cK / NSL) & 1)) {
              dev::tc_fence_after();
              dbg(p, 2, gS);
              const uint64_t ad = dev::umma_desc_sw128(dev::smem_u32(G.slot(s)), 16, 1024);
              const uint64_t bd0 = dev::umma_desc_sw128(dev::smem_u32(G.q(q)), 16, 1024);
#pragma unroll
              for (int kk = 0; kk < 8; ++kk) {  // descriptor start address is addr >> 4
                const uint32_t ch = kk >> 2, w = (kk & 3) * 32;
                const uint64_t a = ad + uint64_t((ch * (kBK * 128) + w) >> 4);
                const uint64_t b = bd0 + uint64_t((ch * (kN * 128) + w) >> 4);
                PSA_DEC_MMA_SS(tS, a, b, idesc_s, kk > 0);
              }
              PSA_DEC_MMA_COMMIT(&sh->s_full);
              PSA_DEC_MMA_COMMIT(&sh->slot_empty[s]);
              ++gS;
              if (++j_s == nb_s) {
                PSA_DEC_MMA_COMMIT(&sh->item_empty[q]);  // Q slot reusable once these S complete
                nb_s = -1;
                ++k_s;
              }
              progress = true;
            }
          }
        }
        // ---- PV stream
        if (gP < gS) {
          const uint32_t q = k_p & 1, b = k_p & 1;
          if (nb_p < 0) { nb_p = nbs_ring[q]; j_p = 0; }
          const uint32_t cV = 2 * gP + 1, s = cV % NSL;
          const bool need_o = j_p == 0;
          if (test(&sh->p_full[gP & 1], (gP >> 1) & 1) &&
              test(&sh->slot_full[s], (cV / NSL) & 1) &&
              (!need_o || test(&sh->o_empty[b], ((k_p >> 1) & 1) ^ 1))) {
            dev::tc_fence_after();
            dbg(p, 3, gP);
            const uint64_t ad = dev::umma_desc_sw128(dev::smem_u32(G.slot(s)), kBK * 128, 1024);
            const uint64_t pd = dev::umma_desc_sw128(pt, 16, 1024);
            const uint32_t tO = tmem + kTmemO + b * kN;
#pragma unroll
            for (int kk = 0; kk < kBK / 16; ++kk) {
              const uint64_t a = ad + uint64_t((kk * (16 * 128)) >> 4);
              const uint64_t bd = pd + uint64_t(((kk >> 2) * (kN * 128) + (kk & 3) * 32) >> 4);
              PSA_DEC_MMA_SS(tO, a, bd, idesc_o, (j_p > 0 || kk > 0));
            }
            PSA_DEC_MMA_COMMIT(&sh->slot_empty[s]);
            PSA_DEC_MMA_COMMIT(&sh->o_done);
            ++gP;
            if (++j_p == nb_p) {
              PSA_DEC_MMA_COMMIT(&sh->o_full[b]);
              nb_p = -1;
              ++k_p;
            }
            progress = true;
          }
        }
        if (s_done && gP == gS) break;
        (void)progress;
      }
    }
  } else if (warp < 4) {
    // ================= softmax + epilogue =================
    const int t = threadIdx.x - 256 * pi;
    const uint32_t lane_base = uint32_t(warp * 32) << 16;
    const uint32_t tS = tmem + kTmemS + lane_base;
    const float sc = float(p.scale) * 1.4426950408889634f;
    uint8_t* pt = G.pt();
    uint32_t g = 0;  // global block counter
    for (uint32_t k = 0;; ++k) {
      const uint32_t q = k & 1, b = k & 1;
      dev::mbar_wait(&sh->item_full[q], (k >> 1) & 1);
      const int idx = sh->item_idx[q];
      if (t == 0) dbg(p, 25, g);
      if (idx < 0) {
        if (t == 0) dev::mq_close(&sh->mq);
        break;
      }
      long long t_item0 = 0;
      if (p.trace_cap > 0 && t == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_item0));
      const auto it = *reinterpret_cast<const decltype(load_item_at(0))*>(sh->item_rec[q]);
      const int64_t it_tok0 = sh->item_tok0[q];
      const int nbA = (it.pk1 - it.pk0 + kBK - 1) / kBK;
      const int nb = nbA + (it.dk1 - it.dk0 + kBK - 1) / kBK;
      const int R = it.nrows;
      // fast merge decided by the producer (its acquire load + this item_full wait order
      // the other contributor's partial rows before the fetch); fetched now, used at the end
      const bool fast_on = sh->item_fast[q] != 0;
      typename Fast::Other other;
      if (fast_on) fast.fetch(sh->item_other[q], t, R, other);
      if (t == 0) dbg(p, 26, g);
      // rows >= R keep m = 0 and x = -inf: their exps are exactly 0, no NaN, and
      // every row's arithmetic stays branch-free (the rows interleave for ILP).
      // kRows (4 or 8, per launch) bounds the rows any VEC item of the plan has
      float m[kR], lp[kR];
#pragma unroll
      for (int r = 0; r < kR; ++r) { m[r] = r < R ? -INFINITY : 0.f; lp[r] = 0.f; }
      // causal prefill (PSA_FLAG_CAUSAL): last visible prefix / distinct key per row
      constexpr bool causal = kCausal;  // a separate kernel: no cost when off
      int limp[kR], limd[kR];
#pragma unroll
      for (int r = 0; r < kR; ++r) { limp[r] = INT_MAX; limd[r] = INT_MAX; }
      if constexpr (causal) {
#pragma unroll
        for (int r = 0; r < kR; ++r) {
          if (r < R) {
            const int64_t tok = it_tok0 + (it.row0 + r) / p.gqa;
            limp[r] = __ldg(p.tok_lim + tok * 2);
            limd[r] = __ldg(p.tok_lim + tok * 2 + 1);
          }
        }
      }
      for (int j = 0; j < nb; ++j, ++g) {
        const int nvalid = block_nvalid(it, nbA, j);
        dev::mbar_wait(&sh->s_full, g & 1);
        if (t == 0) dbg(p, 4, g);
        dev::tc_fence_after();
        uint32_t sr[kN];
        dev::tmem_ld16(tS, sr);
        dev::tmem_wait_ld();
        if (t == 0) dbg(p, 10, g);
        dev::tc_fence_before();
        __syncwarp();
        if (lane == 0) dev::mbar_arrive(&sh->s_free);
        // a shifted partial block holds its nvalid keys in columns [shift, kBK)
        const int shift = j < nbA ? kv_shift(p, it.pk0 + j * kBK, it.pk1, it.pk0, kBK)
                                  : kv_shift(p, it.dk0 + (j - nbA) * kBK, it.dk1, it.dk0, kBK);
        const bool valid = shift ? t >= shift : t < nvalid;
        // block max per row: warp reduce, then across the 4 softmax warps
        float x[kR], v[kR];
        const int key = (j < nbA ? it.pk0 + j * kBK : it.dk0 + (j - nbA) * kBK) + t - shift;
#pragma unroll
        for (int r = 0; r < kRows; ++r) {
          const bool vis = !causal || key <= (j < nbA ? limp[r] : limd[r]);
          x[r] = (valid && r < R && vis) ? __uint_as_float(sr[r]) * sc : -INFINITY;
          v[r] = x[r];
        }
#pragma unroll
        for (int r = 0; r < kRows; ++r) v[r] = dev::warp_max_f32(v[r]);  // one CREDUX.MAX.F32 per row
        if (lane == 0) {
#pragma unroll
          for (int r = 0; r < kRows; ++r) sh->red[g & 1][warp][r] = v[r];
        }
        if (t == 0) dbg(p, 11, g);
        named_sync_softmax(pi);  // red[g & 1] is rewritten two blocks later, after another barrier

        if (t == 0) dbg(p, 12, g);
        const float (&rd)[4][kR] = sh->red[g & 1];
        // the running maxima are identical in every thread, so `any_up` is CTA-uniform
        // and the rescale exponentials run only on blocks that raise a row's maximum
        float alpha[kR], bmax[kR];
        bool any_up = false, any_rescale = false;
#pragma unroll
        for (int r = 0; r < kRows; ++r) {
          bmax[r] = fmaxf(fmaxf(rd[0][r], rd[1][r]), fmaxf(rd[2][r], rd[3][r]));
          alpha[r] = 1.f;
          any_up |= bmax[r] > m[r] + kRescaleThreshold;  // also the first block (m = -inf)
        }
        if (any_up) {
#pragma unroll
          for (int r = 0; r < kRows; ++r) {
            const bool up = bmax[r] > m[r] + kRescaleThreshold;
            alpha[r] = up ? dev::ex2(m[r] - bmax[r]) : 1.f;
            any_rescale |= up && (m[r] != -INFINITY);
            m[r] = up ? bmax[r] : m[r];
          }
        }
        float e[kR];
#pragma unroll
        for (int r = 0; r < kRows; ++r) {
          e[r] = dev::ex2(x[r] - (m[r] == -INFINITY ? 0.f : m[r]));  // all-masked rows: 0
          lp[r] = any_up ? lp[r] * alpha[r] + e[r] : lp[r] + e[r];
        }
        // P^T (single buffer): PV_{g-1} must be done reading it (and O before rescale);
        // it was issued a whole softmax ago, so this wait rarely blocks.
        if (t == 0) dbg(p, 13, g);
        if (g > 0) {
          dev::mbar_wait(&sh->o_done, (g - 1) & 1);
          dev::tc_fence_after();
        }
        if (t == 0) dbg(p, 14, g);
#pragma unroll
        for (int r = 0; r < kRows; ++r) {
          if (r < R) {
            T h;
            if constexpr (sizeof(T) == 2) h = T(e[r]);
            *reinterpret_cast<T*>(pt + sw128_off(r, t, kN)) = h;
          }
        }
        if (any_rescale && j > 0) {
          // O^T lane t (value column t) holds this item's rows as columns
          const uint32_t tO = tmem + kTmemO + b * kN + lane_base;
          uint32_t o[kN];
          dev::tmem_ld16(tO, o);
          dev::tmem_wait_ld();
#pragma unroll
          for (int r = 0; r < kRows; ++r) o[r] = __float_as_uint(__uint_as_float(o[r]) * alpha[r]);
          dev::tmem_st16(tO, o);
          dev::tmem_wait_st();
        }
        if (t == 0) dbg(p, 15, g);
        dev::fence_proxy_async_smem();
        if (t == 0) dbg(p, 16, g);
        dev::tc_fence_before();
        __syncwarp();
        if (lane == 0) dev::mbar_arrive(&sh->p_full[g & 1]);
        if (t == 0) dbg(p, 5, g);
      }
      // ---- item end: l per row, then O^T lane t = value column t
      {
        // lane l holds the warp sum of row l >> (5 - log2 kRows)
        constexpr int kLaneShift = kRows == 8 ? 2 : 3;
        const float s = warp_sum_scatter<kRows>(lp, lane);
        if ((lane & ((1 << kLaneShift) - 1)) == 0) sh->red[g & 1][warp][lane >> kLaneShift] = s;
      }
      named_sync_softmax(pi);
      float L[kR];
      {
        const float (&rd)[4][kR] = sh->red[g & 1];
#pragma unroll
        for (int r = 0; r < kR; ++r)
          L[r] = (r < kRows && r < R) ? (rd[0][r] + rd[1][r]) + (rd[2][r] + rd[3][r]) : 0.f;
      }
      if (t == 0) dbg(p, 7, g - 1);
      dev::mbar_wait(&sh->o_full[b], (k >> 1) & 1);
      if (t == 0) dbg(p, 8, g - 1);
      dev::tc_fence_after();
      uint32_t o[kN];
      dev::tmem_ld16(tmem + kTmemO + b * kN + lane_base, o);
      dev::tmem_wait_ld();
      dev::tc_fence_before();
      __syncwarp();
      if (lane == 0) dev::mbar_arrive(&sh->o_empty[b]);
      if (t == 0) dbg(p, 24, g - 1);
      float ov[kR];
#pragma unroll
      for (int r = 0; r < kR; ++r) ov[r] = __uint_as_float(o[r]);
      const int64_t* oidx = sh->item_oidx[q];
      if (fast_on) fast.finish(it, oidx, t, R, m, L, ov, other);  // merged in registers: final rows
      else finish(it, oidx, idx, t, R, m, L, ov);  // output, or partial rows queued for arrival
      if (t == 0) dbg(p, 9, g - 1);
      named_sync_softmax(pi);      // red[] reuse + item slot release after everyone finished
      if (t == 0) dev::mbar_arrive(&sh->item_empty[q]);
      if (t == 0) dbg(p, 6, g - 1);
      if (p.trace_cap > 0 && t == 0 && idx < p.trace_cap) {
        long long t1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
        uint32_t smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        int64_t* tr = p.trace + int64_t(idx) * 4;
        tr[0] = int64_t(blockIdx.x) | (int64_t(smid) << 32);
        tr[1] = 0;
        tr[2] = t_item0;
        tr[3] = t1;
      }
    }
  }
  // The pipeline's queue is drained by its merge warps (6, 7) from the start; every
  // other warp of the pipeline joins once its role is done and the queue is closed
  // (units with a large fan-in complete late and in bursts).
  __syncwarp();
  if (warp < 6) {
    if (!p.dec_help) return;  // units of <= 2 contributions: the merge warps suffice
    dev::mq_wait_closed(&sh->mq, 1);
  }
  merge_loop(p, sh, merge_unit);
}

}  // namespace dec
}  // namespace psa
