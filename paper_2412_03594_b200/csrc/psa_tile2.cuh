// psa_tile2.cuh — TILE work items of the v2 kernel (1 CTA per SM, 512 threads):
// up to 256 stacked query rows of one (group, kv head) — two 128-row "slots" —
// against one KV range, on the 5th-gen tensor cores. d == dv == 128, bf16/f16.
//
// This is the paper's §2.2 "matrix-vector -> matrix-matrix" transformation
// (reference: the stacked prefix call, attention.py:174-179): all gqa heads x
// tokens of a row range that share a KV range form the M rows of tcgen05 tiles,
// so every K/V byte staged in shared memory feeds 256 rows. With fuse_own plans
// a prefill-chunk request's tiles run over [prefix ++ own distinct KV] in one
// online softmax (attention.py:187-198 merge folded into the block loop).
//
// Roles (warp = threadIdx.x / 32):
//   warps 0-3   softmax WG0: slot 0, thread t = row t = TMEM lane t
//   warps 4-7   softmax WG1: slot 1 (rows 128..255 of the item)
//   warp 8      producer: pulls items (CTA-level queue), Q of both slots by TMA,
//               then K_n, V_n blocks (128 keys) into a ring of 32 KB slots
//   warp 9      MMA issuer (one lane): per block n and slot i,
//                 O_i += P_{i,n-1} V_{n-1}   (A = P from TMEM, B = V MN-major)
//                 S_i  = Q_i K_n^T           (A, B from smem, K-major)
//   warps 10-15 merge workers for units this CTA completes
// TMEM (512 columns): S0 [0,128), S1 [128,256), O0 [256,384), O1 [384,512).
// P_i (bf16 pairs) overwrites S_i columns [0,64) in place; S_{i,n+1} is issued
// after PV_{i,n}, and tcgen05 MMAs of one thread execute in issue order, so the
// buffer is reused without a wait. The two slots ping-pong on the tensor core:
// while WG0 exponentiates S_0 the MMA pipe computes slot 1, and vice versa.
//
// Online softmax (attention.py:95-98 per block, merge :101-119 across blocks)
// runs in base 2 with a lazy rescale: O and l are rescaled only when a row's max
// grows by more than 2^8 (the softmax WG rescales O_i in TMEM itself: s_full of
// block n implies PV_{n-1} completed, and PV_n waits for this WG's p_full).
// A fraction of the exponentials runs as a Cody-Waite + cubic polynomial on the
// FMA pipe so MUFU.EX2 is not the only exp engine.
#pragma once

#include "psa_device.cuh"

#ifndef PSA_MMA_WAIT_SYNC
#define PSA_MMA_WAIT_SYNC 1
#endif

namespace psa {
namespace tile2 {

constexpr int kBN = 128;                  // keys per KV block (S tile N)
constexpr int kM = 128;                   // rows per slot (UMMA M)
constexpr int kD = 128;                   // d == dv
constexpr int kSlotBytes = kBN * kD * 2;  // one K or V block: 32 KB
constexpr int kQBytes = kM * kD * 2;      // one slot's Q tile: 32 KB
constexpr int kMaxRing = 6;
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kTmemO = 256;
constexpr float kRescaleThreshold = 8.0f;  // log2 units
constexpr int kProducerWarp = 8, kMmaWarp = 9, kMergeWarp0 = 10;
constexpr int kThreads = 512;

struct Shared {
  uint64_t item_full[2], item_empty[2];
  uint64_t q_full, q_empty;
  uint64_t ring_full[kMaxRing], ring_empty[kMaxRing];
  uint64_t s_full[2], p_full[2], o_full[2], o_empty[2];
  uint64_t pv_done;  // single-slot items: one phase per PV (the softmax's O-rescale wait)
  int item_idx[2];
  dev::MergeQueue mq;
};

__host__ __device__ constexpr size_t smem_bytes(int ring) {
  return size_t(2) * kQBytes + size_t(ring) * kSlotBytes + 1024;
}

__device__ __forceinline__ void init(Shared* s) {
  for (int i = 0; i < 2; ++i) {
    dev::mbar_init(&s->item_full[i], 1);
    dev::mbar_init(&s->item_empty[i], 3);  // MMA + WG0 + WG1
    dev::mbar_init(&s->s_full[i], 1);
    dev::mbar_init(&s->p_full[i], 4);
    dev::mbar_init(&s->o_full[i], 1);
    dev::mbar_init(&s->o_empty[i], 4);
  }
  dev::mbar_init(&s->pv_done, 1);
  dev::mbar_init(&s->q_full, 1);
  dev::mbar_init(&s->q_empty, 1);
  for (int i = 0; i < kMaxRing; ++i) {
    dev::mbar_init(&s->ring_full[i], 1);
    dev::mbar_init(&s->ring_empty[i], 1);
  }
  dev::mq_init(&s->mq);
  dev::fence_mbar_init();
}

struct Geo {
  uint8_t* base;  // 1024-aligned
  uint32_t ring;
  __device__ __forceinline__ uint8_t* q(int i) const { return base + i * kQBytes; }
  __device__ __forceinline__ uint8_t* slot(uint32_t s) const { return base + 2 * kQBytes + s * kSlotBytes; }
};

__device__ __forceinline__ Geo carve(uint8_t* smem_raw, int ring) {
  Geo g;
  g.ring = uint32_t(ring);
  g.base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                      ~uintptr_t(1023));
  return g;
}

template <typename T> __device__ __forceinline__ uint32_t pack2(float a, float b);
template <> __device__ __forceinline__ uint32_t pack2<__nv_bfloat16>(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}
template <> __device__ __forceinline__ uint32_t pack2<__half>(float a, float b) {
  __half2 h = __floats2half2_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}
template <typename T> struct AbFormat;
template <> struct AbFormat<__nv_bfloat16> { static constexpr uint32_t v = 1; };
template <> struct AbFormat<__half> { static constexpr uint32_t v = 0; };

__device__ __forceinline__ float max3(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}
// (a0, a1) * (b, b) + (c, c) on the packed fp32x2 FMA path.
__device__ __forceinline__ void ffma2(float& x0, float& x1, float a0, float a1, float b, float c) {
  uint64_t r;
  const uint64_t A = (uint64_t(__float_as_uint(a1)) << 32) | __float_as_uint(a0);
  const uint64_t B = (uint64_t(__float_as_uint(b)) << 32) | __float_as_uint(b);
  const uint64_t Cc = (uint64_t(__float_as_uint(c)) << 32) | __float_as_uint(c);
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(A), "l"(B), "l"(Cc));
  x0 = __uint_as_float(uint32_t(r));
  x1 = __uint_as_float(uint32_t(r >> 32));
}
__device__ __forceinline__ void fadd2(float& s0, float& s1, float a0, float a1) {
  uint64_t r;
  const uint64_t A = (uint64_t(__float_as_uint(a1)) << 32) | __float_as_uint(a0);
  const uint64_t S = (uint64_t(__float_as_uint(s1)) << 32) | __float_as_uint(s0);
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(S), "l"(A));
  s0 = __uint_as_float(uint32_t(r));
  s1 = __uint_as_float(uint32_t(r >> 32));
}

// Packed fp32x2 helpers with per-lane operands.
__device__ __forceinline__ uint64_t pk(float a0, float a1) {
  return (uint64_t(__float_as_uint(a1)) << 32) | __float_as_uint(a0);
}
__device__ __forceinline__ uint64_t fma2v(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ uint64_t add2v(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}

// 2^x for x <= 0 on the FMA pipe (two lanes): clamp to -126, x = j + f with
// j = round(x) (magic-number add), f in [-0.5, 0.5]; 2^f by a cubic
// (max rel. error 7.5e-5, far below the bf16 rounding of P), 2^j by adding j to
// the exponent field (t = x + 1.5 * 2^23 holds j in its low bits: t << 23 = j << 23).
__device__ __forceinline__ void exp2_poly2(float& y0, float& y1, float x0, float x1) {
  const float kMagic = 12582912.f;  // 1.5 * 2^23
  const uint64_t X = pk(fmaxf(x0, -126.f), fmaxf(x1, -126.f));
  const uint64_t T = add2v(X, pk(kMagic, kMagic));            // t = x + magic
  const uint64_t J = add2v(T, pk(-kMagic, -kMagic));          // j = round(x)
  const uint64_t F = fma2v(J, pk(-1.f, -1.f), X);              // f = x - j
  const float c3 = 0.05517132f, c2 = 0.24261054f, c1 = 0.69326099f, c0 = 0.99992811f;
  uint64_t P = fma2v(F, pk(c3, c3), pk(c2, c2));
  P = fma2v(P, F, pk(c1, c1));
  P = fma2v(P, F, pk(c0, c0));
  uint32_t r0, r1;
  asm("{\n\t.reg .b32 t0, t1, p0, p1;\n\t"
      "mov.b64 {t0, t1}, %2;\n\t"
      "mov.b64 {p0, p1}, %3;\n\t"
      "shl.b32 t0, t0, 23;\n\t"
      "shl.b32 t1, t1, 23;\n\t"
      "add.u32 %0, p0, t0;\n\t"
      "add.u32 %1, p1, t1;\n\t}"
      : "=r"(r0), "=r"(r1)
      : "l"(T), "l"(P));
  y0 = __uint_as_float(r0);
  y1 = __uint_as_float(r1);
}

// K/V ring positions of global block j. Interleaved (default): K_j = 2j, V_j = 2j + 1.
// Split ring (PSA_TILE_SPLIT_RING=1): K_j in slots [0, NR/2), V_j in [NR/2, NR), each a
// FIFO of its own, loaded in the MMA's consumption order, so a single-slot item's K
// loads never wait behind a V slot held until its PV completes. Measured: c2_prefix
// 40.2 -> 38.3 us but c2 130 -> 135 us (the earlier tile loads compete with the decode
// CTAs for HBM), c3 / c5 unchanged; left off.
#ifndef PSA_TILE_SPLIT_RING
#define PSA_TILE_SPLIT_RING 0
#endif
constexpr bool kSplitRing = PSA_TILE_SPLIT_RING != 0;
struct RingPos {
  uint32_t NR, NH;
  __device__ __forceinline__ explicit RingPos(uint32_t nr) : NR(nr), NH(nr / 2 > 0 ? nr / 2 : 1) {}
  __device__ __forceinline__ uint32_t kslot(uint32_t j) const { return kSplitRing ? j % NH : (2 * j) % NR; }
  __device__ __forceinline__ uint32_t vslot(uint32_t j) const {
    return kSplitRing ? NH + j % NH : (2 * j + 1) % NR;
  }
  __device__ __forceinline__ uint32_t kpar(uint32_t j) const {
    return kSplitRing ? (j / NH) & 1 : ((2 * j) / NR) & 1;
  }
  __device__ __forceinline__ uint32_t vpar(uint32_t j) const {
    return kSplitRing ? (j / NH) & 1 : ((2 * j + 1) / NR) & 1;
  }
};

struct Block {
  const CUtensorMap* km;
  const CUtensorMap* vm;
  bool prefix;
  int64_t base;  // segment base: packed key offset, or page-table offset (paged)
  int key;       // first key of the block within the segment
  int end;       // end of the item's keys within the segment
};

template <typename ItemT>
__device__ __forceinline__ Block block_at(const KParams& p, const ItemT& it, int jb, int nbA,
                                          int64_t pbase, int64_t dbase) {
  Block b;
  b.prefix = jb < nbA;
  if (b.prefix) {
    b.km = &p.tmd_kp;  // (64, 1, 128)-key boxes (paged: page-row boxes), 128-byte swizzle
    b.vm = &p.tmd_vp;
    b.base = pbase;
    b.key = it.pk0 + jb * kBN;
    b.end = it.pk1;
  } else {
    const int j = jb - nbA;
    b.km = &p.tmd_kd;
    b.vm = &p.tmd_vd;
    b.base = dbase;
    b.key = it.dk0 + j * kBN;
    b.end = it.dk1;
  }
  return b;
}

template <typename ItemT>
__device__ __forceinline__ void item_shape(const KParams& p, const ItemT& it, int& nbA, int& nb,
                                           int64_t& pbase, int64_t& dbase) {
  nbA = (it.pk1 - it.pk0 + kBN - 1) / kBN;
  nb = nbA + (it.dk1 - it.dk0 + kBN - 1) / kBN;
  pbase = nbA ? __ldg(p.group_pbase + it.g) : 0;
  dbase = (it.dk1 > it.dk0 && it.req >= 0) ? __ldg(p.req_dbase + it.req) : 0;
}

// Diagnostics: clock64 of per-block events of CTA 0 (first 64 blocks), slot 0.
// Slot = event * 64 + block, after the item records (psa_debug_set_trace).
__device__ __forceinline__ void dbg(const KParams& p, int ev, uint32_t g) {
  if (kTraceEvents && p.trace_cap > 0 && int(blockIdx.x) == p.dbg_cta && g < 64) {
    long long t;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(t));
    p.trace[(int64_t(p.num_items) + 4096) * 4 + ev * 64 + g] = t;
  }
}

__device__ __forceinline__ void named_sync(int id, int threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

// ---------------------------------------------------------------------------
// The tile phase. Returns when the TILE queue is drained and every role is done.
//   load_item(idx)       -> ItemRec
//   arrive(it, slot, r0, r1) : the slot's partial rows [r0, r1) are stored; the
//                              WG (128 threads, after a named barrier) arrives at
//                              the units inside that row range and queues merges
//   merge_unit(u)        : merge worker body (one warp)
// ---------------------------------------------------------------------------
// Roles are separate functions so the kernel can call each inside its own
// setmaxnreg region (ptxas sizes a region by the setmaxnreg that dominates it).
template <typename T, typename LoadItem>
__device__ void run_support(const KParams& p, uint8_t* smem_raw, Shared* sh, uint32_t tmem,
                            LoadItem&& load_item_at) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const Geo G = carve(smem_raw, p.tile_stages);
  const RingPos R(uint32_t(p.tile_stages));
  const int gqa = p.gqa;
  const int tile_rows = gqa * (kM / gqa);

  if (warp == kProducerWarp) {
    // ============================ producer ============================
    uint32_t cb = 0;  // K/V blocks issued (global block index j = cb + item block)
    for (uint32_t k = 0;; ++k) {
      const uint32_t q = k & 1;
      dev::mbar_wait(&sh->item_empty[q], ((k >> 1) & 1) ^ 1);
      int idx = 0;
      if (lane == 0) idx = atomicAdd(&p.ctrl->next_item, 1);
      idx = __shfl_sync(0xffffffffu, idx, 0);
      if (idx >= p.n_tile_items) {
        if (lane == 0) {
          sh->item_idx[q] = -1;
          dev::mbar_arrive(&sh->item_full[q]);
        }
        break;
      }
      if (lane == 0) {
        sh->item_idx[q] = idx;
        dev::mbar_arrive(&sh->item_full[q]);
        const auto it = load_item_at(idx);
        int nbA, nb;
        int64_t pbase, dbase;
        item_shape(p, it, nbA, nb, pbase, dbase);
        const bool two = it.nrows > tile_rows;
        // Q of both slots (the previous item's S MMAs have all completed)
        dev::mbar_wait(&sh->q_empty, (k & 1) ^ 1);
        const int t0 = int(__ldg(p.group_tok0 + it.g) + it.row0 / gqa);
        const uint32_t qbox = uint32_t(tile_rows) * kD * 2;
        dev::mbar_arrive_expect_tx(&sh->q_full, two ? 2 * qbox : qbox);
        for (int i = 0; i < (two ? 2 : 1); ++i)
          for (int ch = 0; ch < 2; ++ch)
            dev::tma_load_4d(G.q(i) + ch * (kM * 128), &p.tm_q, &sh->q_full, ch * 64, 0, it.h,
                             t0 + i * (kM / gqa));
        // K_j / V_j ring loads in the order the MMA issuer consumes them (a split ring
        // never blocks an earlier-needed load behind a later one)
        auto load = [&](int w, int jb) {
          const Block b = block_at(p, it, jb, nbA, pbase, dbase);
          const uint32_t j = cb + uint32_t(jb);
          const uint32_t s = w == 0 ? R.kslot(j) : R.vslot(j);
          dev::mbar_wait(&sh->ring_empty[s], (w == 0 ? R.kpar(j) : R.vpar(j)) ^ 1);
          dev::mbar_arrive_expect_tx(&sh->ring_full[s], kSlotBytes);
          dbg(p, 7 + w, j);
          load_kv_block(p, G.slot(s), w == 0 ? b.km : b.vm, &sh->ring_full[s], it.h, b.prefix,
                        b.base, b.key, b.end, b.key, kBN);  // tiles: forward boxes (no shift)
        };
        if (kSplitRing && !two && p.tile_pp != 0) {  // one slot: S(0), S(1), PV(0), S(2), PV(1) ...
          load(0, 0);
          for (int jb = 1; jb < nb; ++jb) {
            load(0, jb);
            load(1, jb - 1);
          }
          load(1, nb - 1);
        } else {
          for (int jb = 0; jb < nb; ++jb) {
            load(0, jb);
            load(1, jb);
          }
        }
        cb += uint32_t(nb);
      }
      __syncwarp();
    }
  } else if (warp == kMmaWarp) {
    // ============================ MMA issuer ============================
    if (PSA_MMA_WARP_WIDE || lane == 0) {
      // Warp-wide issue: every lane runs each barrier wait, then the warp reconverges
      // (PSA_MMA_WAIT_SYNC) before any lane acts on the phase it observed.
      auto mwait = [&](uint64_t* bar, uint32_t par) {
        dev::mbar_wait(bar, par);
        if (PSA_MMA_WARP_WIDE && PSA_MMA_WAIT_SYNC) __syncwarp();
      };
      constexpr uint32_t fmt = AbFormat<T>::v;
      const uint32_t idesc_s = dev::umma_idesc_f16(fmt, kM, kBN, 0, 0);
      const uint32_t idesc_o = dev::umma_idesc_f16(fmt, kM, kD, 0, 1);
      uint32_t gb = 0;       // K/V blocks consumed (ring position 2 * gb)
      uint32_t nblk[2] = {0u, 0u};  // p_full[b] phases consumed (either mode)
      uint32_t nitem[2] = {0u, 0u}; // items processed per slot (o_empty phases)
      for (uint32_t k = 0;; ++k) {
        const uint32_t q = k & 1;
        mwait(&sh->item_full[q], (k >> 1) & 1);
        const int idx = sh->item_idx[q];
        if (idx < 0) break;
        const auto it = load_item_at(idx);
        if (lane == 0) dev::mbar_arrive(&sh->item_empty[q]);
        int nbA, nb;
        int64_t pbase, dbase;
        item_shape(p, it, nbA, nb, pbase, dbase);
        const int ns = it.nrows > tile_rows ? 2 : 1;
        mwait(&sh->q_full, k & 1);
        dev::tc_fence_after();
        // O_o (+)= P V: 8 K-steps of 16 keys; A = P in TMEM (bf16 pairs) in S buffer pb
        auto issue_pv = [&](int pb, int o, uint32_t vslot, bool first) {
          const uint32_t v_addr = dev::smem_u32(G.slot(vslot));
          const uint32_t tP = tmem + uint32_t(pb) * 128, tO = tmem + kTmemO + uint32_t(o) * 128;
          const uint64_t b0 = dev::umma_desc_sw128(v_addr, kBN * 128, 1024);
#pragma unroll
          for (int kk = 0; kk < kBN / 16; ++kk) {  // descriptor start address is addr >> 4
            const uint64_t b = b0 + uint64_t((kk * (16 * 128)) >> 4);
            PSA_MMA_TS(tO, tP + kk * 8, b, idesc_o, (!first || kk > 0) ? 1u : 0u);
          }
        };
        // S buffer sb = Q_qi K^T
        auto issue_s = [&](int qi, int sb, uint32_t kslot) {
          const uint32_t k_addr = dev::smem_u32(G.slot(kslot));
          const uint32_t q_addr = dev::smem_u32(G.q(qi));
          const uint32_t tS = tmem + uint32_t(sb) * 128;
          const uint64_t a0 = dev::umma_desc_sw128(q_addr, 16, 1024);
          const uint64_t b0 = dev::umma_desc_sw128(k_addr, 16, 1024);
#pragma unroll
          for (int kk = 0; kk < kD / 16; ++kk) {
            const uint32_t ch = kk >> 2, w = (kk & 3) * 32;
            const uint64_t a = a0 + uint64_t((ch * (kM * 128) + w) >> 4);
            const uint64_t b = b0 + uint64_t((ch * (kBN * 128) + w) >> 4);
            PSA_MMA_SS(tS, a, b, idesc_s, kk > 0 ? 1u : 0u);
          }
          PSA_MMA_COMMIT(&sh->s_full[sb]);
        };
        if (ns == 2 || p.tile_pp == 0) {
          // two slots share every K/V block: per block n, slot i: PV_i(n-1) then S_i(n)
          // (S_i(n) overwrites P_i(n-1); MMAs of one thread execute in issue order)
          for (int n = 0; n < nb; ++n) {
            const uint32_t jK = gb + n, sK = R.kslot(jK);
            const uint32_t sV = R.vslot(jK - 1);  // V_{n-1}
            mwait(&sh->ring_full[sK], R.kpar(jK));
            if (n > 0) mwait(&sh->ring_full[sV], R.vpar(jK - 1));
            dev::tc_fence_after();
            for (int i = 0; i < ns; ++i) {
              if (n > 0) {
                if (n == 1) {  // first PV of this item overwrites O_i: the WG read the last one
                  mwait(&sh->o_empty[i], (nitem[i] & 1) ^ 1);
                }
                mwait(&sh->p_full[i], nblk[i] & 1);
                ++nblk[i];
                dev::tc_fence_after();
                dbg(p, i == 0 ? 6 : 13, gb + n - 1);
                issue_pv(i, i, sV, n == 1);
              }
              dbg(p, i == 0 ? 5 : 12, gb + n);
              issue_s(i, i, sK);
            }
            if (n > 0) PSA_MMA_COMMIT(&sh->ring_empty[sV]);
            PSA_MMA_COMMIT(&sh->ring_empty[sK]);
          }
          PSA_MMA_COMMIT(&sh->q_empty);  // every S of this item issued
          const uint32_t sV = R.vslot(gb + nb - 1);
          mwait(&sh->ring_full[sV], R.vpar(gb + nb - 1));
          for (int i = 0; i < ns; ++i) {
            if (nb == 1) mwait(&sh->o_empty[i], (nitem[i] & 1) ^ 1);
            mwait(&sh->p_full[i], nblk[i] & 1);
            ++nblk[i];
            dev::tc_fence_after();
            issue_pv(i, i, sV, nb == 1);
            PSA_MMA_COMMIT(&sh->o_full[i]);
            ++nitem[i];
          }
          PSA_MMA_COMMIT(&sh->ring_empty[sV]);
        } else {
          // one slot: S ping-pongs between both S buffers (block n -> buffer n & 1), so
          // S(n + 1) is computed while the softmax works on block n. Order: S(0), S(1),
          // PV(0), S(2), PV(1), ...: S(n) overwrites P(n - 2) after PV(n - 2) was issued.
          for (int n = 0; n < nb; ++n) {
            const uint32_t jK = gb + n, sK = R.kslot(jK);
            mwait(&sh->ring_full[sK], R.kpar(jK));
            dev::tc_fence_after();
            dbg(p, 5, gb + n);
            issue_s(0, n & 1, sK);
            PSA_MMA_COMMIT(&sh->ring_empty[sK]);
            if (n == nb - 1) PSA_MMA_COMMIT(&sh->q_empty);  // every S of this item issued
            if (n > 0) {
              const uint32_t sV = R.vslot(jK - 1);  // V_{n-1}
              mwait(&sh->ring_full[sV], R.vpar(jK - 1));
              if (n == 1) mwait(&sh->o_empty[0], (nitem[0] & 1) ^ 1);
              const int b = (n - 1) & 1;
              mwait(&sh->p_full[b], nblk[b] & 1);
              ++nblk[b];
              dev::tc_fence_after();
              dbg(p, 6, gb + n - 1);
              issue_pv(b, 0, sV, n == 1);
              PSA_MMA_COMMIT(&sh->pv_done);
              PSA_MMA_COMMIT(&sh->ring_empty[sV]);
            }
          }
          const uint32_t sV = R.vslot(gb + nb - 1);  // V_{nb-1}
          mwait(&sh->ring_full[sV], R.vpar(gb + nb - 1));
          if (nb == 1) mwait(&sh->o_empty[0], (nitem[0] & 1) ^ 1);
          const int b = (nb - 1) & 1;
          mwait(&sh->p_full[b], nblk[b] & 1);
          ++nblk[b];
          dev::tc_fence_after();
          issue_pv(b, 0, sV, nb == 1);
          PSA_MMA_COMMIT(&sh->pv_done);
          PSA_MMA_COMMIT(&sh->o_full[0]);
          ++nitem[0];
          PSA_MMA_COMMIT(&sh->ring_empty[sV]);
        }
        gb += nb;
      }
    }
  }
}

template <typename T, int kEmuEvery, bool kCausal, typename LoadItem>
__device__ void run_softmax(const KParams& p, Shared* sh, uint32_t tmem, LoadItem&& load_item_at) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gqa = p.gqa;
  const int tile_rows = gqa * (kM / gqa);
  {
    // ============================ softmax WG i ============================
    const int i = warp >> 2;
    const int row = threadIdx.x & 127;
    const uint32_t lane_base = uint32_t((warp & 3) * 32) << 16;
    const uint32_t tO = tmem + kTmemO + uint32_t(i) * 128 + lane_base;
    const float sc = float(p.scale) * 1.4426950408889634f;
    uint32_t nblk = 0, nitem = 0;
    // s_full[b] phases consumed as seen by this WG (the other WG / mode consumes some
    // of buffer 1's), and pv_done phases of single-slot items before the current one
    uint32_t hs[2] = {0u, 0u}, npv = 0;
    for (uint32_t k = 0;; ++k) {
      const uint32_t q = k & 1;
      dev::mbar_wait(&sh->item_full[q], (k >> 1) & 1);
      const int idx = sh->item_idx[q];
      if (idx < 0) break;
      const auto it = load_item_at(idx);
      long long t_item0 = 0;
      if (p.trace_cap > 0 && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_item0));
      named_sync(2 + i, 128);  // every thread of the WG has read item_idx[q]
      if (threadIdx.x % 128 == 0) dev::mbar_arrive(&sh->item_empty[q]);
      const int slot_rows = i == 0 ? min(it.nrows, tile_rows) : it.nrows - tile_rows;
      int nbA, nb;
      int64_t pbase, dbase;
      item_shape(p, it, nbA, nb, pbase, dbase);
      const bool two = it.nrows > tile_rows;
      const bool pp = !two && p.tile_pp != 0;  // single slot: S ping-pong over both buffers
      if (slot_rows <= 0) {  // WG1, single-slot item: WG0 uses S buffer 1 for odd blocks
        if (pp) hs[1] += uint32_t(nb) >> 1;
        continue;
      }
      float m = -INFINITY, l0 = 0.f, l1 = 0.f;
      const bool warp_rows = (warp & 3) * 32 < slot_rows;  // this warp has a valid row
      // causal prefill (PSA_FLAG_CAUSAL): last visible prefix / distinct key of this row
      constexpr bool causal = kCausal;  // a separate kernel: no cost when off
      int limp = INT_MAX, limd = INT_MAX;
      if (causal && row < slot_rows) {
        const int64_t tok = __ldg(p.group_tok0 + it.g) + (it.row0 + i * tile_rows + row) / gqa;
        limp = __ldg(p.tok_lim + tok * 2);
        limd = __ldg(p.tok_lim + tok * 2 + 1);
      }
      for (int n = 0; n < nb; ++n, ++nblk) {
        const int nvalid = n < nbA ? min(kBN, it.pk1 - it.pk0 - n * kBN)
                                   : min(kBN, it.dk1 - it.dk0 - (n - nbA) * kBN);
        const int b = pp ? (n & 1) : i;  // S buffer of this block
        dev::mbar_wait(&sh->s_full[b], hs[b] & 1);
        ++hs[b];
        if (!warp_rows) {
          // every row of this warp is past the slot's rows (small groups): keep the
          // barrier pace (one p_full arrival per block, after this block's S) and skip
          // the softmax — its P rows feed only output rows that are never written
          __syncwarp();
          if (lane == 0) dev::mbar_arrive(&sh->p_full[b]);
          continue;
        }
        const uint32_t tS = tmem + uint32_t(b) * 128 + lane_base;
        const bool ev = threadIdx.x == 0;
        if (ev) dbg(p, 0, nblk);
        if (threadIdx.x == 128) dbg(p, 9, nblk);
        dev::tc_fence_after();
        uint32_t r[4][32];
        dev::tmem_ld32(tS + 0, r[0]);
        dev::tmem_ld32(tS + 32, r[1]);
        dev::tmem_ld32(tS + 64, r[2]);
        dev::tmem_ld32(tS + 96, r[3]);
        dev::tmem_wait_ld();
        if (ev) dbg(p, 1, nblk);
        int ncut = nvalid;  // columns >= ncut are masked
        if constexpr (causal) {
          const int key0 = n < nbA ? it.pk0 + n * kBN : it.dk0 + (n - nbA) * kBN;
          ncut = min(ncut, max(0, (n < nbA ? limp : limd) - key0 + 1));
        }
        if (ncut < kBN) {
#pragma unroll
          for (int c = 0; c < 4; ++c)
#pragma unroll
            for (int e = 0; e < 32; ++e)
              if (c * 32 + e >= ncut) r[c][e] = 0xff800000u;
        }
#ifdef PSA_EXP_SKIP  // timing diagnostics only (results wrong): no max / exp work
        const float mraw = 0.f;
#else
        // row max of the raw scores (scale > 0): 8 independent FMNMX3 chains
        float a8[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const uint32_t* v = &r[j >> 1][(j & 1) * 16];
          float acc = fmaxf(__uint_as_float(v[0]), __uint_as_float(v[1]));
#pragma unroll
          for (int e = 2; e < 16; e += 2) acc = max3(acc, __uint_as_float(v[e]), __uint_as_float(v[e + 1]));
          a8[j] = acc;
        }
        const float mraw = max3(max3(a8[0], a8[1], a8[2]), max3(a8[3], a8[4], a8[5]), fmaxf(a8[6], a8[7]));
#endif
        const float mb = mraw * sc;
        if (ev) dbg(p, 2, nblk);
        float alpha = 1.f;
        bool rescale = false;
        if (m == -INFINITY) {
          m = mb;
        } else if (mb > m + kRescaleThreshold) {
          alpha = dev::ex2(m - mb);
          m = mb;
          rescale = true;
        }
        l0 *= alpha;
        l1 *= alpha;
        const float nm = m == -INFINITY ? 0.f : -m;  // a row masked so far: P = 0
        // P = 2^(s*sc - m), packed bf16 pairs into r[c][0..15]; sums in (l0, l1)
#pragma unroll
        for (int c = 0; c < 4; ++c) {
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            float x0, x1, y0, y1;
#ifdef PSA_EXP_SKIP
            y0 = __uint_as_float(r[c][2 * e]); y1 = __uint_as_float(r[c][2 * e + 1]);
            r[c][e] = pack2<T>(y0, y1);
            continue;
#endif
            ffma2(x0, x1, __uint_as_float(r[c][2 * e]), __uint_as_float(r[c][2 * e + 1]), sc, nm);
            if (kEmuEvery > 0 && ((c * 16 + e) % kEmuEvery) == kEmuEvery - 1) {
              exp2_poly2(y0, y1, x0, x1);
            } else {
              y0 = dev::ex2(x0);
              y1 = dev::ex2(x1);
            }
            fadd2(l0, l1, y0, y1);
            r[c][e] = pack2<T>(y0, y1);
          }
        }
        if (ev) dbg(p, 3, nblk);
        if (threadIdx.x == 128) dbg(p, 10, nblk);
        // P_n -> S_i columns [0, 64)
        {
          uint32_t hi[32];
#pragma unroll
          for (int e = 0; e < 16; ++e) { hi[e] = r[2][e]; hi[16 + e] = r[3][e]; }
          uint32_t lo[32];
#pragma unroll
          for (int e = 0; e < 16; ++e) { lo[e] = r[0][e]; lo[16 + e] = r[1][e]; }
          dev::tmem_st32(tS + 0, lo);
          dev::tmem_st32(tS + 32, hi);
        }
        if (__any_sync(0xffffffffu, rescale)) {
          // O_i must hold PV(0 .. n-1) complete. Two slots: S_i(n) was issued after
          // PV_i(n-1). One slot: S(n) only follows PV(n-2), so wait for PV(n-1) (PV(n)
          // waits for this WG's p_full, so the parity cannot alias).
          if (pp && n > 0) {
            dev::mbar_wait(&sh->pv_done, (npv + uint32_t(n) - 1) & 1);
            dev::tc_fence_after();
          }
#pragma unroll 1
          for (int c = 0; c < kD; c += 32) {
            uint32_t o[32];
            dev::tmem_ld32(tO + c, o);
            dev::tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * alpha);
            dev::tmem_st32(tO + c, o);
          }
        }
        dev::tmem_wait_st();
        dev::tc_fence_before();
        __syncwarp();
        if (lane == 0) dev::mbar_arrive(&sh->p_full[b]);
        if (ev) dbg(p, 4, nblk);
        if (threadIdx.x == 128) dbg(p, 11, nblk);
      }
      if (two) {
        if (i == 0) hs[1] += uint32_t(nb);  // WG1 consumed buffer 1's phases
      } else if (pp) {
        npv += uint32_t(nb);
      }
      // ---------------- epilogue: O_i -> output / partial ----------------
      dev::mbar_wait(&sh->o_full[i], nitem & 1);
      ++nitem;
      dev::tc_fence_after();
      const float l = l0 + l1;
      const int slot_row0 = it.row0 + i * tile_rows;
      const bool valid = row < slot_rows;
      const bool partial_out = p.flags & PSA_FLAG_PARTIAL_OUT;
      if (it.ws_row >= 0) {
        float* wo = static_cast<float*>(p.ws_o) + ((int64_t)it.ws_row + i * tile_rows + row) * kD;
#pragma unroll 1
        for (int c = 0; c < kD; c += 32) {
          uint32_t o[32];
          dev::tmem_ld32(tO + c, o);
          dev::tmem_wait_ld();
          if (c == kD - 32) {
            dev::tc_fence_before();
            __syncwarp();
            if (lane == 0) dev::mbar_arrive(&sh->o_empty[i]);
          }
          if (valid) {
#pragma unroll
            for (int e = 0; e < 32; e += 4)
              *reinterpret_cast<float4*>(wo + c + e) =
                  make_float4(__uint_as_float(o[e]), __uint_as_float(o[e + 1]),
                              __uint_as_float(o[e + 2]), __uint_as_float(o[e + 3]));
          }
        }
        if (valid)
          *reinterpret_cast<float2*>(static_cast<float*>(p.ws_ml) +
                                     ((int64_t)it.ws_row + i * tile_rows + row) * 2) = make_float2(m, l);
        // publish the slot's partial rows to the merge warps, which arrive at the
        // units they cover (and merge or queue the units they complete)
        named_sync(2 + i, 128);
        if ((threadIdx.x & 127) == 0) dev::mq_push(&sh->mq, 2 * idx + i);
      } else {
        const int grow = slot_row0 + row;
        const int64_t tok = __ldg(p.group_tok0 + it.g) + grow / gqa;
        const int64_t oidx = tok * p.Hq + (int64_t)it.h * gqa + grow % gqa;
        const float inv = 1.f / l;
#pragma unroll 1
        for (int c = 0; c < kD; c += 32) {
          uint32_t o[32];
          dev::tmem_ld32(tO + c, o);
          dev::tmem_wait_ld();
          if (c == kD - 32) {
            dev::tc_fence_before();
            __syncwarp();
            if (lane == 0) dev::mbar_arrive(&sh->o_empty[i]);
          }
          if (!valid) continue;
          if (partial_out) {
            float* dst = static_cast<float*>(p.out) + oidx * kD + c;
#pragma unroll
            for (int e = 0; e < 32; e += 4)
              *reinterpret_cast<float4*>(dst + e) =
                  make_float4(__uint_as_float(o[e]), __uint_as_float(o[e + 1]),
                              __uint_as_float(o[e + 2]), __uint_as_float(o[e + 3]));
          } else {
            uint8_t* dst = reinterpret_cast<uint8_t*>(static_cast<T*>(p.out) + oidx * kD + c);
#pragma unroll
            for (int e = 0; e < 32; e += 8) {
              uint4 v;
              v.x = pack2<T>(__uint_as_float(o[e]) * inv, __uint_as_float(o[e + 1]) * inv);
              v.y = pack2<T>(__uint_as_float(o[e + 2]) * inv, __uint_as_float(o[e + 3]) * inv);
              v.z = pack2<T>(__uint_as_float(o[e + 4]) * inv, __uint_as_float(o[e + 5]) * inv);
              v.w = pack2<T>(__uint_as_float(o[e + 6]) * inv, __uint_as_float(o[e + 7]) * inv);
              *reinterpret_cast<uint4*>(dst + e * 2) = v;
            }
          }
        }
        if (valid) {
          if (partial_out) {
            static_cast<float*>(p.m_out)[oidx] = m * 0.6931471805599453f;
            static_cast<float*>(p.l_out)[oidx] = l;
          } else {
            if (!(l > 0.f)) atomicOr(&p.ctrl->error, 1);
            if (p.lse) p.lse[oidx] = (m + log2f(l)) * 0.6931471805599453f;
          }
        }
      }
      if (p.trace_cap > 0 && threadIdx.x == 0 && idx < p.trace_cap) {  // diagnostics
        long long t1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
        uint32_t smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        int64_t* tr = p.trace + int64_t(idx) * 4;
        tr[0] = int64_t(blockIdx.x) | (int64_t(smid) << 32);
        tr[1] = 1;
        tr[2] = t_item0;
        tr[3] = t1;
      }
    }
    // this WG will not queue more merges
    named_sync(2 + i, 128);
    if ((threadIdx.x & 127) == 0) dev::mq_close(&sh->mq);
  }
}

}  // namespace tile2
}  // namespace psa
