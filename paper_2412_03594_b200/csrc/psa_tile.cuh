// psa_tile.cuh — TILE work items: a 128-row tile of stacked query rows of one
// (group, kv head) against a KV range, on the 5th-gen tensor cores.
//
// This is the "matrix-vector -> matrix-matrix" transformation of the paper's
// §2.2 (reference: the stacked prefix call, attention.py:174-179): all gqa
// heads x tokens of a group's requests that share the prefix form the M=128
// rows of one tcgen05 tile, so each prefix K/V byte fetched from HBM feeds
// 128 rows.
//
// Per CTA (256 threads) the roles are:
//   warps 0-3  softmax + epilogue: thread t owns row t == TMEM lane t
//   warp 4     TMA producer (one lane): Q tile once, then K and V blocks into
//              two independent 2-stage rings
//   warp 5     MMA issuer (one lane): S = Q K^T (A, B from smem) and
//              O += P V (A = P from TMEM, B = V from smem) with tcgen05.mma
// TMEM (256 columns per CTA, 2 CTAs/SM): S [0, 64), P (bf16 pairs) double-buffered
// [64, 96) / [96, 128), O [128, 128+dv). Shared memory (d = dv = 128): Q 32 KB, K 2 x 16 KB,
// V 2 x 16 KB.
//
// Pipelining: a K stage is released as soon as S_j = Q K_j^T has completed and
// a V stage once O += P_j V_j has, so the producer streams K a block ahead of
// V and never waits for the softmax; in steady state the MMA issuer never
// waits on a fresh TMA.
//
// Online softmax (attention.py:95-98 per block, merge :101-119 across blocks)
// runs in base 2 with a lazy rescale: O and l are rescaled only when a row's
// max grows by more than 2^8, so the common case never touches O in TMEM.
#pragma once

#include "psa_device.cuh"

namespace psa {
namespace tile {

constexpr int kBN = 64;          // keys per KV block (S tile N)
constexpr int kM = 128;          // rows per tile (UMMA M)
constexpr int kMaxStages = 4;    // K/V ring depth: p.tile_stages (2 with 2 CTAs/SM, 4 with 1)
constexpr uint32_t kTmemCols = 256;
constexpr uint32_t kTmemS = 0;
constexpr uint32_t kTmemP = 64;   // two P buffers: [64, 96) and [96, 128)
constexpr uint32_t kTmemO = 128;
constexpr float kRescaleThreshold = 8.0f;  // log2 units

struct Barriers {
  uint64_t q_full;
  uint64_t k_full[kMaxStages];
  uint64_t v_full[kMaxStages];
  uint64_t k_empty[kMaxStages];
  uint64_t v_empty[kMaxStages];
  uint64_t s_full;
  uint64_t s_free;
  uint64_t p_full[2];        // by block parity, so a fast softmax can never lap the MMA waiter
  uint64_t o_done[2];        // PV_n completes phase n >> 1 of o_done[n & 1]
};

// Running phase bookkeeping, identical in every thread of the CTA.
struct State {
  uint32_t blocks;  // KV blocks processed by this CTA's TILE items so far
  uint32_t items;   // TILE items processed so far
  uint32_t tmem;    // TMEM base address
};

__host__ __device__ constexpr size_t smem_bytes(int d, int dv, int stages) {
  // Q + stages * (K + V) + 1 KB alignment slack
  return size_t(kM) * d * 2 + size_t(stages) * kBN * (d + dv) * 2 + 1024;
}

__device__ __forceinline__ void init_barriers(Barriers* b) {
  dev::mbar_init(&b->q_full, 1);
  for (int s = 0; s < kMaxStages; ++s) {
    dev::mbar_init(&b->k_full[s], 1);
    dev::mbar_init(&b->v_full[s], 1);
    dev::mbar_init(&b->k_empty[s], 1);
    dev::mbar_init(&b->v_empty[s], 1);
  }
  dev::mbar_init(&b->p_full[0], 4);
  dev::mbar_init(&b->p_full[1], 4);
  dev::mbar_init(&b->s_full, 1);
  dev::mbar_init(&b->s_free, 4);
  dev::mbar_init(&b->o_done[0], 1);
  dev::mbar_init(&b->o_done[1], 1);
  dev::fence_mbar_init();
}

// Shared-memory layout, computed arithmetically (no runtime-indexed arrays:
// those would live in local memory).
struct Layout {
  uint8_t* base;     // 1024-aligned
  uint32_t q_bytes;  // kM * d * 2
  uint32_t k_bytes;  // kBN * d * 2
  uint32_t v_bytes;  // kBN * dv * 2
  uint32_t stages;
  __device__ __forceinline__ uint8_t* q() const { return base; }
  __device__ __forceinline__ uint8_t* k(uint32_t s) const { return base + q_bytes + s * k_bytes; }
  __device__ __forceinline__ uint8_t* v(uint32_t s) const {
    return base + q_bytes + stages * k_bytes + s * v_bytes;
  }
};

__device__ __forceinline__ Layout carve(uint8_t* smem_raw, int d, int dv, int stages) {
  Layout L;
  L.stages = uint32_t(stages);
  L.base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                      ~uintptr_t(1023));
  L.q_bytes = kM * d * 2;
  L.k_bytes = kBN * d * 2;
  L.v_bytes = kBN * dv * 2;
  return L;
}

// bf16/f16 pack of two floats
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

struct Block {
  const CUtensorMap* km;
  const CUtensorMap* vm;
  int key;     // first key row in the K/V tensor
  int nvalid;  // valid keys in this block (<= kBN)
};

template <typename ItemT>
__device__ __forceinline__ Block block_at(const KParams& p, const ItemT& it, int jb, int nbA,
                                          int64_t pbase, int64_t dbase) {
  Block b;
  if (jb < nbA) {
    b.km = &p.tm_kp;
    b.vm = &p.tm_vp;
    b.key = int(pbase + it.pk0 + jb * kBN);
    b.nvalid = min(kBN, it.pk1 - it.pk0 - jb * kBN);
  } else {
    const int j = jb - nbA;
    b.km = &p.tm_kd;
    b.vm = &p.tm_vd;
    b.key = int(dbase + it.dk0 + j * kBN);
    b.nvalid = min(kBN, it.dk1 - it.dk0 - j * kBN);
  }
  return b;
}

// Diagnostics: clock64 timestamps of the first tile item of CTA 0, written after
// the trace records (psa_debug_set_trace). Slot = event * 64 + block.
enum DbgEvent { kEvProdIssue = 0, kEvSIssue, kEvSoftWait, kEvPArrive, kEvPvIssue, kEvMisc,
                kEvKWaitStart, kEvVWaitStart, kEvVIssue };
__device__ __forceinline__ void dbg_event(const KParams& p, const State& st, int ev, int n) {
  if (p.trace_cap > 0 && blockIdx.x == 0 && st.items == 0 && n < 64) {
    long long t;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(t));
    p.trace[(int64_t(p.num_items) + 4096) * 4 + ev * 64 + n] = t;
  }
}

template <typename T, typename ItemT>
__device__ __forceinline__ State tile_item(const KParams& p, const ItemT& it, uint8_t* smem_raw,
                                           Barriers* bar, State st) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int d = p.d, dv = p.dv;
  const Layout L = carve(smem_raw, d, dv, p.tile_stages);
  const uint32_t NS = uint32_t(p.tile_stages);
  const int nbA = (it.pk1 - it.pk0 + kBN - 1) / kBN;
  const int nbB = (it.dk1 - it.dk0 + kBN - 1) / kBN;
  const int nb = nbA + nbB;
  const int64_t pbase = nbA ? __ldg(p.group_pbase + it.g) : 0;
  const int64_t dbase = (it.req >= 0) ? __ldg(p.req_dbase + it.req) : 0;
  const uint32_t base_blk = st.blocks;
  const int gqa = p.gqa;
  const int tokens_per_tile = kM / gqa;
  const uint32_t k_bytes = kBN * d * 2, v_bytes = kBN * dv * 2;

  if (threadIdx.x == 0) dbg_event(p, st, kEvMisc, 2);
  if (warp == 4) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      const int t_start = int(__ldg(p.group_tok0 + it.g) + it.row0 / gqa);
      dev::mbar_arrive_expect_tx(&bar->q_full, uint32_t(tokens_per_tile * gqa) * d * 2);
      for (int c = 0; c < d / 64; ++c)
        dev::tma_load_4d(L.q() + c * (kM * 128), &p.tm_q, &bar->q_full, c * 64, 0, it.h, t_start);
      auto load_k = [&](int jb) {
        const uint32_t n = base_blk + jb, s = n % NS, ph = (n / NS) & 1;
        const Block b = block_at(p, it, jb, nbA, pbase, dbase);
        dbg_event(p, st, kEvKWaitStart, jb);
        dev::mbar_wait(&bar->k_empty[s], ph ^ 1);  // S_{n-2} has consumed this stage
        dbg_event(p, st, kEvProdIssue, jb);
        dev::mbar_arrive_expect_tx(&bar->k_full[s], k_bytes);
        for (int c = 0; c < d / 64; ++c)
          dev::tma_load_3d(L.k(s) + c * (kBN * 128), b.km, &bar->k_full[s], c * 64, it.h, b.key);
      };
      auto load_v = [&](int jb) {
        const uint32_t n = base_blk + jb, s = n % NS, ph = (n / NS) & 1;
        const Block b = block_at(p, it, jb, nbA, pbase, dbase);
        dbg_event(p, st, kEvVWaitStart, jb);
        dev::mbar_wait(&bar->v_empty[s], ph ^ 1);  // PV_{n-2} has consumed this stage
        dbg_event(p, st, kEvVIssue, jb);
        dev::mbar_arrive_expect_tx(&bar->v_full[s], v_bytes);
        for (int c = 0; c < dv / 64; ++c)
          dev::tma_load_3d(L.v(s) + c * (kBN * 128), b.vm, &bar->v_full[s], c * 64, it.h, b.key);
      };
      // K runs one block ahead of V: K_{j+1} is requested before V_j.
      load_k(0);
      for (int jb = 0; jb < nb; ++jb) {
        if (jb + 1 < nb) load_k(jb + 1);
        load_v(jb);
      }
    }
  } else if (warp == 5) {
    // ---------------- MMA issuer ----------------
    if (lane == 0) {
      constexpr uint32_t fmt = AbFormat<T>::v;
      const uint32_t idesc_s = dev::umma_idesc_f16(fmt, kM, kBN, 0, 0);
      const uint32_t idesc_o = dev::umma_idesc_f16(fmt, kM, uint32_t(dv), 0, 1);
      const uint32_t tS = st.tmem + kTmemS, tP = st.tmem + kTmemP, tO = st.tmem + kTmemO;
      const uint32_t q_addr = dev::smem_u32(L.q());
      dev::mbar_wait(&bar->q_full, st.items & 1);
      dev::tc_fence_after();
      auto issue_s = [&](int jb) {
        const uint32_t n = base_blk + jb, s = n % NS;
        dev::mbar_wait(&bar->k_full[s], (n / NS) & 1);
        dev::tc_fence_after();
        const uint32_t k_addr = dev::smem_u32(L.k(s));
        dbg_event(p, st, kEvSIssue, jb);
        for (int kk = 0; kk < d / 16; ++kk) {
          const uint32_t c = kk >> 2, w = (kk & 3) * 32;
          const uint64_t a = dev::umma_desc_sw128(q_addr + c * (kM * 128) + w, 16, 1024);
          const uint64_t b = dev::umma_desc_sw128(k_addr + c * (kBN * 128) + w, 16, 1024);
          dev::mma_f16_ss(tS, a, b, idesc_s, kk > 0);
        }
        dev::mma_commit(&bar->s_full);
        dev::mma_commit(&bar->k_empty[s]);
      };
      issue_s(0);
      for (int jb = 0; jb < nb; ++jb) {
        const uint32_t n = base_blk + jb, s = n % NS, pb = n & 1;
        if (jb + 1 < nb) {
          dev::mbar_wait(&bar->s_free, n & 1);  // S_n is in registers: S TMEM reusable
          dev::tc_fence_after();
          issue_s(jb + 1);
        }
        dev::mbar_wait(&bar->p_full[pb], (n >> 1) & 1);
        dev::mbar_wait(&bar->v_full[s], (n / NS) & 1);
        dev::tc_fence_after();
        const uint32_t v_addr = dev::smem_u32(L.v(s));
        dbg_event(p, st, kEvPvIssue, jb);
        for (int kk = 0; kk < kBN / 16; ++kk) {
          const uint64_t b = dev::umma_desc_sw128(v_addr + kk * (16 * 128), kBN * 128, 1024);
          dev::mma_f16_ts(tO, tP + pb * 32 + kk * 8, b, idesc_o, (jb > 0 || kk > 0));
        }
        dev::mma_commit(&bar->v_empty[s]);
        dev::mma_commit(&bar->o_done[n & 1]);
      }
    }
  } else if (warp < 4) {
    // ---------------- softmax + epilogue (row = threadIdx.x) ----------------
    const int row = threadIdx.x;
    const uint32_t lane_base = uint32_t(warp * 32) << 16;
    const uint32_t tS = st.tmem + kTmemS + lane_base, tP = st.tmem + kTmemP + lane_base;
    const uint32_t tO = st.tmem + kTmemO + lane_base;
    const float sc = float(p.scale) * 1.4426950408889634f;
    float m = -INFINITY, l = 0.f;
    for (int jb = 0; jb < nb; ++jb) {
      const uint32_t n = base_blk + jb, s = n & 1;  // s: P buffer / p_full parity
      const Block b = block_at(p, it, jb, nbA, pbase, dbase);
      dev::mbar_wait(&bar->s_full, n & 1);
      if (threadIdx.x == 0) dbg_event(p, st, kEvSoftWait, jb);
      dev::tc_fence_after();
      uint32_t r0[32], r1[32];
      dev::tmem_ld32(tS, r0);
      dev::tmem_ld32(tS + 32, r1);
      dev::tmem_wait_ld();
      dev::tc_fence_before();
      __syncwarp();
      if (lane == 0) dev::mbar_arrive(&bar->s_free);
      // Raw S stays in r0/r1 (no second copy: keeps the softmax warps spill-free);
      // masked keys become -inf in place. scale > 0, so max(s) * sc == max(s * sc).
      if (b.nvalid < kBN) {
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          if (i >= b.nvalid) r0[i] = 0xff800000u;
          if (32 + i >= b.nvalid) r1[i] = 0xff800000u;
        }
      }
      float mraw = __uint_as_float(r0[0]);
#pragma unroll
      for (int i = 1; i < 32; ++i) mraw = fmaxf(mraw, __uint_as_float(r0[i]));
#pragma unroll
      for (int i = 0; i < 32; ++i) mraw = fmaxf(mraw, __uint_as_float(r1[i]));
      const float mb = mraw * sc;
      float alpha = 1.f;
      bool rescale = false;
      if (m == -INFINITY) {
        m = mb;
      } else if (mb > m + kRescaleThreshold) {
        alpha = dev::ex2(m - mb);
        m = mb;
        rescale = true;
      }
      l *= alpha;
      // P_n (bf16 pairs) replaces S_n's registers in place: r0[i] = pack(p_2i, p_2i+1).
      const float nm = -m;
      float l4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const float e0 = dev::ex2(fmaf(__uint_as_float(r0[2 * i]), sc, nm));
        const float e1 = dev::ex2(fmaf(__uint_as_float(r0[2 * i + 1]), sc, nm));
        l4[i & 3] += e0 + e1;
        r0[i] = pack2<T>(e0, e1);
      }
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const float e0 = dev::ex2(fmaf(__uint_as_float(r1[2 * i]), sc, nm));
        const float e1 = dev::ex2(fmaf(__uint_as_float(r1[2 * i + 1]), sc, nm));
        l4[i & 3] += e0 + e1;
        r0[16 + i] = pack2<T>(e0, e1);
      }
      l += (l4[0] + l4[1]) + (l4[2] + l4[3]);
      // P is double-buffered in TMEM (P_n in buffer n & 1): PV_{n-2} finished with it
      // before S_n could be computed... except across the wait below, which also
      // orders the rare O rescale after PV_{n-1}.
      if (jb > 1) {
        dev::mbar_wait(&bar->o_done[n & 1], ((n - 2) >> 1) & 1);
        dev::tc_fence_after();
      }
      dev::tmem_st32(tP + s * 32, r0);
      if (__any_sync(0xffffffffu, rescale)) {
        // O holds PV_0..PV_{n-1}: scale rows in place before PV_n accumulates.
        dev::mbar_wait(&bar->o_done[(n - 1) & 1], ((n - 1) >> 1) & 1);
        dev::tc_fence_after();
        for (int c = 0; c < dv; c += 32) {
          uint32_t o[32];
          dev::tmem_ld32(tO + c, o);
          dev::tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
          dev::tmem_st32(tO + c, o);
        }
      }
      dev::tmem_wait_st();
      dev::tc_fence_before();
      __syncwarp();
      if (lane == 0) dev::mbar_arrive(&bar->p_full[s]);
      if (threadIdx.x == 0) dbg_event(p, st, kEvPArrive, jb);
    }
    if (threadIdx.x == 0) dbg_event(p, st, kEvMisc, 0);
    // ---------------- epilogue ----------------
    {
      const uint32_t last = base_blk + nb - 1;
      dev::mbar_wait(&bar->o_done[last & 1], (last >> 1) & 1);
    }
    dev::tc_fence_after();
    const bool valid = row < it.nrows;
    if (it.ws_row >= 0) {
      float* wo = static_cast<float*>(p.ws_o) + ((int64_t)it.ws_row + row) * dv;
      for (int c = 0; c < dv; c += 32) {
        uint32_t o[32];
        dev::tmem_ld32(tO + c, o);
        dev::tmem_wait_ld();
        if (valid) {
#pragma unroll
          for (int i = 0; i < 32; i += 4)
            *reinterpret_cast<float4*>(wo + c + i) =
                make_float4(__uint_as_float(o[i]), __uint_as_float(o[i + 1]),
                            __uint_as_float(o[i + 2]), __uint_as_float(o[i + 3]));
        }
      }
      if (valid) {
        float* ml = static_cast<float*>(p.ws_ml) + ((int64_t)it.ws_row + row) * 2;
        ml[0] = m;
        ml[1] = l;
      }
    } else {
      const int grow = it.row0 + row;
      const int64_t tok = __ldg(p.group_tok0 + it.g) + grow / gqa;
      const int64_t idx = tok * p.Hq + (int64_t)it.h * gqa + grow % gqa;
      const bool partial_out = p.flags & PSA_FLAG_PARTIAL_OUT;
      const float inv = 1.f / l;
      for (int c = 0; c < dv; c += 32) {
        uint32_t o[32];
        dev::tmem_ld32(tO + c, o);
        dev::tmem_wait_ld();
        if (!valid) continue;
        if (partial_out) {
          float* dst = static_cast<float*>(p.out) + idx * dv + c;
#pragma unroll
          for (int i = 0; i < 32; ++i) dst[i] = __uint_as_float(o[i]);
        } else {
          uint8_t* dst = reinterpret_cast<uint8_t*>(static_cast<T*>(p.out) + idx * dv + c);
#pragma unroll
          for (int i = 0; i < 32; i += 8) {
            uint4 v;
            v.x = pack2<T>(__uint_as_float(o[i]) * inv, __uint_as_float(o[i + 1]) * inv);
            v.y = pack2<T>(__uint_as_float(o[i + 2]) * inv, __uint_as_float(o[i + 3]) * inv);
            v.z = pack2<T>(__uint_as_float(o[i + 4]) * inv, __uint_as_float(o[i + 5]) * inv);
            v.w = pack2<T>(__uint_as_float(o[i + 6]) * inv, __uint_as_float(o[i + 7]) * inv);
            *reinterpret_cast<uint4*>(dst + i * 2) = v;
          }
        }
      }
      if (valid) {
        if (partial_out) {
          static_cast<float*>(p.m_out)[idx] = m * 0.6931471805599453f;
          static_cast<float*>(p.l_out)[idx] = l;
        } else {
          if (!(l > 0.f)) atomicOr(&p.ctrl->error, 1);
          if (p.lse) p.lse[idx] = (m + log2f(l)) * 0.6931471805599453f;
        }
      }
    }
  }
  if (threadIdx.x == 0) dbg_event(p, st, kEvMisc, 1);
  st.blocks += nb;
  st.items += 1;
  return st;
}

}  // namespace tile
}  // namespace psa
