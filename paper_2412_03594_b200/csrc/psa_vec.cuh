// psa_vec.cuh — VEC work items on CUDA cores: the memory-bound decode path for
// the per-request distinct KV (and for groups too small for a tensor tile).
//
// A VEC item is <= 8 stacked rows of one (group, kv head) — typically the gqa
// query heads of one decode token — against a KV range (reference:
// partial_attention(q_r, dk_r, dv_r), attention.py:187-189). Every K/V byte is
// read once per item and reused by all its rows.
//
// Granularity: ONE WARP per item. Each warp of the persistent CTA pulls VEC
// items from its own queue cursor and owns a private 3-stage ring in shared
// memory; it streams 8-key blocks of K and V into the ring with TMA
// (cp.async.bulk.tensor, one 2 KB box per operand), so nothing synchronises
// across warps and a warp's TMA stream stays busy for the whole item.
// Math: lane = (key slot, 16-byte d slice); QK^T partial dot products for
// (8 keys x 4 rows) are finished with a butterfly reduce-scatter (15 shuffles
// for 16 sums, each lane ends with one full score), softmax statistics take 3
// xor-shuffles per row, P goes through a 128-byte per-warp scratch and PV
// accumulates with packed fp32x2 FMAs (FFMA2). The warp finishes its rows
// itself: final output, or a partial for the in-kernel merge.
#pragma once

#include "psa_device.cuh"

namespace psa {
namespace vec {

constexpr int kKB = 8;       // keys per block
constexpr int kStages = 3;   // ring depth per warp
constexpr int kRP = 4;       // rows per pass
constexpr int kWarps = 8;
constexpr float kRescaleThreshold = 8.0f;  // log2 units (lazy rescale, see psa_tile.cuh)

template <int D>
struct Geo {
  static constexpr int LPK = D / 8;            // lanes per key row (16 B each)
  static constexpr int KPI = 32 / LPK;         // keys covered by one warp-wide LDS.128
  static constexpr int J = kKB / KPI;          // LDS.128 per operand per block
  static constexpr int BLK = kKB * D * 2;      // bytes of one K (or V) block
  static constexpr int STAGE = 2 * BLK;
  static constexpr int WARP = kStages * STAGE;
  static_assert(J * 4 == LPK, "one finished score per lane");
};

__host__ __device__ constexpr size_t smem_bytes(int d) {
  return size_t(kWarps) * kStages * 2 * kKB * d * 2 + 128;
}

struct alignas(16) Shared {
  uint64_t full[kWarps][kStages];
  alignas(16) float p[kWarps][32];  // read back as float4
};

__device__ __forceinline__ void init_barriers(Shared* s) {
  for (int w = 0; w < kWarps; ++w)
    for (int i = 0; i < kStages; ++i) dev::mbar_init(&s->full[w][i], 1);
  dev::fence_mbar_init();
}

__device__ __forceinline__ uint8_t* warp_ring(uint8_t* smem_raw, int warp, int d) {
  uint8_t* ring = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 127) &
                                             ~uintptr_t(127));
  return ring + size_t(warp) * kStages * 2 * kKB * d * 2;
}

template <typename T> __device__ __forceinline__ float2 unpack2(uint32_t w);
template <> __device__ __forceinline__ float2 unpack2<__nv_bfloat16>(uint32_t w) {
  return make_float2(__uint_as_float(w << 16), __uint_as_float(w & 0xffff0000u));
}
template <> __device__ __forceinline__ float2 unpack2<__half>(uint32_t w) {
  return __half22float2(*reinterpret_cast<__half2*>(&w));
}

// Processes VEC item `it` with the calling warp. `emit8(row_in_item, col, M, L, o[8])`
// receives the 8 finished columns [col, col+8) of each row (M in log2 units).
// Returns the warp's updated block count (ring phase bookkeeping).
template <typename T, int D, typename ItemT, typename Emit8>
__device__ __forceinline__ uint32_t warp_item(const KParams& p, const ItemT& it, uint8_t* ring,
                                              uint64_t* full, float* pscratch, uint32_t cnt,
                                              Emit8&& emit8) {
  using G = Geo<D>;
  const int lane = threadIdx.x & 31;
  const int kg = lane / G::LPK, ds = lane % G::LPK;
  const int npA = it.pk1 - it.pk0, npB = it.dk1 - it.dk0;
  const int nbA = (npA + kKB - 1) / kKB, nb = nbA + (npB + kKB - 1) / kKB;
  const int64_t pbase = npA ? __ldg(p.group_pbase + it.g) + it.pk0 : 0;
  const int64_t dbase = (it.req >= 0) ? __ldg(p.req_dbase + it.req) + it.dk0 : 0;
  const float sc = float(p.scale) * 1.4426950408889634f;
  const int64_t tok0 = __ldg(p.group_tok0 + it.g);
  const T* Q = static_cast<const T*>(p.q);

  auto issue = [&](int b, uint32_t c) {  // lane 0: block b into the stage of count c
    const uint32_t s = c % kStages;
    uint8_t* dst = ring + s * G::STAGE;
    const CUtensorMap *km, *vm;
    int key;
    if (b < nbA) { km = &p.tmv_kp; vm = &p.tmv_vp; key = int(pbase + b * kKB); }
    else { km = &p.tmv_kd; vm = &p.tmv_vd; key = int(dbase + (b - nbA) * kKB); }
    dev::mbar_arrive_expect_tx(&full[s], 2 * G::BLK);
    dev::tma_load_3d(dst, km, &full[s], 0, it.h, key);
    dev::tma_load_3d(dst + G::BLK, vm, &full[s], 0, it.h, key);
  };

  for (int pr = 0; pr < it.nrows; pr += kRP) {
    const int nr = min(kRP, it.nrows - pr);
    if (lane == 0) {
      dev::fence_proxy_async_smem();  // the ring was last read through the generic proxy
      for (int i = 0; i < min(kStages, nb); ++i) issue(i, cnt + i);
    }
    float2 q[kRP][4];
#pragma unroll
    for (int r = 0; r < kRP; ++r) {
      const int row = it.row0 + pr + r;
      if (r < nr) {
        const T* qr = Q + ((tok0 + row / p.gqa) * p.Hq + (int64_t)it.h * p.gqa + row % p.gqa) * D +
                      ds * 8;
        const uint4 w = __ldg(reinterpret_cast<const uint4*>(qr));
        q[r][0] = unpack2<T>(w.x); q[r][1] = unpack2<T>(w.y);
        q[r][2] = unpack2<T>(w.z); q[r][3] = unpack2<T>(w.w);
      } else {
#pragma unroll
        for (int e = 0; e < 4; ++e) q[r][e] = make_float2(0.f, 0.f);
      }
    }
    float2 o[kRP][4];
#pragma unroll
    for (int r = 0; r < kRP; ++r)
#pragma unroll
      for (int e = 0; e < 4; ++e) o[r][e] = make_float2(0.f, 0.f);
    float m = -INFINITY, lp = 0.f;  // running max / partial sum of row (lane & 3)

    for (int b = 0; b < nb; ++b) {
      const uint32_t c = cnt + b, s = c % kStages;
      const int nvalid = b < nbA ? min(kKB, npA - b * kKB) : min(kKB, npB - (b - nbA) * kKB);
      dev::mbar_wait(&full[s], (c / kStages) & 1);
      const uint8_t* kb = ring + s * G::STAGE;
      const uint8_t* vb = kb + G::BLK;
      // ---- scores: partial dots for (J key slots x 4 rows), then reduce-scatter
      float v[G::LPK];
#pragma unroll
      for (int j = 0; j < G::J; ++j) {
        const uint4 w = *reinterpret_cast<const uint4*>(kb + (j * G::KPI + kg) * (D * 2) + ds * 16);
        const float2 k0 = unpack2<T>(w.x), k1 = unpack2<T>(w.y), k2 = unpack2<T>(w.z),
                     k3 = unpack2<T>(w.w);
#pragma unroll
        for (int r = 0; r < kRP; ++r) {
          float2 a = __fmul2_rn(q[r][0], k0);
          a = __ffma2_rn(q[r][1], k1, a);
          a = __ffma2_rn(q[r][2], k2, a);
          a = __ffma2_rn(q[r][3], k3, a);
          v[j * kRP + r] = a.x + a.y;
        }
      }
#pragma unroll
      for (int off = G::LPK / 2, n = G::LPK; off >= 1; off >>= 1, n >>= 1) {
        const bool up = (lane & off) != 0;
#pragma unroll
        for (int t = 0; t < n / 2; ++t) {
          const float send = up ? v[t] : v[t + n / 2];
          const float keep = up ? v[t + n / 2] : v[t];
          v[t] = keep + __shfl_xor_sync(0xffffffffu, send, off);
        }
      }
      // lane holds the score of key slot (ds/4)*KPI + kg, row (lane & 3)
      const int key_local = (ds >> 2) * G::KPI + kg;
      const float x = key_local < nvalid ? v[0] * sc : -INFINITY;
      float bm = x;
      bm = fmaxf(bm, __shfl_xor_sync(0xffffffffu, bm, 4));
      bm = fmaxf(bm, __shfl_xor_sync(0xffffffffu, bm, 8));
      bm = fmaxf(bm, __shfl_xor_sync(0xffffffffu, bm, 16));
      float alpha = 1.f;
      if (bm > m + kRescaleThreshold) {  // also the first block (m = -inf)
        alpha = dev::ex2(m - bm);
        m = bm;
      }
      const float pe = dev::ex2(x - m);
      lp = lp * alpha + pe;
      if (__any_sync(0xffffffffu, alpha != 1.f)) {
#pragma unroll
        for (int r = 0; r < kRP; ++r) {
          const float ar = __shfl_sync(0xffffffffu, alpha, r);
          const float2 a2 = make_float2(ar, ar);
#pragma unroll
          for (int e = 0; e < 4; ++e) o[r][e] = __fmul2_rn(o[r][e], a2);
        }
      }
      // ---- P V
      pscratch[lane] = pe;
      __syncwarp();
#pragma unroll
      for (int j = 0; j < G::J; ++j) {
        const float4 pj = *reinterpret_cast<const float4*>(&pscratch[kg * G::LPK + j * 4]);
        const uint4 w = *reinterpret_cast<const uint4*>(vb + (j * G::KPI + kg) * (D * 2) + ds * 16);
        const float2 v0 = unpack2<T>(w.x), v1 = unpack2<T>(w.y), v2 = unpack2<T>(w.z),
                     v3 = unpack2<T>(w.w);
        const float pr4[4] = {pj.x, pj.y, pj.z, pj.w};
#pragma unroll
        for (int r = 0; r < kRP; ++r) {
          const float2 pp = make_float2(pr4[r], pr4[r]);
          o[r][0] = __ffma2_rn(pp, v0, o[r][0]);
          o[r][1] = __ffma2_rn(pp, v1, o[r][1]);
          o[r][2] = __ffma2_rn(pp, v2, o[r][2]);
          o[r][3] = __ffma2_rn(pp, v3, o[r][3]);
        }
      }
      __syncwarp();  // stage s and the p scratch are free
      if (lane == 0 && b + kStages < nb) {
        dev::fence_proxy_async_smem();
        issue(b + kStages, c + kStages);
      }
    }
    cnt += nb;

    // ---- finish the rows: sum o over key slots, l over lanes of the same row
#pragma unroll
    for (int off = G::LPK; off < 32; off <<= 1)
#pragma unroll
      for (int r = 0; r < kRP; ++r)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          o[r][e].x += __shfl_xor_sync(0xffffffffu, o[r][e].x, off);
          o[r][e].y += __shfl_xor_sync(0xffffffffu, o[r][e].y, off);
        }
    lp += __shfl_xor_sync(0xffffffffu, lp, 4);
    lp += __shfl_xor_sync(0xffffffffu, lp, 8);
    lp += __shfl_xor_sync(0xffffffffu, lp, 16);
#pragma unroll
    for (int r = 0; r < kRP; ++r) {
      const float M = __shfl_sync(0xffffffffu, m, r);
      const float L = __shfl_sync(0xffffffffu, lp, r);
      if (kg == 0 && r < nr) {
        const float ov[8] = {o[r][0].x, o[r][0].y, o[r][1].x, o[r][1].y,
                             o[r][2].x, o[r][2].y, o[r][3].x, o[r][3].y};
        emit8(pr + r, ds * 8, M, L, ov);
      }
    }
  }
  return cnt;
}

}  // namespace vec
}  // namespace psa
