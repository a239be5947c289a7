// psa_kernel.cu — persistent prefix-shared attention kernel for sm_100a.
//
// One launch per call covers every work item of the plan (psa_plan.cpp): the
// CTAs of a grid sized to (SMs x CTAs/SM) pull items from a global atomic
// cursor in LPT order. Each item evaluates rows of one (group, kv head)
// against one KV range — the reference's partial_attention (attention.py:78-98)
// — and either finalises its rows directly (sole contributor) or stores the
// unnormalised partial (o, m, l) in the workspace; the last item to arrive at a
// merge unit combines that unit's partials in fixed contribution order
// (merge, attention.py:101-119) and finalises (attention.py:122-126). No CTA
// ever waits on another, so the single launch cannot deadlock.
//
// Paths:
//   VEC  — CUDA-core decode path (few rows per item): see vec_item_*.
//   TILE — tcgen05/TMEM/TMA tiles for stacked-row tiles of bf16/f16 d=64/128.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cfloat>
#include <climits>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <cstdlib>

#include "../../include/psa.h"
#include "psa_kernel.h"
#include "psa_plan.h"
#include "psa_tile.cuh"
#include "psa_vec.cuh"
#include "psa_dec.cuh"
#include "psa_tile2.cuh"

namespace psa {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kMaxLanesElems = 8;  // generic path: d, dv <= 256

template <typename T> struct AccOf { using type = float; };
template <> struct AccOf<double> { using type = double; };

__device__ __forceinline__ float ld_acc(const float* p) { return *p; }
__device__ __forceinline__ float ld_acc(const __nv_bfloat16* p) { return __bfloat162float(*p); }
__device__ __forceinline__ float ld_acc(const __half* p) { return __half2float(*p); }
__device__ __forceinline__ double ld_acc(const double* p) { return *p; }

template <typename T> __device__ __forceinline__ T from_acc(float x);
template <> __device__ __forceinline__ float from_acc<float>(float x) { return x; }
template <> __device__ __forceinline__ __nv_bfloat16 from_acc<__nv_bfloat16>(float x) { return __float2bfloat16_rn(x); }
template <> __device__ __forceinline__ __half from_acc<__half>(float x) { return __float2half_rn(x); }
template <typename T> __device__ __forceinline__ T from_acc(double x) { return T(x); }

// Softmax domain: float paths work in base 2 on logits pre-multiplied by
// log2(e) (one FFMA per exponent); the float64 path works in base e exactly
// like the reference.
template <typename A> struct Dom;
template <> struct Dom<float> {
  static __device__ __forceinline__ float ex(float x) { return exp2f(x); }
  static __device__ __forceinline__ float lg(float x) { return log2f(x); }
  static constexpr float kLogE = 1.4426950408889634f;  // logits -> domain
  static constexpr float kToNat = 0.6931471805599453f; // domain -> natural
};
template <> struct Dom<double> {
  static __device__ __forceinline__ double ex(double x) { return exp(x); }
  static __device__ __forceinline__ double lg(double x) { return log(x); }
  static constexpr double kLogE = 1.0;
  static constexpr double kToNat = 1.0;
};

template <typename A> __device__ __forceinline__ A neg_inf();
template <> __device__ __forceinline__ float neg_inf<float>() { return -INFINITY; }
template <> __device__ __forceinline__ double neg_inf<double>() { return -HUGE_VAL; }

template <typename A>
__device__ __forceinline__ A warp_sum(A v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

struct ItemRec {
  int32_t kind, g, h, row0, nrows, req, pk0, pk1, dk0, dk1, u0, u1, ws_row, pair;
};

__device__ __forceinline__ ItemRec load_item(const int32_t* rec) {
  ItemRec it;
  it.kind = __ldg(rec + kItKind);
  it.g = __ldg(rec + kItGroup);
  it.h = __ldg(rec + kItHead);
  it.row0 = __ldg(rec + kItRow0);
  it.nrows = __ldg(rec + kItRows);
  it.req = __ldg(rec + kItRequest);
  it.pk0 = __ldg(rec + kItPk0);
  it.pk1 = __ldg(rec + kItPk1);
  it.dk0 = __ldg(rec + kItDk0);
  it.dk1 = __ldg(rec + kItDk1);
  it.u0 = __ldg(rec + kItUnit0);
  it.u1 = __ldg(rec + kItUnit1);
  it.ws_row = __ldg(rec + kItWsRow);
  it.pair = __ldg(rec + kItPair);
  return it;
}

// Final output of one (row, column) of group g / kv head h: out = o / l, or the
// unnormalised partial with PSA_FLAG_PARTIAL_OUT. Column 0 also writes LSE/m/l.
template <typename T, typename A>
__device__ __forceinline__ void write_final(const KParams& p, int g, int h, int row, int c, A M,
                                            A L, A O) {
  const int64_t tok = __ldg(p.group_tok0 + g) + row / p.gqa;
  const int64_t idx = tok * p.Hq + (int64_t)h * p.gqa + row % p.gqa;
  if (p.flags & PSA_FLAG_PARTIAL_OUT) {
    static_cast<A*>(p.out)[idx * p.dv + c] = O;
    if (c == 0) {
      static_cast<A*>(p.m_out)[idx] = M * A(Dom<A>::kToNat);
      static_cast<A*>(p.l_out)[idx] = L;
    }
    return;
  }
  static_cast<T*>(p.out)[idx * p.dv + c] = from_acc<T>(O / L);
  if (c == 0) {
    if (!(L > A(0))) atomicOr(&p.ctrl->error, 1);
    if (p.lse) p.lse[idx] = float((M + Dom<A>::lg(L)) * A(Dom<A>::kToNat));
  }
}

template <typename T> __device__ __forceinline__ void store4(T* dst, float4 v, float s);
template <> __device__ __forceinline__ void store4<float>(float* dst, float4 v, float s) {
  *reinterpret_cast<float4*>(dst) = make_float4(v.x * s, v.y * s, v.z * s, v.w * s);
}
template <> __device__ __forceinline__ void store4<__nv_bfloat16>(__nv_bfloat16* dst, float4 v,
                                                                  float s) {
  __nv_bfloat162 a = __floats2bfloat162_rn(v.x * s, v.y * s), b = __floats2bfloat162_rn(v.z * s, v.w * s);
  uint2 w;
  w.x = *reinterpret_cast<uint32_t*>(&a);
  w.y = *reinterpret_cast<uint32_t*>(&b);
  *reinterpret_cast<uint2*>(dst) = w;
}
template <> __device__ __forceinline__ void store4<__half>(__half* dst, float4 v, float s) {
  __half2 a = __floats2half2_rn(v.x * s, v.y * s), b = __floats2half2_rn(v.z * s, v.w * s);
  uint2 w;
  w.x = *reinterpret_cast<uint32_t*>(&a);
  w.y = *reinterpret_cast<uint32_t*>(&b);
  *reinterpret_cast<uint2*>(dst) = w;
}

// Four consecutive columns (c % 4 == 0, dv % 4 == 0) of a final row, fp32 accumulate.
template <typename T>
__device__ __forceinline__ void write_final4_t(const KParams& p, int64_t tok0, int h, int row,
                                               int c, float M, float L, float4 O) {
  const int64_t tok = tok0 + row / p.gqa;
  const int64_t idx = tok * p.Hq + (int64_t)h * p.gqa + row % p.gqa;
  if (p.flags & PSA_FLAG_PARTIAL_OUT) {
    store4<float>(static_cast<float*>(p.out) + idx * p.dv + c, O, 1.f);
    if (c == 0) {
      static_cast<float*>(p.m_out)[idx] = M * Dom<float>::kToNat;
      static_cast<float*>(p.l_out)[idx] = L;
    }
    return;
  }
  store4<T>(static_cast<T*>(p.out) + idx * p.dv + c, O, 1.f / L);
  if (c == 0) {
    if (!(L > 0.f)) atomicOr(&p.ctrl->error, 1);
    if (p.lse) p.lse[idx] = (M + log2f(L)) * Dom<float>::kToNat;
  }
}

template <typename T>
__device__ __forceinline__ void write_final4(const KParams& p, int g, int h, int row, int c,
                                             float M, float L, float4 O) {
  write_final4_t<T>(p, __ldg(p.group_tok0 + g), h, row, c, M, L, O);
}

// Emits one combined (row, column) value of an item: to the workspace when the
// item shares its merge units, else straight to the output.
template <typename T, typename A>
__device__ __forceinline__ void emit(const KParams& p, const ItemRec& it, int r, int c, A M, A L,
                                     A O) {
  if (it.ws_row >= 0) {
    const int64_t wr = (int64_t)it.ws_row + r;
    static_cast<A*>(p.ws_o)[wr * p.dv + c] = O;
    if (c == 0) {
      static_cast<A*>(p.ws_ml)[wr * 2 + 0] = M;
      static_cast<A*>(p.ws_ml)[wr * 2 + 1] = L;
    }
  } else {
    write_final<T, A>(p, it.g, it.h, it.row0 + r, c, M, L, O);
  }
}

template <typename T>
__device__ __forceinline__ void emit4(const KParams& p, const ItemRec& it, int r, int c, float M,
                                      float L, float4 O) {
  if (it.ws_row >= 0) {
    const int64_t wr = (int64_t)it.ws_row + r;
    store4<float>(static_cast<float*>(p.ws_o) + wr * p.dv + c, O, 1.f);
    if (c == 0) *reinterpret_cast<float2*>(static_cast<float*>(p.ws_ml) + wr * 2) = make_float2(M, L);
  } else {
    write_final4<T>(p, it.g, it.h, it.row0 + r, c, M, L, O);
  }
}

// Combines the per-warp online-softmax states (m, l, o) of `nr` rows held in
// shared memory — sm_o [kWarps][rp][dv], sm_ml [kWarps][rp][2] — and emits
// every (row, column). Row statistics and the per-warp rescale factors are
// computed once per row (s_f [kWarps][rp], s_M / s_L [rp]).
template <typename T, typename A, typename Emit1, typename Emit4>
__device__ __forceinline__ void combine_warps(int nr, int rp, int dv, const A* sm_o, const A* sm_ml,
                                              A* s_f, A* s_M, A* s_L, Emit1&& e1, Emit4&& e4) {
  if (threadIdx.x < nr) {
    const int r = threadIdx.x;
    A M = neg_inf<A>();
#pragma unroll
    for (int w = 0; w < kWarps; ++w) M = max(M, sm_ml[(w * rp + r) * 2]);
    A L = A(0);
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
      const A lw = sm_ml[(w * rp + r) * 2 + 1];
      const A f = lw > A(0) ? Dom<A>::ex(sm_ml[(w * rp + r) * 2] - M) : A(0);
      s_f[w * rp + r] = f;
      L += f * lw;
    }
    s_M[r] = M;
    s_L[r] = L;
  }
  __syncthreads();
  if constexpr (sizeof(A) == 4) {
    if ((dv & 3) == 0) {
      const int q4 = dv >> 2;
      for (int idx = threadIdx.x; idx < nr * q4; idx += kThreads) {
        const int r = idx / q4, c = (idx - r * q4) * 4;
        float4 O = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int w = 0; w < kWarps; ++w) {
          const float f = s_f[w * rp + r];
          const float4 v = *reinterpret_cast<const float4*>(sm_o + (w * rp + r) * dv + c);
          O.x += f * v.x; O.y += f * v.y; O.z += f * v.z; O.w += f * v.w;
        }
        e4(r, c, s_M[r], s_L[r], O);
      }
      return;
    }
  }
  for (int idx = threadIdx.x; idx < nr * dv; idx += kThreads) {
    const int r = idx / dv, c = idx - r * dv;
    A O = A(0);
#pragma unroll
    for (int w = 0; w < kWarps; ++w) O += s_f[w * rp + r] * sm_o[(w * rp + r) * dv + c];
    e1(r, c, s_M[r], s_L[r], O);
  }
}

// ---------------------------------------------------------------------------
// Generic CUDA-core path: any dtype, any d, dv <= 256. Warps stride over keys,
// lanes stride over the head dim; every key is a full online-softmax update
// (exactly partial_attention's math, one key at a time). Rows go in passes of
// RP; the eight warps' states are merged through shared memory.
// ---------------------------------------------------------------------------
template <typename T, typename A, int RP>
__device__ void vec_item_generic(const KParams& p, const ItemRec& it, uint8_t* smem, A* s_f,
                                 A* s_M, A* s_L) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int d = p.d, dv = p.dv;
  const A sc = A(p.scale) * A(Dom<A>::kLogE);
  const T* Q = static_cast<const T*>(p.q);
  const T* KP = static_cast<const T*>(p.kp);
  const T* VP = static_cast<const T*>(p.vp);
  const T* KD = static_cast<const T*>(p.kd);
  const T* VD = static_cast<const T*>(p.vd);
  const int np = it.pk1 - it.pk0, nk = np + (it.dk1 - it.dk0);
  const int64_t pbase = (np > 0) ? __ldg(p.group_pbase + it.g) + it.pk0 : 0;
  const int64_t dbase = (it.req >= 0) ? __ldg(p.req_dbase + it.req) + it.dk0 : 0;
  const int64_t kstride = (int64_t)p.Hkv * d, vstride = (int64_t)p.Hkv * dv;
  const int64_t tok0 = __ldg(p.group_tok0 + it.g);
  A* sm_o = reinterpret_cast<A*>(smem);        // [kWarps][RP][dv]
  A* sm_ml = sm_o + kWarps * RP * dv;          // [kWarps][RP][2]

  for (int pr = 0; pr < it.nrows; pr += RP) {
    const int nr = min(RP, it.nrows - pr);
    A q[RP][kMaxLanesElems], o[RP][kMaxLanesElems], m[RP], l[RP];
#pragma unroll
    for (int r = 0; r < RP; ++r) {
      const int row = it.row0 + pr + r;
      const int64_t tok = tok0 + row / p.gqa;
      const T* qr = Q + (tok * p.Hq + (int64_t)it.h * p.gqa + row % p.gqa) * d;
#pragma unroll
      for (int e = 0; e < kMaxLanesElems; ++e) {
        const int c = lane + 32 * e;
        q[r][e] = (r < nr && c < d) ? ld_acc(qr + c) : A(0);
        o[r][e] = A(0);
      }
      m[r] = neg_inf<A>();
      l[r] = A(0);
    }
    for (int j = warp; j < nk; j += kWarps) {
      const T* kr;
      const T* vr;
      if (j < np) {
        kr = KP + (pbase + j) * kstride + (int64_t)it.h * d;
        vr = VP + (pbase + j) * vstride + (int64_t)it.h * dv;
      } else {
        kr = KD + (dbase + j - np) * kstride + (int64_t)it.h * d;
        vr = VD + (dbase + j - np) * vstride + (int64_t)it.h * dv;
      }
      A kk[kMaxLanesElems], vv[kMaxLanesElems];
#pragma unroll
      for (int e = 0; e < kMaxLanesElems; ++e) {
        const int c = lane + 32 * e;
        kk[e] = c < d ? ld_acc(kr + c) : A(0);
        vv[e] = c < dv ? ld_acc(vr + c) : A(0);
      }
#pragma unroll
      for (int r = 0; r < RP; ++r) {
        A s = A(0);
#pragma unroll
        for (int e = 0; e < kMaxLanesElems; ++e) s += q[r][e] * kk[e];
        s = warp_sum(s);
        const A x = s * sc;
        const A mn = max(m[r], x);
        const A alpha = Dom<A>::ex(m[r] - mn);
        const A pe = Dom<A>::ex(x - mn);
        l[r] = l[r] * alpha + pe;
#pragma unroll
        for (int e = 0; e < kMaxLanesElems; ++e) o[r][e] = o[r][e] * alpha + pe * vv[e];
        m[r] = mn;
      }
    }
#pragma unroll
    for (int r = 0; r < RP; ++r) {
#pragma unroll
      for (int e = 0; e < kMaxLanesElems; ++e) {
        const int c = lane + 32 * e;
        if (c < dv) sm_o[(warp * RP + r) * dv + c] = o[r][e];
      }
      if (lane == 0) {
        sm_ml[(warp * RP + r) * 2 + 0] = m[r];
        sm_ml[(warp * RP + r) * 2 + 1] = l[r];
      }
    }
    __syncthreads();
    combine_warps<T, A>(
        nr, RP, dv, sm_o, sm_ml, s_f, s_M, s_L,
        [&](int r, int c, A M, A L, A O) { emit<T, A>(p, it, pr + r, c, M, L, O); },
        [&](int r, int c, float M, float L, float4 O) { emit4<T>(p, it, pr + r, c, M, L, O); });
    __syncthreads();
  }
}

// Last arriver: combine the unit's partials in contribution order and finalise.
// Phase 1 (thread per row): running max M and sum L over the contributions.
// Phase 2 (thread per 4 columns): O = sum_i 2^(m_i - M) o_i.
template <typename T, typename A>
__device__ void merge_unit(const KParams& p, int u, A* s_M, A* s_L) {
  const int32_t* U = p.units + (int64_t)u * kUnitWords;
  const int g = __ldg(U + kUnGroup), h = __ldg(U + kUnHead);
  const int row0 = __ldg(U + kUnRow0), nrows = __ldg(U + kUnRows);
  const int cb = __ldg(U + kUnContribBegin), cc = __ldg(U + kUnContribCount);
  const int32_t* C = p.contribs + cb;
  const A* WO = static_cast<const A*>(p.ws_o);
  const A* WML = static_cast<const A*>(p.ws_ml);
  const int dv = p.dv;
  for (int r = threadIdx.x; r < nrows; r += kThreads) {
    A M = neg_inf<A>(), L = A(0);
    for (int i = 0; i < cc; ++i) {
      const int64_t wr = (int64_t)__ldg(C + i) + r;
      const A mi = __ldcg(WML + wr * 2), li = __ldcg(WML + wr * 2 + 1);
      if (li > A(0)) {  // online combine in contribution order (attention.py:109-118)
        const A mn = max(M, mi);
        L = L * Dom<A>::ex(M - mn) + li * Dom<A>::ex(mi - mn);
        M = mn;
      }
    }
    s_M[r] = M;
    s_L[r] = L;
  }
  __syncthreads();
  if constexpr (sizeof(A) == 4) {
    if ((dv & 3) == 0) {
      const int q4 = dv >> 2;
      for (int idx = threadIdx.x; idx < nrows * q4; idx += kThreads) {
        const int r = idx / q4, c = (idx - r * q4) * 4;
        const float M = s_M[r];
        float4 O = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int i = 0; i < cc; ++i) {
          const int64_t wr = (int64_t)__ldg(C + i) + r;
          const float2 ml = __ldcg(reinterpret_cast<const float2*>(WML) + wr);
          if (ml.y > 0.f) {
            const float f = exp2f(ml.x - M);
            const float4 v = __ldcg(reinterpret_cast<const float4*>(WO + wr * dv + c));
            O.x += f * v.x; O.y += f * v.y; O.z += f * v.z; O.w += f * v.w;
          }
        }
        write_final4<T>(p, g, h, row0 + r, c, M, s_L[r], O);
      }
      __syncthreads();
      return;
    }
  }
  for (int idx = threadIdx.x; idx < nrows * dv; idx += kThreads) {
    const int r = idx / dv, c = idx - r * dv;
    const A M = s_M[r];
    A O = A(0);
    for (int i = 0; i < cc; ++i) {
      const int64_t wr = (int64_t)__ldg(C + i) + r;
      const A li = __ldcg(WML + wr * 2 + 1);
      if (li > A(0)) O += Dom<A>::ex(__ldcg(WML + wr * 2) - M) * __ldcg(WO + wr * dv + c);
    }
    write_final<T, A>(p, g, h, row0 + r, c, M, s_L[r], O);
  }
  __syncthreads();
}

// Warp-per-row merge of one row of merge unit `u` (fp32 accumulate, dv % 4 == 0,
// dv <= 128): every contribution's (m, l) and o are loaded in one round trip,
// combined in contribution order and finalised (attention.py:101-126).
template <typename T>
__device__ __forceinline__ void merge_row_warp(const KParams& p, int u, int r) {
  const int lane = threadIdx.x & 31;
  const int32_t* U = p.units + (int64_t)u * kUnitWords;
  const int g = __ldg(U + kUnGroup), h = __ldg(U + kUnHead), row0 = __ldg(U + kUnRow0);
  const int cb = __ldg(U + kUnContribBegin), cc = __ldg(U + kUnContribCount);
  const float* WO = static_cast<const float*>(p.ws_o);
  const float2* WML = static_cast<const float2*>(p.ws_ml);
  const int dv = p.dv, c = lane * 4;
  float M = -INFINITY, L = 0.f;
  float4 O = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int base = 0; base < cc; base += 32) {
    const int n = min(32, cc - base);
    int64_t wr = 0;
    float2 ml = make_float2(-INFINITY, 0.f);
    if (lane < n) {
      wr = (int64_t)__ldg(p.contribs + cb + base + lane) + r;
      ml = __ldcg(WML + wr);
    }
    float mc = ml.y > 0.f ? ml.x : -INFINITY;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mc = fmaxf(mc, __shfl_xor_sync(0xffffffffu, mc, o));
    const float mn = fmaxf(M, mc);
    const float fo = M == -INFINITY ? 0.f : exp2f(M - mn);
    float f = ml.y > 0.f ? exp2f(ml.x - mn) : 0.f;
    float lsum = f * ml.y;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) lsum += __shfl_xor_sync(0xffffffffu, lsum, o);
    L = L * fo + lsum;
    O.x *= fo; O.y *= fo; O.z *= fo; O.w *= fo;
    M = mn;
    // 8 contributions per batch: all loads in flight before the first FMA
    for (int i0 = 0; i0 < n; i0 += 8) {
      float4 v[8];
      float fi[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int i = i0 + j;
        fi[j] = __shfl_sync(0xffffffffu, f, i & 31);
        const int64_t wi = __shfl_sync(0xffffffffu, wr, i & 31);
        v[j] = (i < n && fi[j] != 0.f && c < dv)
                   ? __ldcg(reinterpret_cast<const float4*>(WO + wi * dv + c))
                   : make_float4(0.f, 0.f, 0.f, 0.f);
        if (i >= n) fi[j] = 0.f;
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        O.x += fi[j] * v[j].x; O.y += fi[j] * v[j].y; O.z += fi[j] * v[j].z; O.w += fi[j] * v[j].w;
      }
    }
  }
  if (c < dv) write_final4<T>(p, g, h, row0 + r, c, M, L, O);
}

// Warp merge of rows [r0, r0 + nr) of unit u with nr * cc <= 32 (fp32, dv % 4 == 0,
// dv <= 128): lane l < nr * cc loads the (m, l) of (row l / cc, contribution
// l % cc); every o the rows need is then issued before the first FMA, so the
// whole chunk costs two memory round trips. Combination order per row is the
// contribution order (bit-reproducible).
template <typename T>
__device__ __forceinline__ void merge_chunk_warp(const KParams& p, int u, int r0, int nr) {
  const int lane = threadIdx.x & 31;
  const int32_t* U = p.units + (int64_t)u * kUnitWords;
  const int g = __ldg(U + kUnGroup), h = __ldg(U + kUnHead), row0 = __ldg(U + kUnRow0);
  const int cb = __ldg(U + kUnContribBegin), cc = __ldg(U + kUnContribCount);
  const int64_t tok0 = __ldg(p.group_tok0 + g);
  const float* WO = static_cast<const float*>(p.ws_o);
  const float2* WML = static_cast<const float2*>(p.ws_ml);
  const int dv = p.dv, c = lane * 4;
  int64_t wr = 0;
  float2 ml = make_float2(-INFINITY, 0.f);
  if (lane < nr * cc) {
    const int r = lane / cc, i = lane - r * cc;
    wr = (int64_t)__ldg(p.contribs + cb + i) + r0 + r;
  }
  // the partial rows' o are loaded together with their (m, l): one round trip
  float4 v8[8];
  if (cc <= 8) {
    const int np0 = min(8 / cc, nr) * cc;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int64_t wj = __shfl_sync(0xffffffffu, wr, j);
      v8[j] = (j < np0 && c < dv) ? __ldcg(reinterpret_cast<const float4*>(WO + wj * dv + c))
                                  : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
  if (lane < nr * cc) ml = __ldcg(WML + wr);
  const float mv = ml.y > 0.f ? ml.x : -INFINITY;
  // per-row max over the row's cc lanes (lanes of a row are contiguous)
  float M = -INFINITY;
  const int my_r = lane / max(cc, 1);
  for (int i = 0; i < cc; ++i) M = fmaxf(M, __shfl_sync(0xffffffffu, mv, min(my_r * cc + i, 31)));
  const float f = ml.y > 0.f ? dev::ex2(ml.x - M) : 0.f;
  const float fl = __fmul_rn(f, ml.y);
  if (cc <= 8) {
    // groups of rg rows: rg * cc <= 8 (row, contribution) pairs, all loads in flight
    const int rg = 8 / cc;
    for (int rb = 0; rb < nr; rb += rg) {
      const int np = min(rg, nr - rb) * cc;
      float fi[8];
      float4 v[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int src = min(rb * cc + j, 31);
        fi[j] = j < np ? __shfl_sync(0xffffffffu, f, src) : 0.f;
        if (rb == 0) {
          v[j] = fi[j] != 0.f ? v8[j] : make_float4(0.f, 0.f, 0.f, 0.f);
        } else {
          const int64_t wj = __shfl_sync(0xffffffffu, wr, src);
          v[j] = (j < np && fi[j] != 0.f && c < dv)
                     ? __ldcg(reinterpret_cast<const float4*>(WO + wj * dv + c))
                     : make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
      for (int rr = 0; rr < rg && rb + rr < nr; ++rr) {
        float4 O = make_float4(0.f, 0.f, 0.f, 0.f);
        float L = 0.f;
#pragma unroll
        for (int j = 0; j < 8; ++j) {  // contribution order; arithmetic pinned (DecFast)
          const bool mine = j >= rr * cc && j < (rr + 1) * cc;
          const float fj = mine ? fi[j] : 0.f;
          O.x = __fmaf_rn(fj, v[j].x, O.x); O.y = __fmaf_rn(fj, v[j].y, O.y);
          O.z = __fmaf_rn(fj, v[j].z, O.z); O.w = __fmaf_rn(fj, v[j].w, O.w);
        }
        for (int i = 0; i < cc; ++i) L = __fadd_rn(L, __shfl_sync(0xffffffffu, fl, min((rb + rr) * cc + i, 31)));
        const float Mr = __shfl_sync(0xffffffffu, M, min((rb + rr) * cc, 31));
        if (c < dv) write_final4_t<T>(p, tok0, h, row0 + r0 + rb + rr, c, Mr, L, O);
      }
    }
    return;
  }
  for (int rr = 0; rr < nr; ++rr) {
    float L = 0.f;
    float4 O = make_float4(0.f, 0.f, 0.f, 0.f);
    float fi[8];
    float4 v[8];
    for (int i0 = 0; i0 < cc; i0 += 8) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int src = min(rr * cc + i0 + j, 31);
        const bool ok = i0 + j < cc;
        fi[j] = ok ? __shfl_sync(0xffffffffu, f, src) : 0.f;
        const float flj = __shfl_sync(0xffffffffu, fl, src);
        const int64_t wj = __shfl_sync(0xffffffffu, wr, src);
        if (ok) L += flj;
        v[j] = (ok && fi[j] != 0.f && c < dv)
                   ? __ldcg(reinterpret_cast<const float4*>(WO + wj * dv + c))
                   : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        O.x += fi[j] * v[j].x; O.y += fi[j] * v[j].y; O.z += fi[j] * v[j].z; O.w += fi[j] * v[j].w;
      }
    }
    const float Mr = __shfl_sync(0xffffffffu, M, min(rr * cc, 31));
    if (c < dv) write_final4_t<T>(p, tok0, h, row0 + r0 + rr, c, Mr, L, O);
  }
}

// All rows of unit u, by one warp, in chunks of <= 32 (row, contribution) pairs.
template <typename T>
__device__ __noinline__ void merge_unit_warp(const KParams& p, int u) {
  const int32_t* U = p.units + (int64_t)u * kUnitWords;
  const int rows = __ldg(U + kUnRows), cc = __ldg(U + kUnContribCount);
  if (cc > 32) {
    for (int r = 0; r < rows; ++r) merge_row_warp<T>(p, u, r);
    return;
  }
  const int per = max(1, 32 / cc);
  for (int r0 = 0; r0 < rows; r0 += per) merge_chunk_warp<T>(p, u, r0, min(per, rows - r0));
}

template <typename T> struct HasTiles { static constexpr bool v = false; };
template <> struct HasTiles<__nv_bfloat16> { static constexpr bool v = true; };
template <> struct HasTiles<__half> { static constexpr bool v = true; };

// Kernel modes: which item paths are compiled in (keeps register allocation of
// the hot paths free of the generic path's pressure).
enum Mode : int { kModeGeneric = 0, kModeFast = 1, kModeTileGeneric = 2 };

__device__ __forceinline__ void trace_item(const KParams& p, int idx, int kind, int64_t t0) {
  if (idx < p.trace_cap) {
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    int64_t* t = p.trace + int64_t(idx) * 4;
    t[0] = int64_t(blockIdx.x) | (int64_t(smid) << 32) | (int64_t(threadIdx.x >> 5) << 48);
    t[1] = kind;
    t[2] = t0;
    t[3] = int64_t(globaltimer());
  }
}

// CTA-level arrival at the merge units of item `it` (after its partial rows are
// written): the last arriver of a unit merges that unit's rows, one warp per row.
template <typename T, typename A>
__device__ __forceinline__ void cta_arrive_and_merge(const KParams& p, const ItemRec& it,
                                                     int* s_merge, int* s_nmerge, A* s_rowM,
                                                     A* s_rowL) {
  // Publish this item's partial rows: CTA barrier, then the arrivals — one thread per
  // unit, in parallel (a serial loop of returning atomics costs one L2 round trip
  // per unit), each after a gpu-scope fence (release is cumulative over the barrier).
  if (threadIdx.x == 0) *s_nmerge = 0;
  __syncthreads();
  const int nu = it.u1 - it.u0;
  for (int i = threadIdx.x; i < nu; i += kThreads) {
    const int u = it.u0 + i;
    __threadfence();
    const int need = __ldg(p.units + (int64_t)u * kUnitWords + kUnContribCount);
    if (atomicAdd(p.unit_cnt + u, 1) == need - 1) {
      p.unit_cnt[u] = 0;  // every contribution has arrived: reset for the next launch
      s_merge[atomicAdd(s_nmerge, 1)] = u;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0 && *s_nmerge) __threadfence();  // acquire side for the partials
  __syncthreads();
  const int nm = *s_nmerge;
  if (!nm) return;
  if constexpr (sizeof(A) == 4) {
    if ((p.dv & 3) == 0 && p.dv <= 128) {
      const int warp = threadIdx.x >> 5;
      int k = 0;
      for (int i = 0; i < nm; ++i) {
        const int u = s_merge[i];
        const int rows = __ldg(p.units + (int64_t)u * kUnitWords + kUnRows);
        const int cc = __ldg(p.units + (int64_t)u * kUnitWords + kUnContribCount);
        if (cc > 32) {
          for (int r = 0; r < rows; ++r, ++k)
            if ((k & (kWarps - 1)) == warp) merge_row_warp<T>(p, u, r);
          continue;
        }
        const int per = max(1, 32 / cc);
        for (int r0 = 0; r0 < rows; r0 += per, ++k)
          if ((k & (kWarps - 1)) == warp) merge_chunk_warp<T>(p, u, r0, min(per, rows - r0));
      }
      return;
    }
  }
  for (int i = 0; i < nm; ++i) merge_unit<T, A>(p, s_merge[i], s_rowM, s_rowL);
}

// Warp-level arrival for a VEC item processed by one warp.
template <typename T>
__device__ __forceinline__ void warp_arrive_and_merge(const KParams& p, const ItemRec& it) {
  const int lane = threadIdx.x & 31;
  __threadfence();  // one warp-wide fence: publishes every lane's partial rows
  __syncwarp();
  // one lane per unit (items of <= 8 rows cover <= 9 units)
  bool is_last = false;
  const int u = it.u0 + lane;
  if (u < it.u1) {
    const int need = __ldg(p.units + (int64_t)u * kUnitWords + kUnContribCount);
    if (atomicAdd(p.unit_cnt + u, 1) == need - 1) {
      p.unit_cnt[u] = 0;
      is_last = true;
    }
  }
  uint32_t last = __ballot_sync(0xffffffffu, is_last);
  if (last) __threadfence();
  while (last) {
    const int bit = __ffs(last) - 1;
    last &= last - 1;
    merge_unit_warp<T>(p, it.u0 + bit);
  }
}

// Merge-warp arrival on behalf of an item whose partial rows [r0, r1) (group rows)
// were published to this warp through the CTA merge queue: one fence (cumulative
// over the queue handoff), one atomic per unit whose first row lies in the range;
// `on_last(u)` gets every unit this arrival completed (merge it now, or queue it so
// several merge warps share a tile's units). Keeps the gpu-scope fence and the
// merges off the softmax warps' critical path.
__device__ __forceinline__ void dbg_clock(const KParams& p, int ev, int slot) {
  if (kTraceEvents && slot >= 0 && (threadIdx.x & 31) == 0) {
    long long t;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(t));
    p.trace[(int64_t(p.num_items) + 4096) * 4 + ev * 64 + slot] = t;
  }
}

template <typename OnLast>
__device__ __forceinline__ void warp_arrive_rows(const KParams& p, const ItemRec& it, int r0,
                                                 int r1, OnLast&& on_last, int dslot = -1) {
  const int lane = threadIdx.x & 31;
  dev::fence_acq_rel_gpu();
  __syncwarp();
  dbg_clock(p, 36, dslot);
  for (int base = it.u0; base < it.u1; base += 32) {
    const int u = base + lane;
    bool is_last = false;
    if (u < it.u1) {
      const int32_t* U = p.units + (int64_t)u * kUnitWords;
      const int ur0 = __ldg(U + kUnRow0);
      if (ur0 >= r0 && ur0 < r1) {
        const int need = __ldg(U + kUnContribCount);
        if (atomicAdd(p.unit_cnt + u, 1) == need - 1) {
          p.unit_cnt[u] = 0;
          is_last = true;
        }
      }
    }
    uint32_t last = __ballot_sync(0xffffffffu, is_last);
    dbg_clock(p, 37, dslot);
    if (last) dev::fence_acq_rel_gpu();  // acquire: the other contributors' partial rows
    dbg_clock(p, 38, dslot);
    while (last) {
      const int bit = __ffs(last) - 1;
      last &= last - 1;
      on_last(base + bit);
    }
  }
}

// Decode items whose single merge unit has exactly one other contributor (the
// group's prefix tile chunk) that has already arrived: the item merges that partial
// in registers (thread t = value column t) with the same arithmetic, in the same
// contribution order, as merge_chunk_warp — so the result is bit-identical whichever
// side finishes last — and writes the final rows; it never publishes a partial.
template <typename T>
struct DecFast {
  const KParams& p;
  struct Other {
    float m[dec::kR], l[dec::kR], o[dec::kR];
    int first;  // the other contribution precedes this item's in contribution order
  };
  // Producer lane 0. Returns 1 (fast) with `other` = (workspace row of the other
  // contribution) * 2 + (the other contribution comes first in contribution order).
  // The pair (kItPair) is precomputed by the planner, so this is one acquire load.
  __device__ int probe(const ItemRec& it, int& other) const {
    if (!p.dec_fast || it.pair < 0) return 0;
    int cnt;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(cnt) : "l"(p.unit_cnt + it.u0) : "memory");
    if (cnt != 1) return 0;
    other = it.pair;
    return 1;
  }
  // All softmax threads at the item start (ordered after the producer's acquire by the
  // item barrier); the loads are issued here and consumed by finish().
  __device__ void fetch(int other, int t, int R, Other& o) const {
    o.first = other & 1;
    const int64_t base = other >> 1;
    const float* WO = static_cast<const float*>(p.ws_o);
    const float2* WML = static_cast<const float2*>(p.ws_ml);
#pragma unroll
    for (int r = 0; r < dec::kR; ++r) {
      if (r < R) {
        const float2 ml = dev::ld_cg_f32x2(WML + base + r);
        o.m[r] = ml.x;
        o.l[r] = ml.y;
        o.o[r] = dev::ld_cg_f32(WO + (base + r) * 128 + t);
      }
    }
  }
  __device__ void finish(const ItemRec& it, const int64_t* oidx, int t, int R, const float (&m)[dec::kR],
                         const float (&L)[dec::kR], const float (&ov)[dec::kR],
                         const Other& o) const {
    const bool partial_out = p.flags & PSA_FLAG_PARTIAL_OUT;
#pragma unroll
    for (int r = 0; r < dec::kR; ++r) {
      if (r >= R) continue;
      // contributions in order: (m0, l0, o0) then (m1, l1, o1)
      const float m0 = o.first ? o.m[r] : m[r], l0 = o.first ? o.l[r] : L[r];
      const float o0 = o.first ? o.o[r] : ov[r];
      const float m1 = o.first ? m[r] : o.m[r], l1 = o.first ? L[r] : o.l[r];
      const float o1 = o.first ? ov[r] : o.o[r];
      const float M = fmaxf(fmaxf(-INFINITY, l0 > 0.f ? m0 : -INFINITY), l1 > 0.f ? m1 : -INFINITY);
      const float f0 = l0 > 0.f ? dev::ex2(m0 - M) : 0.f;
      const float f1 = l1 > 0.f ? dev::ex2(m1 - M) : 0.f;
      const float Ls = __fadd_rn(__fadd_rn(0.f, __fmul_rn(f0, l0)), __fmul_rn(f1, l1));
      const float O = __fmaf_rn(f1, o1, __fmaf_rn(f0, o0, 0.f));
      const int64_t idx = oidx[r];
      if (partial_out) {
        static_cast<float*>(p.out)[idx * 128 + t] = O;
        if (t == 0) {
          static_cast<float*>(p.m_out)[idx] = M * Dom<float>::kToNat;
          static_cast<float*>(p.l_out)[idx] = Ls;
        }
        continue;
      }
      static_cast<T*>(p.out)[idx * 128 + t] = from_acc<T>(O * (1.f / Ls));
      if (t == 0) {
        if (!(Ls > 0.f)) atomicOr(&p.ctrl->error, 1);
        if (p.lse) p.lse[idx] = (M + log2f(Ls)) * Dom<float>::kToNat;
      }
    }
    if (t == 0) p.unit_cnt[it.u0] = 0;  // every contributor arrived: reset for the next launch
  }
};

// End of a decode item (thread t = value column t of the item's <= 8 rows): the
// partial rows + arrival at the merge units, or the final output.
template <typename T>
__device__ __forceinline__ void dec_finish(const KParams& p, dec::Shared* sh, const ItemRec& it,
                                           const int64_t* oidx, int idx, int t, int R,
                                           const float (&m)[dec::kR],
                                           const float (&L)[dec::kR], const float (&ov)[dec::kR],
                                           int pi) {
  if (it.ws_row >= 0) {
    float* wo = static_cast<float*>(p.ws_o);
#pragma unroll
    for (int r = 0; r < dec::kR; ++r)
      if (r < R) wo[((int64_t)it.ws_row + r) * 128 + t] = ov[r];
    if (t == 0) {
#pragma unroll
      for (int r = 0; r < dec::kR; ++r)
        if (r < R)
          *reinterpret_cast<float2*>(static_cast<float*>(p.ws_ml) + ((int64_t)it.ws_row + r) * 2) =
              make_float2(m[r], L[r]);
    }
    // publish to the pipeline's merge warps, which arrive at the item's units
    dec::named_sync_softmax(pi);
    if (t == 0) dec::enqueue_merge(sh, idx);
    return;
  }
  const bool partial_out = p.flags & PSA_FLAG_PARTIAL_OUT;
#pragma unroll
  for (int r = 0; r < dec::kR; ++r) {
    if (r < R) {
      const int64_t idx = oidx[r];
      if (partial_out) {
        static_cast<float*>(p.out)[idx * 128 + t] = ov[r];
        if (t == 0) {
          static_cast<float*>(p.m_out)[idx] = m[r] * Dom<float>::kToNat;
          static_cast<float*>(p.l_out)[idx] = L[r];
        }
        continue;
      }
      static_cast<T*>(p.out)[idx * 128 + t] = from_acc<T>(ov[r] / L[r]);
      if (t == 0) {
        if (!(L[r] > 0.f)) atomicOr(&p.ctrl->error, 1);
        if (p.lse) p.lse[idx] = (m[r] + log2f(L[r])) * Dom<float>::kToNat;
      }
    }
  }
}

template <typename T, int kMode>
__global__ void __launch_bounds__(kThreads, 2) psa_persistent(const __grid_constant__ KParams p) {
  using A = typename AccOf<T>::type;
  constexpr bool kTiles = HasTiles<T>::v && kMode != kModeGeneric;
  constexpr bool kVecFast = HasTiles<T>::v && kMode == kModeFast;
  constexpr int RP = sizeof(A) == 8 ? 2 : 4;
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ int s_item;
  __shared__ int s_nmerge;
  __shared__ int s_merge[kTileM + 8];
  __shared__ tile::Barriers s_bar;
  __shared__ uint32_t s_tmem;
  __shared__ vec::Shared s_vec;
  __shared__ dec::Shared s_dec;
  __shared__ A s_rowM[kTileM], s_rowL[kTileM];
  __shared__ A s_fac[kWarps * 8];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t t_kernel0 = (p.trace_cap > 0 && threadIdx.x == 0) ? int64_t(globaltimer()) : 0;
  tile::State tst{0u, 0u, 0u};
  const bool tiles = kTiles && p.use_tiles;
  const bool dec_on = kVecFast && p.use_dec;
  const bool tmem_on = tiles || dec_on;
  if (kVecFast) {
    if (threadIdx.x == 0) vec::init_barriers(&s_vec);
    if (threadIdx.x == 32) {
      dev::tma_prefetch_desc(&p.tmv_kp);
      dev::tma_prefetch_desc(&p.tmv_vp);
      dev::tma_prefetch_desc(&p.tmv_kd);
      dev::tma_prefetch_desc(&p.tmv_vd);
    }
    __syncthreads();
  }
  if (kTiles && !tmem_on && warp == 5) dev::tmem_relinquish();
  if (dec_on && threadIdx.x == 0) dec::init_barriers(&s_dec);
  if (dec_on && threadIdx.x == 4 * 32) {
    dev::tma_prefetch_desc(&p.tmd_kp);
    dev::tma_prefetch_desc(&p.tmd_vp);
    dev::tma_prefetch_desc(&p.tmd_kd);
    dev::tma_prefetch_desc(&p.tmd_vd);
  }
  if (tmem_on) {
    if (threadIdx.x == 0) tile::init_barriers(&s_bar);
    if (warp == 4 && lane == 0) {
      dev::tma_prefetch_desc(&p.tm_q);
      dev::tma_prefetch_desc(&p.tm_kp);
      dev::tma_prefetch_desc(&p.tm_vp);
      dev::tma_prefetch_desc(&p.tm_kd);
      dev::tma_prefetch_desc(&p.tm_vd);
    }
    if (warp == 5) dev::tmem_alloc<tile::kTmemCols>(&s_tmem);
    dev::tc_fence_before();
    __syncthreads();
    dev::tc_fence_after();
    tst.tmem = s_tmem;
  }

  // ---- CTA-level items from cursor `next_item`, indices [0, n) ------------------
  auto cta_phase = [&](int n) {
    if (tiles && threadIdx.x == 4 * 32) dev::fence_proxy_async_smem();
    for (;;) {
      if (threadIdx.x == 0) s_item = atomicAdd(&p.ctrl->next_item, 1);
      __syncthreads();
      const int idx = s_item;
      if (idx >= n) break;
      const ItemRec it = load_item(p.items + (int64_t)idx * kItemWords);
      int64_t t0 = 0;
      if (p.trace_cap > 0 && threadIdx.x == 0) t0 = int64_t(globaltimer());
      if constexpr (kTiles) {
        if (it.kind == kItemTile) tst = tile::tile_item<T>(p, it, smem, &s_bar, tst);
        else if constexpr (!kVecFast) vec_item_generic<T, A, RP>(p, it, smem, s_fac, s_rowM, s_rowL);
      } else {
        vec_item_generic<T, A, RP>(p, it, smem, s_fac, s_rowM, s_rowL);
      }
      if (it.ws_row >= 0) cta_arrive_and_merge<T, A>(p, it, s_merge, &s_nmerge, s_rowM, s_rowL);
      if (p.trace_cap > 0 && threadIdx.x == 0) trace_item(p, idx, it.kind, t0);
      if (tiles) dev::tc_fence_before();
      __syncthreads();
      if (tiles) dev::tc_fence_after();
    }
  };

  if constexpr (kVecFast) {
    // Two queues: TILE items [0, n_tile) are CTA-level, VEC items [n_tile, n) are
    // warp-level. CTAs below n_tile_ctas start on the tile queue, the rest on the
    // VEC queue; each drains the other queue once its own is empty.
    auto warp_phase = [&]() {
      uint8_t* ring = vec::warp_ring(smem, warp, p.d);
      uint32_t vcnt = 0;  // ring phase bookkeeping (barriers are fresh every launch)
      for (;;) {
        int i = 0;
        if (lane == 0) i = atomicAdd(&p.ctrl->next_vec, 1);
        i = __shfl_sync(0xffffffffu, i, 0);
        const int idx = p.n_tile_items + i;
        if (idx >= p.num_items) break;
        const ItemRec it = load_item(p.items + (int64_t)idx * kItemWords);
        int64_t t0 = 0;
        if (p.trace_cap > 0 && lane == 0) t0 = int64_t(globaltimer());
        auto em = [&](int r, int c, float M, float L, const float (&o)[8]) {
          emit4<T>(p, it, r, c, M, L, make_float4(o[0], o[1], o[2], o[3]));
          emit4<T>(p, it, r, c + 4, M, L, make_float4(o[4], o[5], o[6], o[7]));
        };
        if (p.d == 128)
          vcnt = vec::warp_item<T, 128>(p, it, ring, s_vec.full[warp], s_vec.p[warp], vcnt, em);
        else
          vcnt = vec::warp_item<T, 64>(p, it, ring, s_vec.full[warp], s_vec.p[warp], vcnt, em);
        if (it.ws_row >= 0) warp_arrive_and_merge<T>(p, it);
        if (p.trace_cap > 0 && lane == 0) trace_item(p, idx, it.kind, t0);
      }
    };
    auto dec_phase = [&]() {
      auto load_at = [&](int idx) { return load_item(p.items + (int64_t)idx * kItemWords); };
      auto finish = [&](const ItemRec& it, const int64_t* oidx, int idx, int t, int R, const float (&m)[dec::kR],
                        const float (&L)[dec::kR], const float (&ov)[dec::kR]) {
        dec_finish<T>(p, &s_dec, it, oidx, idx, t, R, m, L, ov, 0);
      };
      auto arrive = [&](int idx) {
        warp_arrive_rows(p, load_at(idx), INT_MIN, INT_MAX,
                         [&](int u) { merge_unit_warp<T>(p, u); });
      };
      dec::run<T>(p, smem, &s_dec, tst.tmem, 0, load_at, finish, arrive);
    };
    if (dec_on) {
      cta_phase(p.n_tile_items);
      __syncthreads();
      dec_phase();
    } else if (int(blockIdx.x) < p.n_tile_ctas) {
      cta_phase(p.n_tile_items);
      warp_phase();
    } else {
      warp_phase();
      __syncthreads();
      cta_phase(p.n_tile_items);
    }
  } else {
    cta_phase(p.num_items);
  }
  // Every warp of this CTA must be done pulling from the queues before the CTA
  // counts itself out: the last CTA out resets the cursors for the next launch.
  __syncthreads();
  if (p.trace_cap > 0 && threadIdx.x == 0)  // per-CTA residency record after the items
    trace_item(p, p.num_items + int(blockIdx.x), -1, t_kernel0);
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&p.ctrl->done, 1) == (int)gridDim.x - 1) {
      p.ctrl->next_item = 0;
      p.ctrl->next_vec = 0;
      p.ctrl->done = 0;
      __threadfence();
    }
  }
  if (tmem_on) {
    dev::tc_fence_before();
    __syncthreads();
    if (warp == 5) dev::tmem_dealloc<tile::kTmemCols>(tst.tmem);
  }
}

// ---------------------------------------------------------------------------
// v2 kernel (bf16/f16, d == dv == 128): ONE CTA per SM, 512 threads.
//   tile phase  — tile2::run: two 128-row softmax slots share every K/V block
//                 (warps 0-7 softmax, 8 producer, 9 MMA, 10-15 merges), all
//                 512 TMEM columns;
//   decode phase — two independent dec pipelines (warps 0-7 and 8-15), each
//                 with its own K/V ring in one half of shared memory.
// The tile phase drains the CTA-level TILE queue, the decode phase the VEC
// queue; the last CTA out resets both cursors.
// ---------------------------------------------------------------------------
constexpr int kV2Threads = 512;
#ifndef PSA_EMU_EVERY
#define PSA_EMU_EVERY 4
#endif
constexpr int kV2EmuEvery = PSA_EMU_EVERY;  // every 4th exp pair of the tile softmax on the FMA pipe

__device__ __forceinline__ void setmaxnreg_inc_168() { asm volatile("setmaxnreg.inc.sync.aligned.u32 168;"); }
__device__ __forceinline__ void setmaxnreg_dec_88() { asm volatile("setmaxnreg.dec.sync.aligned.u32 88;"); }
__device__ __forceinline__ void setmaxnreg_inc_128() { asm volatile("setmaxnreg.inc.sync.aligned.u32 128;"); }

template <typename T, int kEmu, bool kCausal, int kRows>
__global__ void __launch_bounds__(kV2Threads, 1) psa_v2(const __grid_constant__ KParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ tile2::Shared s_t2;
  __shared__ dec::Shared s_dec[2];
  __shared__ uint32_t s_tmem;
  __shared__ int s_dbg_n;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t t_kernel0 = (p.trace_cap > 0 && threadIdx.x == 0) ? int64_t(globaltimer()) : 0;
  if (threadIdx.x == 0) {
    s_dbg_n = 0;
    tile2::init(&s_t2);
    dec::init_barriers(&s_dec[0]);
    dec::init_barriers(&s_dec[1]);
  }
  if (warp == tile2::kProducerWarp && lane == 0) {
    if (p.use_tiles) dev::tma_prefetch_desc(&p.tm_q);
    {
      dev::tma_prefetch_desc(&p.tmd_kp);
      dev::tma_prefetch_desc(&p.tmd_vp);
      dev::tma_prefetch_desc(&p.tmd_kd);
      dev::tma_prefetch_desc(&p.tmd_vd);
    }
  }
  if (warp == tile2::kMmaWarp) dev::tmem_alloc<tile2::kTmemCols>(&s_tmem);
  dev::tc_fence_before();
  __syncthreads();
  dev::tc_fence_after();
  const uint32_t tmem = s_tmem;
  auto load_at = [&](int idx) { return load_item(p.items + (int64_t)idx * kItemWords); };
  // Merge-queue tasks. Decode pipelines: an item index (arrive at all its units,
  // merge the completed ones). Tile phase: 2 * item + slot (arrive at the units of
  // that slot's rows) or ~u (merge unit u): a slot can complete dozens of units, so
  // they go back to the queue and all six merge warps share them.
  auto merge_now = [&](int u) { merge_unit_warp<T>(p, u); };
  auto arrive_dec = [&](int idx) {
    int dslot = -1;  // diagnostics: CTA 0, pipeline 0, ticket < 64
    if (p.trace_cap > 0 && blockIdx.x == 0 && threadIdx.x < 256) {
      int n = 0;
      if ((threadIdx.x & 31) == 0) n = atomicAdd(&s_dbg_n, 1);
      n = __shfl_sync(0xffffffffu, n, 0);
      if (n < 64) dslot = n;
    }
    warp_arrive_rows(p, load_at(idx), INT_MIN, INT_MAX, merge_now, dslot);
    if (dslot >= 0) dbg_clock(p, 39, dslot);
  };
  auto tile_task = [&](int task) {
    if (task < 0) {
      merge_unit_warp<T>(p, ~task);
      return;
    }
    const ItemRec it = load_at(task >> 1);
    const int tile_rows = p.gqa * (tile2::kM / p.gqa);
    const int i = task & 1;
    const int r0 = it.row0 + i * tile_rows;
    const int r1 = i == 0 ? it.row0 + min(it.nrows, tile_rows) : it.row0 + it.nrows;
    warp_arrive_rows(p, it, r0, r1, [&](int u) {
      int queued = 0;
      if ((threadIdx.x & 31) == 0 && dev::mq_pending(&s_t2.mq) < dev::MergeQueue::kCap / 2) {
        dev::mq_push(&s_t2.mq, ~u);
        queued = 1;
      }
      if (!__shfl_sync(0xffffffffu, queued, 0)) merge_unit_warp<T>(p, u);
    });
  };

  // diagnostics: per-CTA phase record {t(softmax done), t(producer/MMA done), t(merge
  // warps done), t(tile phase barrier passed)} at trace row num_items + 2048 + CTA
  auto phase_mark = [&](int field, int row = 2048) {
    if (p.trace_cap > 0 && (threadIdx.x & 31) == 0)
      atomicMax(reinterpret_cast<unsigned long long*>(
                    p.trace + (int64_t(p.num_items) + row + blockIdx.x) * 4 + field),
                (unsigned long long)globaltimer());
  };
  auto tile_phase = [&]() {
    if (warp < 8) {
      setmaxnreg_inc_168();
      tile2::run_softmax<T, kEmu, kCausal>(p, &s_t2, tmem, load_at);
      phase_mark(0);
      setmaxnreg_dec_88();
    } else {
      setmaxnreg_dec_88();
      if (warp < tile2::kMergeWarp0) {
        tile2::run_support<T>(p, smem, &s_t2, tmem, load_at);
        phase_mark(1);
      }
    }
    // Merge workers: warps 10-15 from the start; every other warp joins once its tile
    // role is done and both softmax WGs closed the queue — a tile slot can complete
    // dozens of merge units at once (a long prefix split into many chunks: fan-in
    // ~17), which six warps of one CTA would otherwise work off alone.
    __syncwarp();
    if (warp < tile2::kMergeWarp0) dev::mq_wait_closed(&s_t2.mq, 2);
    dev::mq_drain(&s_t2.mq, 2, tile_task);
    phase_mark(2);
    setmaxnreg_inc_128();
  };
  auto dec_phase = [&]() {
    if ((warp >> 3) >= p.dec_pipes) return;
    const int pi = warp >> 3;
    const size_t half = dec::pipe_stride(p.dec_slots);
    auto finish = [&](const ItemRec& it, const int64_t* oidx, int idx, int t, int R, const float (&m)[dec::kR],
                      const float (&L)[dec::kR], const float (&ov)[dec::kR]) {
      dec_finish<T>(p, &s_dec[pi], it, oidx, idx, t, R, m, L, ov, pi);
    };
    dec::run<T, kCausal, kRows>(p, smem + pi * half, &s_dec[pi], tmem + 64u * uint32_t(pi), pi, load_at, finish,
                arrive_dec, DecFast<T>{p});
    // diagnostics: decode-phase record at trace row num_items + 3072 + CTA:
    // {softmax warps, producer, MMA warp, merge warps} done
    const int rw = (warp & 7) < 4 ? 0 : (warp & 7) == 4 ? 1 : (warp & 7) == 5 ? 2 : 3;
    phase_mark(rw, 3072);
  };
  // Tile phase, then decode phase. Between them every role of the tile phase is done
  // (its TMA loads were all consumed, its TMEM reads/writes completed) before the
  // decode pipelines reuse shared memory and TMEM. (Each phase body is inlined once:
  // the kernel's instruction footprint is itself a measured cost.)
  if (p.use_tiles) {
    tile_phase();
    dev::tc_fence_before();
    __syncthreads();
    dev::tc_fence_after();
    if (threadIdx.x == 0) phase_mark(3);
  }
  if (p.use_dec) dec_phase();
  __syncthreads();
  if (p.trace_cap > 0 && threadIdx.x == 0) trace_item(p, p.num_items + int(blockIdx.x), -1, t_kernel0);
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&p.ctrl->done, 1) == (int)gridDim.x - 1) {
      p.ctrl->next_item = 0;
      p.ctrl->next_vec = 0;
      p.ctrl->done = 0;
      __threadfence();
    }
  }
  dev::tc_fence_before();
  __syncthreads();
  if (warp == tile2::kMmaWarp) dev::tmem_dealloc<tile2::kTmemCols>(tmem);
}

// ---- standalone building blocks (PartialResult API) -----------------------

template <typename A>
__global__ void merge_kernel(int64_t rows, int32_t dv, const A* oa, const A* ma, const A* la,
                             const A* ob, const A* mb, const A* lb, A* o, A* m, A* l) {
  // One block per row, threads over columns (blockDim >= dv).
  for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
    const A a_m = ma[r], b_m = mb[r], a_l = la[r], b_l = lb[r];
    const A mm = max(a_m, b_m);
    // attention.py:109-114: rows with l == 0 contribute nothing (exp(-inf - -inf) is masked).
    const A fa = a_l > A(0) ? A(exp(double(a_m - mm))) : A(0);
    const A fb = b_l > A(0) ? A(exp(double(b_m - mm))) : A(0);
    const int c = threadIdx.x;
    if (c < dv) o[r * dv + c] = fa * oa[r * dv + c] + fb * ob[r * dv + c];
    __syncthreads();  // m/l outputs may alias inputs: every thread has read them
    if (c == 0) {
      m[r] = mm;
      l[r] = fa * a_l + fb * b_l;
    }
    __syncthreads();
  }
}

template <typename A, typename T>
__global__ void finalize_kernel(int64_t rows, int32_t dv, const A* o, const A* l, T* out,
                                int32_t* bad) {
  const int64_t n = rows * dv;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / dv;
    const A lr = l[r];
    out[i] = T(o[i] / lr);
    if (i % dv == 0 && !(lr > A(0))) atomicAdd(bad, 1);
  }
}

template <typename T>
__global__ void nonfinite_kernel(const T* x, int64_t n, int32_t* count) {
  int local = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    local += !isfinite((double)ld_acc(x + i));
  local = __reduce_add_sync(0xffffffffu, local);
  if ((threadIdx.x & 31) == 0 && local) atomicAdd(count, local);
}

// Dynamic shared memory per CTA and the ring depths that fit it: 2 CTAs/SM get
// ~110 KB each (tile: 2 K/V stages, decode: 3 slots), 1 CTA/SM gets ~220 KB
// (tile: 4 stages, decode: 6 slots).
template <typename T>
size_t smem_for(KParams& p, int mode, int ctas_per_sm) {
  using A = typename AccOf<T>::type;
  constexpr int RP = sizeof(A) == 8 ? 2 : 4;
  const size_t budget = (ctas_per_sm >= 2 ? size_t(227) * 1024 / 2 : size_t(227) * 1024) - 6 * 1024;
  size_t smem = mode == kModeFast ? 0 : size_t(kWarps) * RP * (p.dv + 2) * sizeof(A);
  p.tile_stages = 2;
  p.dec_slots = 3;
  if (HasTiles<T>::v && mode != kModeGeneric && p.use_tiles) {
    while (p.tile_stages < tile::kMaxStages &&
           tile::smem_bytes(p.d, p.dv, p.tile_stages + 1) <= budget)
      ++p.tile_stages;
    const size_t t = tile::smem_bytes(p.d, p.dv, p.tile_stages);
    if (t > smem) smem = t;
  }
  if (HasTiles<T>::v && mode == kModeFast) {
    if (p.use_dec) {
      while (p.dec_slots < dec::kMaxSlots && dec::smem_bytes(p.dec_slots + 1) <= budget)
        ++p.dec_slots;
    }
    const size_t v = p.use_dec ? dec::smem_bytes(p.dec_slots) : vec::smem_bytes(p.d);
    if (v > smem) smem = v;
  }
  return smem;
}

template <typename T, int kMode>
int launch_mode(const KParams& p_in, int32_t num_sms, int32_t ctas_per_sm, void* stream) {
  KParams p = p_in;
  const size_t smem = smem_for<T>(p, kMode, ctas_per_sm);
  cudaError_t e = cudaFuncSetAttribute(psa_persistent<T, kMode>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  if (e != cudaSuccess) return e;
  // Two CTAs per SM only fit with the maximum shared-memory carveout.
  e = cudaFuncSetAttribute(psa_persistent<T, kMode>,
                           cudaFuncAttributePreferredSharedMemoryCarveout,
                           int(cudaSharedmemCarveoutMaxShared));
  if (e != cudaSuccess) return e;
  const int grid = num_sms * ctas_per_sm;
  psa_persistent<T, kMode><<<grid, kThreads, smem, static_cast<cudaStream_t>(stream)>>>(p);
  return cudaGetLastError();
}

// v2: 227 KB of dynamic shared memory per CTA; the tile ring and the two decode
// rings take as many 32 KB slots as fit.
template <typename T>
int launch_v2(const KParams& p_in, int32_t num_sms, void* stream) {
  KParams p = p_in;
  const size_t budget = size_t(227) * 1024 - 4 * 1024;  // minus static shared memory
  p.tile_stages = 2;
  while (p.tile_stages < tile2::kMaxRing && tile2::smem_bytes(p.tile_stages + 1) <= budget)
    ++p.tile_stages;
  p.dec_slots = 2;
  while (p.dec_slots < dec::kMaxSlots && 2 * dec::pipe_stride(p.dec_slots + 1) <= budget)
    ++p.dec_slots;
  // Diagnostics (PSA_DEBUG bit mask): 1 = one decode pipeline per CTA, 2 = two ring slots.
  const char* dbg_env = std::getenv("PSA_DEBUG");
  const int dbg = dbg_env ? std::atoi(dbg_env) : 0;
  p.dec_pipes = (dbg & 1) ? 1 : 2;
  p.tile_pp = (dbg & 32) ? 0 : 1;
  p.dec_fast = (dbg & 256) ? 0 : 1;
  const char* dbg_cta = std::getenv("PSA_DBG_CTA");
  p.dbg_cta = dbg_cta ? std::atoi(dbg_cta) : 0;
  if (dbg & 2) p.dec_slots = 2;
  if (const char* tr = std::getenv("PSA_TILE_RING"))  // diagnostics: a shallower tile ring
    p.tile_stages = std::max(2, std::min(p.tile_stages, std::atoi(tr)));
  if (dbg & 128) {  // one decode pipeline with the whole ring (diagnostics)
    p.dec_pipes = 1;
    while (p.dec_slots < dec::kMaxSlots && dec::pipe_stride(p.dec_slots + 1) <= budget) ++p.dec_slots;
  }
  size_t smem = 0;
  if (p.use_tiles) smem = tile2::smem_bytes(p.tile_stages);
  if (p.use_dec) {
    smem = std::max(smem, size_t(p.dec_pipes) * dec::pipe_stride(p.dec_slots));
  }
  // decode rows per item: 4 (one token of gqa <= 4 heads) or 8
  const bool r4 = p.max_vec_rows <= 4;
  auto kern = (p.flags & PSA_FLAG_CAUSAL)
                  ? (r4 ? psa_v2<T, kV2EmuEvery, true, 4> : psa_v2<T, kV2EmuEvery, true, 8>)
                  : (r4 ? psa_v2<T, kV2EmuEvery, false, 4> : psa_v2<T, kV2EmuEvery, false, 8>);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       int(smem));
  if (e != cudaSuccess) return e;
  kern<<<num_sms, kV2Threads, smem, static_cast<cudaStream_t>(stream)>>>(p);
  return cudaGetLastError();
}

template <typename T>
int launch_typed(const KParams& p, int32_t num_sms, int32_t ctas_per_sm, void* stream) {
  if constexpr (HasTiles<T>::v) {
    if (p.use_v2) return launch_v2<T>(p, num_sms, stream);
    if (p.use_vec_fast) return launch_mode<T, kModeFast>(p, num_sms, ctas_per_sm, stream);
    if (p.use_tiles) return launch_mode<T, kModeTileGeneric>(p, num_sms, ctas_per_sm, stream);
  }
  return launch_mode<T, kModeGeneric>(p, num_sms, ctas_per_sm, stream);
}

inline int grid_for(int64_t n) {
  int64_t b = (n + 255) / 256;
  return int(b < 1 ? 1 : (b > 4096 ? 4096 : b));
}

}  // namespace

int launch_psa(const KParams& p, int32_t dtype, int32_t num_sms, int32_t ctas_per_sm,
               bool use_tiles, void* stream) {
  (void)use_tiles;
  switch (dtype) {
    case PSA_DTYPE_F32: return launch_typed<float>(p, num_sms, ctas_per_sm, stream);
    case PSA_DTYPE_BF16: return launch_typed<__nv_bfloat16>(p, num_sms, ctas_per_sm, stream);
    case PSA_DTYPE_F16: return launch_typed<__half>(p, num_sms, ctas_per_sm, stream);
    case PSA_DTYPE_F64: return launch_typed<double>(p, num_sms, ctas_per_sm, stream);
    default: return cudaErrorInvalidValue;
  }
}

size_t kernel_smem_bytes(int32_t dtype, bool use_tiles) {
  (void)use_tiles;
  return dtype == PSA_DTYPE_F64 ? size_t(kWarps) * 2 * (256 + 2) * 8
                                : size_t(kWarps) * 4 * (256 + 2) * 4;
}

namespace {
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                              const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                              const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeFn encode_fn() {
  static EncodeFn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return reinterpret_cast<EncodeFn>(f);
  }();
  return fn;
}

// rank-3 (d, Hkv, keys) map with a (box_inner, 1, box_rows) box.
int encode_kv(CUtensorMap* m, CUtensorMapDataType dt, const void* base, int64_t keys, int heads,
              int dim, int box_inner, int box_rows, bool swizzle128) {
  std::memset(m, 0, sizeof(*m));
  if (keys <= 0 || base == nullptr) return 0;
  cuuint64_t gdim[3] = {cuuint64_t(dim), cuuint64_t(heads), cuuint64_t(keys)};
  cuuint64_t gstride[2] = {cuuint64_t(dim) * 2, cuuint64_t(dim) * heads * 2};
  cuuint32_t box[3] = {cuuint32_t(box_inner), 1, cuuint32_t(box_rows)};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = encode_fn()(m, dt, 3, const_cast<void*>(base), gdim, gstride, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE,
                           swizzle128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : int(cudaErrorInvalidValue);
}
}  // namespace

bool dec_supported(int32_t dtype, int32_t d, int32_t dv) {
  return (dtype == PSA_DTYPE_BF16 || dtype == PSA_DTYPE_F16) && d == 128 && dv == 128;
}

bool v2_supported(int32_t dtype, int32_t d, int32_t dv) { return dec_supported(dtype, d, dv); }

bool vec_fast_supported(int32_t dtype, int32_t d, int32_t dv) {
  return (dtype == PSA_DTYPE_BF16 || dtype == PSA_DTYPE_F16) && d == dv && (d == 64 || d == 128);
}

int encode_tile_maps(KParams& p, int32_t dtype, int64_t T, int64_t prefix_keys,
                     int64_t distinct_keys) {
  if (!encode_fn()) return int(cudaErrorNotSupported);
  const CUtensorMapDataType dt = dtype == PSA_DTYPE_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                                         : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  int e = 0;
  if (p.use_tiles) {
    std::memset(&p.tm_q, 0, sizeof(p.tm_q));
    const int gqa = p.gqa;
    cuuint64_t gdim[4] = {cuuint64_t(p.d), cuuint64_t(gqa), cuuint64_t(p.Hkv), cuuint64_t(T)};
    cuuint64_t gstride[3] = {cuuint64_t(p.d) * 2, cuuint64_t(p.d) * gqa * 2,
                             cuuint64_t(p.d) * p.Hq * 2};
    cuuint32_t box[4] = {64, cuuint32_t(gqa), 1, cuuint32_t(tile::kM / gqa)};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    CUresult r = encode_fn()(&p.tm_q, dt, 4, const_cast<void*>(p.q), gdim, gstride, box, estr,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return int(cudaErrorInvalidValue);
    e = encode_kv(&p.tm_kp, dt, p.kp, prefix_keys, p.Hkv, p.d, 64, tile::kBN, true);
    if (!e) e = encode_kv(&p.tm_vp, dt, p.vp, prefix_keys, p.Hkv, p.dv, 64, tile::kBN, true);
    if (!e) e = encode_kv(&p.tm_kd, dt, p.kd, distinct_keys, p.Hkv, p.d, 64, tile::kBN, true);
    if (!e) e = encode_kv(&p.tm_vd, dt, p.vd, distinct_keys, p.Hkv, p.dv, 64, tile::kBN, true);
  }
  if (!e && (p.use_dec || p.use_v2)) {
    std::memset(&p.tmd_q, 0, sizeof(p.tmd_q));
    const int gqa = p.gqa;
    p.dec_q_tma = 0;
    if (gqa <= dec::kN && (dec::kN % gqa) == 0 && T > 0) {
      cuuint64_t gdim[4] = {cuuint64_t(p.d), cuuint64_t(gqa), cuuint64_t(p.Hkv), cuuint64_t(T)};
      cuuint64_t gstride[3] = {cuuint64_t(p.d) * 2, cuuint64_t(p.d) * gqa * 2,
                               cuuint64_t(p.d) * p.Hq * 2};
      cuuint32_t box[4] = {64, cuuint32_t(gqa), 1, cuuint32_t(dec::kN / gqa)};
      cuuint32_t estr[4] = {1, 1, 1, 1};
      CUresult r = encode_fn()(&p.tmd_q, dt, 4, const_cast<void*>(p.q), gdim, gstride, box, estr,
                               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) return int(cudaErrorInvalidValue);
      p.dec_q_tma = 1;
    }
    const int rows = p.page_size ? p.page_size : dec::kBK;  // paged: one box per page
    e = encode_kv(&p.tmd_kp, dt, p.kp, prefix_keys, p.Hkv, p.d, 64, rows, true);
    if (!e) e = encode_kv(&p.tmd_vp, dt, p.vp, prefix_keys, p.Hkv, p.dv, 64, rows, true);
    if (!e) e = encode_kv(&p.tmd_kd, dt, p.kd, distinct_keys, p.Hkv, p.d, 64, rows, true);
    if (!e) e = encode_kv(&p.tmd_vd, dt, p.vd, distinct_keys, p.Hkv, p.dv, 64, rows, true);
  }
  if (!e && p.use_vec_fast) {
    e = encode_kv(&p.tmv_kp, dt, p.kp, prefix_keys, p.Hkv, p.d, p.d, vec::kKB, false);
    if (!e) e = encode_kv(&p.tmv_vp, dt, p.vp, prefix_keys, p.Hkv, p.dv, p.dv, vec::kKB, false);
    if (!e) e = encode_kv(&p.tmv_kd, dt, p.kd, distinct_keys, p.Hkv, p.d, p.d, vec::kKB, false);
    if (!e) e = encode_kv(&p.tmv_vd, dt, p.vd, distinct_keys, p.Hkv, p.dv, p.dv, vec::kKB, false);
  }
  return e;
}

int launch_merge(int64_t rows, int32_t dv, int32_t dtype, const void* oa, const void* ma,
                 const void* la, const void* ob, const void* mb, const void* lb, void* o,
                 void* m, void* l, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // One block per row keeps the alias-safe barrier inside a row.
  if (dv > 1024) return cudaErrorInvalidValue;
  const int threads = ((dv + 31) / 32) * 32;
  const int grid = int(rows < 65535 ? rows : 65535);
  if (rows == 0) return cudaSuccess;
  if (dtype == PSA_DTYPE_F64)
    merge_kernel<double><<<grid, threads, 0, s>>>(
        rows, dv, (const double*)oa, (const double*)ma, (const double*)la, (const double*)ob,
        (const double*)mb, (const double*)lb, (double*)o, (double*)m, (double*)l);
  else
    merge_kernel<float><<<grid, threads, 0, s>>>(
        rows, dv, (const float*)oa, (const float*)ma, (const float*)la, (const float*)ob,
        (const float*)mb, (const float*)lb, (float*)o, (float*)m, (float*)l);
  return cudaGetLastError();
}

int launch_finalize(int64_t rows, int32_t dv, int32_t dtype, const void* o, const void* l,
                    void* out, int32_t* bad, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t n = rows * dv;
  if (n == 0) return cudaSuccess;
  if (dtype == PSA_DTYPE_F64)
    finalize_kernel<double, double><<<grid_for(n), 256, 0, s>>>(rows, dv, (const double*)o,
                                                              (const double*)l, (double*)out, bad);
  else
    finalize_kernel<float, float><<<grid_for(n), 256, 0, s>>>(rows, dv, (const float*)o,
                                                            (const float*)l, (float*)out, bad);
  return cudaGetLastError();
}

int launch_count_nonfinite(const void* data, int64_t n, int32_t dtype, int32_t* count,
                           void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (n == 0) return cudaSuccess;
  switch (dtype) {
    case PSA_DTYPE_F32: nonfinite_kernel<<<grid_for(n), 256, 0, s>>>((const float*)data, n, count); break;
    case PSA_DTYPE_BF16: nonfinite_kernel<<<grid_for(n), 256, 0, s>>>((const __nv_bfloat16*)data, n, count); break;
    case PSA_DTYPE_F16: nonfinite_kernel<<<grid_for(n), 256, 0, s>>>((const __half*)data, n, count); break;
    case PSA_DTYPE_F64: nonfinite_kernel<<<grid_for(n), 256, 0, s>>>((const double*)data, n, count); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace psa
