// common.cuh — device helpers for the sm_100a DDP kernels: 128-bit vector
// access, fp32/bf16 lane conversion, and the CTA-cooperative multi-source /
// multi-destination transfer used by pack, the P2P reduction
// and unpack.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../internal.h"

namespace b200ddp {

// Slot table passed BY VALUE (__grid_constant__): the gradients of one bucket
// (or of a run of its slots) and their element offsets inside the bucket.
template <int MAXS>
struct SlotArgs {
  void* grad[MAXS];
  int64_t off[MAXS + 1];
  int32_t n;
};

// ---- 128-bit memory access -------------------------------------------------
// Gradients are not written by anyone while a kernel reads them: read-only path.
__device__ __forceinline__ uint4 ld_nc_v4(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
// Staging / bucket data written by peers during the kernel: L2-coherent load.
__device__ __forceinline__ uint4 ld_cg_v4(const void* p) {
  uint4 r;
  asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p) : "memory");
  return r;
}
__device__ __forceinline__ void st_v4(void* p, const uint4& v) {
  asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w) : "memory");
}

// ---- element conversions (fp32 accumulate, RNE back; reading C-4) ----------
template <typename T> struct Elem;
template <> struct Elem<float> {
  static constexpr int VE = 4;  // elements per 16 bytes
  __device__ static __forceinline__ float to_f(float x) { return x; }
  __device__ static __forceinline__ float from_f(float x) { return x; }
  __device__ static __forceinline__ void unpack(const uint4& v, float (&f)[8]) {
    f[0] = __uint_as_float(v.x); f[1] = __uint_as_float(v.y);
    f[2] = __uint_as_float(v.z); f[3] = __uint_as_float(v.w);
  }
  __device__ static __forceinline__ uint4 pack(const float (&f)[8]) {
    return make_uint4(__float_as_uint(f[0]), __float_as_uint(f[1]), __float_as_uint(f[2]),
                      __float_as_uint(f[3]));
  }
};
template <> struct Elem<__nv_bfloat16> {
  static constexpr int VE = 8;
  __device__ static __forceinline__ float to_f(__nv_bfloat16 x) { return __bfloat162float(x); }
  __device__ static __forceinline__ __nv_bfloat16 from_f(float x) { return __float2bfloat16_rn(x); }
  __device__ static __forceinline__ void unpack(const uint4& v, float (&f)[8]) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      f[2 * i] = __uint_as_float(w[i] << 16);
      f[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
    }
  }
  __device__ static __forceinline__ uint4 pack(const float (&f)[8]) {
    uint32_t w[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint32_t lo = __bfloat16_as_ushort(__float2bfloat16_rn(f[2 * i]));
      const uint32_t hi = __bfloat16_as_ushort(__float2bfloat16_rn(f[2 * i + 1]));
      w[i] = lo | (hi << 16);
    }
    return make_uint4(w[0], w[1], w[2], w[3]);
  }
};

// ---- CTA-cooperative transfer ------------------------------------------------
// For i in [0, n):  y = sum_{k<NS} src_k[i]  (fp32, in k order; a plain load
// when NS == 1), optionally y = fl(y * s), then dst_j[i] = RNE_T(y), j < ND.
// Vectorized (16 B) when every pointer has the same address mod 16, with a
// scalar head/tail; scalar otherwise.  SRC_NC: sources are read-only for the
// kernel's lifetime (gradients) -> non-coherent path; else L2-coherent loads
// (data written by peers inside the kernel).  NS / ND are compile-time so the
// pointer and value arrays live in registers; U vectors per source are kept
// in flight per thread (U * NS >= 4).
// EACH (with SCALE): every operand is scaled and rounded to T BEFORE the sum,
//   y = RNE_T( sum_k RNE_T(src_k[i] * s) )        (oracle O-3b written out),
// so raw gradients can be reduced with the 1/W of pack applied on the fly.
// grp_xfer: the same over a GROUP of nt threads of the CTA (thread index tid in
// [0, nt)), for warp-specialized kernels; cta_xfer = the whole CTA.
template <typename T, int NS, int ND, bool SRC_NC, bool SCALE, bool EACH = false, int UF = 0>
__device__ __forceinline__ void grp_xfer(T* const (&dst)[ND], const T* const (&src)[NS], int64_t n, float s,
                                         const int tid, const int nt) {
  using E = Elem<T>;
  constexpr int VE = E::VE;
  // 4 vectors per thread in flight for a plain copy: with many small CTAs this
  // measured best on B200 (tools/local_probe.cu; profiles/r01_local_u.md)
  constexpr int U = UF ? UF : NS <= 2 ? 4 : (NS >= 4 ? 1 : 4 / NS);
  if (n <= 0) return;
  const uintptr_t a0 = reinterpret_cast<uintptr_t>(dst[0]) & 15;
  uintptr_t mis = 0;
#pragma unroll
  for (int j = 0; j < ND; ++j) mis |= (reinterpret_cast<uintptr_t>(dst[j]) & 15) ^ a0;
#pragma unroll
  for (int k = 0; k < NS; ++k) mis |= (reinterpret_cast<uintptr_t>(src[k]) & 15) ^ a0;

  auto ld1 = [&](const T* p) -> float { return E::to_f(SRC_NC ? __ldg(p) : __ldcg(p)); };
  auto each = [&](float x) -> float { return E::to_f(E::from_f(__fmul_rn(x, s))); };
  auto scalar = [&](int64_t i) {
    float acc = ld1(src[0] + i);
    if (EACH) acc = each(acc);
#pragma unroll
    for (int k = 1; k < NS; ++k) acc = __fadd_rn(acc, EACH ? each(ld1(src[k] + i)) : ld1(src[k] + i));
    if (SCALE && !EACH) acc = __fmul_rn(acc, s);
    const T y = E::from_f(acc);
#pragma unroll
    for (int j = 0; j < ND; ++j) dst[j][i] = y;
  };

  if (mis != 0) {
    for (int64_t i = tid; i < n; i += nt) scalar(i);
    return;
  }
  int64_t head = a0 ? (int64_t)((16 - a0) / sizeof(T)) : 0;
  if (head > n) head = n;
  for (int64_t i = tid; i < head; i += nt) scalar(i);
  const int64_t nv = (n - head) / VE;
  auto vec = [&](int64_t v, const uint4 (&in)[NS]) {
    float acc[8], f[8];
    E::unpack(in[0], acc);
    if (EACH) {
#pragma unroll
      for (int e = 0; e < VE; ++e) acc[e] = each(acc[e]);
    }
#pragma unroll
    for (int k = 1; k < NS; ++k) {
      E::unpack(in[k], f);
#pragma unroll
      for (int e = 0; e < VE; ++e) acc[e] = __fadd_rn(acc[e], EACH ? each(f[e]) : f[e]);
    }
    if (SCALE && !EACH) {
#pragma unroll
      for (int e = 0; e < VE; ++e) acc[e] = __fmul_rn(acc[e], s);
    }
    const uint4 y = E::pack(acc);
#pragma unroll
    for (int j = 0; j < ND; ++j) st_v4(dst[j] + head + v * VE, y);
  };
  auto ldv = [&](const T* p) -> uint4 { return SRC_NC ? ld_nc_v4(p) : ld_cg_v4(p); };
  // U vectors per source in flight per thread; the last round is predicated so a
  // partial round still keeps its loads in flight together
  for (int64_t v = tid; v < nv; v += (int64_t)U * nt) {
    uint4 in[U][NS];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (v + (int64_t)u * nt < nv) {
#pragma unroll
        for (int k = 0; k < NS; ++k) in[u][k] = ldv(src[k] + head + (v + (int64_t)u * nt) * VE);
      }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (v + (int64_t)u * nt < nv) vec(v + (int64_t)u * nt, in[u]);
  }
  for (int64_t i = head + nv * VE + tid; i < n; i += nt) scalar(i);
}

template <typename T, int NS, int ND, bool SRC_NC, bool SCALE, bool EACH = false, int UF = 0>
__device__ __forceinline__ void cta_xfer(T* const (&dst)[ND], const T* const (&src)[NS], int64_t n,
                                         float s) {
  grp_xfer<T, NS, ND, SRC_NC, SCALE, EACH, UF>(dst, src, n, s, (int)threadIdx.x, (int)blockDim.x);
}

// First slot k with off[k] <= x < off[k+1]  (CTA-uniform binary search).
template <int MAXS>
__device__ __forceinline__ int find_slot(const SlotArgs<MAXS>& sa, int64_t x) {
  int a = 0, b = sa.n - 1;
  while (a < b) {
    const int m = (a + b + 1) >> 1;
    if (sa.off[m] <= x) a = m; else b = m - 1;
  }
  return a;
}

// Pack the bucket range [lo, hi) from the gradients into ND buffers:
// element x goes to dst_j[x - base], scaled by s (Alg. 1, C-2).
template <typename T, int ND, int MAXS>
__device__ __forceinline__ void walk_pack(const SlotArgs<MAXS>& sa, int64_t lo, int64_t hi,
                                          T* const (&dstb)[ND], int64_t base, float s, int64_t gstride) {
  if (lo >= hi) return;
  for (int k = find_slot(sa, lo); k < sa.n && lo < hi; ++k) {
    const int64_t s0 = sa.off[k], e = min(hi, sa.off[k + 1]);
    if (e <= lo) continue;
    const T* g = reinterpret_cast<const T*>(static_cast<const char*>(sa.grad[k]) + gstride) + (lo - s0);
    T* d[ND];
#pragma unroll
    for (int j = 0; j < ND; ++j) d[j] = dstb[j] + (lo - base);
    const T* sp[1] = {g};
    cta_xfer<T, 1, ND, true, true>(d, sp, e - lo, s);
    lo = e;
  }
}

// Unpack / reduce the bucket range [lo, hi) into the gradients:
// grad(x) = RNE(sum_k src_k[x - base]) (NS == 1: plain copy back).
template <typename T, int NS, int MAXS>
__device__ __forceinline__ void walk_unpack(const SlotArgs<MAXS>& sa, int64_t lo, int64_t hi,
                                            const T* const (&srcb)[NS], int64_t base, int64_t gstride) {
  if (lo >= hi) return;
  for (int k = find_slot(sa, lo); k < sa.n && lo < hi; ++k) {
    const int64_t s0 = sa.off[k], e = min(hi, sa.off[k + 1]);
    if (e <= lo) continue;
    T* g = reinterpret_cast<T*>(static_cast<char*>(sa.grad[k]) + gstride) + (lo - s0);
    T* d[1] = {g};
    const T* sp[NS];
#pragma unroll
    for (int j = 0; j < NS; ++j) sp[j] = srcb[j] + (lo - base);
    cta_xfer<T, NS, 1, false, false>(d, sp, e - lo, 1.0f);
    lo = e;
  }
}

}  // namespace b200ddp
