// wire.cu — compressed wire for the copy-engine exchange (§8(f) N-3; PAPER.md
// L571-L573 "communicating gradients with the necessary precision"): fp32
// gradients travel as bf16 (half the NVLink and slot bytes).  Reading C-14 /
// oracle O-8, written out:
//   wire_gather:  slot_r[wire_k + i] = RNE_bf16( g_k[i] * fl(1/W) )      (pack)
//   wire_reduce:  g_k[i] = sum_{q=0..W-1} fp32(v_q)  in rank order, fp32,
//                 v_r = RNE_bf16(g_k[i] * fl(1/W)) recomputed locally (the same
//                 value rank r sent), v_q = slot q (bf16, from peer q)
// No final rounding: the gradient stays fp32.  HBM-bound: gather 1.5 S,
// reduce (1 + (W-1)/2 + 1) S for S = fp32 bucket bytes.
#include "common.cuh"

namespace b200ddp {

namespace {

constexpr int kTile = kThreads * 8 * 4;  // elements per CTA tile (8 per vector step, 4 steps)

template <int MAXS>
struct WArgs {
  float* grad[MAXS];
  int64_t wire[MAXS];
  int64_t vo[MAXS + 1];
  int32_t n;
};

template <int MAXS>
__device__ __forceinline__ int find_w(const WArgs<MAXS>& a, int64_t x) {
  int lo = 0, hi = a.n - 1;
  while (lo < hi) {
    const int m = (lo + hi + 1) >> 1;
    if (a.vo[m] <= x) lo = m; else hi = m - 1;
  }
  return lo;
}

__device__ __forceinline__ uint32_t pack2(float a, float b) {
  return (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(a)) |
         ((uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(b)) << 16);
}
__device__ __forceinline__ float q(float x, float s) {  // RNE_bf16(x * s), back to fp32
  return __bfloat162float(__float2bfloat16_rn(__fmul_rn(x, s)));
}

// Visit n elements of a slot: a scalar head up to the first index where both g
// (fp32) and w (bf16) are 16-B aligned (possible when their misalignments agree,
// e.g. 16-B aligned gradient and slot bases), 8-element vector steps, a scalar
// tail; scalar throughout otherwise.  fv(i) handles i..i+7, fs(i) element i.
template <typename FV, typename FS>
__device__ __forceinline__ void walk8(const float* g, const __nv_bfloat16* w, int64_t n, FV fv, FS fs) {
  int64_t h = 0;
  while (h < 8 && h < n && ((reinterpret_cast<uintptr_t>(g + h) & 15) || (reinterpret_cast<uintptr_t>(w + h) & 15))) ++h;
  const bool al = h < 8 && !((reinterpret_cast<uintptr_t>(g + h) & 15) || (reinterpret_cast<uintptr_t>(w + h) & 15));
  if (!al) h = n;
  h = min(h, n);
  for (int64_t i = threadIdx.x; i < h; i += blockDim.x) fs(i);
  const int64_t nv = (n - h) / 8;
  for (int64_t v = threadIdx.x; v < nv; v += blockDim.x) fv(h + v * 8);
  for (int64_t i = h + nv * 8 + threadIdx.x; i < n; i += blockDim.x) fs(i);
}

template <int MAXS>
__global__ void __launch_bounds__(kThreads) wire_gather_kernel(const __grid_constant__ WArgs<MAXS> a,
                                                               __nv_bfloat16* __restrict__ slot, float s) {
  const int64_t total = a.vo[a.n];
  for (int64_t t = (int64_t)blockIdx.x * kTile; t < total; t += (int64_t)gridDim.x * kTile) {
    const int64_t hi = min(t + (int64_t)kTile, total);
    for (int k = find_w(a, t); k < a.n && a.vo[k] < hi; ++k) {
      const int64_t x0 = max(t, a.vo[k]), x1 = min(hi, a.vo[k + 1]);
      if (x0 >= x1) continue;
      const float* g = a.grad[k] + (x0 - a.vo[k]);
      __nv_bfloat16* w = slot + a.wire[k] + (x0 - a.vo[k]);
      walk8(g, w, x1 - x0,
            [&](int64_t i) {
              const uint4 u0 = ld_nc_v4(g + i), u1 = ld_nc_v4(g + i + 4);
              st_v4(w + i, make_uint4(pack2(__fmul_rn(__uint_as_float(u0.x), s), __fmul_rn(__uint_as_float(u0.y), s)),
                                      pack2(__fmul_rn(__uint_as_float(u0.z), s), __fmul_rn(__uint_as_float(u0.w), s)),
                                      pack2(__fmul_rn(__uint_as_float(u1.x), s), __fmul_rn(__uint_as_float(u1.y), s)),
                                      pack2(__fmul_rn(__uint_as_float(u1.z), s), __fmul_rn(__uint_as_float(u1.w), s))));
            },
            [&](int64_t i) { w[i] = __float2bfloat16_rn(__fmul_rn(__ldg(g + i), s)); });
    }
  }
}

template <int W, int MAXS>
__global__ void __launch_bounds__(kThreads) wire_reduce_kernel(const __grid_constant__ WArgs<MAXS> a,
                                                               const char* __restrict__ slot0, int64_t stride,
                                                               int rank, float s) {
  const int64_t total = a.vo[a.n];
  for (int64_t t = (int64_t)blockIdx.x * kTile; t < total; t += (int64_t)gridDim.x * kTile) {
    const int64_t hi = min(t + (int64_t)kTile, total);
    for (int k = find_w(a, t); k < a.n && a.vo[k] < hi; ++k) {
      const int64_t x0 = max(t, a.vo[k]), x1 = min(hi, a.vo[k + 1]);
      if (x0 >= x1) continue;
      const int64_t i0 = x0 - a.vo[k];
      float* g = a.grad[k] + i0;
      const __nv_bfloat16* w[W];
#pragma unroll
      for (int qq = 0; qq < W; ++qq)
        w[qq] = reinterpret_cast<const __nv_bfloat16*>(slot0 + qq * stride) + a.wire[k] + i0;
      walk8(g, w[rank == 0 ? 1 : 0], x1 - x0,
            [&](int64_t i) {
              const uint4 u0 = ld_cg_v4(g + i), u1 = ld_cg_v4(g + i + 4);
              const float own[8] = {__uint_as_float(u0.x), __uint_as_float(u0.y), __uint_as_float(u0.z),
                                    __uint_as_float(u0.w), __uint_as_float(u1.x), __uint_as_float(u1.y),
                                    __uint_as_float(u1.z), __uint_as_float(u1.w)};
              float acc[8], f[8];
#pragma unroll
              for (int qq = 0; qq < W; ++qq) {
                if (qq == rank) {
#pragma unroll
                  for (int e = 0; e < 8; ++e) f[e] = q(own[e], s);
                } else {
                  Elem<__nv_bfloat16>::unpack(ld_cg_v4(w[qq] + i), f);
                }
#pragma unroll
                for (int e = 0; e < 8; ++e) acc[e] = qq == 0 ? f[e] : __fadd_rn(acc[e], f[e]);
              }
              st_v4(g + i, make_uint4(__float_as_uint(acc[0]), __float_as_uint(acc[1]), __float_as_uint(acc[2]),
                                      __float_as_uint(acc[3])));
              st_v4(g + i + 4, make_uint4(__float_as_uint(acc[4]), __float_as_uint(acc[5]),
                                          __float_as_uint(acc[6]), __float_as_uint(acc[7])));
            },
            [&](int64_t i) {
              float acc = 0.f;
#pragma unroll
              for (int qq = 0; qq < W; ++qq) {
                const float f = qq == rank ? q(g[i], s) : __bfloat162float(w[qq][i]);
                acc = qq == 0 ? f : __fadd_rn(acc, f);
              }
              g[i] = acc;
            });
    }
  }
}

template <int MAXS>
WArgs<MAXS> make_args(const CeView& v, int first, int n) {
  WArgs<MAXS> a;
  a.n = n;
  int64_t pos = 0;
  for (int k = 0; k < n; ++k) {
    a.grad[k] = static_cast<float*>(v.grad[first + k]);
    a.wire[k] = v.wire[first + k];
    a.vo[k] = pos;
    pos += v.numel[first + k];
  }
  a.vo[n] = pos;
  return a;
}

int grid_of(int64_t elems, int max_ctas) {
  int64_t g = (elems + kTile - 1) / kTile;
  return (int)(g < 1 ? 1 : g > max_ctas ? max_ctas : g);
}

template <int MAXS>
cudaError_t gather_n(const CeView& v, int first, int n, void* slot, float s, int max_ctas, cudaStream_t st) {
  const WArgs<MAXS> a = make_args<MAXS>(v, first, n);
  wire_gather_kernel<MAXS><<<grid_of(a.vo[n], max_ctas), kThreads, 0, st>>>(a, static_cast<__nv_bfloat16*>(slot), s);
  return cudaGetLastError();
}

template <int W, int MAXS>
cudaError_t reduce_n(const CeView& v, int first, int n, const void* slot0, int64_t stride, int rank, float s,
                     int max_ctas, cudaStream_t st) {
  const WArgs<MAXS> a = make_args<MAXS>(v, first, n);
  wire_reduce_kernel<W, MAXS><<<grid_of(a.vo[n], max_ctas), kThreads, 0, st>>>(
      a, static_cast<const char*>(slot0), stride, rank, s);
  return cudaGetLastError();
}

template <int W>
cudaError_t reduce_w(const CeView& v, const void* slot0, int64_t stride, int rank, float s, int max_ctas,
                     cudaStream_t st) {
  for (int first = 0; first < v.n; first += kMaxSlotsPerLaunch) {
    const int n = v.n - first < kMaxSlotsPerLaunch ? v.n - first : kMaxSlotsPerLaunch;
    cudaError_t e = n <= 32    ? reduce_n<W, 32>(v, first, n, slot0, stride, rank, s, max_ctas, st)
                    : n <= 256 ? reduce_n<W, 256>(v, first, n, slot0, stride, rank, s, max_ctas, st)
                               : reduce_n<W, 1024>(v, first, n, slot0, stride, rank, s, max_ctas, st);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace

cudaError_t launch_wire_gather(const CeView& v, void* own_slot, float scale, int max_ctas, cudaStream_t s) {
  for (int first = 0; first < v.n; first += kMaxSlotsPerLaunch) {
    const int n = v.n - first < kMaxSlotsPerLaunch ? v.n - first : kMaxSlotsPerLaunch;
    cudaError_t e = n <= 32    ? gather_n<32>(v, first, n, own_slot, scale, max_ctas, s)
                    : n <= 256 ? gather_n<256>(v, first, n, own_slot, scale, max_ctas, s)
                               : gather_n<1024>(v, first, n, own_slot, scale, max_ctas, s);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t launch_wire_reduce(int world, int rank, const CeView& v, const void* slot0, int64_t stride_bytes,
                               float scale, int max_ctas, cudaStream_t s) {
  switch (world) {
    case 2: return reduce_w<2>(v, slot0, stride_bytes, rank, scale, max_ctas, s);
    case 3: return reduce_w<3>(v, slot0, stride_bytes, rank, scale, max_ctas, s);
    case 4: return reduce_w<4>(v, slot0, stride_bytes, rank, scale, max_ctas, s);
    case 5: return reduce_w<5>(v, slot0, stride_bytes, rank, scale, max_ctas, s);
    case 6: return reduce_w<6>(v, slot0, stride_bytes, rank, scale, max_ctas, s);
    case 7: return reduce_w<7>(v, slot0, stride_bytes, rank, scale, max_ctas, s);
    case 8: return reduce_w<8>(v, slot0, stride_bytes, rank, scale, max_ctas, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace b200ddp
