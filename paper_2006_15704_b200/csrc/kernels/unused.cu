// unused.cu — write-back of locally-unused parameters after the bitmap
// allreduce (find_unused_parameters, §3.2.3, §4.2).
//
// A parameter with no local gradient in the pass contributed zeros through a
// library scratch slot; its averaged value sits in that slot after its bucket's
// allreduce.  Once the participation bitmap has been summed across ranks:
//     grad_p[i] = scratch_p[i]   if global_used[p] > 0
//     (untouched)                otherwise ("DDP should only touch
//                                 gradients that are indeed involved")
// One launch for all such parameters; HBM-bound, 2 x bytes of the copied ones.
// The participation bitmaps themselves travel as W slots per rank (copy-engine
// transfers ordered by stream memory operations, core/exchange.cpp) and are
// summed here in one small kernel (bitmap_sum_kernel).
#include "common.cuh"

namespace b200ddp {

namespace {

constexpr int64_t kTileBytes = (int64_t)kThreads * 16 * 4;

template <int MAXS>
struct FixArgs {
  const void* src[MAXS];
  void* dst[MAXS];
  int32_t param[MAXS];
  int64_t off[MAXS + 1];  // virtual element offsets of the concatenated slots
  int32_t n;
};

template <typename T, int MAXS>
__global__ void __launch_bounds__(kThreads) unused_fixup_kernel(const __grid_constant__ FixArgs<MAXS> fa,
                                                                const int32_t* __restrict__ global_used) {
  constexpr int64_t tile = kTileBytes / sizeof(T);
  const int64_t total = fa.off[fa.n];
  for (int64_t t = (int64_t)blockIdx.x * tile; t < total; t += (int64_t)gridDim.x * tile) {
    const int64_t hi = min(t + tile, total);
    int a = 0, b = fa.n - 1;  // first slot with off[k] <= t
    while (a < b) {
      const int m = (a + b + 1) >> 1;
      if (fa.off[m] <= t) a = m; else b = m - 1;
    }
    for (int k = a; k < fa.n && fa.off[k] < hi; ++k) {
      const int64_t x0 = max(t, fa.off[k]), x1 = min(hi, fa.off[k + 1]);
      if (x0 >= x1 || global_used[fa.param[k]] == 0) continue;
      T* d[1] = {static_cast<T*>(fa.dst[k]) + (x0 - fa.off[k])};
      const T* s[1] = {static_cast<const T*>(fa.src[k]) + (x0 - fa.off[k])};
      cta_xfer<T, 1, 1, true, false>(d, s, x1 - x0, 1.0f);
    }
  }
}

template <typename T, int MAXS>
cudaError_t run(const UnusedView& uv, int first, int n, const int32_t* global_used, int max_ctas,
                cudaStream_t st) {
  FixArgs<MAXS> a;
  a.n = n;
  int64_t pos = 0;
  for (int k = 0; k < n; ++k) {
    a.src[k] = uv.src[first + k];
    a.dst[k] = uv.dst[first + k];
    a.param[k] = uv.param[first + k];
    a.off[k] = pos;
    pos += uv.numel[first + k];
  }
  a.off[n] = pos;
  const int64_t tile = kTileBytes / sizeof(T);
  int64_t grid = (pos + tile - 1) / tile;
  if (grid > max_ctas) grid = max_ctas;
  if (grid < 1) grid = 1;
  unused_fixup_kernel<T, MAXS><<<(int)grid, kThreads, 0, st>>>(a, global_used);
  return cudaGetLastError();
}

template <typename T>
cudaError_t dispatch(const UnusedView& uv, const int32_t* global_used, int max_ctas, cudaStream_t st) {
  for (int first = 0; first < uv.n; first += kMaxSlotsPerLaunch) {
    const int n = uv.n - first < kMaxSlotsPerLaunch ? uv.n - first : kMaxSlotsPerLaunch;
    cudaError_t e = n <= 32    ? run<T, 32>(uv, first, n, global_used, max_ctas, st)
                    : n <= 256 ? run<T, 256>(uv, first, n, global_used, max_ctas, st)
                               : run<T, 1024>(uv, first, n, global_used, max_ctas, st);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

__global__ void __launch_bounds__(kThreads) bitmap_sum_kernel(const char* __restrict__ slot0, int64_t stride,
                                                             int world, int32_t* __restrict__ global, int32_t n) {
  for (int32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) {
    int32_t s = 0;
    for (int q = 0; q < world; ++q) s += __ldcg(reinterpret_cast<const int32_t*>(slot0 + q * stride) + p);
    global[p] = s;
  }
}

}  // namespace

cudaError_t launch_bitmap_sum(int world, const void* slot0, int64_t stride_bytes, int32_t* global, int32_t n,
                              cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  int grid = (n + kThreads - 1) / kThreads;
  if (grid > 148) grid = 148;
  bitmap_sum_kernel<<<grid, kThreads, 0, s>>>(static_cast<const char*>(slot0), stride_bytes, world, global, n);
  return cudaGetLastError();
}

cudaError_t launch_unused_fixup(int dtype, const UnusedView& uv, const int32_t* global_used, int max_ctas,
                                cudaStream_t s) {
  if (uv.n == 0) return cudaSuccess;
  return dtype == 0 ? dispatch<float>(uv, global_used, max_ctas, s)
                    : dispatch<__nv_bfloat16>(uv, global_used, max_ctas, s);
}

}  // namespace b200ddp
