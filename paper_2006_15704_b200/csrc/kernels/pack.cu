// pack.cu — multi-tensor pack (+ scale by 1/world) and unpack kernels for the
// NCCL bucket path.
//
//   pack:   bucket[off_p + i] = RNE(grad_p[i] * fl(1/W))   Alg. 1,
//           P:L304 "tensors are copied from all parameter gradients to
//           buckets", average P:L166 with the scale placed here (reading C-2)
//   unpack: grad_p[i] = bucket[off_p + i]
//           "averaged gradients are copied back after AllReduce"
//
// One launch per bucket (not per gradient, as the paper's per-hook
// view.copy_): the slot table travels by value (__grid_constant__), each CTA
// takes 32 KiB tiles of the bucket grid-stride and walks the slots overlapping
// its tile with 128-bit loads/stores.  HBM-bound: 2 * bucket bytes per launch.
#include "common.cuh"

namespace b200ddp {

namespace {

constexpr int64_t kTileBytes = (int64_t)kThreads * 16 * 4;  // 4 vectors per thread

template <typename T, int MAXS>
__global__ void __launch_bounds__(kThreads, 2) pack_kernel(const __grid_constant__ SlotArgs<MAXS> sa,
                                                        T* __restrict__ bucket, float s) {
  constexpr int64_t tile = kTileBytes / sizeof(T);
  const int64_t lo0 = sa.off[0], hi0 = sa.off[sa.n];
  T* d[1] = {bucket};
  for (int64_t t = lo0 + (int64_t)blockIdx.x * tile; t < hi0; t += (int64_t)gridDim.x * tile)
    walk_pack<T, 1, MAXS>(sa, t, min(t + tile, hi0), d, 0, s, 0);
}

template <typename T, int MAXS>
__global__ void __launch_bounds__(kThreads) unpack_kernel(const __grid_constant__ SlotArgs<MAXS> sa,
                                                          const T* __restrict__ bucket) {
  constexpr int64_t tile = kTileBytes / sizeof(T);
  const int64_t lo0 = sa.off[0], hi0 = sa.off[sa.n];
  const T* src[1] = {bucket};
  for (int64_t t = lo0 + (int64_t)blockIdx.x * tile; t < hi0; t += (int64_t)gridDim.x * tile)
    walk_unpack<T, 1, MAXS>(sa, t, min(t + tile, hi0), src, 0, 0);
}

template <int MAXS>
SlotArgs<MAXS> make_args(const SlotView& sv, int first, int n) {
  SlotArgs<MAXS> a;
  a.n = n;
  for (int k = 0; k < n; ++k) {
    a.grad[k] = sv.grad[first + k];
    a.off[k] = sv.off[first + k];
  }
  a.off[n] = sv.off[first + n];
  return a;
}

int grid_for(int64_t elems, int64_t tile, int max_ctas) {
  int64_t g = (elems + tile - 1) / tile;
  if (g > max_ctas) g = max_ctas;
  return g < 1 ? 1 : (int)g;
}

template <typename T, int MAXS>
cudaError_t run(bool is_pack, const SlotView& sv, int first, int n, void* bucket, float s,
                int max_ctas, cudaStream_t st) {
  const SlotArgs<MAXS> a = make_args<MAXS>(sv, first, n);
  const int grid = grid_for(a.off[n] - a.off[0], kTileBytes / sizeof(T), max_ctas);
  if (is_pack)
    pack_kernel<T, MAXS><<<grid, kThreads, 0, st>>>(a, static_cast<T*>(bucket), s);
  else
    unpack_kernel<T, MAXS><<<grid, kThreads, 0, st>>>(a, static_cast<const T*>(bucket));
  return cudaGetLastError();
}

template <typename T>
cudaError_t dispatch(bool is_pack, const SlotView& sv, void* bucket, float s, int max_ctas,
                     cudaStream_t st) {
  // Split tables larger than the biggest by-value class into several launches.
  for (int first = 0; first < sv.n; first += kMaxSlotsPerLaunch) {
    const int n = sv.n - first < kMaxSlotsPerLaunch ? sv.n - first : kMaxSlotsPerLaunch;
    cudaError_t e;
    if (n <= 16) e = run<T, 16>(is_pack, sv, first, n, bucket, s, max_ctas, st);
    else if (n <= 64) e = run<T, 64>(is_pack, sv, first, n, bucket, s, max_ctas, st);
    else if (n <= 256) e = run<T, 256>(is_pack, sv, first, n, bucket, s, max_ctas, st);
    else e = run<T, 1024>(is_pack, sv, first, n, bucket, s, max_ctas, st);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace

cudaError_t launch_pack(int dtype, const SlotView& sv, void* bucket, float scale, int max_ctas,
                        cudaStream_t s) {
  return dtype == 0 ? dispatch<float>(true, sv, bucket, scale, max_ctas, s)
                    : dispatch<__nv_bfloat16>(true, sv, bucket, scale, max_ctas, s);
}

cudaError_t launch_unpack(int dtype, const SlotView& sv, const void* bucket, int max_ctas,
                          cudaStream_t s) {
  return dtype == 0
             ? dispatch<float>(false, sv, const_cast<void*>(bucket), 1.0f, max_ctas, s)
             : dispatch<__nv_bfloat16>(false, sv, const_cast<void*>(bucket), 1.0f, max_ctas, s);
}

}  // namespace b200ddp
