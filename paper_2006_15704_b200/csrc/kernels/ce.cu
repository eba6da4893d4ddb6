// ce.cu — the SM part of the copy-engine (CE) bucket allreduce.
//
// In the CE algorithm the NVLink traffic is moved by the copy engines
// (cudaMemcpyAsync into the peers' slots) and ordered by stream memory
// operations, so no SM spins or pushes while backward runs (overlap,
// P:L184-L186).  What remains on the SMs is pack (pack.cu) and this
// reduction, which sums the W slots of a bucket in rank order in fp32 and
// writes the result straight into the gradients (fused unpack):
//     grad_p[i] = RNE( sum_{q=0..W-1} slot_q[off_p + i] )      (oracle O-3b)
#include "common.cuh"

namespace b200ddp {

namespace {

constexpr int64_t kTileBytes = (int64_t)kThreads * 16 * 4;

template <typename T, int W, int MAXS>
__global__ void __launch_bounds__(kThreads) reduce_slots_kernel(const __grid_constant__ SlotArgs<MAXS> sa,
                                                                const T* __restrict__ slot0, int64_t stride) {
  constexpr int64_t tile = kTileBytes / sizeof(T);
  const T* src[W];
#pragma unroll
  for (int q = 0; q < W; ++q) src[q] = slot0 + q * stride;
  const int64_t lo0 = sa.off[0], hi0 = sa.off[sa.n];
  for (int64_t t = lo0 + (int64_t)blockIdx.x * tile; t < hi0; t += (int64_t)gridDim.x * tile)
    walk_unpack<T, W, MAXS>(sa, t, min(t + tile, hi0), src, 0, 0);
}

template <typename T, int W, int MAXS>
cudaError_t run(const SlotView& sv, int first, int n, const void* slot0, int64_t stride, int max_ctas,
                cudaStream_t st) {
  SlotArgs<MAXS> a;
  a.n = n;
  for (int k = 0; k < n; ++k) {
    a.grad[k] = sv.grad[first + k];
    a.off[k] = sv.off[first + k];
  }
  a.off[n] = sv.off[first + n];
  const int64_t tile = kTileBytes / sizeof(T);
  int64_t grid = (a.off[n] - a.off[0] + tile - 1) / tile;
  if (grid > max_ctas) grid = max_ctas;
  if (grid < 1) grid = 1;
  reduce_slots_kernel<T, W, MAXS><<<(int)grid, kThreads, 0, st>>>(a, static_cast<const T*>(slot0), stride);
  return cudaGetLastError();
}

template <typename T, int W>
cudaError_t by_slots(const SlotView& sv, const void* slot0, int64_t stride, int max_ctas, cudaStream_t st) {
  for (int first = 0; first < sv.n; first += kMaxSlotsPerLaunch) {
    const int n = sv.n - first < kMaxSlotsPerLaunch ? sv.n - first : kMaxSlotsPerLaunch;
    cudaError_t e = n <= 32    ? run<T, W, 32>(sv, first, n, slot0, stride, max_ctas, st)
                    : n <= 256 ? run<T, W, 256>(sv, first, n, slot0, stride, max_ctas, st)
                               : run<T, W, 1024>(sv, first, n, slot0, stride, max_ctas, st);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

template <typename T>
cudaError_t by_world(int world, const SlotView& sv, const void* slot0, int64_t stride, int max_ctas,
                     cudaStream_t st) {
  switch (world) {
    case 2: return by_slots<T, 2>(sv, slot0, stride, max_ctas, st);
    case 3: return by_slots<T, 3>(sv, slot0, stride, max_ctas, st);
    case 4: return by_slots<T, 4>(sv, slot0, stride, max_ctas, st);
    case 5: return by_slots<T, 5>(sv, slot0, stride, max_ctas, st);
    case 6: return by_slots<T, 6>(sv, slot0, stride, max_ctas, st);
    case 7: return by_slots<T, 7>(sv, slot0, stride, max_ctas, st);
    case 8: return by_slots<T, 8>(sv, slot0, stride, max_ctas, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace

cudaError_t launch_ce_reduce(int dtype, int world, const SlotView& sv, const void* slot0, int64_t stride_elems,
                             int max_ctas, cudaStream_t s) {
  return dtype == 0 ? by_world<float>(world, sv, slot0, stride_elems, max_ctas, s)
                    : by_world<__nv_bfloat16>(world, sv, slot0, stride_elems, max_ctas, s);
}

}  // namespace b200ddp
