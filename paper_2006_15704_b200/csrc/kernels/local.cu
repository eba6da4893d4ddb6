// local.cu — world-1 fused bucket sync for a group of buckets in one launch.
//
// With one replica the allreduce of the packed value s = RNE(g * fl(1/1)) is s
// itself (reading C-12), so for every element the kernel does, in registers:
//   pack   bucket[off_p + i] = s          (Alg. 1)
//   reduce sum over the single rank = s
//   unpack grad_p[i] = s
// i.e. one read of the gradient and two writes (bucket, gradient): 3 x bytes.
// All buckets that become ready in the same call are one launch (their slots
// concatenated into a virtual range split evenly over the CTAs), which removes
// the per-bucket launch ramp of separate kernels.  HBM-bound.
#include "common.cuh"

namespace b200ddp {

namespace {

template <int MAXS>
struct GroupArgs {
  void* grad[MAXS];
  int64_t dst[MAXS];
  int64_t off[MAXS + 1];
  int32_t n;
};

template <typename T, int MAXS, int U>
__global__ void __launch_bounds__(kThreads, 2)
    local_kernel(const __grid_constant__ GroupArgs<MAXS> ga, char* __restrict__ storage, int64_t chunk) {
  const int64_t total = ga.off[ga.n];
  const int64_t lo = min((int64_t)blockIdx.x * chunk, total), hi = min(lo + chunk, total);
  if (lo >= hi) return;
  int a = 0, b = ga.n - 1;  // first slot with off[k] <= lo (CTA-uniform binary search)
  while (a < b) {
    const int m = (a + b + 1) >> 1;
    if (ga.off[m] <= lo) a = m; else b = m - 1;
  }
  for (int k = a; k < ga.n; ++k) {
    const int64_t s0 = ga.off[k];
    if (s0 >= hi) break;
    const int64_t x0 = max(lo, s0), x1 = min(hi, ga.off[k + 1]);
    if (x0 >= x1) continue;
    T* g = static_cast<T*>(ga.grad[k]) + (x0 - s0);
    T* d[2] = {reinterpret_cast<T*>(storage + ga.dst[k]) + (x0 - s0), g};
    const T* sp[1] = {g};
    cta_xfer<T, 1, 2, true, true, false, U>(d, sp, x1 - x0, 1.0f);
  }
}

template <typename T, int MAXS>
cudaError_t run(const GroupView& gv, void* storage, int max_ctas, cudaStream_t st) {
  GroupArgs<MAXS> a;
  a.n = gv.n;
  for (int k = 0; k < gv.n; ++k) {
    a.grad[k] = gv.grad[k];
    a.dst[k] = gv.dst[k];
    a.off[k] = gv.off[k];
  }
  a.off[gv.n] = gv.off[gv.n];
  const int64_t total = gv.off[gv.n];
  int64_t ctas = (total + 4095) / 4096;
  if (ctas > max_ctas) ctas = max_ctas;
  if (ctas < 1) ctas = 1;
  int64_t chunk = (total + ctas - 1) / ctas;
  chunk = (chunk + kAlignElems - 1) / kAlignElems * kAlignElems;
  ctas = (total + chunk - 1) / chunk;
  local_kernel<T, MAXS, 4><<<(int)ctas, kThreads, 0, st>>>(a, static_cast<char*>(storage), chunk);
  return cudaGetLastError();
}

template <typename T>
cudaError_t dispatch(const GroupView& gv, void* storage, int max_ctas, cudaStream_t st) {
  if (gv.n <= 32) return run<T, 32>(gv, storage, max_ctas, st);
  if (gv.n <= 256) return run<T, 256>(gv, storage, max_ctas, st);
  if (gv.n <= kMaxSlotsPerLaunch) return run<T, 1024>(gv, storage, max_ctas, st);
  return cudaErrorInvalidValue;
}

}  // namespace

cudaError_t launch_local(int dtype, const GroupView& gv, void* storage, int max_ctas, cudaStream_t s) {
  return dtype == 0 ? dispatch<float>(gv, storage, max_ctas, s) : dispatch<__nv_bfloat16>(gv, storage, max_ctas, s);
}

}  // namespace b200ddp
