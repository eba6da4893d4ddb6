// nvlink_probe.cu — measures what NVLink 5 / NVSwitch gives a kernel on this
// box: peer copy engine bandwidth and SM-driven remote stores (push) / remote
// loads (pull) vs CTA count and vectors in flight, one direction and both.
// Single process, two GPUs, peer access enabled: no kernel ever waits on
// another, so there is no cross-launch co-residency hazard.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o nvlink_probe nvlink_probe.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                       \
  do {                                                                              \
    cudaError_t e = (x);                                                            \
    if (e != cudaSuccess) {                                                         \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e)); \
      exit(1);                                                                      \
    }                                                                               \
  } while (0)

template <int U>
__global__ void __launch_bounds__(512) copy_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst,
                                                   size_t n) {
  const size_t stride = (size_t)gridDim.x * blockDim.x * U;
  for (size_t i = (size_t)blockIdx.x * blockDim.x * U + threadIdx.x; i < n; i += stride) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const size_t k = i + (size_t)u * blockDim.x;
      if (k < n) v[u] = src[k];
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const size_t k = i + (size_t)u * blockDim.x;
      if (k < n) dst[k] = v[u];
    }
  }
}

typedef void (*kfn)(const uint4*, uint4*, size_t);

static float time_kernel(int dev, kfn f, int ctas, const uint4* s, uint4* d, size_t n, int reps) {
  CK(cudaSetDevice(dev));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  f<<<ctas, 512>>>(s, d, n);
  CK(cudaEventRecord(a));
  for (int r = 0; r < reps; ++r) f<<<ctas, 512>>>(s, d, n);
  CK(cudaEventRecord(b));
  CK(cudaEventSynchronize(b));
  float ms;
  CK(cudaEventElapsedTime(&ms, a, b));
  return ms / reps;
}

int main(int argc, char** argv) {
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  if (ndev < 2) {
    printf("need 2 GPUs\n");
    return 0;
  }
  const size_t bytes = (argc > 1 ? atoll(argv[1]) : 256ll) << 20;
  const size_t n = bytes / 16;
  uint4 *a0, *b0, *a1, *b1;
  CK(cudaSetDevice(0));
  CK(cudaDeviceEnablePeerAccess(1, 0));
  CK(cudaMalloc(&a0, bytes));
  CK(cudaMalloc(&b0, bytes));
  CK(cudaMemset(a0, 1, bytes));
  CK(cudaSetDevice(1));
  CK(cudaDeviceEnablePeerAccess(0, 0));
  CK(cudaMalloc(&a1, bytes));
  CK(cudaMalloc(&b1, bytes));
  CK(cudaMemset(a1, 2, bytes));
  const int reps = 10;

  // copy engine
  {
    CK(cudaSetDevice(0));
    cudaStream_t s0;
    CK(cudaStreamCreate(&s0));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaMemcpyPeerAsync(b1, 1, a0, 0, bytes, s0));
    CK(cudaEventRecord(e0, s0));
    for (int r = 0; r < reps; ++r) CK(cudaMemcpyPeerAsync(b1, 1, a0, 0, bytes, s0));
    CK(cudaEventRecord(e1, s0));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    printf("copy-engine peer 0->1 %zu MiB: %.1f GB/s\n", bytes >> 20, bytes / (ms / reps * 1e-3) / 1e9);
  }
  // copy engines in both directions at once (what a 2-rank copy-engine exchange does),
  // one 256 MiB transfer and 25 MiB transfers (bucket-sized), timed on each device
  for (size_t chunk : {bytes, (size_t)25 << 20}) {
    cudaStream_t s[2];
    cudaEvent_t ev[2][2];
    for (int d = 0; d < 2; ++d) {
      CK(cudaSetDevice(d));
      CK(cudaStreamCreate(&s[d]));
      CK(cudaEventCreate(&ev[d][0]));
      CK(cudaEventCreate(&ev[d][1]));
    }
    const int nrep = (int)(bytes / chunk) * reps;
    for (int d = 0; d < 2; ++d) {
      CK(cudaSetDevice(d));
      CK(cudaEventRecord(ev[d][0], s[d]));
      for (int r = 0; r < nrep; ++r)
        CK(d == 0 ? cudaMemcpyPeerAsync(b1, 1, a0, 0, chunk, s[0]) : cudaMemcpyPeerAsync(b0, 0, a1, 1, chunk, s[1]));
      CK(cudaEventRecord(ev[d][1], s[d]));
    }
    for (int d = 0; d < 2; ++d) {
      CK(cudaSetDevice(d));
      CK(cudaEventSynchronize(ev[d][1]));
      float ms;
      CK(cudaEventElapsedTime(&ms, ev[d][0], ev[d][1]));
      printf("copy-engine bidirectional %zu MiB transfers: gpu%d -> peer %.1f GB/s per direction\n", chunk >> 20, d,
             (double)chunk * nrep / (ms * 1e-3) / 1e9);
    }
  }
  CK(cudaSetDevice(0));
  const int ctas_list[] = {8, 16, 32, 64, 96, 128, 148, 296};
  kfn fns[] = {copy_kernel<1>, copy_kernel<4>, copy_kernel<8>};
  const int us[] = {1, 4, 8};
  printf("%-6s %-4s %-5s %12s %12s %12s\n", "mode", "U", "ctas", "push GB/s", "pull GB/s", "local GB/s");
  for (int fi = 0; fi < 3; ++fi) {
    for (int ctas : ctas_list) {
      float push = time_kernel(0, fns[fi], ctas, a0, b1, n, reps);   // GPU0 SMs store into GPU1
      float pull = time_kernel(0, fns[fi], ctas, a1, b0, n, reps);   // GPU0 SMs load from GPU1
      float local = time_kernel(0, fns[fi], ctas, a0, b0, n, reps);
      printf("%-6s %-4d %-5d %12.1f %12.1f %12.1f\n", "uni", us[fi], ctas, bytes / (push * 1e-3) / 1e9,
             bytes / (pull * 1e-3) / 1e9, 2.0 * bytes / (local * 1e-3) / 1e9);
    }
  }
  // bidirectional push: both GPUs store into the other at once
  for (int ctas : {32, 64, 128, 148}) {
    cudaStream_t s[2];
    cudaEvent_t ev[2][2];
    for (int d = 0; d < 2; ++d) {
      CK(cudaSetDevice(d));
      CK(cudaStreamCreate(&s[d]));
      CK(cudaEventCreate(&ev[d][0]));
      CK(cudaEventCreate(&ev[d][1]));
    }
    for (int d = 0; d < 2; ++d) {
      CK(cudaSetDevice(d));
      CK(cudaEventRecord(ev[d][0], s[d]));
      for (int r = 0; r < reps; ++r)
        copy_kernel<8><<<ctas, 512, 0, s[d]>>>(d == 0 ? a0 : a1, d == 0 ? b1 : b0, n);
      CK(cudaEventRecord(ev[d][1], s[d]));
    }
    float ms[2];
    for (int d = 0; d < 2; ++d) {
      CK(cudaSetDevice(d));
      CK(cudaEventSynchronize(ev[d][1]));
      CK(cudaEventElapsedTime(&ms[d], ev[d][0], ev[d][1]));
    }
    printf("bidir push U=8 ctas=%d: gpu0 %.1f GB/s, gpu1 %.1f GB/s (per direction)\n", ctas,
           bytes / (ms[0] / reps * 1e-3) / 1e9, bytes / (ms[1] / reps * 1e-3) / 1e9);
  }
  return 0;
}
