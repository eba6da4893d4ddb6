// sync_probe.cu — latency of the cross-GPU synchronization primitives the P2P
// kernels use, on two GPUs of one process (each GPU runs its own kernel, so no
// two waiting kernels share a GPU):
//   (1) flag ping-pong round trip (st.release.sys remote / ld.acquire.sys local)
//   (2) cost of one thread's __threadfence_system() after the CTA pushed B bytes
//       of remote stores (bar.sync first), vs the same with every thread fencing
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o sync_probe sync_probe.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                        \
  do {                                                                               \
    cudaError_t e_ = (x);                                                            \
    if (e_ != cudaSuccess) {                                                         \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      exit(1);                                                                       \
    }                                                                                \
  } while (0)

__device__ __forceinline__ void st_rel(unsigned* p, unsigned v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acq(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// side 0 starts: for i in 1..n: write peer[0] = i (remote), wait mine[0] >= i.
__global__ void pingpong(unsigned* mine, unsigned* peer, int n, int side, unsigned long long* out) {
  if (threadIdx.x) return;
  unsigned long long t0 = gtimer();
  for (int i = 1; i <= n; ++i) {
    if (side == 0) {
      st_rel(peer, i);
      while (ld_acq(mine) < (unsigned)i) {}
    } else {
      while (ld_acq(mine) < (unsigned)i) {}
      st_rel(peer, i);
    }
  }
  if (side == 0) *out = gtimer() - t0;
}

// Each CTA pushes `bytes_per_cta` into the peer with 16-B stores, then fences.
// mode 0: bar.sync then thread 0 fences; mode 1: every thread fences then bar.sync.
__global__ void push_then_fence(uint4* peer, size_t bytes_per_cta, int mode, unsigned long long* out) {
  const size_t n = bytes_per_cta / 16;
  uint4* d = peer + blockIdx.x * n;
  uint4 v = make_uint4(threadIdx.x, 1, 2, 3);
  __syncthreads();
  unsigned long long t0 = gtimer();
  for (size_t i = threadIdx.x; i < n; i += blockDim.x) d[i] = v;
  unsigned long long t1 = gtimer();
  if (mode == 1) __threadfence_system();
  __syncthreads();
  if (mode == 0 && threadIdx.x == 0) __threadfence_system();
  __syncthreads();
  unsigned long long t2 = gtimer();
  if (threadIdx.x == 0) {
    out[blockIdx.x * 2] = t1 - t0;
    out[blockIdx.x * 2 + 1] = t2 - t1;
  }
}

int main() {
  int nd = 0;
  CK(cudaGetDeviceCount(&nd));
  if (nd < 2) {
    printf("need 2 GPUs\n");
    return 0;
  }
  unsigned *f0, *f1;
  unsigned long long *o0, *o1;
  CK(cudaSetDevice(0));
  CK(cudaDeviceEnablePeerAccess(1, 0));
  CK(cudaMalloc(&f0, 4096));
  CK(cudaMemset(f0, 0, 4096));
  CK(cudaMallocManaged(&o0, 1 << 20));
  CK(cudaSetDevice(1));
  CK(cudaDeviceEnablePeerAccess(0, 0));
  CK(cudaMalloc(&f1, 4096));
  CK(cudaMemset(f1, 0, 4096));
  CK(cudaMallocManaged(&o1, 1 << 20));
  const int n = 2000;
  CK(cudaSetDevice(1));
  pingpong<<<1, 32>>>(f1, f0, n, 1, o1);
  CK(cudaSetDevice(0));
  pingpong<<<1, 32>>>(f0, f1, n, 0, o0);
  CK(cudaDeviceSynchronize());
  CK(cudaSetDevice(1));
  CK(cudaDeviceSynchronize());
  printf("flag ping-pong round trip: %.2f us\n", o0[0] / 1000.0 / n);

  uint4* buf1;
  CK(cudaSetDevice(1));
  CK(cudaMalloc(&buf1, 512ull << 20));
  CK(cudaSetDevice(0));
  for (int mode = 0; mode < 2; ++mode) {
    for (size_t kb : {0, 32, 128, 512}) {
      for (int ctas : {1, 32, 128}) {
        push_then_fence<<<ctas, 512>>>(buf1, kb << 10, mode, o0);
        CK(cudaDeviceSynchronize());
        push_then_fence<<<ctas, 512>>>(buf1, kb << 10, mode, o0);
        CK(cudaDeviceSynchronize());
        double issue = 0, fence = 0;
        for (int c = 0; c < ctas; ++c) {
          issue += o0[2 * c];
          fence += o0[2 * c + 1];
        }
        printf("mode=%s push %4zu KB/CTA ctas=%3d: issue %.2f us, fence %.2f us (avg per CTA)\n",
               mode ? "all-threads-fence" : "one-thread-fence", kb, ctas, issue / ctas / 1000,
               fence / ctas / 1000);
      }
    }
  }
  return 0;
}
