// ce_probe.cu — copy-engine (CE) peer copies and stream memory operations on
// B200 / NVLink 5, as a substrate for an SM-free bucket exchange:
//   (1) cudaMemcpyAsync peer pushes from GPU0 to 1..P peers concurrently
//       (one stream per peer), bandwidth per GPU;
//   (2) cuStreamWriteValue32 into a peer's flag + cuStreamWaitValue32 on the
//       peer: ping-pong round trip through the GPU front ends (no SM).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ce_probe ce_probe.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                        \
  do {                                                                               \
    cudaError_t e_ = (x);                                                            \
    if (e_ != cudaSuccess) {                                                         \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      exit(1);                                                                       \
    }                                                                                \
  } while (0)

typedef CUresult (*WriteFn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
typedef CUresult (*WaitFn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);

int main(int argc, char** argv) {
  int nd = 0;
  CK(cudaGetDeviceCount(&nd));
  if (nd < 2) {
    printf("need >= 2 GPUs\n");
    return 0;
  }
  WriteFn wr = nullptr;
  WaitFn wt = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuStreamWriteValue32", (void**)&wr, cudaEnableDefault, &q));
  CK(cudaGetDriverEntryPoint("cuStreamWaitValue32", (void**)&wt, cudaEnableDefault, &q));
  for (int i = 0; i < nd; ++i) {
    CK(cudaSetDevice(i));
    for (int j = 0; j < nd; ++j)
      if (i != j) CK(cudaDeviceEnablePeerAccess(j, 0));
    int memops = 0;
    cudaDeviceGetAttribute(&memops, (cudaDeviceAttr)CU_DEVICE_ATTRIBUTE_CAN_USE_STREAM_MEM_OPS_V1, i);
  }
  const size_t bytes = (argc > 1 ? atoll(argv[1]) : 25ll) << 20;
  std::vector<char*> src(nd), dst(nd);
  std::vector<unsigned*> flag(nd);
  for (int i = 0; i < nd; ++i) {
    CK(cudaSetDevice(i));
    CK(cudaMalloc(&src[i], bytes));
    CK(cudaMalloc(&dst[i], bytes * nd));
    CK(cudaMalloc(&flag[i], 4096));
    CK(cudaMemset(flag[i], 0, 4096));
    CK(cudaMemset(src[i], i, bytes));
  }
  // (1) GPU0 pushes to P peers concurrently
  CK(cudaSetDevice(0));
  std::vector<cudaStream_t> st(nd);
  for (int i = 0; i < nd; ++i) CK(cudaStreamCreateWithFlags(&st[i], cudaStreamNonBlocking));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  for (int P = 1; P < nd; ++P) {
    const int reps = 10;
    CK(cudaEventRecord(e0, st[0]));
    for (int p = 1; p <= P; ++p) CK(cudaStreamWaitEvent(st[p], e0, 0));
    for (int r = 0; r < reps; ++r)
      for (int p = 1; p <= P; ++p) CK(cudaMemcpyAsync(dst[p], src[0], bytes, cudaMemcpyDeviceToDevice, st[p]));
    for (int p = 1; p <= P; ++p) {
      cudaEvent_t ep;
      CK(cudaEventCreate(&ep));
      CK(cudaEventRecord(ep, st[p]));
      CK(cudaStreamWaitEvent(st[0], ep, 0));
    }
    CK(cudaEventRecord(e1, st[0]));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    printf("CE push %zu MiB from GPU0 to %d peer(s) concurrently: %.1f GB/s out of GPU0 (%.1f us per round)\n",
           bytes >> 20, P, (double)bytes * P * reps / (ms * 1e-3) / 1e9, ms * 1e3 / reps);
  }
  // all GPUs push to all peers at once (all-to-all, like a one-shot exchange)
  {
    const int reps = 10;
    std::vector<std::vector<cudaStream_t>> ss(nd, std::vector<cudaStream_t>(nd));
    std::vector<cudaEvent_t> a(nd), b(nd);
    for (int i = 0; i < nd; ++i) {
      CK(cudaSetDevice(i));
      for (int j = 0; j < nd; ++j) CK(cudaStreamCreateWithFlags(&ss[i][j], cudaStreamNonBlocking));
      CK(cudaEventCreate(&a[i]));
      CK(cudaEventCreate(&b[i]));
    }
    for (int i = 0; i < nd; ++i) {
      CK(cudaSetDevice(i));
      CK(cudaEventRecord(a[i], ss[i][0]));
      for (int j = 0; j < nd; ++j) {
        if (j == i) continue;
        CK(cudaStreamWaitEvent(ss[i][j], a[i], 0));
        for (int r = 0; r < reps; ++r)
          CK(cudaMemcpyAsync(dst[j] + (size_t)i * bytes, src[i], bytes, cudaMemcpyDeviceToDevice, ss[i][j]));
        cudaEvent_t ep;
        CK(cudaEventCreate(&ep));
        CK(cudaEventRecord(ep, ss[i][j]));
        CK(cudaStreamWaitEvent(ss[i][0], ep, 0));
      }
      CK(cudaEventRecord(b[i], ss[i][0]));
    }
    for (int i = 0; i < nd; ++i) {
      CK(cudaSetDevice(i));
      CK(cudaEventSynchronize(b[i]));
      float ms;
      CK(cudaEventElapsedTime(&ms, a[i], b[i]));
      printf("all-to-all CE push, GPU%d: %.1f GB/s out (%d peers, %zu MiB each)\n", i,
             (double)bytes * (nd - 1) * reps / (ms * 1e-3) / 1e9, nd - 1, bytes >> 20);
    }
  }
  // (2) stream-memop ping-pong GPU0 <-> GPU1
  {
    const int n = 1000;
    cudaStream_t s0, s1;
    CK(cudaSetDevice(0));
    CK(cudaStreamCreateWithFlags(&s0, cudaStreamNonBlocking));
    CK(cudaSetDevice(1));
    CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
    CK(cudaSetDevice(0));
    CK(cudaEventRecord(e0, s0));
    for (int i = 1; i <= n; ++i) {
      CK(cudaSetDevice(0));
      if (wr((CUstream)s0, (CUdeviceptr)flag[1], i, 0) != CUDA_SUCCESS) { printf("write failed\n"); return 1; }
      if (wt((CUstream)s0, (CUdeviceptr)flag[0], i, CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS) { printf("wait failed\n"); return 1; }
      CK(cudaSetDevice(1));
      if (wt((CUstream)s1, (CUdeviceptr)flag[1], i, CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS) { printf("wait failed\n"); return 1; }
      if (wr((CUstream)s1, (CUdeviceptr)flag[0], i, 0) != CUDA_SUCCESS) { printf("write failed\n"); return 1; }
    }
    CK(cudaSetDevice(0));
    CK(cudaEventRecord(e1, s0));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    printf("stream-memop flag ping-pong round trip: %.2f us\n", ms * 1e3 / n);
    // one-way: copy then write flag; peer waits then measures
  }
  printf("ok\n");
  return 0;
}
