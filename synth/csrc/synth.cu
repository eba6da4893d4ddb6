// synth.cu — device implementation of the seeded synthetic gradient recipe of
// synth/gen.py.  Input generation only: no
// arithmetic of the method.  Checked bit-for-bit against the host generator
// by tests/test_gpu_synth.py.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace {

constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;

__device__ __forceinline__ uint64_t fmix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// dist 0 = grid, 1 = normal; dtype 0 = fp32, 1 = bf16
__global__ void fill_kernel(void* out, int64_t n, int dtype, int dist, uint64_t key, float sigma,
                            int exp_p, int64_t K) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t h = fmix64(key + (uint64_t)(i + 1) * kGolden);
    float v;
    if (dist == 0) {
      const int64_t k = (int64_t)(h % (uint64_t)(2 * K + 1)) - K;
      v = ldexpf((float)k, -exp_p);  // exact: |k| <= 2^16
    } else {
      const float s = 1.0f / 65536.0f;
      const float u0 = __fmul_rn((float)(h & 0xFFFF), s);
      const float u1 = __fmul_rn((float)((h >> 16) & 0xFFFF), s);
      const float u2 = __fmul_rn((float)((h >> 32) & 0xFFFF), s);
      const float u3 = __fmul_rn((float)((h >> 48) & 0xFFFF), s);
      const float z = __fsub_rn(__fadd_rn(__fadd_rn(u0, u1), __fadd_rn(u2, u3)), 2.0f);
      v = __fmul_rn(z, sigma);
    }
    if (dtype == 0) static_cast<float*>(out)[i] = v;
    else static_cast<__nv_bfloat16*>(out)[i] = __float2bfloat16_rn(v);
  }
}

}  // namespace

extern "C" int synth_fill(void* out, int64_t n, int dtype, int dist, uint64_t key, float sigma, int exp_p,
                          int64_t K, void* stream) {
  if (n <= 0) return 0;
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  fill_kernel<<<(int)blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(out, n, dtype, dist, key, sigma,
                                                                          exp_p, K);
  return (int)cudaGetLastError();
}
