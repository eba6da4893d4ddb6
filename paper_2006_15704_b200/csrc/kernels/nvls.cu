// nvls.cu — bucket allreduce through NVSwitch multicast (NVLS), fused with pack
// (x 1/W) and unpack.  One launch per bucket; CTA c of every rank owns chunk c
// of every shard (shard length L, 256-element aligned):
//
//   A  pack + scale chunk c of every shard into this rank's bucket
//      (Alg. 1, reading C-2);                       barrier (kind 0)
//   B  rank r: for its own shard, chunk c:
//        v = multimem.ld_reduce.add [mc + x]   (the switch sums the W ranks'
//                                               buckets)
//        multimem.st [mc + x], v               (the switch writes the sum into
//                                               every rank's bucket)
//                                                              barrier (kind 1)
//   C  unpack chunk c of every shard from the local bucket into .grad.
//
// NVLink bytes per GPU and direction: S (ld_reduce operands) + S/W (result) —
// (1 + 1/W) S, against 2(W-1)/W S for a ring / two-shot.  The in-switch sum
// order is the switch's: results are bit-identical on every rank (one
// multicast store) and within the north_star tolerance of oracle O-3 (like
// NCCL), not bit-identical to O-3b.  fp32 buckets sum in fp32; bf16 buckets
// use the .acc::f32 form (fp32 accumulation, one rounding, reading C-4).
#include "barrier.cuh"

namespace b200ddp {

namespace {

template <typename T> struct Mm;
template <> struct Mm<float> {
  __device__ static __forceinline__ uint4 ld_reduce(const void* p) {
    uint4 r;
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p) : "memory");
    return r;
  }
  __device__ static __forceinline__ void st(void* p, const uint4& v) {
    asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y),
                 "r"(v.z), "r"(v.w) : "memory");
  }
};
template <> struct Mm<__nv_bfloat16> {
  __device__ static __forceinline__ uint4 ld_reduce(const void* p) {
    uint4 r;
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v4.bf16x2 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p) : "memory");
    return r;
  }
  __device__ static __forceinline__ void st(void* p, const uint4& v) {
    asm volatile("multimem.st.relaxed.sys.global.v4.bf16x2 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y),
                 "r"(v.z), "r"(v.w) : "memory");
  }
};

template <typename T, int W, int MAXS>
__global__ void __launch_bounds__(kThreads, 1)
    nvls_kernel(const __grid_constant__ SlotArgs<MAXS> sa, const __grid_constant__ P2PLaunch a) {
  constexpr int VE = 16 / sizeof(T);
  const int r = a.rank;
  const int c = blockIdx.x;
  const int64_t L = a.shard, N = a.numel, Q = a.chunk;
  auto rng = [&](int j, int64_t& lo, int64_t& hi) {
    const int64_t c0 = (int64_t)c * Q, c1 = min(c0 + Q, L);
    lo = min(j * L + c0, N);
    hi = min(j * L + c1, N);
  };
  T* own = at<T>(a.storage[r], a.bucket_byte_off);
  // A: pack + scale chunk c of every shard into the local bucket
  {
    T* d[1] = {own};
#pragma unroll 1
    for (int j = 0; j < W; ++j) {
      int64_t lo, hi;
      rng(j, lo, hi);
      if (lo < hi) walk_pack<T, 1, MAXS>(sa, lo, hi, d, 0, a.scale, 0);
    }
  }
  p2p_signal<W>(a, r, 0, a.seq + 1u);
  p2p_wait<W>(a, r, 0, a.seq + 1u);
  // B: in-switch reduction of chunk c of the own shard, multicast back to every rank.
  // 16-B vectors; the bucket region is padded to 256 B, so rounding the end of
  // the bucket up to a whole vector stays inside it (padding is never unpacked).
  {
    int64_t lo, hi;
    rng(r, lo, hi);
    if (lo < hi) {
      hi = (hi + VE - 1) / VE * VE;
      char* mcb = static_cast<char*>(a.mc) + a.bucket_byte_off;
      const int64_t v0 = lo / VE, nv = hi / VE - v0;
      constexpr int U = 8;  // ld_reduce is a round trip through the switch: keep many in flight
      int64_t v = threadIdx.x;
      for (; v + (U - 1) * (int64_t)blockDim.x < nv; v += U * (int64_t)blockDim.x) {
        uint4 x[U];
#pragma unroll
        for (int u = 0; u < U; ++u) x[u] = Mm<T>::ld_reduce(mcb + (v0 + v + u * (int64_t)blockDim.x) * 16);
#pragma unroll
        for (int u = 0; u < U; ++u) Mm<T>::st(mcb + (v0 + v + u * (int64_t)blockDim.x) * 16, x[u]);
      }
      for (; v < nv; v += blockDim.x) Mm<T>::st(mcb + (v0 + v) * 16, Mm<T>::ld_reduce(mcb + (v0 + v) * 16));
    }
  }
  p2p_signal<W>(a, r, 1, a.seq + 1u);
  p2p_wait<W>(a, r, 1, a.seq + 1u);
  // C: unpack chunk c of every shard from the local bucket
  {
    const T* b[1] = {own};
#pragma unroll 1
    for (int j = 0; j < W; ++j) {
      int64_t lo, hi;
      rng(j, lo, hi);
      if (lo < hi) walk_unpack<T, 1, MAXS>(sa, lo, hi, b, 0, 0);
    }
  }
}

template <int MAXS>
SlotArgs<MAXS> make_args(const SlotView& sv) {
  SlotArgs<MAXS> s;
  s.n = sv.n;
  for (int k = 0; k < sv.n; ++k) {
    s.grad[k] = sv.grad[k];
    s.off[k] = sv.off[k];
  }
  s.off[sv.n] = sv.off[sv.n];
  return s;
}

template <typename T, int MAXS>
cudaError_t run(const SlotView& sv, const P2PLaunch& a, cudaStream_t st) {
  const SlotArgs<MAXS> sargs = make_args<MAXS>(sv);
  P2PLaunch pa = a;
  void* args[] = {const_cast<SlotArgs<MAXS>*>(&sargs), &pa};
  void* fn = nullptr;
  switch (a.world) {
    case 2: fn = reinterpret_cast<void*>(nvls_kernel<T, 2, MAXS>); break;
    case 3: fn = reinterpret_cast<void*>(nvls_kernel<T, 3, MAXS>); break;
    case 4: fn = reinterpret_cast<void*>(nvls_kernel<T, 4, MAXS>); break;
    case 5: fn = reinterpret_cast<void*>(nvls_kernel<T, 5, MAXS>); break;
    case 6: fn = reinterpret_cast<void*>(nvls_kernel<T, 6, MAXS>); break;
    case 7: fn = reinterpret_cast<void*>(nvls_kernel<T, 7, MAXS>); break;
    case 8: fn = reinterpret_cast<void*>(nvls_kernel<T, 8, MAXS>); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaLaunchKernel(fn, dim3(a.ctas), dim3(kThreads), args, 0, st);
}

template <typename T>
cudaError_t dispatch(const SlotView& sv, const P2PLaunch& a, cudaStream_t st) {
  if (!a.mc || a.emulated) return cudaErrorInvalidValue;
  if (sv.n <= 32) return run<T, 32>(sv, a, st);
  if (sv.n <= 256) return run<T, 256>(sv, a, st);
  if (sv.n <= kMaxSlotsPerLaunch) return run<T, 1024>(sv, a, st);
  return cudaErrorInvalidValue;
}

}  // namespace

cudaError_t launch_nvls(int dtype, const SlotView& sv, const P2PLaunch& a, cudaStream_t s) {
  return dtype == 0 ? dispatch<float>(sv, a, s) : dispatch<__nv_bfloat16>(sv, a, s);
}

}  // namespace b200ddp
