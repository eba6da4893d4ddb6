// ce.cu — the SM part of the copy-engine (CE) bucket allreduce.
//
// In the CE algorithm the NVLink traffic is moved by the copy engines
// (cudaMemcpyAsync into the peers' slots, straight from .grad for large
// gradients) and ordered by stream memory operations, so no SM spins or
// pushes while backward runs (overlap).  The bucket is carried on
// the wire in "wire layout": large gradients first, then the small ones,
// each at a 64-element aligned wire offset.  What remains on the SMs:
//
//   ce_gather_kernel:  small gradients -> this rank's own slot (raw copy, so
//                      one copy-engine transfer carries all of them);
//   ce_reduce_kernel:  grad_p[i] = RNE( sum_{q=0..W-1} RNE(v_q[i] * fl(1/W)) )
//                      in rank order, v_r = grad_p (own, raw), v_q = slot q at
//                      the wire offset (raw, pushed by rank q) — the pack
//                      scale of Alg. 1 L231-L232 applied on the fly per
//                      operand, i.e. exactly oracle O-3b, written straight
//                      into the gradients (fused unpack).
#include "common.cuh"

namespace b200ddp {

namespace {

constexpr int64_t kTileBytes = (int64_t)kThreads * 16 * 4;

template <int MAXS>
struct CeArgs {
  void* grad[MAXS];
  int64_t wire[MAXS];     // element offset inside a slot
  int64_t vo[MAXS + 1];   // virtual offsets: concatenation of the listed gradients
  int32_t n;
};

template <int MAXS>
__device__ __forceinline__ int find_v(const CeArgs<MAXS>& a, int64_t x) {
  int lo = 0, hi = a.n - 1;
  while (lo < hi) {
    const int m = (lo + hi + 1) >> 1;
    if (a.vo[m] <= x) lo = m; else hi = m - 1;
  }
  return lo;
}

template <typename T, int MAXS>
__global__ void __launch_bounds__(kThreads) ce_gather_kernel(const __grid_constant__ CeArgs<MAXS> a,
                                                             T* __restrict__ own_slot) {
  constexpr int64_t tile = kTileBytes / sizeof(T);
  const int64_t total = a.vo[a.n];
  for (int64_t t = (int64_t)blockIdx.x * tile; t < total; t += (int64_t)gridDim.x * tile) {
    const int64_t hi = min(t + tile, total);
    for (int k = find_v(a, t); k < a.n && a.vo[k] < hi; ++k) {
      const int64_t x0 = max(t, a.vo[k]), x1 = min(hi, a.vo[k + 1]);
      if (x0 >= x1) continue;
      const int64_t i0 = x0 - a.vo[k];
      T* d[1] = {own_slot + a.wire[k] + i0};
      const T* s[1] = {static_cast<const T*>(a.grad[k]) + i0};
      cta_xfer<T, 1, 1, true, false>(d, s, x1 - x0, 1.0f);
    }
  }
}

template <typename T, int W, int MAXS>
__global__ void __launch_bounds__(kThreads) ce_reduce_kernel(const __grid_constant__ CeArgs<MAXS> a,
                                                             const char* __restrict__ slot0, int64_t stride,
                                                             int rank, float s) {
  constexpr int64_t tile = kTileBytes / sizeof(T);
  const int64_t total = a.vo[a.n];
  for (int64_t t = (int64_t)blockIdx.x * tile; t < total; t += (int64_t)gridDim.x * tile) {
    const int64_t hi = min(t + tile, total);
    for (int k = find_v(a, t); k < a.n && a.vo[k] < hi; ++k) {
      const int64_t x0 = max(t, a.vo[k]), x1 = min(hi, a.vo[k + 1]);
      if (x0 >= x1) continue;
      const int64_t i0 = x0 - a.vo[k];
      T* g = static_cast<T*>(a.grad[k]) + i0;
      T* d[1] = {g};
      const T* src[W];
#pragma unroll
      for (int q = 0; q < W; ++q)
        src[q] = q == rank ? g : reinterpret_cast<const T*>(slot0 + q * stride) + a.wire[k] + i0;
      cta_xfer<T, W, 1, false, true, true>(d, src, x1 - x0, s);
    }
  }
}

// SM push (DDP_ALGO_PUSH): one read of every gradient, NP remote stores (the
// same wire offset in slot `rank` of each peer).  No waiting inside the kernel:
// the ready flags are stream memory operations after it completes.
struct PeerDst {
  char* p[kMaxWorld];
};

template <typename T, int NP, int MAXS>
__global__ void __launch_bounds__(kThreads) ce_push_kernel(const __grid_constant__ CeArgs<MAXS> a,
                                                           const __grid_constant__ PeerDst pd) {
  constexpr int64_t tile = kTileBytes / sizeof(T);
  const int64_t total = a.vo[a.n];
  for (int64_t t = (int64_t)blockIdx.x * tile; t < total; t += (int64_t)gridDim.x * tile) {
    const int64_t hi = min(t + tile, total);
    for (int k = find_v(a, t); k < a.n && a.vo[k] < hi; ++k) {
      const int64_t x0 = max(t, a.vo[k]), x1 = min(hi, a.vo[k + 1]);
      if (x0 >= x1) continue;
      const int64_t i0 = x0 - a.vo[k];
      T* d[NP];
#pragma unroll
      for (int j = 0; j < NP; ++j) d[j] = reinterpret_cast<T*>(pd.p[j]) + a.wire[k] + i0;
      const T* s[1] = {static_cast<const T*>(a.grad[k]) + i0};
      cta_xfer<T, 1, NP, true, false>(d, s, x1 - x0, 1.0f);
    }
  }
}

template <int MAXS>
CeArgs<MAXS> make_args(const CeView& v, int first, int n) {
  CeArgs<MAXS> a;
  a.n = n;
  int64_t pos = 0;
  for (int k = 0; k < n; ++k) {
    a.grad[k] = v.grad[first + k];
    a.wire[k] = v.wire[first + k];
    a.vo[k] = pos;
    pos += v.numel[first + k];
  }
  a.vo[n] = pos;
  return a;
}

int grid_for(int64_t elems, int64_t tile, int max_ctas) {
  int64_t g = (elems + tile - 1) / tile;
  if (g > max_ctas) g = max_ctas;
  return g < 1 ? 1 : (int)g;
}

template <typename T, int W, int MAXS>
cudaError_t run_reduce(const CeView& v, int first, int n, const void* slot0, int64_t stride, int rank,
                       float s, int max_ctas, cudaStream_t st) {
  const CeArgs<MAXS> a = make_args<MAXS>(v, first, n);
  const int grid = grid_for(a.vo[n], kTileBytes / sizeof(T), max_ctas);
  ce_reduce_kernel<T, W, MAXS><<<grid, kThreads, 0, st>>>(a, static_cast<const char*>(slot0), stride, rank, s);
  return cudaGetLastError();
}

template <typename T, int W>
cudaError_t reduce_by_slots(const CeView& v, const void* slot0, int64_t stride, int rank, float s, int max_ctas,
                            cudaStream_t st) {
  for (int first = 0; first < v.n; first += kMaxSlotsPerLaunch) {
    const int n = v.n - first < kMaxSlotsPerLaunch ? v.n - first : kMaxSlotsPerLaunch;
    cudaError_t e = n <= 32    ? run_reduce<T, W, 32>(v, first, n, slot0, stride, rank, s, max_ctas, st)
                    : n <= 256 ? run_reduce<T, W, 256>(v, first, n, slot0, stride, rank, s, max_ctas, st)
                               : run_reduce<T, W, 1024>(v, first, n, slot0, stride, rank, s, max_ctas, st);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

template <typename T>
cudaError_t reduce_by_world(int world, const CeView& v, const void* slot0, int64_t stride, int rank, float s,
                            int max_ctas, cudaStream_t st) {
  switch (world) {
    case 2: return reduce_by_slots<T, 2>(v, slot0, stride, rank, s, max_ctas, st);
    case 3: return reduce_by_slots<T, 3>(v, slot0, stride, rank, s, max_ctas, st);
    case 4: return reduce_by_slots<T, 4>(v, slot0, stride, rank, s, max_ctas, st);
    case 5: return reduce_by_slots<T, 5>(v, slot0, stride, rank, s, max_ctas, st);
    case 6: return reduce_by_slots<T, 6>(v, slot0, stride, rank, s, max_ctas, st);
    case 7: return reduce_by_slots<T, 7>(v, slot0, stride, rank, s, max_ctas, st);
    case 8: return reduce_by_slots<T, 8>(v, slot0, stride, rank, s, max_ctas, st);
    default: return cudaErrorInvalidValue;
  }
}

template <typename T, int MAXS>
cudaError_t run_gather(const CeView& v, int first, int n, void* own_slot, int max_ctas, cudaStream_t st) {
  const CeArgs<MAXS> a = make_args<MAXS>(v, first, n);
  const int grid = grid_for(a.vo[n], kTileBytes / sizeof(T), max_ctas);
  ce_gather_kernel<T, MAXS><<<grid, kThreads, 0, st>>>(a, static_cast<T*>(own_slot));
  return cudaGetLastError();
}

template <typename T>
cudaError_t gather(const CeView& v, void* own_slot, int max_ctas, cudaStream_t st) {
  for (int first = 0; first < v.n; first += kMaxSlotsPerLaunch) {
    const int n = v.n - first < kMaxSlotsPerLaunch ? v.n - first : kMaxSlotsPerLaunch;
    cudaError_t e = n <= 32    ? run_gather<T, 32>(v, first, n, own_slot, max_ctas, st)
                    : n <= 256 ? run_gather<T, 256>(v, first, n, own_slot, max_ctas, st)
                               : run_gather<T, 1024>(v, first, n, own_slot, max_ctas, st);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

template <typename T, int NP, int MAXS>
cudaError_t run_push(const CeView& v, int first, int n, const PeerDst& pd, int max_ctas, cudaStream_t st) {
  const CeArgs<MAXS> a = make_args<MAXS>(v, first, n);
  const int grid = grid_for(a.vo[n], kTileBytes / sizeof(T), max_ctas);
  ce_push_kernel<T, NP, MAXS><<<grid, kThreads, 0, st>>>(a, pd);
  return cudaGetLastError();
}

template <typename T, int NP>
cudaError_t push_by_slots(const CeView& v, const PeerDst& pd, int max_ctas, cudaStream_t st) {
  for (int first = 0; first < v.n; first += kMaxSlotsPerLaunch) {
    const int n = v.n - first < kMaxSlotsPerLaunch ? v.n - first : kMaxSlotsPerLaunch;
    cudaError_t e = n <= 32    ? run_push<T, NP, 32>(v, first, n, pd, max_ctas, st)
                    : n <= 256 ? run_push<T, NP, 256>(v, first, n, pd, max_ctas, st)
                               : run_push<T, NP, 1024>(v, first, n, pd, max_ctas, st);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

template <typename T>
cudaError_t push_by_world(int npeers, const CeView& v, const PeerDst& pd, int max_ctas, cudaStream_t st) {
  switch (npeers) {
    case 1: return push_by_slots<T, 1>(v, pd, max_ctas, st);
    case 2: return push_by_slots<T, 2>(v, pd, max_ctas, st);
    case 3: return push_by_slots<T, 3>(v, pd, max_ctas, st);
    case 4: return push_by_slots<T, 4>(v, pd, max_ctas, st);
    case 5: return push_by_slots<T, 5>(v, pd, max_ctas, st);
    case 6: return push_by_slots<T, 6>(v, pd, max_ctas, st);
    case 7: return push_by_slots<T, 7>(v, pd, max_ctas, st);
    default: return cudaErrorInvalidValue;
  }
}

// CE2: dst[i] = RNE( sum_{q<W} src_q[i] ), rank order, fp32 (the values are
// pre-scaled by pack); dst may alias src_rank (same element, same thread).
// EACH (gradient-as-bucket-view: raw operands): RNE( sum_q RNE(src_q[i] * s) ) = O-3b.
struct ShardSrc {
  const void* p[kMaxWorld];
};

template <typename T, int W, bool EACH>
__global__ void __launch_bounds__(kThreads) shard_reduce_kernel(const __grid_constant__ ShardSrc ss,
                                                                T* dst, int64_t n, float s) {
  constexpr int64_t tile = kTileBytes / sizeof(T);
  for (int64_t t = (int64_t)blockIdx.x * tile; t < n; t += (int64_t)gridDim.x * tile) {
    const int64_t m = min(tile, n - t);
    T* d[1] = {dst + t};
    const T* src[W];
#pragma unroll
    for (int q = 0; q < W; ++q) src[q] = static_cast<const T*>(ss.p[q]) + t;
    cta_xfer<T, W, 1, false, EACH, EACH>(d, src, m, s);
  }
}

template <typename T, bool EACH>
cudaError_t shard_reduce(int world, const ShardSrc& ss, void* dst, int64_t n, float s, int max_ctas,
                         cudaStream_t st) {
  const int grid = grid_for(n, kTileBytes / sizeof(T), max_ctas);
  T* d = static_cast<T*>(dst);
  switch (world) {
    case 2: shard_reduce_kernel<T, 2, EACH><<<grid, kThreads, 0, st>>>(ss, d, n, s); break;
    case 3: shard_reduce_kernel<T, 3, EACH><<<grid, kThreads, 0, st>>>(ss, d, n, s); break;
    case 4: shard_reduce_kernel<T, 4, EACH><<<grid, kThreads, 0, st>>>(ss, d, n, s); break;
    case 5: shard_reduce_kernel<T, 5, EACH><<<grid, kThreads, 0, st>>>(ss, d, n, s); break;
    case 6: shard_reduce_kernel<T, 6, EACH><<<grid, kThreads, 0, st>>>(ss, d, n, s); break;
    case 7: shard_reduce_kernel<T, 7, EACH><<<grid, kThreads, 0, st>>>(ss, d, n, s); break;
    case 8: shard_reduce_kernel<T, 8, EACH><<<grid, kThreads, 0, st>>>(ss, d, n, s); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_shard_reduce(int dtype, int world, const void* const* src, void* dst, int64_t n, float scale,
                                int max_ctas, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  ShardSrc ss{};
  for (int q = 0; q < world && q < kMaxWorld; ++q) ss.p[q] = src[q];
  if (scale != 1.0f)
    return dtype == 0 ? shard_reduce<float, true>(world, ss, dst, n, scale, max_ctas, s)
                      : shard_reduce<__nv_bfloat16, true>(world, ss, dst, n, scale, max_ctas, s);
  return dtype == 0 ? shard_reduce<float, false>(world, ss, dst, n, 1.0f, max_ctas, s)
                    : shard_reduce<__nv_bfloat16, false>(world, ss, dst, n, 1.0f, max_ctas, s);
}

cudaError_t launch_ce_push(int dtype, const CeView& v, void* const* peer_slots, int npeers, int max_ctas,
                           cudaStream_t s) {
  PeerDst pd{};
  for (int j = 0; j < npeers && j < kMaxWorld; ++j) pd.p[j] = static_cast<char*>(peer_slots[j]);
  return dtype == 0 ? push_by_world<float>(npeers, v, pd, max_ctas, s)
                    : push_by_world<__nv_bfloat16>(npeers, v, pd, max_ctas, s);
}

cudaError_t launch_ce_gather(int dtype, const CeView& v, void* own_slot, int max_ctas, cudaStream_t s) {
  if (v.n == 0) return cudaSuccess;
  return dtype == 0 ? gather<float>(v, own_slot, max_ctas, s) : gather<__nv_bfloat16>(v, own_slot, max_ctas, s);
}

cudaError_t launch_ce_reduce(int dtype, int world, int rank, const CeView& v, const void* slot0,
                             int64_t stride_bytes, float scale, int max_ctas, cudaStream_t s) {
  return dtype == 0 ? reduce_by_world<float>(world, v, slot0, stride_bytes, rank, scale, max_ctas, s)
                    : reduce_by_world<__nv_bfloat16>(world, v, slot0, stride_bytes, rank, scale, max_ctas, s);
}

}  // namespace b200ddp
