// p2p.cu — hand-written sm_100a bucket allreduce over NVLink 5 / NVSwitch peer
// memory, fused with pack (x 1/W) and unpack.  One launch per bucket.
//
// What it computes ("gradient summation across all processes",
// L166 average, Alg. 1): for every element x of bucket b,
//     grad_r(x) <- RNE( sum_{q=0..W-1} RNE(g_q(x) * fl(1/W)) )   on every rank r,
// accumulated in fp32 in fixed rank order q = 0..W-1 (readings C-2, C-3, C-4),
// i.e. exactly oracle O-3b, bit-identical on all ranks.
//
// Memory (per rank, symmetric storage, see core/reducer.cpp):
//   flags    uint32 [kMaxCtas][kMaxWorld]   barrier counters, [cta][src rank]
//   bucket   per-bucket flat buffers         two-shot all-gather target
//   staging  [W][...] per-source slots        push targets
//
// Two-shot (reduce-scatter + all-gather, 2(W-1)/W * S per direction):
//   A  CTA c of rank r packs chunk c of every shard j and PUSHES it (remote
//      st.global.v4) into rank j's staging slot r;
//   B  barrier among CTA c of all ranks;
//   C  rank r reduces chunk c of its own shard from its W local staging slots
//      and pushes the result into every rank's bucket;
//   D  barrier;
//   E  rank r unpacks chunk c of every shard from its own bucket into .grad.
// One-shot (small buckets, latency bound): A pushes the whole chunk c to every
// rank; B barrier; C each rank reduces chunk c from its W local slots straight
// into .grad (fused unpack).  Staging is double-buffered by launch parity, so
// no closing barrier is needed (the next launch's barrier orders reuse).
//
// Barriers: per CTA index, monotonic uint32 counters written with
// st.release.sys into the peer's flag table and polled with ld.acquire.sys;
// all writers fence.acq_rel.sys first.  A bounded spin (30 s of %globaltimer)
// sets the error word instead of hanging.  All remote traffic is stores.
#include <cooperative_groups.h>

#include "barrier.cuh"

namespace b200ddp {

namespace {

// Two-shot, software-pipelined over `stages` sub-chunks of the CTA's chunk:
// iteration k pushes reduce-scatter data of stage k, reduces + all-gathers
// stage k-1 and unpacks stage k-2, so NVLink stores of one stage overlap the
// local reduction / unpack of the previous ones.
template <typename T, int W, int MAXS>
__global__ void __launch_bounds__(kThreads, 1)
    twoshot_kernel(const __grid_constant__ SlotArgs<MAXS> sa, const __grid_constant__ P2PLaunch a) {
  const int r = a.emulated ? (int)blockIdx.y : a.rank;
  if (a.emulated && r == a.dead_rank) return;  // test support: a peer that never arrives
  const int64_t gstride = a.emulated ? (int64_t)r * a.grad_rank_stride : 0;
  const int c = blockIdx.x;
  const int64_t L = a.shard, N = a.numel, Q = a.chunk, SUB = a.sub;
  const int K = a.stages;
  // stage k of chunk c of shard j: [j*L + c*Q + k*SUB, ...) clipped to the chunk, shard and bucket
  auto rng = [&](int j, int k, int64_t& lo, int64_t& hi) {
    const int64_t c0 = (int64_t)c * Q, c1 = min(c0 + Q, L);
    lo = min(j * L + min(c0 + (int64_t)k * SUB, c1), N);
    hi = min(j * L + min(c0 + (int64_t)(k + 1) * SUB, c1), N);
  };

#pragma unroll 1
  for (int k = 0; k <= K + 1; ++k) {
    if (k < K) {  // A: pack + scale, push stage k of every shard j into rank j's slot r
#pragma unroll
      for (int i = 1; i <= W; ++i) {
        const int j = (r + i) % W;  // peers in rotated order, self last
        int64_t lo, hi;
        rng(j, k, lo, hi);
        if (lo >= hi) continue;
        T* d[1] = {at<T>(a.storage[j], a.stage_byte_off + (int64_t)r * a.stage_stride)};
        walk_pack<T, 1, MAXS>(sa, lo, hi, d, j * L, a.scale, gstride);
      }
    }
    if (k >= 1 && k <= K) {  // C: reduce own shard, stage k-1; all-gather into every bucket
      p2p_wait<W>(a, r, 0, a.seq + (uint32_t)k);
      int64_t lo, hi;
      rng(r, k - 1, lo, hi);
      if (lo < hi) {
        const T* src[W];
        T* dst[W];
#pragma unroll
        for (int q = 0; q < W; ++q) {
          src[q] = at<T>(a.storage[r], a.stage_byte_off + (int64_t)q * a.stage_stride) + (lo - r * L);
          dst[q] = at<T>(a.storage[(r + 1 + q) % W], a.bucket_byte_off) + lo;
        }
        cta_xfer<T, W, W, false, false>(dst, src, hi - lo, 1.0f);
      }
    }
    if (k >= 2) {  // E: unpack stage k-2 of every shard from the local bucket
      p2p_wait<W>(a, r, 1, a.seq + (uint32_t)(k - 1));
      const T* b[1] = {at<T>(a.storage[r], a.bucket_byte_off)};
#pragma unroll
      for (int j = 0; j < W; ++j) {
        int64_t lo, hi;
        rng(j, k - 2, lo, hi);
        if (lo < hi) walk_unpack<T, 1, MAXS>(sa, lo, hi, b, 0, gstride);
      }
    }
    if (W == 1) {
      __syncthreads();
    } else if (k <= K) {
      p2p_signal<W>(a, r, 0, a.seq + (uint32_t)(k + 1));  // through stage k (k == K: harmless)
      if (k >= 1) {
        const int t = threadIdx.x;  // all-gather of stage k-1 is covered by the same fence
        if (t < W && t != r) {
          uint32_t* f = flag_ptr(a.storage[t], a.flags_byte_off, 1, blockIdx.x, r);
          asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(f), "r"(a.seq + (uint32_t)k) : "memory");
        }
      }
    }
  }
}

// One-shot, software-pipelined: iteration k pushes stage k of the chunk to
// slot r of every rank and reduces stage k-1 (W local slots, rank order)
// straight into the gradients.  Staging is double-buffered by launch parity.
template <typename T, int W, int MAXS>
__global__ void __launch_bounds__(kThreads, 1)
    oneshot_kernel(const __grid_constant__ SlotArgs<MAXS> sa, const __grid_constant__ P2PLaunch a) {
  const int r = a.emulated ? (int)blockIdx.y : a.rank;
  if (a.emulated && r == a.dead_rank) return;  // test support: a peer that never arrives
  const int64_t gstride = a.emulated ? (int64_t)r * a.grad_rank_stride : 0;
  const int64_t lo0 = min((int64_t)blockIdx.x * a.chunk, a.numel);
  const int64_t hi0 = min(lo0 + a.chunk, a.numel);

  if (W == 1) {
    // A world of one: the allreduce of the packed value s = RNE(g * 1) is s
    // itself, so each thread packs into the bucket and writes the reduced
    // value back to .grad from registers (pack, 1-rank reduce, unpack fused).
    T* st = at<T>(a.storage[r], a.stage_byte_off);
    for (int k = find_slot(sa, lo0); k < sa.n; ++k) {
      const int64_t s0 = sa.off[k];
      if (s0 >= hi0) break;
      const int64_t x0 = max(lo0, s0), x1 = min(hi0, sa.off[k + 1]);
      if (x0 >= x1) continue;
      T* g = reinterpret_cast<T*>(static_cast<char*>(sa.grad[k]) + gstride) + (x0 - s0);
      T* dd[2] = {st + x0, g};
      const T* sp[1] = {g};
      cta_xfer<T, 1, 2, true, true>(dd, sp, x1 - x0, a.scale);
    }
    return;
  }

  const int K = a.stages;
  T* d[W];
  const T* s[W];
#pragma unroll
  for (int q = 0; q < W; ++q) {
    d[q] = at<T>(a.storage[(r + 1 + q) % W], a.stage_byte_off + (int64_t)r * a.stage_stride);
    s[q] = at<T>(a.storage[r], a.stage_byte_off + (int64_t)q * a.stage_stride);
  }
#pragma unroll 1
  for (int k = 0; k <= K; ++k) {
    if (k < K) {  // A: pack + scale stage k once, push to slot r of every rank
      const int64_t lo = min(lo0 + (int64_t)k * a.sub, hi0), hi = min(lo + a.sub, hi0);
      walk_pack<T, W, MAXS>(sa, lo, hi, d, 0, a.scale, gstride);
    }
    if (k >= 1) {  // C: stage k-1 from every rank -> reduce in rank order -> .grad
      p2p_wait<W>(a, r, 0, a.seq + (uint32_t)k);
      const int64_t lo = min(lo0 + (int64_t)(k - 1) * a.sub, hi0), hi = min(lo + a.sub, hi0);
      walk_unpack<T, W, MAXS>(sa, lo, hi, s, 0, gstride);
    }
    if (k < K) p2p_signal<W>(a, r, 0, a.seq + (uint32_t)(k + 1));
  }
}

template <int MAXS>
SlotArgs<MAXS> make_args(const SlotView& sv) {
  SlotArgs<MAXS> a;
  a.n = sv.n;
  for (int k = 0; k < sv.n; ++k) {
    a.grad[k] = sv.grad[k];
    a.off[k] = sv.off[k];
  }
  a.off[sv.n] = sv.off[sv.n];
  return a;
}

template <typename T, int MAXS>
void* kernel_ptr(int algo, int world) {
#define B200DDP_K(WW)                                                      \
  case WW:                                                                 \
    return algo == 3 ? reinterpret_cast<void*>(twoshot_kernel<T, WW, MAXS>) \
                     : reinterpret_cast<void*>(oneshot_kernel<T, WW, MAXS>);
  switch (world) {
    B200DDP_K(1) B200DDP_K(2) B200DDP_K(3) B200DDP_K(4) B200DDP_K(5) B200DDP_K(6) B200DDP_K(7) B200DDP_K(8)
    default: return nullptr;
  }
#undef B200DDP_K
}

template <typename T>
void* kernel_for(int algo, int world, int n_slots) {
  if (n_slots <= 32) return kernel_ptr<T, 32>(algo, world);
  if (n_slots <= 256) return kernel_ptr<T, 256>(algo, world);
  return kernel_ptr<T, 1024>(algo, world);
}

template <typename T, int MAXS>
cudaError_t run(int algo, const SlotView& sv, const P2PLaunch& a, cudaStream_t st) {
  const SlotArgs<MAXS> sargs = make_args<MAXS>(sv);
  P2PLaunch pa = a;
  void* args[] = {const_cast<SlotArgs<MAXS>*>(&sargs), &pa};
  void* fn = kernel_ptr<T, MAXS>(algo, a.world);
  if (!fn) return cudaErrorInvalidValue;
  if (a.emulated) {
    return cudaLaunchCooperativeKernel(fn, dim3(a.ctas, a.world), dim3(kThreads), args, 0, st);
  }
  return cudaLaunchKernel(fn, dim3(a.ctas), dim3(kThreads), args, 0, st);
}

template <typename T>
cudaError_t dispatch(int algo, const SlotView& sv, const P2PLaunch& a, cudaStream_t st) {
  if (sv.n <= 32) return run<T, 32>(algo, sv, a, st);
  if (sv.n <= 256) return run<T, 256>(algo, sv, a, st);
  if (sv.n <= kMaxSlotsPerLaunch) return run<T, 1024>(algo, sv, a, st);
  return cudaErrorInvalidValue;
}

template <typename T>
int occupancy(int algo, int world, int n_slots) {
  int blocks = 0;
  void* fn = kernel_for<T>(algo, world, n_slots);
  if (!fn || cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, fn, kThreads, 0) != cudaSuccess) return 0;
  return blocks;
}

}  // namespace

cudaError_t launch_p2p(int algo, int dtype, const SlotView& sv, const P2PLaunch& a, cudaStream_t s) {
  if ((a.pull || a.view) && a.world > 1) return launch_pull(algo, dtype, sv, a, s);
  return dtype == 0 ? dispatch<float>(algo, sv, a, s) : dispatch<__nv_bfloat16>(algo, sv, a, s);
}

int emulated_max_ctas(int algo, int dtype, int n_slots, int world, bool pull, bool view) {
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 0;
  const int occ = view && world > 1   ? pull_view_occupancy(dtype, world)
                  : pull && world > 1 ? pull_occupancy(algo, dtype, world, n_slots)
                  : dtype == 0 ? occupancy<float>(algo, world, n_slots)
                               : occupancy<__nv_bfloat16>(algo, world, n_slots);
  return occ * sms / (world > 0 ? world : 1);
}

}  // namespace b200ddp
