// pull.cu — the fused bucket allreduce over NVLink 5 / NVSwitch peer memory,
// "pull" form: every rank packs into its OWN bucket buffer, and ranks READ each
// other's buffers (peer loads, 775 GB/s per GPU on B200-class parts, B300_MICROARCH
// "peer BW (kernel LDG.128)").  One launch per bucket, pack (x 1/W) and unpack
// fused in.
//
// What it computes ("gradient summation across all processes",
// L166 average, Alg. 1): for every element x of bucket b,
//     grad_r(x) <- RNE( sum_{q=0..W-1} RNE(g_q(x) * fl(1/W)) )   on every rank r,
// accumulated in fp32 in fixed rank order q = 0..W-1 (readings C-2, C-3, C-4):
// exactly oracle O-3b, bit-identical on all ranks.
//
// Why pull (vs pushing into peers' staging): a rank signals "my stores are done"
// only for LOCAL stores (its own buffer), so the system-scope release before
// each flag drains local HBM writes, not remote NVLink writes; the all-gather
// reads land straight in .grad (no unpack pass, no closing barrier).  Reuse of a
// buffer is ordered by double buffering: pass v uses buffer v % 2 of the bucket,
// and a rank rewrites buffer v % 2 in pass v + 2 only after its pass-(v+1)
// kernel saw every peer's pass-(v+1) "packed" flag, which each peer raised
// after its pass-v kernel (all of whose reads of this rank's buffer) completed
// (same bucket -> same lane stream -> launches in order).
//
// One-shot (small buckets, and W = 2 at any size: it moves (W-1) S = S per
// direction, like two-shot, with ONE sync):
//   P  CTA c packs chunk c (stage k) into its own buffer;      flag kind 0
//   R  reads chunk c (stage k) of all W buffers (W-1 remote) and writes the
//      rank-order sum straight into .grad.
// Two-shot (reduce-scatter + all-gather, 2(W-1)/W S per direction):
//   P  CTA c packs chunk c of every shard into its own buffer;  flag kind 0
//   R  sums chunk c of its OWN shard r over the W buffers (W-1 remote), writes
//      it into its own buffer (in place: the same thread loads then stores an
//      element) and into .grad;                                  flag kind 1
//   G  reads chunk c of every other shard j from rank j's buffer (the sums)
//      straight into .grad.
// Stages: each CTA chunk is split into `stages` sub-chunks and the phases are
// software-pipelined (iteration k: P(k), R(k-1), G(k-2)), so local packing of a
// stage overlaps the NVLink reads of the previous one.
#include "barrier.cuh"

namespace b200ddp {

namespace {

// Publish "this CTA's stores through here are done": kind-0 value v0 and / or
// kind-1 value v1 (0 = not this time) for the same CTA index of every peer.
// bar.sync first orders every thread's stores before the publishing thread(s).
// a.sig_mode (DDP_OPT_P2P_SIGNAL): 0 fence.sc.sys + st.release.sys into each
// peer; 1 st.release.sys alone; 2 fence.acq_rel.gpu + st.relaxed.sys (the stores
// being published are LOCAL and already performed at this GPU's L2, which also
// serves the peers' reads); 3 st.release.gpu into the OWN flag table, polled by
// the peers over NVLink.
template <int W>
__device__ __forceinline__ void pull_signal(const P2PLaunch& a, int r, uint32_t v0, uint32_t v1) {
  __syncthreads();
  const int t = threadIdx.x;
  if (a.sig_mode == 3) {
    if (t == 0) {
      if (v0) {
        uint32_t* f = flag_ptr(a.storage[r], a.flags_byte_off, 0, blockIdx.x, r);
        asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(f), "r"(v0) : "memory");
      }
      if (v1) {
        uint32_t* f = flag_ptr(a.storage[r], a.flags_byte_off, 1, blockIdx.x, r);
        asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(f), "r"(v1) : "memory");
      }
    }
    return;
  }
  if (t < W && t != r) {
    if (a.sig_mode == 0) __threadfence_system();
    if (a.sig_mode == 2) asm volatile("fence.acq_rel.gpu;" ::: "memory");
    for (int kind = 0; kind < 2; ++kind) {
      const uint32_t v = kind ? v1 : v0;
      if (!v) continue;
      uint32_t* f = flag_ptr(a.storage[t], a.flags_byte_off, kind, blockIdx.x, r);
      if (a.sig_mode == 2) asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(f), "r"(v) : "memory");
      else asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(f), "r"(v) : "memory");
    }
  }
}

// Wait until every peer's same-index CTA has published >= val (bounded spin);
// sig_mode 3 polls the peers' own flag tables over NVLink.
template <int W>
__device__ __forceinline__ void pull_wait(const P2PLaunch& a, int r, int kind, uint32_t val) {
  const int t = threadIdx.x;
  if (t < W && t != r) {
    const uint32_t* f = a.sig_mode == 3 ? flag_ptr(a.storage[t], a.flags_byte_off, kind, blockIdx.x, t)
                                        : flag_ptr(a.storage[r], a.flags_byte_off, kind, blockIdx.x, t);
    const uint64_t t0 = globaltimer();
    while (true) {
      uint32_t v;
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
      if ((int32_t)(v - val) >= 0) break;
      if (globaltimer() - t0 > a.timeout_ns) {
        atomicExch(a.err, 1u);
        break;
      }
    }
  }
  __syncthreads();
}

// grad(x) = RNE( sum_{k<NS} src_k[x - base] ) for x in [lo, hi) (rank order), also
// written to extra[x - base] when EXTRA (the two-shot's own shard, in place).
template <typename T, int NS, bool EXTRA, int MAXS>
__device__ __forceinline__ void walk_sum(const SlotArgs<MAXS>& sa, int64_t lo, int64_t hi,
                                         const T* const (&srcb)[NS], T* extra, int64_t base, int64_t gstride) {
  if (lo >= hi) return;
  for (int k = find_slot(sa, lo); k < sa.n && lo < hi; ++k) {
    const int64_t s0 = sa.off[k], e = min(hi, sa.off[k + 1]);
    if (e <= lo) continue;
    T* g = reinterpret_cast<T*>(static_cast<char*>(sa.grad[k]) + gstride) + (lo - s0);
    const T* sp[NS];
#pragma unroll
    for (int j = 0; j < NS; ++j) sp[j] = srcb[j] + (lo - base);
    if (EXTRA) {
      T* d[2] = {g, extra + (lo - base)};
      cta_xfer<T, NS, 2, false, false>(d, sp, e - lo, 1.0f);
    } else {
      T* d[1] = {g};
      cta_xfer<T, NS, 1, false, false>(d, sp, e - lo, 1.0f);
    }
    lo = e;
  }
}

template <typename T, int W, int MAXS>
__global__ void __launch_bounds__(kThreads, 1)
    pull_oneshot_kernel(const __grid_constant__ SlotArgs<MAXS> sa, const __grid_constant__ P2PLaunch a) {
  const int r = a.emulated ? (int)blockIdx.y : a.rank;
  if (a.emulated && r == a.dead_rank) return;  // test support: a peer that never arrives
  const int64_t gstride = a.emulated ? (int64_t)r * a.grad_rank_stride : 0;
  const int64_t lo0 = min((int64_t)blockIdx.x * a.chunk, a.numel);
  const int64_t hi0 = min(lo0 + a.chunk, a.numel);
  T* own = at<T>(a.storage[r], a.bucket_byte_off);
  const T* buf[W];
#pragma unroll
  for (int q = 0; q < W; ++q) buf[q] = at<T>(a.storage[q], a.bucket_byte_off);
  const int K = a.stages;
#pragma unroll 1
  for (int k = 0; k <= K; ++k) {
    if (k < K) {  // P: pack + scale stage k into the own buffer, then publish it
      const int64_t lo = min(lo0 + (int64_t)k * a.sub, hi0), hi = min(lo + a.sub, hi0);
      T* d[1] = {own};
      if (!(a.debug & 2)) walk_pack<T, 1, MAXS>(sa, lo, hi, d, 0, a.scale, gstride);
      pull_signal<W>(a, r, a.seq + (uint32_t)(k + 1), 0);
    }
    if (k >= 1) {  // R: stage k-1 of every rank's buffer -> rank-order sum -> .grad
      pull_wait<W>(a, r, 0, a.seq + (uint32_t)k);
      const int64_t lo = min(lo0 + (int64_t)(k - 1) * a.sub, hi0), hi = min(lo + a.sub, hi0);
      if (!(a.debug & 1)) walk_sum<T, W, false, MAXS>(sa, lo, hi, buf, nullptr, 0, gstride);
    }
  }
}

template <typename T, int W, int MAXS>
__global__ void __launch_bounds__(kThreads, 1)
    pull_twoshot_kernel(const __grid_constant__ SlotArgs<MAXS> sa, const __grid_constant__ P2PLaunch a) {
  const int r = a.emulated ? (int)blockIdx.y : a.rank;
  if (a.emulated && r == a.dead_rank) return;
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
  T* own = at<T>(a.storage[r], a.bucket_byte_off);
  const T* buf[W];
#pragma unroll
  for (int q = 0; q < W; ++q) buf[q] = at<T>(a.storage[q], a.bucket_byte_off);

#pragma unroll 1
  for (int k = 0; k <= K + 1; ++k) {
    if (k < K) {  // P: pack + scale stage k of chunk c of every shard into the own buffer
      T* d[1] = {own};
#pragma unroll 1
      for (int j = 0; j < W; ++j) {
        int64_t lo, hi;
        rng(j, k, lo, hi);
        if (!(a.debug & 2)) walk_pack<T, 1, MAXS>(sa, lo, hi, d, 0, a.scale, gstride);
      }
    }
    if (k >= 1 && k <= K) {  // R: own shard, stage k-1: sum over the W buffers -> own buffer + .grad
      pull_wait<W>(a, r, 0, a.seq + (uint32_t)k);
      int64_t lo, hi;
      rng(r, k - 1, lo, hi);
      if (!(a.debug & 1)) walk_sum<T, W, true, MAXS>(sa, lo, hi, buf, own, 0, gstride);
    }
    // publish: "packed through stage k" (kind 0) and "reduced through stage k-1" (kind 1);
    // one CTA barrier + one release covers both (local stores only)
    if (k <= K) pull_signal<W>(a, r, k < K ? a.seq + (uint32_t)(k + 1) : 0u, k >= 1 ? a.seq + (uint32_t)k : 0u);
    if (k >= 2) {  // G: every other shard j, stage k-2, from rank j's buffer -> .grad
      pull_wait<W>(a, r, 1, a.seq + (uint32_t)(k - 1));
#pragma unroll 1
      for (int i = 1; i < W; ++i) {
        const int j = (r + i) % W;
        int64_t lo, hi;
        rng(j, k - 2, lo, hi);
        const T* src[1] = {buf[j]};
        if (!(a.debug & 1)) walk_sum<T, 1, false, MAXS>(sa, lo, hi, src, nullptr, 0, gstride);
      }
    }
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
#define B200DDP_K(WW)                                                           \
  case WW:                                                                      \
    return algo == 3 ? reinterpret_cast<void*>(pull_twoshot_kernel<T, WW, MAXS>) \
                     : reinterpret_cast<void*>(pull_oneshot_kernel<T, WW, MAXS>);
  switch (world) {
    B200DDP_K(2) B200DDP_K(3) B200DDP_K(4) B200DDP_K(5) B200DDP_K(6) B200DDP_K(7) B200DDP_K(8)
    default: return nullptr;
  }
#undef B200DDP_K
}

template <typename T, int MAXS>
cudaError_t run(int algo, const SlotView& sv, const P2PLaunch& a, cudaStream_t st) {
  const SlotArgs<MAXS> sargs = make_args<MAXS>(sv);
  P2PLaunch pa = a;
  void* args[] = {const_cast<SlotArgs<MAXS>*>(&sargs), &pa};
  void* fn = kernel_ptr<T, MAXS>(algo, a.world);
  if (!fn) return cudaErrorInvalidValue;
  if (a.emulated) return cudaLaunchCooperativeKernel(fn, dim3(a.ctas, a.world), dim3(kThreads), args, 0, st);
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
  void* fn = n_slots <= 32 ? kernel_ptr<T, 32>(algo, world)
             : n_slots <= 256 ? kernel_ptr<T, 256>(algo, world) : kernel_ptr<T, 1024>(algo, world);
  if (!fn || cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, fn, kThreads, 0) != cudaSuccess) return 0;
  return blocks;
}

}  // namespace

cudaError_t launch_pull(int algo, int dtype, const SlotView& sv, const P2PLaunch& a, cudaStream_t s) {
  return dtype == 0 ? dispatch<float>(algo, sv, a, s) : dispatch<__nv_bfloat16>(algo, sv, a, s);
}

int pull_occupancy(int algo, int dtype, int world, int n_slots) {
  return dtype == 0 ? occupancy<float>(algo, world, n_slots) : occupancy<__nv_bfloat16>(algo, world, n_slots);
}

}  // namespace b200ddp
