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
// only for LOCAL stores (its own buffer), so a gpu-scope fence before each flag
// suffices (reading A-1; ~1 us against 5-8 us for the system-scope
// fence remote stores need); the all-gather reads land straight in .grad (no
// unpack pass, no closing barrier).  Pulling needs many CTAs to keep enough loads
// in flight, so by default it runs the last bucket of a pass (every SM); the
// buckets beside backward keep the push kernels (kernels/p2p.cu).  Reuse of a
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
// Stages + warp specialization: each CTA chunk is split into `stages` sub-chunks;
// a quarter (or half) of the CTA's warps pack stage after stage (P) and publish
// each, the others read and reduce one stage behind (R, G), so local packing
// overlaps the NVLink reads.  A third form, pull_view_twoshot_kernel, runs the
// two-shot in place on gradients that ARE the bucket (DDP_OPT_GRAD_VIEW).
#include "barrier.cuh"

namespace b200ddp {

namespace {

// Warp specialization: the first a.pack_threads threads of a CTA pack stage after
// stage into the own buffer and publish each one; the other kThreads -
// a.pack_threads read (over NVLink) and reduce, one stage behind, so local packing
// overlaps the NVLink reads.  Named barriers: 1 = pack group, 2 = read group.
// The host picks the split: a quarter of the CTA packs when the grid covers the
// SMs (each CTA's chunk is small), half when it is capped (COMM_CTAS): there the
// pack of a large per-CTA chunk would otherwise hold the reads back.

__device__ __forceinline__ void group_sync(int id, int nt) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nt) : "memory");
}

// Publish "this group's stores through stage v are done" for the same CTA index
// of every peer: kind-`kind` value v.  Called by EVERY thread of the group (the
// group barrier orders all of its stores before the publishing threads).
// a.sig_mode (DDP_OPT_P2P_SIGNAL): 0 (default) fence.acq_rel.gpu + st.relaxed.sys
// into each peer: the published stores are LOCAL, so once the gpu-scope fence has
// them performed at this GPU's L2 — which is also where every peer's read of them
// is served (peer loads bypass the reader's L2, B300_MICROARCH "NVLink") — the
// flag store that follows cannot overtake them; 1 fence.sc.sys + st.release.sys
// (the formal system-scope release; measured ~7 us per publish, profiles/r02_pull.md);
// 2 st.release.sys alone; 3 st.release.gpu into the OWN flag table, polled by the
// peers over NVLink.  `smem` (optional): the group's progress for the other group
// of this CTA, written after the fence.
template <int W>
__device__ __forceinline__ void group_publish(const P2PLaunch& a, int r, int kind, uint32_t v, int bar_id, int gt,
                                              int nt, volatile uint32_t* smem, uint32_t smem_v) {
  group_sync(bar_id, nt);
  if (a.sig_mode == 3) {
    if (gt == 0) {
      uint32_t* f = flag_ptr(a.storage[r], a.flags_byte_off, kind, blockIdx.x, r);
      asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(f), "r"(v) : "memory");
      if (smem) *smem = smem_v;
    }
    return;
  }
  if (gt < W && (gt != r || smem)) {
    if (a.sig_mode == 1) __threadfence_system();
    else if (a.sig_mode == 0) asm volatile("fence.acq_rel.gpu;" ::: "memory");
    if (gt != r) {
      uint32_t* f = flag_ptr(a.storage[gt], a.flags_byte_off, kind, blockIdx.x, r);
      if (a.sig_mode == 0) asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(f), "r"(v) : "memory");
      else asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(f), "r"(v) : "memory");
    } else {
      __threadfence();  // own group's progress for the other group (gpu scope suffices: same SM)
      *smem = smem_v;
    }
  }
}

// Wait (whole group) until every peer's same-index CTA has published kind >= val
// and, if `smem`, this CTA's other group has reached smem_v.  Bounded spin.
template <int W>
__device__ __forceinline__ void group_wait(const P2PLaunch& a, int r, int kind, uint32_t val, int bar_id, int gt,
                                           int nt, volatile uint32_t* smem, uint32_t smem_v) {
  if (gt < W) {
    const uint64_t t0 = globaltimer();
    if (gt != r) {
      const uint32_t* f = a.sig_mode == 3 ? flag_ptr(a.storage[gt], a.flags_byte_off, kind, blockIdx.x, gt)
                                          : flag_ptr(a.storage[r], a.flags_byte_off, kind, blockIdx.x, gt);
      while (true) {
        uint32_t v;
        asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
        if ((int32_t)(v - val) >= 0) break;
        if (globaltimer() - t0 > a.timeout_ns) {
          atomicExch(a.err, 1u);
          break;
        }
      }
    } else if (smem) {
      while ((int32_t)(*smem - smem_v) < 0) {
        if (globaltimer() - t0 > a.timeout_ns) {
          atomicExch(a.err, 1u);
          break;
        }
      }
      __threadfence_block();
    }
  }
  group_sync(bar_id, nt);
}

// Measurement only (DDP_OPT_P2P_DEBUG bit 2 = 4): one thread per CTA records
// %globaltimer at point i (0 entry, 1 stage 0 packed, 2 stage 0 published,
// 3 stage 0 seen from every peer, 4 stage 0 read, 5 last stage read, 6 end) into
// uint64 [kMaxCtas][8] at byte 40 KiB of the lane's flag region (scratch).
__device__ __forceinline__ void trace_point(const P2PLaunch& a, int r, int i, bool who) {
  if ((a.debug & 4) && who)
    reinterpret_cast<uint64_t*>(static_cast<char*>(a.storage[r]) + a.flags_byte_off + 40 * 1024)[blockIdx.x * 8 + i] =
        globaltimer();
}

// Pack the bucket range [lo, hi) from the gradients (x s) into dst[x], by a group.
template <typename T, int MAXS, int U>
__device__ __forceinline__ void grp_pack(const SlotArgs<MAXS>& sa, int64_t lo, int64_t hi, T* dst, float s,
                                         int64_t gstride, int gt, int nt) {
  if (lo >= hi) return;
  for (int k = find_slot(sa, lo); k < sa.n && lo < hi; ++k) {
    const int64_t s0 = sa.off[k], e = min(hi, sa.off[k + 1]);
    if (e <= lo) continue;
    const T* g = reinterpret_cast<const T*>(static_cast<const char*>(sa.grad[k]) + gstride) + (lo - s0);
    T* d[1] = {dst + lo};
    const T* sp[1] = {g};
    grp_xfer<T, 1, 1, true, true, false, U>(d, sp, e - lo, s, gt, nt);
    lo = e;
  }
}

// grad(x) = RNE( sum_{k<NS} src_k[x] ) for x in [lo, hi) (rank order), by a group;
// also written to extra[x] when EXTRA (the two-shot's own shard, in place).
template <typename T, int NS, bool EXTRA, int MAXS>
__device__ __forceinline__ void grp_sum(const SlotArgs<MAXS>& sa, int64_t lo, int64_t hi,
                                        const T* const (&srcb)[NS], T* extra, int64_t gstride, int gt, int nt) {
  if (lo >= hi) return;
  // remote loads are latency-bound: keep ~16 16-B loads in flight per thread
  // (EXTRA, the two-shot's reduce with two destinations: fewer, to stay in 128 registers)
  constexpr int UF = EXTRA ? (NS <= 2 ? 4 : NS <= 4 ? 3 : NS <= 6 ? 2 : 1) : (NS <= 2 ? 8 : NS <= 4 ? 4 : 2);
  for (int k = find_slot(sa, lo); k < sa.n && lo < hi; ++k) {
    const int64_t s0 = sa.off[k], e = min(hi, sa.off[k + 1]);
    if (e <= lo) continue;
    T* g = reinterpret_cast<T*>(static_cast<char*>(sa.grad[k]) + gstride) + (lo - s0);
    const T* sp[NS];
#pragma unroll
    for (int j = 0; j < NS; ++j) sp[j] = srcb[j] + lo;
    if (EXTRA) {
      T* d[2] = {g, extra + lo};
      grp_xfer<T, NS, 2, false, false, false, UF>(d, sp, e - lo, 1.0f, gt, nt);
    } else {
      T* d[1] = {g};
      grp_xfer<T, NS, 1, false, false, false, UF>(d, sp, e - lo, 1.0f, gt, nt);
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
  __shared__ uint32_t packed;  // stages packed by this CTA's pack group
  if (threadIdx.x == 0) packed = 0;
  __syncthreads();
  trace_point(a, r, 0, threadIdx.x == 0);
  auto stage = [&](int k, int64_t& lo, int64_t& hi) {
    lo = min(lo0 + (int64_t)k * a.sub, hi0);
    hi = min(lo + a.sub, hi0);
  };
  const int np = a.pack_threads, nr = kThreads - np;
  if (threadIdx.x < np) {  // P: pack + scale every stage into the own buffer, publish each
    const int gt = threadIdx.x;
#pragma unroll 1
    for (int k = 0; k < K; ++k) {
      int64_t lo, hi;
      stage(k, lo, hi);
      if (!(a.debug & 2)) grp_pack<T, MAXS, 16>(sa, lo, hi, own, a.scale, gstride, gt, np);
      if (k == 0) trace_point(a, r, 1, gt == 0);
      group_publish<W>(a, r, 0, a.seq + (uint32_t)(k + 1), 1, gt, np, &packed, (uint32_t)(k + 1));
      if (k == 0) trace_point(a, r, 2, gt == 0);
    }
  } else {  // R: each stage of every rank's buffer -> rank-order sum -> .grad
    const int gt = threadIdx.x - np;
#pragma unroll 1
    for (int k = 0; k < K; ++k) {
      group_wait<W>(a, r, 0, a.seq + (uint32_t)(k + 1), 2, gt, nr, &packed, (uint32_t)(k + 1));
      if (k == 0) trace_point(a, r, 3, gt == 0);
      int64_t lo, hi;
      stage(k, lo, hi);
      if (!(a.debug & 1)) grp_sum<T, W, false, MAXS>(sa, lo, hi, buf, nullptr, gstride, gt, nr);
      if (k == 0) trace_point(a, r, 4, gt == 0);
    }
    trace_point(a, r, 5, gt == 0);
  }
  __syncthreads();
  trace_point(a, r, 6, threadIdx.x == 0);
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
  __shared__ uint32_t packed;
  if (threadIdx.x == 0) packed = 0;
  __syncthreads();
  trace_point(a, r, 0, threadIdx.x == 0);
  const int np = a.pack_threads, nr = kThreads - np;
  if (threadIdx.x < np) {  // P: pack + scale stage k of chunk c of every shard, publish (kind 0)
    const int gt = threadIdx.x;
#pragma unroll 1
    for (int k = 0; k < K; ++k) {
#pragma unroll 1
      for (int j = 0; j < W; ++j) {
        int64_t lo, hi;
        rng((r + 1 + j) % W, k, lo, hi);  // own shard last: the peers need theirs first
        if (!(a.debug & 2)) grp_pack<T, MAXS, 8>(sa, lo, hi, own, a.scale, gstride, gt, np);
      }
      if (k == 0) trace_point(a, r, 1, gt == 0);
      group_publish<W>(a, r, 0, a.seq + (uint32_t)(k + 1), 1, gt, np, &packed, (uint32_t)(k + 1));
      if (k == 0) trace_point(a, r, 2, gt == 0);
    }
  } else {
    const int gt = threadIdx.x - np;
#pragma unroll 1
    for (int k = 0; k <= K; ++k) {
      if (k < K) {  // R: own shard, stage k: sum over the W buffers -> own buffer + .grad; publish (kind 1)
        group_wait<W>(a, r, 0, a.seq + (uint32_t)(k + 1), 2, gt, nr, &packed, (uint32_t)(k + 1));
        if (k == 0) trace_point(a, r, 3, gt == 0);
        int64_t lo, hi;
        rng(r, k, lo, hi);
        if (!(a.debug & 1)) grp_sum<T, W, true, MAXS>(sa, lo, hi, buf, own, gstride, gt, nr);
        if (k == 0) trace_point(a, r, 4, gt == 0);
        group_publish<W>(a, r, 1, a.seq + (uint32_t)(k + 1), 2, gt, nr, nullptr, 0);
      }
      if (k >= 1) {  // G: every other shard j, stage k-1, from rank j's buffer (its sums) -> .grad
        group_wait<W>(a, r, 1, a.seq + (uint32_t)k, 2, gt, nr, nullptr, 0);
#pragma unroll 1
        for (int i = 1; i < W; ++i) {
          const int j = (r + i) % W;
          int64_t lo, hi;
          rng(j, k - 1, lo, hi);
          const T* src[1] = {buf[j]};
          if (!(a.debug & 1)) grp_sum<T, 1, false, MAXS>(sa, lo, hi, src, nullptr, gstride, gt, nr);
        }
      }
    }
    trace_point(a, r, 5, gt == 0);
  }
  __syncthreads();
  trace_point(a, r, 6, threadIdx.x == 0);
}

// Gradient-as-bucket-view form of the two-shot (DDP_OPT_GRAD_VIEW, §8(f) N-3,
// zero-copy): every rank's gradients ARE its bucket region, so there is no pack
// and no second buffer, and the average is written in place:
//   publish kind 0: this rank's (raw) gradients are final — prior work on the
//      launching stream produced them;
//   R  own shard r, stage k: RNE( sum_q RNE(g_q(x) * fl(1/W)) ) over the W ranks'
//      raw gradients (W-1 read over NVLink), written in place into the own shard
//      (no peer reads the own shard's raw values: in R each rank reads only its
//      own shard); publish kind 1 (stage k summed);
//   G  every other shard j, stage k: rank j's sums -> the own region, once rank j
//      has published kind 1 for the stage, i.e. finished reading this rank's raw
//      shard j;
//   kind 2 at the end: this rank has read every peer's sums; wait for every
//      peer's, so no sum is still being read when the caller's next backward
//      overwrites the gradients.
// Arithmetic = oracle O-3b (each operand x fl(1/W), rank-order fp32 sum, one rounding).
template <typename T, int W>
__global__ void __launch_bounds__(kThreads, 1) pull_view_twoshot_kernel(const __grid_constant__ P2PLaunch a) {
  const int r = a.emulated ? (int)blockIdx.y : a.rank;
  if (a.emulated && r == a.dead_rank) return;
  const int c = blockIdx.x;
  const int64_t L = a.shard, N = a.numel, Q = a.chunk, SUB = a.sub;
  const int K = a.stages;
  auto rng = [&](int j, int k, int64_t& lo, int64_t& hi) {
    const int64_t c0 = (int64_t)c * Q, c1 = min(c0 + Q, L);
    lo = min(j * L + min(c0 + (int64_t)k * SUB, c1), N);
    hi = min(j * L + min(c0 + (int64_t)(k + 1) * SUB, c1), N);
  };
  T* own = at<T>(a.storage[r], a.bucket_byte_off);
  const T* buf[W];
#pragma unroll
  for (int q = 0; q < W; ++q) buf[q] = at<T>(a.storage[q], a.bucket_byte_off);
  const int gt = threadIdx.x, nt = kThreads;
  constexpr int UR = W <= 2 ? 4 : W <= 4 ? 3 : W <= 6 ? 2 : 1;
  group_publish<W>(a, r, 0, a.seq + (uint32_t)K, 0, gt, nt, nullptr, 0);
  group_wait<W>(a, r, 0, a.seq + (uint32_t)K, 0, gt, nt, nullptr, 0);
#pragma unroll 1
  for (int k = 0; k <= K; ++k) {
    if (k < K) {  // R
      int64_t lo, hi;
      rng(r, k, lo, hi);
      if (lo < hi && !(a.debug & 1)) {
        T* d[1] = {own + lo};
        const T* sp[W];
#pragma unroll
        for (int q = 0; q < W; ++q) sp[q] = buf[q] + lo;
        grp_xfer<T, W, 1, false, true, true, UR>(d, sp, hi - lo, a.scale, gt, nt);
      }
      group_publish<W>(a, r, 1, a.seq + (uint32_t)(k + 1), 0, gt, nt, nullptr, 0);
    }
    if (k >= 1) {  // G, stage k-1
      group_wait<W>(a, r, 1, a.seq + (uint32_t)k, 0, gt, nt, nullptr, 0);
#pragma unroll 1
      for (int i = 1; i < W; ++i) {
        const int j = (r + i) % W;
        int64_t lo, hi;
        rng(j, k - 1, lo, hi);
        if (lo >= hi || (a.debug & 1)) continue;
        T* d[1] = {own + lo};
        const T* sp[1] = {buf[j] + lo};
        grp_xfer<T, 1, 1, false, false, false, 8>(d, sp, hi - lo, 1.0f, gt, nt);
      }
    }
  }
  group_publish<W>(a, r, 2, a.seq + 1u, 0, gt, nt, nullptr, 0);
  group_wait<W>(a, r, 2, a.seq + 1u, 0, gt, nt, nullptr, 0);
}

template <typename T>
cudaError_t run_view(const P2PLaunch& a, cudaStream_t st) {
  P2PLaunch pa = a;
  void* args[] = {&pa};
  void* fn = nullptr;
  switch (a.world) {
    case 2: fn = reinterpret_cast<void*>(pull_view_twoshot_kernel<T, 2>); break;
    case 3: fn = reinterpret_cast<void*>(pull_view_twoshot_kernel<T, 3>); break;
    case 4: fn = reinterpret_cast<void*>(pull_view_twoshot_kernel<T, 4>); break;
    case 5: fn = reinterpret_cast<void*>(pull_view_twoshot_kernel<T, 5>); break;
    case 6: fn = reinterpret_cast<void*>(pull_view_twoshot_kernel<T, 6>); break;
    case 7: fn = reinterpret_cast<void*>(pull_view_twoshot_kernel<T, 7>); break;
    case 8: fn = reinterpret_cast<void*>(pull_view_twoshot_kernel<T, 8>); break;
    default: return cudaErrorInvalidValue;
  }
  if (a.emulated) return cudaLaunchCooperativeKernel(fn, dim3(a.ctas, a.world), dim3(kThreads), args, 0, st);
  return cudaLaunchKernel(fn, dim3(a.ctas), dim3(kThreads), args, 0, st);
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
  if (a.view) return dtype == 0 ? run_view<float>(a, s) : run_view<__nv_bfloat16>(a, s);
  return dtype == 0 ? dispatch<float>(algo, sv, a, s) : dispatch<__nv_bfloat16>(algo, sv, a, s);
}

int pull_view_occupancy(int dtype, int world) {
  int blocks = 0;
  void* fn = nullptr;
#define B200DDP_V(WW) \
  case WW: fn = dtype == 0 ? reinterpret_cast<void*>(pull_view_twoshot_kernel<float, WW>) \
                           : reinterpret_cast<void*>(pull_view_twoshot_kernel<__nv_bfloat16, WW>); break;
  switch (world) { B200DDP_V(2) B200DDP_V(3) B200DDP_V(4) B200DDP_V(5) B200DDP_V(6) B200DDP_V(7) B200DDP_V(8) default: return 0; }
#undef B200DDP_V
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, fn, kThreads, 0) != cudaSuccess) return 0;
  return blocks;
}

int pull_occupancy(int algo, int dtype, int world, int n_slots) {
  return dtype == 0 ? occupancy<float>(algo, world, n_slots) : occupancy<__nv_bfloat16>(algo, world, n_slots);
}

}  // namespace b200ddp
