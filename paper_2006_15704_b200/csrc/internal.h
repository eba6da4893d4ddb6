// internal.h — declarations shared by the host core (core/reducer.cpp) and
// the sm_100a kernels (kernels/*.cu).  Not part of the public ABI.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace b200ddp {

constexpr int kMaxWorld = 8;
constexpr int kMaxCtas = 256;                  // rows of the barrier flag table
constexpr int64_t kFlagsBytes = 64 * 1024;     // 2 flag arrays of kMaxCtas * kMaxWorld uint32 + scratch
constexpr int64_t kFlagArrayBytes = kMaxCtas * kMaxWorld * 4;
constexpr int kMaxSlotsPerLaunch = 1024;       // largest by-value slot table
constexpr int64_t kAlignElems = 256;           // shard / chunk granularity (elements)
constexpr int kThreads = 512;                  // threads per CTA for every kernel

// Host view of the slots of one bucket (or of a contiguous run of them).
struct SlotView {
  const int64_t* off;   // n+1 element offsets inside the bucket; off[n] = end
  void* const* grad;    // n gradient pointers (rank-0 pointers in emulation)
  int32_t n;
};

// Per-launch description of a P2P allreduce (one-shot or two-shot).
struct P2PLaunch {
  void* storage[kMaxWorld];   // every rank's symmetric storage base (peer-mapped)
  int64_t flags_byte_off;     // flags: uint32 [2][kMaxCtas][kMaxWorld] = [stage kind][cta][src rank]
  int64_t bucket_byte_off;    // this bucket inside the bucket region
  int64_t stage_byte_off;     // staging region for this launch (parity applied)
  int64_t stage_stride;       // bytes between per-source staging slots
  int64_t numel;              // bucket elements
  int64_t shard;              // two-shot shard length L (elements); unused by one-shot
  int64_t chunk;              // per-CTA chunk Q (elements)
  int64_t sub;                // pipeline sub-chunk (elements); stages = ceil(chunk / sub)
  int32_t stages;
  int32_t world;
  int32_t rank;               // this rank (ignored when emulated: rank = blockIdx.y)
  int32_t ctas;               // gridDim.x
  int32_t emulated;
  uint32_t seq;               // barrier values seq (first) and seq+1 (second)
  float scale;                // fl(1/world)
  int64_t grad_rank_stride;   // emulation: byte distance between ranks' gradients
  uint32_t* err;              // device-visible error word (mapped pinned host memory)
  void* mc;                   // NVLS: multicast address of the storage base (NULL otherwise)
  uint64_t timeout_ns;        // bound of every barrier spin (%globaltimer), then *err = 1
  int32_t dead_rank;          // test support (emulation): this rank returns at once, never signals
  int32_t pull;               // 1: pull kernels (kernels/pull.cu; bucket_byte_off = this pass's buffer)
  int32_t sig_mode;           // pull kernels: how a flag is published (DDP_OPT_P2P_SIGNAL)
  int32_t debug;              // measurement only (DDP_OPT_P2P_DEBUG): 1 skip reads, 2 skip pack
  int32_t pack_threads;       // pull kernels: threads of the pack group (multiple of 32, < kThreads)
  int32_t view;               // pull two-shot in place on the gradients (DDP_OPT_GRAD_VIEW); no slot table
};

// Several buckets launched together at world 1: slot k covers virtual elements
// [off[k], off[k+1]) of the concatenated buckets and packs to storage byte
// offset dst[k].
struct GroupView {
  const int64_t* off;   // n+1 virtual offsets
  void* const* grad;    // n gradient pointers
  const int64_t* dst;   // n bucket byte offsets (inside the storage)
  int32_t n;
};

// dtype: 0 = fp32, 1 = bf16 (ddp_dtype_t).
cudaError_t launch_local(int dtype, const GroupView& gv, void* storage, int max_ctas, cudaStream_t s);
cudaError_t launch_pack(int dtype, const SlotView& sv, void* bucket, float scale, int max_ctas,
                        cudaStream_t s);
cudaError_t launch_unpack(int dtype, const SlotView& sv, const void* bucket, int max_ctas,
                          cudaStream_t s);
cudaError_t launch_p2p(int algo, int dtype, const SlotView& sv, const P2PLaunch& a, cudaStream_t s);
// Pull form of the same two algorithms (kernels/pull.cu): ranks read each other's buffers.
cudaError_t launch_pull(int algo, int dtype, const SlotView& sv, const P2PLaunch& a, cudaStream_t s);
int pull_occupancy(int algo, int dtype, int world, int n_slots);
int pull_view_occupancy(int dtype, int world);
// NVLS (NVSwitch multicast) two-shot: pack -> multimem.ld_reduce + multimem.st -> unpack.
cudaError_t launch_nvls(int dtype, const SlotView& sv, const P2PLaunch& a, cudaStream_t s);
// Copy-engine algorithm, SM part.  A list of gradients with their element
// offsets inside a slot ("wire layout").
struct CeView {
  void* const* grad;
  const int64_t* wire;
  const int64_t* numel;
  int32_t n;
};
// own_slot[wire_k + i] = grad_k[i] (raw) for the listed (small) gradients.
cudaError_t launch_ce_gather(int dtype, const CeView& v, void* own_slot, int max_ctas, cudaStream_t s);
// CE2: dst[i] = RNE(sum_q src_q[i]) in rank order q = 0..world-1 (fp32 accumulate);
// scale != 1: every operand scaled and rounded first, RNE(sum_q RNE(src_q[i] * scale)).
cudaError_t launch_shard_reduce(int dtype, int world, const void* const* src, void* dst, int64_t n, float scale,
                                int max_ctas, cudaStream_t s);
// SM push: every listed gradient (raw) to peer_slots[j] + wire_k, j < npeers.
cudaError_t launch_ce_push(int dtype, const CeView& v, void* const* peer_slots, int npeers, int max_ctas,
                           cudaStream_t s);
// Compressed wire (fp32 gradients, bf16 slots): gather converts RNE_bf16(g * scale);
// reduce sums fp32(v_q) in rank order, v_rank recomputed from .grad, fp32 result.
cudaError_t launch_wire_gather(const CeView& v, void* own_slot, float scale, int max_ctas, cudaStream_t s);
cudaError_t launch_wire_reduce(int world, int rank, const CeView& v, const void* slot0, int64_t stride_bytes,
                               float scale, int max_ctas, cudaStream_t s);
// grad_k[i] = RNE( sum_q RNE(v_q * scale) ), rank order; v_rank = grad_k[i],
// v_q = slot q (slot0 + q * stride_bytes) at wire_k + i.
cudaError_t launch_ce_reduce(int dtype, int world, int rank, const CeView& v, const void* slot0,
                             int64_t stride_bytes, float scale, int max_ctas, cudaStream_t s);
// find_unused bitmap exchange: global[p] = sum_{q<world} slot_q[p] (int32), slot_q =
// slot0 + q * stride_bytes (each rank's local participation bitmap).
cudaError_t launch_bitmap_sum(int world, const void* slot0, int64_t stride_bytes, int32_t* global, int32_t n,
                              cudaStream_t s);
// Locally-unused parameters (find_unused): copy src (library scratch holding the
// average) -> dst (the caller's gradient) where global_used[param] > 0.
struct UnusedView {
  const void* const* src;
  void* const* dst;
  const int32_t* param;
  const int64_t* numel;
  int32_t n;
};
cudaError_t launch_unused_fixup(int dtype, const UnusedView& uv, const int32_t* global_used, int max_ctas,
                                cudaStream_t s);
// Largest number of CTAs per rank an emulated launch of `world` ranks may use.
int emulated_max_ctas(int algo, int dtype, int n_slots, int world, bool pull, bool view = false);

}  // namespace b200ddp
