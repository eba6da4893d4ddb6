// exchange.cpp — device side of the host core: what a launched bucket does
// (Alg. 1: pack into the bucket, AllReduce, copy back),
// per algorithm, on the comm stream / lanes / copy-engine
// streams after the producer streams (overlap), and the
// find_unused bitmap step.  Called from core/reducer.cpp.
#include <algorithm>
#include <cstring>

#include "ctx.h"

namespace b200ddp {

// ---- profiling -------------------------------------------------------------
cudaEvent_t pool_event(ddp_ctx* c) {
  if (!c->event_pool.empty()) {
    cudaEvent_t e = c->event_pool.back();
    c->event_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}
void prof_begin(ddp_ctx* c, int kind, cudaStream_t s) {
  if (!c->profile) return;
  ProfRec r{kind, pool_event(c), pool_event(c), (int)c->prof_ready.size() - 1};
  cudaEventRecord(r.a, s ? s : c->comm);
  c->prof.push_back(r);
}
void prof_end(ddp_ctx* c, cudaStream_t s) {
  if (!c->profile || c->prof.empty()) return;
  cudaEventRecord(c->prof.back().b, s ? s : c->comm);
}

typedef CUresult (*StreamValueFn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);

// ce flags of bucket b in a rank's storage: [0][b][src] ready, [1][b][src] consumed,
// [2][b][src] gathered (CE2), [3][0][src] participation bitmap delivered (find_unused)
uint32_t* ce_flag(const ddp_ctx* c, int r, int kind, int b, int src) {
  return reinterpret_cast<uint32_t*>(static_cast<char*>(c->storage[r]) + c->ce_flags_off) +
         ((size_t)kind * c->buckets.size() + b) * kMaxWorld + src;  // kind < kCeFlagKinds
}

ddp_status_t ce_write(ddp_ctx* c, cudaStream_t s, uint32_t* addr, uint32_t v) {
  // default flags: a memory fence precedes the write (stream-scoped __threadfence_system)
  CUresult r = reinterpret_cast<StreamValueFn>(c->fn_write32)((CUstream)s, (CUdeviceptr)addr, v, 0);
  if (r != CUDA_SUCCESS) return cuda_fail(c, cudaErrorUnknown, "cuStreamWriteValue32");
  if (c->peer_emu) emu_issued(c, addr, v);
  return DDP_OK;
}
// The wait is invisible to the CUDA scheduler.  Across processes each rank issues
// its writes of a step before its waits of that step, so every wait's write is
// enqueued somewhere; with every rank in ONE process (peer emulation) the host
// additionally holds the wait back until the matching write has been issued, so
// streams that share a hardware queue can never hold a wait ahead of its write.
ddp_status_t ce_wait(ddp_ctx* c, cudaStream_t s, uint32_t* addr, uint32_t v) {
  if (c->peer_emu)
    if (ddp_status_t st = emu_await_issue(c, addr, v)) return st;
  CUresult r = reinterpret_cast<StreamValueFn>(c->fn_wait32)((CUstream)s, (CUdeviceptr)addr, v,
                                                              CU_STREAM_WAIT_VALUE_GEQ);
  if (r != CUDA_SUCCESS) return cuda_fail(c, cudaErrorUnknown, "cuStreamWaitValue32");
  return DDP_OK;
}

// Copy-engine one-shot (SM-free exchange).  Rank r's raw gradients go to slot r
// of every peer: large ones by one cudaMemcpyAsync each straight from .grad,
// the small ones gathered (kernel) into r's own slot and sent as one region.
// Stream memory operations order everything, so no SM spins while waiting:
//   comm stream:    [wait: peers consumed pass v-1] -> copies -> ready flags to peers
//   reduce stream:  [wait: own copies issued, peers' ready flags] -> rank-order
//                   reduce x 1/W per operand straight into .grad -> consumed flags
ddp_status_t launch_ce_view(ddp_ctx* c, int b);

// Gradient-as-bucket-view: maximal runs [k0, k1) of the bucket's slots whose
// gradient was handed over somewhere else than its slot in `region`.
std::vector<std::pair<int, int>> alias_runs(const ddp_ctx* c, const Bucket& bk, const char* region) {
  const int n = (int)bk.params.size();
  std::vector<std::pair<int, int>> runs;
  for (int k = 0; k < n;) {
    if (bk.grads[k] == region + bk.off[k] * c->esize) {
      ++k;
      continue;
    }
    int e = k;
    while (e < n && bk.grads[e] != region + bk.off[e] * c->esize) ++e;
    runs.emplace_back(k, e);
    k = e;
  }
  return runs;
}

// raw copies of those runs into the region (before) / back out of it (after)
ddp_status_t copy_runs(ddp_ctx* c, const Bucket& bk, const std::vector<std::pair<int, int>>& runs, char* region,
                       bool in, cudaStream_t s) {
  if (runs.empty()) return DDP_OK;
  prof_begin(c, in ? 0 : 2, s);
  for (auto& q : runs) {
    const SlotView sv{bk.off.data() + q.first, bk.grads.data() + q.first, q.second - q.first};
    if (in) CUDA_TRY(c, launch_pack(c->dtype, sv, region, 1.0f, (int)c->pack_ctas, s));
    else CUDA_TRY(c, launch_unpack(c->dtype, sv, region, (int)c->pack_ctas, s));
  }
  prof_end(c, s);
  return DDP_OK;
}

ddp_status_t launch_ce(ddp_ctx* c, int b) {
  Bucket& bk = c->buckets[b];
  if (c->grad_view) return launch_ce_view(c, b);
  const int W = c->world, r = c->rank;
  char* mine = static_cast<char*>(c->storage[r]);
  char* own_slot = mine + bk.ce_off + r * bk.ce_stride;
  const uint32_t v = ++bk.ce_count;
  const size_t ns = bk.params.size();
  const bool push = bk.algo == DDP_ALGO_PUSH;
  c->ce_grad.clear();
  c->ce_wire.clear();
  c->ce_numel.clear();
  for (size_t k = 0; k < ns && !push; ++k) {
    if (bk.ce_direct[k]) continue;
    c->ce_grad.push_back(bk.grads[k]);
    c->ce_wire.push_back(bk.ce_wire[k]);
    c->ce_numel.push_back(bk.off[k + 1] - bk.off[k]);
  }
  const bool any_small = !c->ce_grad.empty();
  const int64_t we = c->wire_bf16 ? 2 : c->esize;  // wire element bytes
  const float scale = 1.0f / (float)W;
  if (any_small) {  // gather on its own stream so it overlaps the previous bucket's copies
    const CeView gv{c->ce_grad.data(), c->ce_wire.data(), c->ce_numel.data(), (int32_t)c->ce_grad.size()};
    prof_begin(c, 0, c->ce_pack);
    if (c->wire_bf16) CUDA_TRY(c, launch_wire_gather(gv, own_slot, scale, (int)c->pack_ctas, c->ce_pack));
    else CUDA_TRY(c, launch_ce_gather(c->dtype, gv, own_slot, (int)c->pack_ctas, c->ce_pack));
    prof_end(c, c->ce_pack);
    CUDA_TRY(c, cudaEventRecord(c->ce_packed[b], c->ce_pack));
  }
  // reuse guard: every peer has consumed (reduced) its slot r of this bucket from pass v-1
  if (v > 1)
    for (int i = 1; i < W; ++i)
      if (ddp_status_t st = ce_wait(c, c->comm, ce_flag(c, r, 1, b, (r + i) % W), v - 1)) return st;
  prof_begin(c, 4);
  if (push) {  // SM push: one kernel reads each gradient once and stores it into every peer
    void* peers[kMaxWorld];
    for (int i = 1; i < W; ++i)
      peers[i - 1] = static_cast<char*>(c->storage[(r + i) % W]) + bk.ce_off + r * bk.ce_stride;
    c->ce_grad.assign(bk.grads.begin(), bk.grads.end());
    c->ce_wire.assign(bk.ce_wire.begin(), bk.ce_wire.end());
    for (size_t k = 0; k < ns; ++k) c->ce_numel.push_back(bk.off[k + 1] - bk.off[k]);
    const CeView pv{c->ce_grad.data(), c->ce_wire.data(), c->ce_numel.data(), (int32_t)ns};
    CUDA_TRY(c, launch_ce_push(c->dtype, pv, peers, W - 1, (int)std::min<int64_t>(c->comm_ctas, 148), c->comm));
  } else {
    // copy engines: the large gradients straight from .grad first (they do not wait
    // for the gather), then the gathered region of the small ones
    for (int i = 1; i < W; ++i) {
      char* dst = static_cast<char*>(c->storage[(r + i) % W]) + bk.ce_off + r * bk.ce_stride;
      for (size_t k = 0; k < ns; ++k)
        if (bk.ce_direct[k])
          CUDA_TRY(c, cudaMemcpyAsync(dst + bk.ce_wire[k] * c->esize, bk.grads[k],
                                      (size_t)((bk.off[k + 1] - bk.off[k]) * c->esize), cudaMemcpyDeviceToDevice,
                                      c->comm));
    }
    if (any_small) {
      CUDA_TRY(c, cudaStreamWaitEvent(c->comm, c->ce_packed[b], 0));
      for (int i = 1; i < W; ++i) {
        char* dst = static_cast<char*>(c->storage[(r + i) % W]) + bk.ce_off + r * bk.ce_stride;
        CUDA_TRY(c, cudaMemcpyAsync(dst + bk.ce_small0 * we, own_slot + bk.ce_small0 * we,
                                    (size_t)((bk.ce_wire_numel - bk.ce_small0) * we), cudaMemcpyDeviceToDevice,
                                    c->comm));
      }
    }
  }
  prof_end(c);
  for (int i = 1; i < W; ++i) {
    const int j = (r + i) % W;
    if (ddp_status_t st = ce_write(c, c->comm, ce_flag(c, j, 0, b, r), v)) return st;
  }
  // the reduction overwrites .grad, which the copies above read: order after them
  CUDA_TRY(c, cudaEventRecord(c->ce_copied[b], c->comm));
  CUDA_TRY(c, cudaStreamWaitEvent(c->ce_red, c->ce_copied[b], 0));
  for (int i = 1; i < W; ++i)
    if (ddp_status_t st = ce_wait(c, c->ce_red, ce_flag(c, r, 0, b, (r + i) % W), v)) return st;
  c->ce_grad.assign(bk.grads.begin(), bk.grads.end());
  c->ce_wire.assign(bk.ce_wire.begin(), bk.ce_wire.end());
  c->ce_numel.clear();
  for (size_t k = 0; k < ns; ++k) c->ce_numel.push_back(bk.off[k + 1] - bk.off[k]);
  const CeView rv{c->ce_grad.data(), c->ce_wire.data(), c->ce_numel.data(), (int32_t)ns};
  prof_begin(c, 5, c->ce_red);
  if (c->wire_bf16)
    CUDA_TRY(c, launch_wire_reduce(W, r, rv, mine + bk.ce_off, bk.ce_stride, scale, (int)c->pack_ctas, c->ce_red));
  else
    CUDA_TRY(c, launch_ce_reduce(c->dtype, W, r, rv, mine + bk.ce_off, bk.ce_stride, scale, (int)c->pack_ctas,
                                 c->ce_red));
  prof_end(c, c->ce_red);
  for (int i = 1; i < W; ++i) {
    const int j = (r + i) % W;
    if (ddp_status_t st = ce_write(c, c->ce_red, ce_flag(c, j, 1, b, r), v)) return st;
  }
  c->ce_used = true;
  return DDP_OK;
}

// Copy-engine one-shot with gradient-as-bucket-view (N-3 zero-copy): the
// gradients are the bucket region, so the gather disappears, the whole region
// travels as ONE copy per peer into slot r (wire layout = bucket layout) and
// the rank-order reduce (x 1/W per operand, O-3b) writes back into the region
// as one flat range.  Gradients handed over elsewhere are packed raw into the
// region first (comm stream) and unpacked after the reduce (reduce stream).
// Ordering as launch_ce: consumed flags guard slot reuse, ready flags the
// reduce, and the reduce follows this rank's own copies out of the region.
ddp_status_t launch_ce_view(ddp_ctx* c, int b) {
  Bucket& bk = c->buckets[b];
  const int W = c->world, r = c->rank;
  char* mine = static_cast<char*>(c->storage[r]);
  char* region = mine + bk.byte_off;
  const uint32_t v = ++bk.ce_count;
  const auto runs = alias_runs(c, bk, region);
  if (ddp_status_t st = copy_runs(c, bk, runs, region, true, c->comm)) return st;
  if (v > 1)
    for (int i = 1; i < W; ++i)
      if (ddp_status_t st = ce_wait(c, c->comm, ce_flag(c, r, 1, b, (r + i) % W), v - 1)) return st;
  prof_begin(c, 4);
  for (int i = 1; i < W; ++i) {
    char* dst = static_cast<char*>(c->storage[(r + i) % W]) + bk.ce_off + r * bk.ce_stride;
    CUDA_TRY(c, cudaMemcpyAsync(dst, region, (size_t)(bk.numel * c->esize), cudaMemcpyDeviceToDevice, c->comm));
  }
  prof_end(c);
  for (int i = 1; i < W; ++i)
    if (ddp_status_t st = ce_write(c, c->comm, ce_flag(c, (r + i) % W, 0, b, r), v)) return st;
  CUDA_TRY(c, cudaEventRecord(c->ce_copied[b], c->comm));
  CUDA_TRY(c, cudaStreamWaitEvent(c->ce_red, c->ce_copied[b], 0));
  for (int i = 1; i < W; ++i)
    if (ddp_status_t st = ce_wait(c, c->ce_red, ce_flag(c, r, 0, b, (r + i) % W), v)) return st;
  void* flat[1] = {region};
  const int64_t wire0[1] = {0}, numel[1] = {bk.numel};
  const CeView rv{flat, wire0, numel, 1};
  prof_begin(c, 5, c->ce_red);
  CUDA_TRY(c, launch_ce_reduce(c->dtype, W, r, rv, mine + bk.ce_off, bk.ce_stride, 1.0f / (float)W,
                               (int)c->pack_ctas, c->ce_red));
  prof_end(c, c->ce_red);
  for (int i = 1; i < W; ++i)
    if (ddp_status_t st = ce_write(c, c->ce_red, ce_flag(c, (r + i) % W, 1, b, r), v)) return st;
  if (ddp_status_t st = copy_runs(c, bk, runs, region, false, c->ce_red)) return st;
  c->ce_used = true;
  return DDP_OK;
}

// Copy-engine two-shot (CE2): the reduce-scatter and all-gather of a ring /
// two-shot, 2 (W-1)/W S NVLink bytes per direction, moved by copy engines and
// ordered by stream memory operations (no SM waits):
//   pack stream:    pack x 1/W into the own bucket
//   comm stream:    shard j of the own bucket -> peer j's staging slot r (half v%2);
//                   ready flags
//   reduce stream:  [wait all ready] own shard = rank-order sum of the W values
//                   (slot q, own bucket for q = r), in place in the own bucket
//   all-gather:     [after the reduce] own shard -> shard r of every peer's bucket;
//                   gathered flags
//   unpack stream:  [wait all gathered] own bucket -> .grad
// Staging is double-buffered by pass parity, so no "consumed" flags are needed:
// writing half v%2 again (pass v+2) follows, through this rank's own finalize,
// every peer's all-gather of pass v+1, which follows its reduce of pass v.
ddp_status_t launch_ce2(ddp_ctx* c, int b, const SlotView& sv, float scale) {
  Bucket& bk = c->buckets[b];
  const int W = c->world, r = c->rank;
  const uint32_t v = ++bk.ce_count;
  char* mine = static_cast<char*>(c->storage[r]);
  char* own = mine + bk.byte_off;
  const int64_t L = bk.shard, e = c->esize;
  const int64_t half = (int64_t)(v & 1) * W * bk.ce_stride;
  auto shard_len = [&](int j) { return std::max<int64_t>(0, std::min<int64_t>(L, bk.numel - j * L)); };
  // gradient-as-bucket-view: the gradients are the bucket region, so no pack /
  // unpack (only raw copies for gradients handed over elsewhere); the reduce
  // scales every operand instead (O-3b).  The all-gather from peer j writes
  // only shard j, which this rank's reduce-scatter copy has already sent to j.
  const bool view = c->grad_view != 0;
  const auto runs = view ? alias_runs(c, bk, own) : std::vector<std::pair<int, int>>();
  if (view) {
    if (ddp_status_t st = copy_runs(c, bk, runs, own, true, c->ce_pack)) return st;
  } else {
    prof_begin(c, 0, c->ce_pack);
    CUDA_TRY(c, launch_pack(c->dtype, sv, own, scale, (int)c->pack_ctas, c->ce_pack));
    prof_end(c, c->ce_pack);
  }
  CUDA_TRY(c, cudaEventRecord(c->ce_packed[b], c->ce_pack));
  // reduce-scatter on the CE2 copy stream(s); each transfer is followed by its peer's flag
  const size_t nst = c->ce2_rs.size();
  for (int i = 1; i < W; ++i) {
    const int j = (r + i) % W;
    cudaStream_t q = c->ce2_rs[(i - 1) % nst];
    if ((size_t)(i - 1) < nst) CUDA_TRY(c, cudaStreamWaitEvent(q, c->ce_packed[b], 0));  // once per stream
    prof_begin(c, 4, q);
    if (shard_len(j) > 0)
      CUDA_TRY(c, cudaMemcpyAsync(static_cast<char*>(c->storage[j]) + bk.ce_off + half + r * bk.ce_stride,
                                  own + j * L * e, (size_t)(shard_len(j) * e), cudaMemcpyDeviceToDevice, q));
    prof_end(c, q);
    if (ddp_status_t st = ce_write(c, q, ce_flag(c, j, 0, b, r), v)) return st;
  }
  // reduce own shard r in rank order
  CUDA_TRY(c, cudaStreamWaitEvent(c->ce_red, c->ce_packed[b], 0));
  for (int i = 1; i < W; ++i)
    if (ddp_status_t st = ce_wait(c, c->ce_red, ce_flag(c, r, 0, b, (r + i) % W), v)) return st;
  const void* src[kMaxWorld];
  for (int q = 0; q < W; ++q)
    src[q] = q == r ? static_cast<const void*>(own + r * L * e)
                    : static_cast<const void*>(mine + bk.ce_off + half + q * bk.ce_stride);
  prof_begin(c, 5, c->ce_red);
  CUDA_TRY(c, launch_shard_reduce(c->dtype, W, src, own + r * L * e, shard_len(r), view ? scale : 1.0f,
                                  (int)c->pack_ctas, c->ce_red));
  prof_end(c, c->ce_red);
  CUDA_TRY(c, cudaEventRecord(c->ce_reduced[b], c->ce_red));
  // all-gather the reduced own shard into every peer's bucket
  for (int i = 1; i < W; ++i) {
    const int j = (r + i) % W;
    cudaStream_t q = c->ce2_ag[(i - 1) % nst];
    if ((size_t)(i - 1) < nst) CUDA_TRY(c, cudaStreamWaitEvent(q, c->ce_reduced[b], 0));
    prof_begin(c, 4, q);
    if (shard_len(r) > 0)
      CUDA_TRY(c, cudaMemcpyAsync(static_cast<char*>(c->storage[j]) + bk.byte_off + r * L * e, own + r * L * e,
                                  (size_t)(shard_len(r) * e), cudaMemcpyDeviceToDevice, q));
    prof_end(c, q);
    if (ddp_status_t st = ce_write(c, q, ce_flag(c, j, 2, b, r), v)) return st;
  }
  // unpack once every shard has arrived
  CUDA_TRY(c, cudaStreamWaitEvent(c->ce_up, c->ce_reduced[b], 0));
  for (int i = 1; i < W; ++i)
    if (ddp_status_t st = ce_wait(c, c->ce_up, ce_flag(c, r, 2, b, (r + i) % W), v)) return st;
  if (view) {
    if (ddp_status_t st = copy_runs(c, bk, runs, own, false, c->ce_up)) return st;
  } else {
    prof_begin(c, 2, c->ce_up);
    CUDA_TRY(c, launch_unpack(c->dtype, sv, own, (int)c->pack_ctas, c->ce_up));
    prof_end(c, c->ce_up);
  }
  c->ce2_used = true;
  return DDP_OK;
}

// Gradient-as-bucket-view (N-3, zero-copy): the gradients normally ARE the
// bucket's slots, so pack (Alg. 1) and the copy back (L246) vanish and
// the bucket is averaged in place: ncclAvg multiplies every operand by fl(1/W)
// before summing (oracle O-3b up to NCCL's summation order).  A gradient handed
// over at another address (e.g. .grad re-created after zero_grad(set_to_none))
// is copied raw into its slot first and the average copied back after, per
// maximal run of such slots.
ddp_status_t launch_nccl_view(ddp_ctx* c, const Bucket& bk, char* buf, ncclComm_t comm, cudaStream_t s) {
  const auto runs = alias_runs(c, bk, buf);
  if (ddp_status_t st = copy_runs(c, bk, runs, buf, true, s)) return st;
  prof_begin(c, 1, s);
  NCCL_TRY(c, ncclAllReduce(buf, buf, (size_t)bk.numel, c->dtype == DDP_FP32 ? ncclFloat32 : ncclBfloat16,
                            ncclAvg, comm, s));
  prof_end(c, s);
  return copy_runs(c, bk, runs, buf, false, s);
}

// ---- a3/a4/a6 device work for one bucket -------------------------------------
ddp_status_t launch_device(ddp_ctx* c, int b) {
  Bucket& bk = c->buckets[b];
  const SlotView sv{bk.off.data(), bk.grads.data(), (int32_t)bk.params.size()};
  const float scale = 1.0f / (float)c->world;  // fl(1/W), reading C-2
  char* mine = static_cast<char*>(c->storage[c->rank]);
  if (bk.algo == DDP_ALGO_CE || bk.algo == DDP_ALGO_PUSH) return launch_ce(c, b);
  if (bk.algo == DDP_ALGO_CE2) return launch_ce2(c, b, sv, scale);
  if (bk.algo == DDP_ALGO_NCCL) {
    void* buf = mine + bk.byte_off;
    const size_t k = c->rr_comm.empty() ? 0 : (size_t)b % c->rr_comm.size();
    cudaStream_t s = k == 0 ? c->comm : c->rr_stream[k];
    ncclComm_t comm = k == 0 ? c->nccl : c->rr_comm[k];
    if (k) c->rr_used[k] = 1;
    if (c->grad_view) return launch_nccl_view(c, bk, static_cast<char*>(buf), comm, s);
    prof_begin(c, 0, s);
    CUDA_TRY(c, launch_pack(c->dtype, sv, buf, scale, (int)c->pack_ctas, s));
    prof_end(c, s);
    prof_begin(c, 1, s);
    NCCL_TRY(c, ncclAllReduce(buf, buf, (size_t)bk.numel, c->dtype == DDP_FP32 ? ncclFloat32 : ncclBfloat16,
                              ncclSum, comm, s));
    prof_end(c, s);
    prof_begin(c, 2, s);
    CUDA_TRY(c, launch_unpack(c->dtype, sv, buf, (int)c->pack_ctas, s));
    prof_end(c, s);
    return DDP_OK;
  }
  // lane: its stream, flag table, sequence and staging (identical choice on every rank)
  const int nl = lanes_in_use(c);
  const int ln = (c->emulated || c->world == 1) ? 0 : b % nl;
  cudaStream_t ls = ln == 0 ? c->comm : c->lane_stream[ln];
  if (ln) c->lane_used[ln] = true;
  const bool last = b == (int)c->buckets.size() - 1 && c->world > 1 && !c->emulated;
  // The last bucket holds the first-registered parameters: its ready signal is the
  // end of backward, so nothing is left to overlap with.  Launched from that signal
  // it runs on the PRODUCER stream itself, after every library stream has been
  // joined into it: the pass then ends on the producer stream, and the two
  // cross-stream hops (producer -> comm, comm -> producer) of its sync disappear.
  const bool on_producer = last && c->last_on_producer && c->from_signal && c->producer && !c->find_unused;
  if (c->lone_last && !on_producer) return fail(DDP_ERR_STATE, "internal: lone last bucket off its producer");
  auto join = [&](cudaStream_t q, cudaStream_t into, size_t& k) -> ddp_status_t {
    if (!q || q == into) return DDP_OK;
    if (k >= c->join_ev.size()) return fail(DDP_ERR_STATE, "join event pool exhausted");
    CUDA_TRY(c, cudaEventRecord(c->join_ev[k], q));
    CUDA_TRY(c, cudaStreamWaitEvent(into, c->join_ev[k++], 0));
    return DDP_OK;
  };
  size_t nj = 0;
  if (on_producer) ls = c->producer;
  if (last && !c->lone_last) {
    // The last bucket's kernel uses every SM (max_ctas_for) and spins until the
    // peers arrive.  Everything this rank launched before it must be finished
    // first: the other lanes' spinning kernels (so all of its CTAs can be
    // resident), and the copy-engine paths' kernels of earlier buckets (else
    // they would wait for SMs behind a kernel that waits for peers — measured
    // as a 0.8 ms stall at W=4, profiles/r01_n4.md).
    for (int k = 0; k < nl; ++k) {
      cudaStream_t ks = k == 0 ? c->comm : c->lane_stream[k];
      if (ks == ls && !on_producer) continue;
      if (ddp_status_t st = join(ks, ls, nj)) return st;
    }
    for (cudaStream_t ks : {c->ce_pack, c->ce_red, c->ce_up})
      if (ddp_status_t st = join(ks, ls, nj)) return st;
    if (!on_producer && ln != 0 && c->ce_used)  // CE copies run on the comm stream
      if (ddp_status_t st = join(c->comm, ls, nj)) return st;
  }
  P2PLaunch a{};
  for (int r = 0; r < c->world; ++r) a.storage[r] = c->storage[r];
  a.flags_byte_off = c->flags_off + ln * kFlagsBytes;
  a.bucket_byte_off = bk.byte_off;
  a.pull = bk.pull ? 1 : 0;
  a.view = c->grad_view && bk.algo == DDP_ALGO_TWOSHOT && c->world > 1 ? 1 : 0;
  if (a.view) {  // in place on the gradients (they are the bucket region)
    a.stage_byte_off = 0;
    a.stage_stride = 0;
  } else if (a.pull) {  // this pass's buffer of the bucket (pass parity, identical on every rank)
    a.bucket_byte_off = (bk.p2p_count++ & 1) ? bk.alt_off : bk.byte_off;
    a.stage_byte_off = 0;
    a.stage_stride = 0;
  } else if (bk.algo == DDP_ALGO_TWOSHOT) {
    a.stage_byte_off = c->stage2_off + ln * c->world * c->stage2_stride;
    a.stage_stride = c->stage2_stride;
  } else if (c->world == 1) {
    a.stage_byte_off = bk.byte_off;  // world 1 packs straight into the bucket
    a.stage_stride = 0;
  } else {
    a.stage_byte_off = c->stage1_off + (int64_t)(2 * ln + (c->p2p_launches[ln] & 1)) * c->world * c->stage1_stride;
    a.stage_stride = c->stage1_stride;
  }
  a.numel = bk.numel;
  a.shard = bk.shard;
  a.chunk = bk.chunk;
  a.world = c->world;
  a.rank = c->rank;
  a.ctas = bk.ctas;
  a.emulated = c->emulated ? 1 : 0;
  a.sub = bk.sub;
  a.stages = bk.stages;
  a.seq = c->p2p_seq[ln];
  a.scale = scale;
  a.grad_rank_stride = c->grad_rank_stride;
  a.err = c->err_dev;
  a.mc = c->mc;
  a.timeout_ns = (uint64_t)c->p2p_timeout_ms * 1000000ull;
  a.dead_rank = (int32_t)c->emu_dead_rank;
  a.sig_mode = (int32_t)c->p2p_signal;
  a.pack_threads = bk.ctas >= 96 ? kThreads / 4 : kThreads / 2;
  a.debug = (int32_t)c->p2p_debug;
  c->p2p_seq[ln] += (uint32_t)bk.stages + 2;  // flag values used: seq .. seq + stages + 1
  c->p2p_launches[ln] += 1;
  // gradient-as-bucket-view: gradients handed over elsewhere are copied raw into
  // their slots first and back after (on the launching stream, in order)
  const auto runs = a.view ? alias_runs(c, bk, mine + bk.byte_off) : std::vector<std::pair<int, int>>();
  if (ddp_status_t st = copy_runs(c, bk, runs, mine + bk.byte_off, true, ls)) return st;
  prof_begin(c, 3, ls);
  if (c->peer_emu) {  // the ranks meet on the host; one cooperative kernel runs them all
    if (ddp_status_t st = emu_p2p_launch(c, bk.algo, sv, a, ls, ln)) return st;
  } else if (bk.algo == DDP_ALGO_NVLS) {
    CUDA_TRY(c, launch_nvls(c->dtype, sv, a, ls));
  } else {
    CUDA_TRY(c, launch_p2p(bk.algo, c->dtype, sv, a, ls));
  }
  prof_end(c, ls);
  if (ddp_status_t st = copy_runs(c, bk, runs, mine + bk.byte_off, false, ls)) return st;
  if (on_producer && !c->lone_last) {  // the copy-only streams join after the kernel (they hold no SMs)
    for (cudaStream_t ks : {c->ce_ag})
      if (ddp_status_t st = join(ks, ls, nj)) return st;
    for (cudaStream_t ks : c->ce2_rs)
      if (ddp_status_t st = join(ks, ls, nj)) return st;
    for (cudaStream_t ks : c->ce2_ag)
      if (ddp_status_t st = join(ks, ls, nj)) return st;
    for (size_t k = 1; k < c->rr_stream.size(); ++k)
      if (ddp_status_t st = join(c->rr_stream[k], ls, nj)) return st;
  }
  if (on_producer) c->last_on = ls;
  return DDP_OK;
}

// World 1: buckets [b0, b1) launched by one call run as ONE fused kernel over
// the concatenation of their slots (pack into each bucket, 1-rank reduce and
// unpack from registers); the values equal per-bucket launches bit for bit.
ddp_status_t launch_local_group(ddp_ctx* c, int b0, int b1) {
  c->g_off.clear();
  c->g_grad.clear();
  c->g_dst.clear();
  int64_t base = 0;
  for (int b = b0; b < b1; ++b) {
    const Bucket& bk = c->buckets[b];
    for (size_t s = 0; s < bk.params.size(); ++s) {
      c->g_off.push_back(base + bk.off[s]);
      c->g_grad.push_back(bk.grads[s]);
      c->g_dst.push_back(bk.byte_off + bk.off[s] * c->esize);
    }
    base += bk.numel;
  }
  c->g_off.push_back(base);
  const GroupView gv{c->g_off.data(), c->g_grad.data(), c->g_dst.data(), (int32_t)c->g_grad.size()};
  prof_begin(c, 3);
  CUDA_TRY(c, launch_local(c->dtype, gv, c->storage[c->rank], (int)c->pack_ctas, c->comm));
  prof_end(c);
  return DDP_OK;
}

ddp_status_t device_range(ddp_ctx* c, int b0, int b1);

ddp_status_t device_range(ddp_ctx* c, int b0, int b1) {
  if (b0 >= b1) return DDP_OK;
  if (c->profile) {  // when the producer reached this launch point (timeline "ready")
    cudaEvent_t ev = pool_event(c);
    CUDA_TRY(c, cudaEventRecord(ev, c->unwaited.empty() ? c->comm : c->unwaited.front()));
    c->prof_ready.push_back(ev);
  }
  // A pass whose first device work is the last bucket alone (a one-bucket model,
  // or every other bucket synced earlier... i.e. nothing else launched) runs that
  // bucket on its producer stream with no cross-stream hop at all (launch_device):
  // the producer only has to follow the previous pass's end.
  const Bucket& lb = c->buckets.back();
  c->lone_last = !c->pass_launched && b0 == (int)c->buckets.size() - 1 && b1 == (int)c->buckets.size() &&
                 c->world > 1 && !c->emulated && c->last_on_producer && c->from_signal && c->producer &&
                 !c->find_unused &&
                 (lb.algo == DDP_ALGO_ONESHOT || lb.algo == DDP_ALGO_TWOSHOT || lb.algo == DDP_ALGO_NVLS);
  if (c->lone_last) {
    c->pass_launched = true;
    c->unwaited.clear();
    if (c->comm_done_valid && c->done_stream != c->producer)
      CUDA_TRY(c, cudaStreamWaitEvent(c->producer, c->comm_done, 0));
  }
  // comm stream waits for everything the producers enqueued so far
  for (cudaStream_t s : c->unwaited) {
    cudaEvent_t ev = nullptr;
    for (auto& se : c->stream_events)
      if (se.first == s) ev = se.second;
    if (!ev) {
      CUDA_TRY(c, cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
      c->stream_events.emplace_back(s, ev);
    }
    CUDA_TRY(c, cudaEventRecord(ev, s));
    CUDA_TRY(c, cudaStreamWaitEvent(c->comm, ev, 0));
    if (c->ce_pack) CUDA_TRY(c, cudaStreamWaitEvent(c->ce_pack, ev, 0));
    if (c->ce_up) CUDA_TRY(c, cudaStreamWaitEvent(c->ce_up, ev, 0));  // unpack writes .grad
    for (size_t k = 1; k < c->rr_stream.size(); ++k) CUDA_TRY(c, cudaStreamWaitEvent(c->rr_stream[k], ev, 0));
    for (int k = 1; k < kMaxLanes; ++k)
      if (c->lane_stream[k]) CUDA_TRY(c, cudaStreamWaitEvent(c->lane_stream[k], ev, 0));
    for (cudaStream_t q : c->ce2_rs) CUDA_TRY(c, cudaStreamWaitEvent(q, ev, 0));
  }
  c->unwaited.clear();
  if (!c->pass_launched) {
    // first launch of a pass: the library's side streams reuse staging / slots /
    // flags the previous pass used, so order them after that pass's end even if
    // the caller's producer stream is not ordered after its consumer stream
    c->pass_launched = true;
    if (c->comm_done_valid) {
      for (cudaStream_t q : {c->comm, c->ce_pack, c->ce_red, c->ce_up, c->ce_ag})
        if (q) CUDA_TRY(c, cudaStreamWaitEvent(q, c->comm_done, 0));
      for (cudaStream_t q : c->ce2_rs) CUDA_TRY(c, cudaStreamWaitEvent(q, c->comm_done, 0));
      for (cudaStream_t q : c->ce2_ag) CUDA_TRY(c, cudaStreamWaitEvent(q, c->comm_done, 0));
      for (int k = 1; k < kMaxLanes; ++k)
        if (c->lane_stream[k]) CUDA_TRY(c, cudaStreamWaitEvent(c->lane_stream[k], c->comm_done, 0));
      for (size_t k = 1; k < c->rr_stream.size(); ++k) CUDA_TRY(c, cudaStreamWaitEvent(c->rr_stream[k], c->comm_done, 0));
    }
  }
  if (c->world == 1 && !c->emulated) {
    // group maximal runs of world-1 fused buckets (slot table <= kMaxSlotsPerLaunch)
    int b = b0;
    while (b < b1) {
      if (c->buckets[b].algo != DDP_ALGO_ONESHOT) {
        if (ddp_status_t st = launch_device(c, b)) return st;
        ++b;
        continue;
      }
      int e = b;
      size_t slots = 0;
      while (e < b1 && c->buckets[e].algo == DDP_ALGO_ONESHOT &&
             slots + c->buckets[e].params.size() <= (size_t)kMaxSlotsPerLaunch)
        slots += c->buckets[e++].params.size();
      if (ddp_status_t st = launch_local_group(c, b, e)) return st;
      b = e;
    }
    return DDP_OK;
  }
  for (int b = b0; b < b1; ++b)
    if (ddp_status_t st = launch_device(c, b)) return st;
  return DDP_OK;
}

// find_unused, end of a synced pass: the local participation bitmap
// (pinned host -> own slot, non-blocking) is sent to slot r of every peer by the
// copy engines (one transfer per peer, then a ready flag; double-buffered by pass
// parity), the W slots are summed once every peer's flag has arrived (ONE extra
// "allreduce" of the bitmap after every bucket, on the comm stream), the
// locally-unused parameters that some rank used get their average, and the
// summed bitmap goes back to the host for ddp_global_unused.  Then the local
// bitmap restarts (next synced window).  Slot reuse: writing half v%2 again (pass
// v+2) follows this rank's wait for the peer's pass-(v+1) flag, which the peer
// wrote on its comm stream after its pass-v sum.
ddp_status_t finish_unused(ddp_ctx* c) {
  const int32_t n = (int32_t)c->numel.size();
  const int W = c->world, r = c->rank;
  if (c->bitmap_valid) CUDA_TRY(c, cudaEventSynchronize(c->bitmap_done));  // host buffers reusable
  for (int32_t p = 0; p < n; ++p) c->bitmap_host[p] = c->used_local[p];
  char* mine = static_cast<char*>(c->storage[r]);
  int32_t* global = reinterpret_cast<int32_t*>(mine + c->global_off);
  if (W == 1) {
    CUDA_TRY(c, cudaMemcpyAsync(global, c->bitmap_host, (size_t)n * 4, cudaMemcpyHostToDevice, c->comm));
  } else {
    const uint32_t v = ++c->un_count;
    const int64_t half = (int64_t)(v & 1) * W * c->bitmap_stride;
    char* own = mine + c->bitmap_off + half + r * c->bitmap_stride;
    CUDA_TRY(c, cudaMemcpyAsync(own, c->bitmap_host, (size_t)n * 4, cudaMemcpyHostToDevice, c->comm));
    for (int i = 1; i < W; ++i) {
      const int j = (r + i) % W;
      char* dst = static_cast<char*>(c->storage[j]) + c->bitmap_off + half + r * c->bitmap_stride;
      CUDA_TRY(c, cudaMemcpyAsync(dst, own, (size_t)n * 4, cudaMemcpyDeviceToDevice, c->comm));
      if (ddp_status_t st = ce_write(c, c->comm, ce_flag(c, j, 3, 0, r), v)) return st;
    }
    for (int i = 1; i < W; ++i)
      if (ddp_status_t st = ce_wait(c, c->comm, ce_flag(c, r, 3, 0, (r + i) % W), v)) return st;
    CUDA_TRY(c, launch_bitmap_sum(W, mine + c->bitmap_off + half, c->bitmap_stride, global, n, c->comm));
  }
  std::vector<const void*> src;
  std::vector<void*> dst;
  std::vector<int32_t> prm;
  std::vector<int64_t> cnt;
  for (size_t k = 0; k < c->un_param.size(); ++k) {
    if (!c->un_dst[k]) continue;  // no gradient buffer: nothing to write back
    src.push_back(c->un_src[k]);
    dst.push_back(c->un_dst[k]);
    prm.push_back(c->un_param[k]);
    cnt.push_back(c->un_numel[k]);
  }
  const UnusedView uv{src.data(), dst.data(), prm.data(), cnt.data(), (int32_t)src.size()};
  CUDA_TRY(c, launch_unused_fixup(c->dtype, uv, global, (int)c->pack_ctas, c->comm));
  CUDA_TRY(c, cudaMemcpyAsync(c->global_host, global, (size_t)n * 4, cudaMemcpyDeviceToHost, c->comm));
  CUDA_TRY(c, cudaEventRecord(c->bitmap_done, c->comm));
  c->bitmap_valid = true;
  std::fill(c->used_local.begin(), c->used_local.end(), 0);
  return DDP_OK;
}

}  // namespace b200ddp
