// reducer.cpp — host core of the B200-native DDP Reducer (C ABI in
// include/b200ddp.h).  Plays the role of the paper's reducer.cpp (PAPER.md
// §4.2): parameter-to-bucket map (a1), per-gradient ready tracking
// — the autograd-hook entry point — and in-order bucket launch (a2), finalize,
// no_sync (a7), unused parameters (N-1), options and introspection.  The device
// work of a launched bucket (a3-a6) is in exchange.cpp; the shared state in
// ctx.h.  The per-bucket algorithm is a deterministic function of bucket bytes
// and options, so it is identical on every rank (same order and
// content on all ranks).
#include <cuda.h>
#include <nccl.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <new>
#include <string>
#include <utility>
#include <vector>

#include "b200ddp_emu.h"
#include "ctx.h"

namespace b200ddp {

namespace {
thread_local std::string g_err;
}  // namespace

ddp_status_t fail(ddp_status_t st, const std::string& msg) {
  g_err = msg;
  return st;
}

ddp_status_t cuda_fail(ddp_ctx* c, cudaError_t e, const char* what) {
  if (c) c->poisoned = true;
  return fail(DDP_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
ddp_status_t nccl_fail(ddp_ctx* c, ncclResult_t r, const char* what) {
  if (c) c->poisoned = true;
  return fail(DDP_ERR_NCCL, std::string(what) + ": " + ncclGetErrorString(r));
}

// The previous pass's end event has completed (or failed: the caller's next
// check reports that).  cudaErrorNotReady is cleared, not left for the caller.
static bool pass_complete(ddp_ctx* c) {
  if (cudaEventQuery(c->comm_done) != cudaErrorNotReady) return true;
  (void)cudaGetLastError();
  return false;
}

}  // namespace b200ddp

namespace {

// ---- a1: bucket assignment (readings C-1, C-6) ----
void assign(ddp_ctx* c) {
  const int n = (int)c->numel.size();
  c->buckets.clear();
  Bucket cur;
  for (int i = 0; i < n; ++i) {
    const int p = c->scan[i];
    if (!cur.params.empty() && (cur.numel + c->numel[p]) * c->esize > c->cap) {
      c->buckets.push_back(std::move(cur));
      cur = Bucket();
    }
    cur.params.push_back(p);
    cur.off.push_back(cur.numel);
    cur.numel += c->numel[p];
  }
  c->buckets.push_back(std::move(cur));
  c->p_bucket.assign(n, -1);
  c->p_slot.assign(n, -1);
  c->p_off.assign(n, -1);
  for (int b = 0; b < (int)c->buckets.size(); ++b) {
    Bucket& bk = c->buckets[b];
    bk.off.push_back(bk.numel);
    bk.grads.assign(bk.params.size(), nullptr);
    for (int s = 0; s < (int)bk.params.size(); ++s) {
      c->p_bucket[bk.params[s]] = b;
      c->p_slot[bk.params[s]] = s;
      c->p_off[bk.params[s]] = bk.off[s];
    }
  }
}

int resolve_algo(const ddp_ctx* c, const Bucket& bk) {
  const int64_t bytes = bk.numel * c->esize;
  // gradient-as-bucket-view: in place on the slots the gradients live in — the
  // copy-engine exchanges (one-shot CE at world 2, two-shot CE2 wider) unless
  // NCCL is forced; NCCL at world 1
  if (c->grad_view) {
    if (c->world == 1 || c->algo == DDP_ALGO_NCCL) return DDP_ALGO_NCCL;
    if (c->algo == DDP_ALGO_CE || c->algo == DDP_ALGO_CE2) return (int)c->algo;
    // beside a running backward (fp32 overlap policy): the SM-free copy engines;
    // otherwise, and for the last bucket, the fused two-shot in place
    // (kernels/pull.cu pull_view_twoshot_kernel: no pack, no copy back)
    if (c->prefer_overlap == 1 && &bk != &c->buckets.back()) return c->world == 2 ? DDP_ALGO_CE : DDP_ALGO_CE2;
    return (int)bk.params.size() > kMaxSlotsPerLaunch ? DDP_ALGO_NCCL : DDP_ALGO_TWOSHOT;
  }
  int a;
  if (c->algo != DDP_ALGO_AUTO) {
    a = (int)c->algo;
    if (c->world == 1 && (a == DDP_ALGO_CE || a == DDP_ALGO_NVLS || a == DDP_ALGO_PUSH || a == DDP_ALGO_CE2))
      a = DDP_ALGO_ONESHOT;
    if (c->world > 1 && c->wire_bf16) a = DDP_ALGO_CE;  // the compressed wire is a CE feature
    if (a == DDP_ALGO_NVLS && !c->multicast) a = DDP_ALGO_TWOSHOT;
  } else if (c->world == 1) {
    a = DDP_ALGO_ONESHOT;
  } else if (c->wire_bf16) {
    a = DDP_ALGO_CE;
  } else if (bytes <= (c->oneshot_max >= 0 ? c->oneshot_max : (1 << 20))) {
    a = DDP_ALGO_ONESHOT;  // latency-bound: one fused kernel, one barrier
  } else if (bytes <= c->twoshot_max) {
    // world 2: the copy-engine exchange moves the same (W-1) S = S bytes as any
    // algorithm, keeps the SMs free for backward and pipelines buckets
    // (profiles/r01_n2.md).  Wider: two-shot, 2(W-1)/W S per direction — best
    // measured at W=4 (profiles/r01_n4.md).  NVLS moves only (1+1/W) S, but the
    // switch path ran at ~0.7x the per-byte rate of SM stores at W=4 (both the
    // fused and the stream-ordered kernel), so it is an option, not a default
    // With the pull kernels (round 2) the fused one-shot moves the same S per
    // direction at W=2 with ONE sync and is faster than the copy engines on the
    // whole sync (profiles/r02_pull.md), so it is the W=2 choice at every size
    a = c->world == 2 ? (c->p2p_pull ? DDP_ALGO_ONESHOT : DDP_ALGO_CE) : DDP_ALGO_TWOSHOT;
    // PREFER_OVERLAP (buckets synced while backward still runs): the copy-engine
    // two-shot keeps the SMs with autograd (lowest exposed time at W=4,
    // profiles/r01_n4.md); the last bucket overlaps nothing and keeps the
    // fastest kernel on every SM
    if (c->prefer_overlap == 1 && &bk != &c->buckets.back()) a = c->world > 2 ? DDP_ALGO_CE2 : DDP_ALGO_CE;
    // PREFER_OVERLAP=2 (SM kernels under backward): at world 2 the one-shot kernel
    // instead of the copy engines — measured better for bf16 models (profiles/r01_n2.md)
    if (c->prefer_overlap == 2 && c->world == 2) a = DDP_ALGO_ONESHOT;
  } else {
    a = DDP_ALGO_NCCL;
  }
  if (a != DDP_ALGO_NCCL &&
      (int)bk.params.size() > kMaxSlotsPerLaunch)
    a = DDP_ALGO_NCCL;
  return a;
}

// Grid of a P2P launch: per-CTA chunks of >= kMinChunkElems, 256-element aligned.
void grid_for(const ddp_ctx* c, Bucket& bk, int max_ctas) {
  if (bk.algo == DDP_ALGO_NCCL || bk.algo == DDP_ALGO_CE2) {
    bk.ctas = 0;
    bk.chunk = 0;
    if (bk.algo == DDP_ALGO_NCCL) bk.shard = 0;
    return;
  }
  const bool sharded = bk.algo == DDP_ALGO_TWOSHOT || bk.algo == DDP_ALGO_NVLS;
  const int64_t L = sharded ? align_up(cdiv(bk.numel, c->world), kAlignElems) : align_up(bk.numel, kAlignElems);
  int64_t C = std::min<int64_t>(max_ctas, std::max<int64_t>(1, cdiv(L, kMinChunkElems)));
  const int64_t Q = align_up(cdiv(L, C), kAlignElems);
  C = std::max<int64_t>(1, cdiv(L, Q));
  bk.shard = L;
  bk.chunk = Q;
  bk.ctas = (int)C;
  // pipeline stage: DDP_OPT_P2P_STAGE_BYTES, else (pull kernels: the pack warps run
  // ahead of the read warps stage by stage) kPullStageBytes, else the whole chunk
  const bool pull = bk.pull || (c->grad_view && bk.algo == DDP_ALGO_TWOSHOT);
  // (the two-shot packs a stage of EVERY shard before publishing it: W x the stage)
  const int64_t pull_stage = bk.algo == DDP_ALGO_TWOSHOT
                                 ? std::max<int64_t>(8 << 10, 2 * kPullStageBytes / c->world) : kPullStageBytes;
  const int64_t stage = c->stage_bytes > 0 ? c->stage_bytes : pull ? pull_stage : 0;
  bk.sub = stage > 0 ? std::max<int64_t>(kAlignElems, std::min<int64_t>(Q, stage / c->esize)) : Q;
  bk.stages = (int32_t)cdiv(Q, bk.sub);
}

// The last bucket holds the first-registered parameters: its sync starts when
// backward has ended and overlaps nothing, so its kernel takes every SM (it is
// launched after the other lanes have drained, exchange.cpp).
int max_ctas_for(const ddp_ctx* c, const Bucket& bk) {
  const bool last = &bk == &c->buckets.back() && c->world > 1;
  int m = c->world == 1 ? (int)c->pack_ctas : last ? std::min(148, kMaxCtas) : (int)std::min<int64_t>(c->comm_ctas, kMaxCtas);
  if (c->emulated || c->peer_emu) {
    // every rank of a launch in one cooperative kernel; in peer emulation the
    // lanes' kernels must also fit side by side (they spin independently)
    const int e = emulated_max_ctas(bk.algo, c->dtype, (int)bk.params.size(), c->world, bk.pull,
                                    c->grad_view && bk.algo == DDP_ALGO_TWOSHOT);
    m = std::min(m, std::max(1, e / (c->peer_emu ? lanes_in_use(c) : 1)));
  }
  return std::max(1, m);
}

void plan(ddp_ctx* c) {
  int64_t pos = c->lanes * kFlagsBytes;  // one flag table per lane
  c->flags_off = 0;
  c->buckets_off = pos;
  int64_t l2max = 0, n1max = 0;
  for (Bucket& bk : c->buckets) {
    bk.algo = resolve_algo(c, bk);
    bk.byte_off = pos;
    pos += align_up(bk.numel * c->esize, 256);
    // which fused buckets run the pull kernels (DDP_OPT_P2P_PULL): they read the
    // peers' buffers, so a CTA's remote throughput is bounded by loads in flight
    // (~5-8 GB/s per SM measured) — best with every SM, i.e. for the LAST bucket;
    // the push kernels' fire-and-forget stores are ~3x more SM-efficient, so the
    // buckets that run beside backward on COMM_CTAS CTAs keep them.  Exception
    // (measured, profiles/r02_pull.md): with every bucket ready at once at W=2 (the
    // throughput policy) the lanes' pull one-shots together saturate the links and
    // beat both the push one-shot and the copy engines on the step
    bk.pull = c->world > 1 && !c->grad_view && (bk.algo == DDP_ALGO_ONESHOT || bk.algo == DDP_ALGO_TWOSHOT) &&
              (c->p2p_pull == 2 ||
               (c->p2p_pull == 1 &&
                (&bk == &c->buckets.back() || (c->world == 2 && c->prefer_overlap == 0))));
    if (bk.pull || c->grad_view) continue;  // pull kernels: no staging (second buffer below); view: in place
    if (bk.algo == DDP_ALGO_TWOSHOT) l2max = std::max(l2max, align_up(cdiv(bk.numel, c->world), kAlignElems));
    if (bk.algo == DDP_ALGO_ONESHOT && c->world > 1) n1max = std::max(n1max, align_up(bk.numel, kAlignElems));
  }
  c->stage2_stride = align_up(l2max * c->esize, 256);
  c->stage2_off = pos;
  pos += c->lanes * c->world * c->stage2_stride;  // per lane
  c->stage1_stride = align_up(n1max * c->esize, 256);
  c->stage1_off = pos;
  pos += c->lanes * 2 * c->world * c->stage1_stride;  // per lane, double-buffered by the lane's launch parity
  // pull kernels: a second buffer per fused bucket; pass v uses buffer v % 2 (kernels/pull.cu)
  for (Bucket& bk : c->buckets) {
    bk.alt_off = bk.byte_off;
    if (bk.pull) {
      bk.alt_off = pos;
      pos += align_up(bk.numel * c->esize, 256);
    }
  }
  // copy-engine buckets: W slots each (dedicated per bucket) + ready/consumed flags
  c->ce_flags_off = pos;
  pos += align_up((int64_t)c->buckets.size() * kMaxWorld * kCeFlagKinds * 4, 256);  // ready, consumed, gathered, bitmap
  for (Bucket& bk : c->buckets) {
    bk.ce_stride = 0;
    bk.ce_wire.clear();
    bk.ce_direct.clear();
    if (bk.algo == DDP_ALGO_CE2) {  // double-buffered reduce-scatter staging: [2][W] shard slots
      const int64_t L = align_up(cdiv(bk.numel, c->world), kAlignElems);
      bk.shard = L;
      bk.ce_stride = align_up(L * c->esize, 256);
      bk.ce_off = pos;
      pos += 2 * c->world * bk.ce_stride;
      continue;
    }
    if (bk.algo != DDP_ALGO_CE && bk.algo != DDP_ALGO_PUSH) continue;
    const size_t ns = bk.params.size();
    bk.ce_wire.assign(ns, 0);
    bk.ce_direct.assign(ns, 0);
    if (c->grad_view) {  // wire layout = bucket layout: the bucket region travels as one copy
      for (size_t k = 0; k < ns; ++k) bk.ce_wire[k] = bk.off[k];
      bk.ce_small0 = 0;
      bk.ce_wire_numel = bk.numel;
      bk.ce_stride = align_up(bk.numel * c->esize, 256);
      bk.ce_off = pos;
      pos += c->world * bk.ce_stride;
      continue;
    }
    int64_t w = 0;
    for (int pass = 0; pass < 2; ++pass) {  // direct gradients first, then the small ones
      if (pass == 1) bk.ce_small0 = w;
      for (size_t k = 0; k < ns; ++k) {
        const int64_t n = bk.off[k + 1] - bk.off[k];
        const bool direct = bk.algo == DDP_ALGO_CE && !c->wire_bf16 && n * c->esize >= c->ce_direct;
        if (direct != (pass == 0)) continue;
        bk.ce_direct[k] = direct;
        bk.ce_wire[k] = w;
        w = align_up(w + n, kCeWireAlign);
      }
    }
    bk.ce_wire_numel = w;
    bk.ce_stride = align_up(w * (c->wire_bf16 ? 2 : c->esize), 256);
    bk.ce_off = pos;
    pos += c->world * bk.ce_stride;
  }
  // find_unused: participation bitmaps (int32 per param; [2 pass parities][W source
  // ranks] slots at world > 1, exchanged by the copy engines), the summed bitmap, and
  // a scratch copy of the bucket region (locally-unused parameters pack zeros from,
  // and receive the average into, it)
  c->bitmap_off = c->global_off = c->scratch_off = c->bitmap_stride = 0;
  if (c->find_unused) {
    c->bitmap_stride = align_up((int64_t)c->numel.size() * 4, 256);
    c->bitmap_off = pos;
    pos += (c->world > 1 ? 2 * c->world : 0) * c->bitmap_stride;
    c->global_off = pos;
    pos += c->bitmap_stride;
    c->scratch_off = pos;
    pos += c->stage2_off - c->buckets_off;  // = the bucket region
  }
  c->storage_bytes = pos;
  for (Bucket& bk : c->buckets) grid_for(c, bk, max_ctas_for(c, bk));
}

void regrid(ddp_ctx* c) {
  for (Bucket& bk : c->buckets) grid_for(c, bk, max_ctas_for(c, bk));
}

ddp_status_t check_ctx(const ddp_ctx* c) {
  if (!c) return fail(DDP_ERR_INVALID_ARG, "null context");
  if (c->poisoned) return fail(DDP_ERR_POISONED, "context poisoned by an earlier fatal error");
  return DDP_OK;
}

// ---- a2/a5: launch buckets [b0, b1) (in order), triggered by ready signal t --
// Inside ddp_grads_ready (a batch of ready signals that arrive together) the
// device launch is deferred to the end of the batch so consecutive buckets can
// share launches; the launch order and trace are unchanged.
ddp_status_t launch_range(ddp_ctx* c, int b0, int b1, int32_t trigger) {
  for (int b = b0; b < b1; ++b) c->trace.emplace_back(b, trigger);
  if (c->dry_run || b0 >= b1) return DDP_OK;
  if (c->defer) {
    if (c->defer_b0 == c->defer_b1) c->defer_b0 = b0;
    c->defer_b1 = b1;
    return DDP_OK;
  }
  return device_range(c, b0, b1);
}

void open_pass(ddp_ctx* c) {
  c->state = State::IN_PASS;
  c->pass_launched = false;
  c->last_on = nullptr;
  c->lone_last = false;
  c->pass_no_sync = c->no_sync;  // reading C-9
  std::fill(c->ready.begin(), c->ready.end(), 0);
  for (size_t b = 0; b < c->buckets.size(); ++b) c->pending[b] = (int32_t)c->buckets[b].params.size();
  c->cursor = 0;
  c->n_ready = 0;
  c->trace.clear();
  c->order.clear();
  c->un_param.clear();
  c->un_dst.clear();
  c->un_src.clear();
  c->un_numel.clear();
}


// Scratch slot of parameter p (find_unused): mirrors its bucket position.
char* scratch_of(ddp_ctx* c, int32_t p) {
  const Bucket& bk = c->buckets[c->p_bucket[p]];
  return static_cast<char*>(c->storage[c->rank]) + c->scratch_off + (bk.byte_off - c->buckets_off) +
         c->p_off[p] * c->esize;
}

// One ready signal (a2).  unused: ddp_mark_unused (Alg. 1 forward L224-L225).
ddp_status_t grad_ready_one(ddp_ctx* c, int32_t p, void* grad, cudaStream_t s, bool unused = false) {
  if (p < 0 || p >= (int32_t)c->numel.size()) return fail(DDP_ERR_INVALID_ARG, "param index out of range");
  if (!unused && !grad && !c->dry_run) return fail(DDP_ERR_INVALID_ARG, "null gradient pointer");
  if (unused && !c->find_unused) return fail(DDP_ERR_STATE, "ddp_mark_unused needs DDP_OPT_FIND_UNUSED");
  if (unused && !grad && c->used_local[p] && !c->dry_run)
    return fail(DDP_ERR_INVALID_ARG, "param " + std::to_string(p) +
                                         " has an accumulated gradient from a no_sync pass: pass it");
  if (c->state != State::IN_PASS) open_pass(c);
  if (c->ready[p]) return fail(DDP_ERR_DUPLICATE, "param " + std::to_string(p) + " marked ready twice");
  c->ready[p] = 1;
  c->order.push_back(p);
  const int32_t t = c->n_ready++;
  const int32_t b = c->p_bucket[p];
  c->pending[b] -= 1;  // P:L306 pending count
  if (!unused) c->used_local[p] = 1;  // participation bitmap, accumulated across no_sync
  void* src = grad;
  if (unused && !c->used_local[p] && !c->pass_no_sync) {
    // no local contribution: the slot packs zeros from scratch and receives the average there
    src = c->dry_run ? nullptr : scratch_of(c, p);
    if (!c->dry_run) {
      CUDA_TRY(c, cudaMemsetAsync(src, 0, (size_t)(c->numel[p] * c->esize), s));
      c->un_param.push_back(p);
      c->un_dst.push_back(grad);
      c->un_src.push_back(src);
      c->un_numel.push_back(c->numel[p]);
    }
  }
  c->buckets[b].grads[c->p_slot[p]] = src;
  if (c->pass_no_sync) return DDP_OK;  // hooks disabled
  if (std::find(c->unwaited.begin(), c->unwaited.end(), s) == c->unwaited.end()) c->unwaited.push_back(s);
  c->producer = s;
  if (!c->overlap) return DDP_OK;
  const int32_t nb = (int32_t)c->buckets.size();
  int32_t e = c->cursor;
  while (e < nb && c->pending[e] == 0) ++e;  // every consecutive ready bucket (C-7)
  const int32_t b0 = c->cursor;
  c->cursor = e;
  c->from_signal = true;
  const ddp_status_t st = launch_range(c, b0, e, t);
  c->from_signal = false;
  return st;
}

bool is_layout_key(int32_t k) {
  return k == DDP_OPT_P2P_ONESHOT_MAX || k == DDP_OPT_P2P_TWOSHOT_MAX || k == DDP_OPT_ALGO ||
         k == DDP_OPT_FIND_UNUSED || k == DDP_OPT_MULTICAST || k == DDP_OPT_CE_DIRECT_BYTES ||
         k == DDP_OPT_WIRE_BF16 || k == DDP_OPT_LANES || k == DDP_OPT_PREFER_OVERLAP || k == DDP_OPT_GRAD_VIEW ||
         k == DDP_OPT_P2P_PULL;
}

}  // namespace

// =============================== C ABI ========================================
extern "C" {

const char* ddp_last_error(void) { return g_err.c_str(); }
const char* ddp_version(void) { return "b200ddp 0.1 (sm_100a)"; }

ddp_status_t ddp_create(const int64_t* param_numel, int32_t n_params, int32_t dtype,
                        int64_t bucket_cap_bytes, int32_t world, int32_t rank, ddp_ctx_t** out) {
  return ddp_create_ordered(param_numel, n_params, nullptr, dtype, bucket_cap_bytes, world, rank, out);
}

ddp_status_t ddp_create_ordered(const int64_t* param_numel, int32_t n_params, const int32_t* scan_order,
                                int32_t dtype, int64_t bucket_cap_bytes, int32_t world, int32_t rank,
                                ddp_ctx_t** out) {
  if (!out || !param_numel || n_params < 1) return fail(DDP_ERR_INVALID_ARG, "need >= 1 parameter");
  if (scan_order) {
    std::vector<uint8_t> seen(n_params, 0);
    for (int32_t i = 0; i < n_params; ++i) {
      const int32_t p = scan_order[i];
      if (p < 0 || p >= n_params || seen[p]) return fail(DDP_ERR_INVALID_ARG, "scan_order is not a permutation");
      seen[p] = 1;
    }
  }
  if (dtype != DDP_FP32 && dtype != DDP_BF16) return fail(DDP_ERR_INVALID_ARG, "dtype must be FP32 or BF16");
  if (bucket_cap_bytes < 0) return fail(DDP_ERR_INVALID_ARG, "bucket_cap_bytes < 0");
  if (world < 1 || world > kMaxWorld || rank < 0 || rank >= world)
    return fail(DDP_ERR_INVALID_ARG, "need 1 <= world <= 8 and 0 <= rank < world");
  for (int32_t i = 0; i < n_params; ++i)
    if (param_numel[i] < 1) return fail(DDP_ERR_INVALID_ARG, "param numel must be >= 1");
  ddp_ctx* c = new (std::nothrow) ddp_ctx();
  if (!c) return fail(DDP_ERR_NOMEM, "out of host memory");
  try {
    c->world = world;
    c->rank = rank;
    c->dtype = dtype;
    c->esize = dtype == DDP_FP32 ? 4 : 2;
    c->cap = bucket_cap_bytes;
    c->numel.assign(param_numel, param_numel + n_params);
    c->scan.resize(n_params);
    for (int32_t i = 0; i < n_params; ++i) c->scan[i] = scan_order ? scan_order[i] : n_params - 1 - i;
    assign(c);
    c->ready.assign(n_params, 0);
    c->used_local.assign(n_params, 0);
    c->pending.assign(c->buckets.size(), 0);
    plan(c);
  } catch (const std::bad_alloc&) {
    delete c;
    return fail(DDP_ERR_NOMEM, "out of host memory");
  }
  *out = c;
  return DDP_OK;
}

void ddp_destroy(ddp_ctx_t* c) {
  if (!c) return;
  if (c->bound && !c->emulated) {
    if (!c->poisoned && c->comm) cudaStreamSynchronize(c->comm);
    for (size_t k = 1; k < c->rr_comm.size(); ++k) {
      if (c->rr_stream[k] && !c->poisoned) cudaStreamSynchronize(c->rr_stream[k]);
      if (c->rr_comm[k]) {
        if (c->poisoned) ncclCommAbort(c->rr_comm[k]);
        else ncclCommDestroy(c->rr_comm[k]);
      }
      if (c->rr_stream[k]) cudaStreamDestroy(c->rr_stream[k]);
      if (c->rr_done[k]) cudaEventDestroy(c->rr_done[k]);
    }
    if (c->nccl) {
      if (c->poisoned) ncclCommAbort(c->nccl);
      else ncclCommDestroy(c->nccl);
    }
  } else if (c->bound && c->comm && !c->poisoned) {
    cudaStreamSynchronize(c->comm);
  }
  for (auto& se : c->stream_events) cudaEventDestroy(se.second);
  for (auto& r : c->prof) {
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  for (cudaEvent_t e : c->event_pool) cudaEventDestroy(e);
  for (cudaEvent_t e : c->prof_ready) cudaEventDestroy(e);
  if (c->comm_done) cudaEventDestroy(c->comm_done);
  std::vector<cudaStream_t> own(c->ce2_rs.begin(), c->ce2_rs.end());
  own.insert(own.end(), c->ce2_ag.begin(), c->ce2_ag.end());
  own.push_back(c->ce_ag);
  own.push_back(c->ce_up);
  own.push_back(c->ce_red);
  own.push_back(c->ce_pack);
  for (cudaStream_t s : own) {
    if (!s) continue;
    if (!c->poisoned) cudaStreamSynchronize(s);
    cudaStreamDestroy(s);
  }
  for (cudaEvent_t e : c->ce_reduced) cudaEventDestroy(e);
  for (cudaEvent_t e : c->ce2_done) cudaEventDestroy(e);
  for (cudaEvent_t e : c->join_ev) cudaEventDestroy(e);
  for (int k = 1; k < kMaxLanes; ++k) {
    if (c->lane_stream[k]) {
      if (!c->poisoned) cudaStreamSynchronize(c->lane_stream[k]);
      cudaStreamDestroy(c->lane_stream[k]);
    }
    if (c->lane_done[k]) cudaEventDestroy(c->lane_done[k]);
  }
  for (cudaEvent_t e : c->ce_packed) cudaEventDestroy(e);
  for (cudaEvent_t e : c->ce_copied) cudaEventDestroy(e);
  if (c->ce_red_done) cudaEventDestroy(c->ce_red_done);
  if (c->err_host) cudaFreeHost(c->err_host);
  if (c->bitmap_host) cudaFreeHost(c->bitmap_host);
  if (c->global_host) cudaFreeHost(c->global_host);
  if (c->bitmap_done) cudaEventDestroy(c->bitmap_done);
  for (cudaEvent_t e : c->emu_pre)
    if (e) cudaEventDestroy(e);
  emu_leave(c);
  delete c;
}

int32_t ddp_num_buckets(const ddp_ctx_t* c) { return c ? (int32_t)c->buckets.size() : -1; }

ddp_status_t ddp_bucket_info(const ddp_ctx_t* c, int32_t b, int64_t* numel, int32_t* n_slots) {
  if (!c || b < 0 || b >= (int32_t)c->buckets.size()) return fail(DDP_ERR_INVALID_ARG, "bad bucket");
  if (numel) *numel = c->buckets[b].numel;
  if (n_slots) *n_slots = (int32_t)c->buckets[b].params.size();
  return DDP_OK;
}

ddp_status_t ddp_bucket_slot(const ddp_ctx_t* c, int32_t b, int32_t s, int32_t* param, int64_t* offset) {
  if (!c || b < 0 || b >= (int32_t)c->buckets.size()) return fail(DDP_ERR_INVALID_ARG, "bad bucket");
  const Bucket& bk = c->buckets[b];
  if (s < 0 || s >= (int32_t)bk.params.size()) return fail(DDP_ERR_INVALID_ARG, "bad slot");
  if (param) *param = bk.params[s];
  if (offset) *offset = bk.off[s];
  return DDP_OK;
}

ddp_status_t ddp_param_location(const ddp_ctx_t* c, int32_t p, int32_t* bucket, int64_t* offset) {
  if (!c || p < 0 || p >= (int32_t)c->numel.size()) return fail(DDP_ERR_INVALID_ARG, "bad param");
  if (bucket) *bucket = c->p_bucket[p];
  if (offset) *offset = c->p_off[p];
  return DDP_OK;
}

ddp_status_t ddp_param_storage_offset(const ddp_ctx_t* c, int32_t p, int64_t* byte_offset) {
  if (!c || !byte_offset || p < 0 || p >= (int32_t)c->numel.size()) return fail(DDP_ERR_INVALID_ARG, "bad param");
  *byte_offset = c->buckets[c->p_bucket[p]].byte_off + c->p_off[p] * c->esize;
  return DDP_OK;
}

ddp_status_t ddp_storage_bytes(const ddp_ctx_t* c, int64_t* bytes) {
  if (!c || !bytes) return fail(DDP_ERR_INVALID_ARG, "null argument");
  *bytes = c->storage_bytes;
  return DDP_OK;
}

ddp_status_t ddp_bucket_algo(const ddp_ctx_t* c, int32_t b, int32_t* algo) {
  if (!c || !algo || b < 0 || b >= (int32_t)c->buckets.size()) return fail(DDP_ERR_INVALID_ARG, "bad bucket");
  *algo = c->buckets[b].algo;
  return DDP_OK;
}

ddp_status_t ddp_get_nccl_id(uint8_t out[128]) {
  if (!out) return fail(DDP_ERR_INVALID_ARG, "null out");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  ncclUniqueId id;
  ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) return nccl_fail(nullptr, r, "ncclGetUniqueId");
  std::memcpy(out, &id, 128);
  return DDP_OK;
}

static ddp_status_t bind_common(ddp_ctx* c, int32_t device, void* comm_stream) {
  CUDA_TRY(c, cudaSetDevice(device));
  c->device = device;
  c->comm = static_cast<cudaStream_t>(comm_stream);
  CUDA_TRY(c, cudaHostAlloc(reinterpret_cast<void**>(&c->err_host), sizeof(uint32_t), cudaHostAllocMapped));
  *c->err_host = 0;
  CUDA_TRY(c, cudaHostGetDevicePointer(reinterpret_cast<void**>(&c->err_dev), c->err_host, 0));
  CUDA_TRY(c, cudaEventCreateWithFlags(&c->comm_done, cudaEventDisableTiming));
  if (c->find_unused) {
    const size_t nb = c->numel.size() * sizeof(int32_t);
    CUDA_TRY(c, cudaHostAlloc(reinterpret_cast<void**>(&c->bitmap_host), nb, cudaHostAllocDefault));
    CUDA_TRY(c, cudaHostAlloc(reinterpret_cast<void**>(&c->global_host), nb, cudaHostAllocDefault));
    CUDA_TRY(c, cudaEventCreateWithFlags(&c->bitmap_done, cudaEventDisableTiming));
  }
  return DDP_OK;
}

}  // extern "C"

namespace b200ddp {

// Zeroes this rank's barrier / stream-memop flags (on the comm stream) and creates
// the library's side streams: lanes for the fused P2P kernels, the copy-engine
// streams and events, and the stream-memory-operation entry points (world > 1).
ddp_status_t create_side_streams(ddp_ctx* c) {
  char* mine = static_cast<char*>(c->storage[c->rank]);
  CUDA_TRY(c, cudaMemsetAsync(mine + c->flags_off, 0, c->lanes * kFlagsBytes, c->comm));
  CUDA_TRY(c, cudaMemsetAsync(mine + c->ce_flags_off, 0, (size_t)c->buckets.size() * kMaxWorld * kCeFlagKinds * 4,
                              c->comm));
  int lo = 0, hi = 0;
  CUDA_TRY(c, cudaDeviceGetStreamPriorityRange(&lo, &hi));
  if (c->low_priority) hi = lo;  // side streams at the lowest priority
  if (c->world > 1 && c->lanes > 1) {
    for (int k = 1; k < c->lanes; ++k) {
      CUDA_TRY(c, cudaStreamCreateWithPriority(&c->lane_stream[k], cudaStreamNonBlocking, hi));
      CUDA_TRY(c, cudaEventCreateWithFlags(&c->lane_done[k], cudaEventDisableTiming));
    }
  }
  bool any_ce = false;
  for (const Bucket& bk : c->buckets)
    any_ce |= bk.algo == DDP_ALGO_CE || bk.algo == DDP_ALGO_PUSH || bk.algo == DDP_ALGO_CE2;
  if (any_ce) {
    CUDA_TRY(c, cudaStreamCreateWithPriority(&c->ce_red, cudaStreamNonBlocking, hi));
    CUDA_TRY(c, cudaStreamCreateWithPriority(&c->ce_pack, cudaStreamNonBlocking, hi));
    c->ce_packed.assign(c->buckets.size(), nullptr);
    for (auto& e : c->ce_packed) CUDA_TRY(c, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    c->ce_copied.assign(c->buckets.size(), nullptr);
    for (auto& e : c->ce_copied) CUDA_TRY(c, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    CUDA_TRY(c, cudaStreamCreateWithPriority(&c->ce_ag, cudaStreamNonBlocking, hi));
    // CE2 copy streams: CE_STREAMS of them (peers round-robin).  One per peer was
    // measured slower at W=4 (profiles/r01_n4.md): the copy engines do not overlap
    // transfers usefully, the extra streams only add ordering hops
    const size_t nst = (size_t)std::max<int64_t>(1, std::min<int64_t>(c->ce_streams, c->world - 1));
    c->ce2_rs.assign(nst, nullptr);
    c->ce2_ag.assign(nst, nullptr);
    for (auto& q : c->ce2_rs) CUDA_TRY(c, cudaStreamCreateWithPriority(&q, cudaStreamNonBlocking, hi));
    for (auto& q : c->ce2_ag) CUDA_TRY(c, cudaStreamCreateWithPriority(&q, cudaStreamNonBlocking, hi));
    c->ce2_done.assign(2 * nst, nullptr);
    for (auto& e : c->ce2_done) CUDA_TRY(c, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    CUDA_TRY(c, cudaStreamCreateWithPriority(&c->ce_up, cudaStreamNonBlocking, hi));
    c->ce_reduced.assign(c->buckets.size(), nullptr);
    for (auto& e : c->ce_reduced) CUDA_TRY(c, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    CUDA_TRY(c, cudaEventCreateWithFlags(&c->ce_red_done, cudaEventDisableTiming));
  }
  if (c->world > 1) {  // joins of the library streams before / after the last bucket (exchange.cpp)
    c->join_ev.assign(48, nullptr);
    for (auto& e : c->join_ev) CUDA_TRY(c, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  if (c->world > 1) {  // copy-engine exchanges and the find_unused bitmap exchange
    cudaDriverEntryPointQueryResult q1, q2;
    CUDA_TRY(c, cudaGetDriverEntryPoint("cuStreamWriteValue32", &c->fn_write32, cudaEnableDefault, &q1));
    CUDA_TRY(c, cudaGetDriverEntryPoint("cuStreamWaitValue32", &c->fn_wait32, cudaEnableDefault, &q2));
    if (q1 != cudaDriverEntryPointSuccess || q2 != cudaDriverEntryPointSuccess || !c->fn_write32 || !c->fn_wait32)
      return fail(DDP_ERR_UNSUPPORTED, "stream memory operations unavailable (copy-engine exchange)");
  }
  return DDP_OK;
}

}  // namespace b200ddp

extern "C" {

ddp_status_t ddp_bind_device(ddp_ctx_t* c, int32_t device, const uint8_t nccl_id[128], void* comm_stream,
                             void* const* peer_storage, void* multicast_ptr) {
  if (ddp_status_t st = check_ctx(c)) return st;
  if (c->multicast && (!multicast_ptr || (reinterpret_cast<uintptr_t>(multicast_ptr) & 255)))
    return fail(DDP_ERR_INVALID_ARG, "DDP_OPT_MULTICAST needs a 256-B aligned multicast address");
  c->mc = c->multicast ? multicast_ptr : nullptr;
  if (c->bound || c->state != State::CREATED) return fail(DDP_ERR_STATE, "already bound");
  if (c->dry_run) return fail(DDP_ERR_STATE, "dry-run context cannot be bound");
  if (!nccl_id || !peer_storage) return fail(DDP_ERR_INVALID_ARG, "null argument");
  for (int r = 0; r < c->world; ++r) {
    if (!peer_storage[r] || (reinterpret_cast<uintptr_t>(peer_storage[r]) & 255))
      return fail(DDP_ERR_INVALID_ARG, "peer storage must be non-null and 256-B aligned");
    c->storage[r] = peer_storage[r];
  }
  if (ddp_status_t st = bind_common(c, device, comm_stream)) return st;
  ncclUniqueId id;
  std::memcpy(&id, nccl_id, 128);
  NCCL_TRY(c, ncclCommInitRank(&c->nccl, c->world, id, c->rank));
  if (c->nccl_comms > 1) {  // round-robin groups: split k-1 more communicators off the first
    int lo = 0, hi = 0;
    CUDA_TRY(c, cudaDeviceGetStreamPriorityRange(&lo, &hi));
    if (c->low_priority) hi = lo;  // side streams at the lowest priority
    c->rr_comm.assign((size_t)c->nccl_comms, nullptr);
    c->rr_stream.assign((size_t)c->nccl_comms, nullptr);
    c->rr_done.assign((size_t)c->nccl_comms, nullptr);
    c->rr_used.assign((size_t)c->nccl_comms, 0);
    c->rr_comm[0] = c->nccl;
    c->rr_stream[0] = c->comm;
    for (size_t k = 1; k < c->rr_comm.size(); ++k) {
      NCCL_TRY(c, ncclCommSplit(c->nccl, 0, c->rank, &c->rr_comm[k], nullptr));
      CUDA_TRY(c, cudaStreamCreateWithPriority(&c->rr_stream[k], cudaStreamNonBlocking, hi));
      CUDA_TRY(c, cudaEventCreateWithFlags(&c->rr_done[k], cudaEventDisableTiming));
    }
  }
  if (ddp_status_t st = create_side_streams(c)) return st;
  char* mine = static_cast<char*>(c->storage[c->rank]);
  // every rank's flags are zero before anyone's first P2P launch
  NCCL_TRY(c, ncclAllReduce(mine + kBarrierScratch, mine + kBarrierScratch, 1, ncclInt32, ncclSum, c->nccl, c->comm));
  CUDA_TRY(c, cudaStreamSynchronize(c->comm));
  c->bound = true;
  c->state = State::IDLE;
  return DDP_OK;
}

ddp_status_t ddp_bind_emulated(ddp_ctx_t* c, int32_t device, void* comm_stream, void* const* storages,
                               int64_t grad_rank_stride_bytes) {
  if (ddp_status_t st = check_ctx(c)) return st;
  if (c->bound || c->state != State::CREATED) return fail(DDP_ERR_STATE, "already bound");
  if (c->dry_run) return fail(DDP_ERR_STATE, "dry-run context cannot be bound");
  if (c->rank != 0) return fail(DDP_ERR_INVALID_ARG, "emulated context must be created with rank 0");
  if (!storages) return fail(DDP_ERR_INVALID_ARG, "null storages");
  for (int r = 0; r < c->world; ++r) {
    if (!storages[r] || (reinterpret_cast<uintptr_t>(storages[r]) & 255))
      return fail(DDP_ERR_INVALID_ARG, "storages must be non-null and 256-B aligned");
  }
  for (const Bucket& bk : c->buckets)
    if (bk.algo == DDP_ALGO_NCCL || bk.algo == DDP_ALGO_CE || bk.algo == DDP_ALGO_PUSH || bk.algo == DDP_ALGO_CE2)
      return fail(DDP_ERR_UNSUPPORTED, "cooperative emulation runs the one-shot / two-shot kernels only (set "
                                       "DDP_OPT_ALGO, or use ddp_bind_peer_emulated)");
  if (c->find_unused) return fail(DDP_ERR_UNSUPPORTED, "find_unused needs a real communicator (no emulation)");
  if (c->grad_view) return fail(DDP_ERR_UNSUPPORTED, "gradient-as-bucket-view needs one context per rank (ddp_bind_peer_emulated)");
  if (c->multicast) return fail(DDP_ERR_UNSUPPORTED, "NVLS needs real multicast memory (no emulation)");
  if (ddp_status_t st = bind_common(c, device, comm_stream)) return st;
  for (int r = 0; r < c->world; ++r) c->storage[r] = storages[r];
  c->grad_rank_stride = grad_rank_stride_bytes;
  c->emulated = true;
  regrid(c);
  for (int r = 0; r < c->world; ++r)
    CUDA_TRY(c, cudaMemsetAsync(static_cast<char*>(c->storage[r]) + c->flags_off, 0, c->lanes * kFlagsBytes, c->comm));
  CUDA_TRY(c, cudaStreamSynchronize(c->comm));
  c->bound = true;
  c->state = State::IDLE;
  return DDP_OK;
}

ddp_status_t ddp_bind_peer_emulated(ddp_ctx_t* c, int32_t device, void* comm_stream, void* const* storages) {
  if (ddp_status_t st = check_ctx(c)) return st;
  if (c->bound || c->state != State::CREATED) return fail(DDP_ERR_STATE, "already bound");
  if (c->dry_run) return fail(DDP_ERR_STATE, "dry-run context cannot be bound");
  if (c->world < 2) return fail(DDP_ERR_INVALID_ARG, "peer emulation needs world >= 2");
  if (!storages) return fail(DDP_ERR_INVALID_ARG, "null storages");
  for (int r = 0; r < c->world; ++r)
    if (!storages[r] || (reinterpret_cast<uintptr_t>(storages[r]) & 255))
      return fail(DDP_ERR_INVALID_ARG, "storages must be non-null and 256-B aligned");
  if (c->multicast) return fail(DDP_ERR_UNSUPPORTED, "NVLS needs real multicast memory (no emulation)");
  for (size_t b = 0; b < c->buckets.size(); ++b)
    if (c->buckets[b].algo == DDP_ALGO_NCCL)
      return fail(DDP_ERR_UNSUPPORTED, "peer emulation has no NCCL communicator: bucket " + std::to_string(b) +
                                           " resolves to NCCL (> 1024 slots, TWOSHOT_MAX or DDP_OPT_ALGO)");
  if (ddp_status_t st = bind_common(c, device, comm_stream)) return st;
  for (int r = 0; r < c->world; ++r) c->storage[r] = storages[r];
  c->peer_emu = true;
  regrid(c);
  if (ddp_status_t st = create_side_streams(c)) return st;
  for (int k = 0; k < c->lanes; ++k) CUDA_TRY(c, cudaEventCreateWithFlags(&c->emu_pre[k], cudaEventDisableTiming));
  CUDA_TRY(c, cudaStreamSynchronize(c->comm));
  // every rank's flags are zero before any rank issues work (host barrier)
  if (ddp_status_t st = emu_join(c)) return st;
  c->bound = true;
  c->state = State::IDLE;
  return DDP_OK;
}

ddp_status_t ddp_grad_ready(ddp_ctx_t* c, int32_t p, void* grad, void* producer_stream) {
  if (ddp_status_t st = check_ctx(c)) return st;
  if (!c->bound && !c->dry_run) return fail(DDP_ERR_STATE, "context not bound to a device");
  return grad_ready_one(c, p, grad, static_cast<cudaStream_t>(producer_stream));
}

ddp_status_t ddp_grads_ready(ddp_ctx_t* c, int32_t n, const int32_t* params, void* const* grads,
                             void* producer_stream) {
  if (ddp_status_t st = check_ctx(c)) return st;
  if (!c->bound && !c->dry_run) return fail(DDP_ERR_STATE, "context not bound to a device");
  if (n < 0 || (n > 0 && (!params || (!grads && !c->dry_run)))) return fail(DDP_ERR_INVALID_ARG, "bad batch");
  c->defer = true;
  c->defer_b0 = c->defer_b1 = 0;
  ddp_status_t st = DDP_OK;
  for (int32_t i = 0; i < n && st == DDP_OK; ++i)
    st = grad_ready_one(c, params[i], grads ? grads[i] : nullptr, static_cast<cudaStream_t>(producer_stream));
  c->defer = false;
  // buckets completed by the batch are launched even if a later signal failed:
  // their launch is already part of the (cross-rank) launch sequence
  const std::string err = g_err;
  c->from_signal = true;  // the batch's buckets were completed by its ready signals
  ddp_status_t st2 = device_range(c, c->defer_b0, c->defer_b1);
  c->from_signal = false;
  if (st != DDP_OK) {
    g_err = err;
    return st;
  }
  return st2;
}

ddp_status_t ddp_mark_unused(ddp_ctx_t* c, int32_t p, void* grad, void* producer_stream) {
  if (ddp_status_t st = check_ctx(c)) return st;
  if (!c->bound && !c->dry_run) return fail(DDP_ERR_STATE, "context not bound to a device");
  return grad_ready_one(c, p, grad, static_cast<cudaStream_t>(producer_stream), true);
}

ddp_status_t ddp_global_unused(ddp_ctx_t* c, uint8_t* out, int32_t n) {
  if (ddp_status_t st = check_ctx(c)) return st;
  if (!out || n < 0 || n > (int32_t)c->numel.size()) return fail(DDP_ERR_INVALID_ARG, "bad output");
  if (!c->bitmap_valid) return fail(DDP_ERR_STATE, "no synced find_unused pass has finished");
  CUDA_TRY(c, cudaEventSynchronize(c->bitmap_done));
  for (int32_t p = 0; p < n; ++p) out[p] = c->global_host[p] == 0 ? 1 : 0;
  return DDP_OK;
}

ddp_status_t ddp_finalize_backward(ddp_ctx_t* c, void* consumer_stream) {
  if (ddp_status_t st = check_ctx(c)) return st;
  if (c->state != State::IN_PASS) return fail(DDP_ERR_STATE, "no backward pass is open");
  if (c->n_ready != (int32_t)c->numel.size()) {
    c->poisoned = true;  // peers may be blocked in a collective
    c->last_trace = c->trace;
    c->state = State::IDLE;
    return fail(DDP_ERR_INCOMPLETE, std::to_string(c->numel.size() - c->n_ready) +
                                        " parameter(s) never marked ready in this pass");
  }
  if (!c->pass_no_sync) {
    const int32_t nb = (int32_t)c->buckets.size();
    const int32_t b0 = c->cursor;  // OVERLAP=0: all launches at finalize, in order
    c->cursor = nb;
    if (ddp_status_t st = launch_range(c, b0, nb, c->n_ready)) return st;
    if (!c->dry_run && !c->last_on) {
      // join the side streams (copy-engine reductions and round-robin NCCL buckets
      // write .grad / scratch there) into the comm stream: one event then covers all
      if (c->ce_used) {
        CUDA_TRY(c, cudaEventRecord(c->ce_red_done, c->ce_red));
        CUDA_TRY(c, cudaStreamWaitEvent(c->comm, c->ce_red_done, 0));
        c->ce_used = false;
      }
      if (c->ce2_used) {  // CE2 writes .grad on the unpack stream; its copies read the bucket
        CUDA_TRY(c, cudaEventRecord(c->ce_red_done, c->ce_up));
        CUDA_TRY(c, cudaStreamWaitEvent(c->comm, c->ce_red_done, 0));
        for (size_t k = 0; k < c->ce2_rs.size(); ++k) {
          CUDA_TRY(c, cudaEventRecord(c->ce2_done[2 * k], c->ce2_rs[k]));
          CUDA_TRY(c, cudaStreamWaitEvent(c->comm, c->ce2_done[2 * k], 0));
          CUDA_TRY(c, cudaEventRecord(c->ce2_done[2 * k + 1], c->ce2_ag[k]));
          CUDA_TRY(c, cudaStreamWaitEvent(c->comm, c->ce2_done[2 * k + 1], 0));
        }
        c->ce2_used = false;
      }
      for (size_t k = 1; k < c->rr_stream.size(); ++k) {
        if (!c->rr_used[k]) continue;
        CUDA_TRY(c, cudaEventRecord(c->rr_done[k], c->rr_stream[k]));
        CUDA_TRY(c, cudaStreamWaitEvent(c->comm, c->rr_done[k], 0));
        c->rr_used[k] = 0;
      }
      for (int k = 1; k < kMaxLanes; ++k) {
        if (!c->lane_used[k]) continue;
        CUDA_TRY(c, cudaEventRecord(c->lane_done[k], c->lane_stream[k]));
        CUDA_TRY(c, cudaStreamWaitEvent(c->comm, c->lane_done[k], 0));
        c->lane_used[k] = false;
      }
    }
    if (c->find_unused) {
      if (!c->dry_run) {
        if (ddp_status_t st = finish_unused(c)) return st;
      } else {
        std::fill(c->used_local.begin(), c->used_local.end(), 0);
      }
    }
    if (!c->dry_run) {
      // the last bucket ran on its producer stream, after every library stream was
      // joined into it (exchange.cpp): that stream alone marks the end of the pass
      cudaStream_t end = c->last_on ? c->last_on : c->comm;
      // watchdog (ddp_check_device_errors): time from the finalize of the oldest
      // pass not yet seen complete; a later pass completes after it (stream order)
      if (!c->watch || pass_complete(c)) c->done_since = std::chrono::steady_clock::now();
      c->watch = true;
      CUDA_TRY(c, cudaEventRecord(c->comm_done, end));
      c->comm_done_valid = true;
      c->done_stream = end;
      if (static_cast<cudaStream_t>(consumer_stream) != end)
        CUDA_TRY(c, cudaStreamWaitEvent(static_cast<cudaStream_t>(consumer_stream), c->comm_done, 0));
      c->ce_used = c->ce2_used = false;
      std::fill(c->lane_used, c->lane_used + kMaxLanes, false);
      std::fill(c->rr_used.begin(), c->rr_used.end(), 0);
    }
  }
  c->unwaited.clear();
  for (Bucket& bk : c->buckets) std::fill(bk.grads.begin(), bk.grads.end(), nullptr);
  c->last_trace = c->trace;
  c->last_order = c->order;
  c->state = State::IDLE;  // pending counts are replenished at the next pass open
  return DDP_OK;
}

ddp_status_t ddp_no_sync_begin(ddp_ctx_t* c) {
  if (ddp_status_t st = check_ctx(c)) return st;
  if (c->state == State::IN_PASS) return fail(DDP_ERR_STATE, "no_sync toggled inside a backward pass");
  if (c->no_sync) return fail(DDP_ERR_STATE, "nested no_sync");
  c->no_sync = true;
  return DDP_OK;
}

ddp_status_t ddp_no_sync_end(ddp_ctx_t* c) {
  if (ddp_status_t st = check_ctx(c)) return st;
  if (c->state == State::IN_PASS) return fail(DDP_ERR_STATE, "no_sync toggled inside a backward pass");
  if (!c->no_sync) return fail(DDP_ERR_STATE, "no_sync_end without no_sync_begin");
  c->no_sync = false;
  return DDP_OK;
}

ddp_status_t ddp_set_option(ddp_ctx_t* c, int32_t key, int64_t v) {
  if (ddp_status_t st = check_ctx(c)) return st;
  if (c->state == State::IN_PASS) return fail(DDP_ERR_STATE, "options cannot change inside a pass");
  if (is_layout_key(key) && c->bound) return fail(DDP_ERR_STATE, "layout options are fixed once bound");
  switch (key) {
    case DDP_OPT_OVERLAP: c->overlap = v ? 1 : 0; return DDP_OK;
    case DDP_OPT_PROFILE: c->profile = v ? 1 : 0; return DDP_OK;
    case DDP_OPT_DRY_RUN:
      if (c->bound) return fail(DDP_ERR_STATE, "dry-run only before binding");
      c->dry_run = v ? 1 : 0;
      return DDP_OK;
    case DDP_OPT_P2P_ONESHOT_MAX:
      if (v < 0) return fail(DDP_ERR_INVALID_ARG, "negative threshold");
      c->oneshot_max = v;
      break;
    case DDP_OPT_P2P_TWOSHOT_MAX:
      if (v < 0) return fail(DDP_ERR_INVALID_ARG, "negative threshold");
      c->twoshot_max = v;
      break;
    case DDP_OPT_ALGO:
      if (v < DDP_ALGO_AUTO || v > DDP_ALGO_CE2) return fail(DDP_ERR_INVALID_ARG, "bad algo");
      c->algo = v;
      break;
    case DDP_OPT_FIND_UNUSED:
      if (v && c->grad_view) return fail(DDP_ERR_UNSUPPORTED, "FIND_UNUSED with GRAD_VIEW");
      c->find_unused = v ? 1 : 0;
      break;
    case DDP_OPT_GRAD_VIEW:
      if (v && (c->find_unused || c->wire_bf16))
        return fail(DDP_ERR_UNSUPPORTED, "GRAD_VIEW with FIND_UNUSED or WIRE_BF16");
      c->grad_view = v ? 1 : 0;
      break;
    case DDP_OPT_MULTICAST:
      c->multicast = v ? 1 : 0;
      break;
    case DDP_OPT_CE_DIRECT_BYTES:
      if (v < 0) return fail(DDP_ERR_INVALID_ARG, "negative CE_DIRECT_BYTES");
      c->ce_direct = v;
      break;
    case DDP_OPT_PREFER_OVERLAP:
      if (v < 0 || v > 2) return fail(DDP_ERR_INVALID_ARG, "PREFER_OVERLAP must be 0, 1 or 2");
      c->prefer_overlap = v;
      break;
    case DDP_OPT_LOW_PRIORITY:
      if (c->bound) return fail(DDP_ERR_STATE, "LOW_PRIORITY is fixed once bound");
      c->low_priority = v ? 1 : 0;
      return DDP_OK;
    case DDP_OPT_LANES:
      if (v < 1 || v > kMaxLanes) return fail(DDP_ERR_INVALID_ARG, "LANES must be in [1, 4]");
      c->lanes = v;
      break;
    case DDP_OPT_WIRE_BF16:
      if (v && c->dtype != DDP_FP32) return fail(DDP_ERR_INVALID_ARG, "WIRE_BF16 compresses fp32 gradients only");
      if (v && c->grad_view) return fail(DDP_ERR_UNSUPPORTED, "WIRE_BF16 with GRAD_VIEW");
      c->wire_bf16 = v ? 1 : 0;
      break;
    case DDP_OPT_NCCL_COMMS:
      if (c->bound) return fail(DDP_ERR_STATE, "NCCL_COMMS is fixed once bound");
      if (v < 1 || v > 8) return fail(DDP_ERR_INVALID_ARG, "NCCL_COMMS must be in [1, 8]");
      c->nccl_comms = v;
      return DDP_OK;
    case DDP_OPT_CE_STREAMS:
      if (c->bound) return fail(DDP_ERR_STATE, "CE_STREAMS is fixed once bound");
      if (v < 1 || v > 16) return fail(DDP_ERR_INVALID_ARG, "CE_STREAMS must be in [1, 16]");
      c->ce_streams = v;
      return DDP_OK;
    case DDP_OPT_COMM_CTAS:
      if (v < 1 || v > 148) return fail(DDP_ERR_INVALID_ARG, "COMM_CTAS must be in [1, 148]");
      c->comm_ctas = v;
      regrid(c);
      return DDP_OK;
    case DDP_OPT_PACK_CTAS:
      if (v < 1 || v > 148 * 64) return fail(DDP_ERR_INVALID_ARG, "PACK_CTAS must be in [1, 9472]");
      c->pack_ctas = v;
      regrid(c);
      return DDP_OK;
    case DDP_OPT_P2P_TIMEOUT_MS:
      if (v < 1) return fail(DDP_ERR_INVALID_ARG, "P2P_TIMEOUT_MS must be >= 1");
      c->p2p_timeout_ms = v;
      return DDP_OK;
    case DDP_OPT_WAIT_TIMEOUT_MS:
      if (v < 1) return fail(DDP_ERR_INVALID_ARG, "WAIT_TIMEOUT_MS must be >= 1");
      c->wait_timeout_ms = v;
      return DDP_OK;
    case DDP_OPT_P2P_PULL:
      if (v < 0 || v > 2) return fail(DDP_ERR_INVALID_ARG, "P2P_PULL must be 0, 1 or 2");
      c->p2p_pull = v;
      break;
    case DDP_OPT_P2P_SIGNAL:
      if (v < 0 || v > 3) return fail(DDP_ERR_INVALID_ARG, "P2P_SIGNAL must be 0..3");
      c->p2p_signal = v;
      return DDP_OK;
    case DDP_OPT_LAST_ON_PRODUCER:
      c->last_on_producer = v ? 1 : 0;
      return DDP_OK;
    case DDP_OPT_P2P_DEBUG:
      if (v < 0 || v > 7) return fail(DDP_ERR_INVALID_ARG, "P2P_DEBUG must be 0..7");
      c->p2p_debug = v;
      return DDP_OK;
    case DDP_OPT_EMU_DEAD_RANK:
      if (v < -1 || v >= c->world) return fail(DDP_ERR_INVALID_ARG, "EMU_DEAD_RANK must be -1 or a rank");
      c->emu_dead_rank = v;
      return DDP_OK;
    case DDP_OPT_P2P_STAGE_BYTES:
      if (v < 0) return fail(DDP_ERR_INVALID_ARG, "negative stage bytes");
      c->stage_bytes = v;
      regrid(c);
      return DDP_OK;
    default:
      return fail(DDP_ERR_INVALID_ARG, "unknown option key");
  }
  plan(c);  // layout keys
  return DDP_OK;
}

ddp_status_t ddp_get_option(const ddp_ctx_t* c, int32_t key, int64_t* v) {
  if (!c || !v) return fail(DDP_ERR_INVALID_ARG, "null argument");
  switch (key) {
    case DDP_OPT_OVERLAP: *v = c->overlap; break;
    case DDP_OPT_P2P_ONESHOT_MAX: *v = c->oneshot_max; break;
    case DDP_OPT_P2P_TWOSHOT_MAX: *v = c->twoshot_max; break;
    case DDP_OPT_COMM_CTAS: *v = c->comm_ctas; break;
    case DDP_OPT_DRY_RUN: *v = c->dry_run; break;
    case DDP_OPT_PROFILE: *v = c->profile; break;
    case DDP_OPT_ALGO: *v = c->algo; break;
    case DDP_OPT_PACK_CTAS: *v = c->pack_ctas; break;
    case DDP_OPT_P2P_STAGE_BYTES: *v = c->stage_bytes; break;
    case DDP_OPT_FIND_UNUSED: *v = c->find_unused; break;
    case DDP_OPT_MULTICAST: *v = c->multicast; break;
    case DDP_OPT_CE_STREAMS: *v = c->ce_streams; break;
    case DDP_OPT_NCCL_COMMS: *v = c->nccl_comms; break;
    case DDP_OPT_CE_DIRECT_BYTES: *v = c->ce_direct; break;
    case DDP_OPT_WIRE_BF16: *v = c->wire_bf16; break;
    case DDP_OPT_LANES: *v = c->lanes; break;
    case DDP_OPT_LOW_PRIORITY: *v = c->low_priority; break;
    case DDP_OPT_PREFER_OVERLAP: *v = c->prefer_overlap; break;
    case DDP_OPT_GRAD_VIEW: *v = c->grad_view; break;
    case DDP_OPT_P2P_TIMEOUT_MS: *v = c->p2p_timeout_ms; break;
    case DDP_OPT_WAIT_TIMEOUT_MS: *v = c->wait_timeout_ms; break;
    case DDP_OPT_EMU_DEAD_RANK: *v = c->emu_dead_rank; break;
    case DDP_OPT_P2P_PULL: *v = c->p2p_pull; break;
    case DDP_OPT_P2P_SIGNAL: *v = c->p2p_signal; break;
    case DDP_OPT_P2P_DEBUG: *v = c->p2p_debug; break;
    case DDP_OPT_LAST_ON_PRODUCER: *v = c->last_on_producer; break;
    default: return fail(DDP_ERR_INVALID_ARG, "unknown option key");
  }
  return DDP_OK;
}

ddp_status_t ddp_launch_trace(const ddp_ctx_t* c, int32_t* buckets, int32_t* triggers, int32_t cap, int32_t* n) {
  if (!c || !n || cap < 0) return fail(DDP_ERR_INVALID_ARG, "bad argument");
  const auto& t = c->state == State::IN_PASS ? c->trace : c->last_trace;
  *n = (int32_t)t.size();
  for (int32_t i = 0; i < cap && i < (int32_t)t.size(); ++i) {
    if (buckets) buckets[i] = t[i].first;
    if (triggers) triggers[i] = t[i].second;
  }
  return DDP_OK;
}

ddp_status_t ddp_ready_order(const ddp_ctx_t* c, int32_t* out, int32_t cap, int32_t* n) {
  if (!c || !n || cap < 0) return fail(DDP_ERR_INVALID_ARG, "bad argument");
  const auto& o = c->state == State::IN_PASS ? c->order : c->last_order;
  *n = (int32_t)o.size();
  for (int32_t i = 0; i < cap && i < (int32_t)o.size(); ++i)
    if (out) out[i] = o[i];
  return DDP_OK;
}

ddp_status_t ddp_broadcast(ddp_ctx_t* c, void* const* bufs, const int64_t* bytes, int32_t n, int32_t root,
                           void* stream) {
  if (ddp_status_t st = check_ctx(c)) return st;
  if (!c->bound || c->emulated || !c->nccl) return fail(DDP_ERR_STATE, "ddp_broadcast needs a bound communicator");
  if (c->state == State::IN_PASS) return fail(DDP_ERR_STATE, "ddp_broadcast inside a backward pass");
  if (n < 0 || (n > 0 && (!bufs || !bytes)) || root < 0 || root >= c->world)
    return fail(DDP_ERR_INVALID_ARG, "bad broadcast arguments");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  NCCL_TRY(c, ncclGroupStart());
  for (int32_t i = 0; i < n; ++i) {
    if (bytes[i] < 0 || (bytes[i] > 0 && !bufs[i])) {
      ncclGroupEnd();
      return fail(DDP_ERR_INVALID_ARG, "bad broadcast buffer");
    }
    if (bytes[i] == 0) continue;
    NCCL_TRY(c, ncclBroadcast(bufs[i], bufs[i], (size_t)bytes[i], ncclUint8, root, c->nccl, s));
  }
  NCCL_TRY(c, ncclGroupEnd());
  return DDP_OK;
}

ddp_status_t ddp_profile_read(ddp_ctx_t* c, double ms[6], int64_t launches[6]) {
  if (ddp_status_t st = check_ctx(c)) return st;
  if (!ms || !launches) return fail(DDP_ERR_INVALID_ARG, "null argument");
  for (int k = 0; k < 6; ++k) {
    ms[k] = 0;
    launches[k] = 0;
  }
  for (auto& r : c->prof) {
    CUDA_TRY(c, cudaEventSynchronize(r.b));
    float t = 0;
    CUDA_TRY(c, cudaEventElapsedTime(&t, r.a, r.b));
    ms[r.kind] += t;
    launches[r.kind] += 1;
  }
  return ddp_profile_timeline(c, 0, nullptr, nullptr, nullptr, nullptr, nullptr);
}

ddp_status_t ddp_profile_timeline(ddp_ctx_t* c, int32_t cap, int32_t* kinds, double* ready_ms, double* start_ms,
                                  double* end_ms, int32_t* n) {
  if (ddp_status_t st = check_ctx(c)) return st;
  if (cap < 0) return fail(DDP_ERR_INVALID_ARG, "negative cap");
  if (n) *n = (int32_t)c->prof.size();
  cudaEvent_t base = c->prof_ready.empty() ? nullptr : c->prof_ready.front();
  for (size_t i = 0; i < c->prof.size(); ++i) {
    const ProfRec& r = c->prof[i];
    CUDA_TRY(c, cudaEventSynchronize(r.b));
    if ((int32_t)i < cap && base) {
      float t0 = 0, t1 = 0, t2 = 0;
      if (r.ready >= 0) CUDA_TRY(c, cudaEventElapsedTime(&t0, base, c->prof_ready[r.ready]));
      CUDA_TRY(c, cudaEventElapsedTime(&t1, base, r.a));
      CUDA_TRY(c, cudaEventElapsedTime(&t2, base, r.b));
      if (kinds) kinds[i] = r.kind;
      if (ready_ms) ready_ms[i] = t0;
      if (start_ms) start_ms[i] = t1;
      if (end_ms) end_ms[i] = t2;
    }
  }
  for (auto& r : c->prof) {
    c->event_pool.push_back(r.a);
    c->event_pool.push_back(r.b);
  }
  for (cudaEvent_t e : c->prof_ready) c->event_pool.push_back(e);
  c->prof.clear();
  c->prof_ready.clear();
  return DDP_OK;
}

ddp_status_t ddp_check_device_errors(ddp_ctx_t* c) {
  if (ddp_status_t st = check_ctx(c)) return st;
  if ((c->err_host && *reinterpret_cast<volatile uint32_t*>(c->err_host)) || emu_error_word(c)) {
    c->poisoned = true;
    return fail(DDP_ERR_TIMEOUT, "a peer never reached a P2P barrier (timeout)");
  }
  if (c->nccl) {
    ncclResult_t ar = ncclSuccess;
    if (ncclCommGetAsyncError(c->nccl, &ar) == ncclSuccess && ar != ncclSuccess && ar != ncclInProgress)
      return nccl_fail(c, ar, "NCCL async error");
  }
  // Host watchdog over the waits that have no device-side bound (the copy-engine
  // exchanges' cuStreamWaitValue32, NCCL): a finalized pass that has not completed
  // DDP_OPT_WAIT_TIMEOUT_MS later is reported, and the context poisoned, so the
  // caller can tear down instead of blocking forever ("could hang").
  if (c->watch) {
    const cudaError_t q = cudaEventQuery(c->comm_done);
    if (q == cudaSuccess) {
      c->watch = false;
    } else if (q == cudaErrorNotReady) {
      (void)cudaGetLastError();  // not an error: do not leave it for the caller's next check
      const auto ms = std::chrono::duration_cast<std::chrono::milliseconds>(std::chrono::steady_clock::now() -
                                                                            c->done_since).count();
      if (ms > c->wait_timeout_ms) {
        c->poisoned = true;
        return fail(DDP_ERR_TIMEOUT, "a finalized pass has not completed " + std::to_string(ms) +
                                         " ms after ddp_finalize_backward (a peer never raised a flag this "
                                         "rank waits on, or a collective is stuck)");
      }
    } else {
      return cuda_fail(c, q, "cudaEventQuery(pass end)");
    }
  }
  return DDP_OK;
}

}  // extern "C"
