// ctx.h — private state of the host core (not part of the ABI): the
// per-bucket plan, the protocol state of a pass (§3.2, Alg. 1), the
// device resources (streams, events, flags) and the helpers shared by
// core/reducer.cpp (assignment, protocol, C ABI) and core/exchange.cpp (the
// device work launched per bucket).
#pragma once

#include <cuda.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <string>
#include <utility>
#include <vector>

#include "../internal.h"
#include "b200ddp.h"

namespace b200ddp {

// thread-local error message for ddp_last_error(); returns st
ddp_status_t fail(ddp_status_t st, const std::string& msg);

inline int64_t align_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }
inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

constexpr int64_t kMinChunkElems = 4096;   // smallest per-CTA chunk worth a CTA
// Pipeline stage per CTA.  A cross-GPU sync point costs ~4-8 us of fence plus
// ~3 us of flag flight (tools/sync_probe.cu on B200), so the default is one
// stage per chunk (one sync for one-shot, two for two-shot); DDP_OPT_P2P_STAGE_BYTES
// splits chunks for experiments.
constexpr int64_t kBarrierScratch = 32 * 1024;  // scratch int inside the flags region
constexpr int64_t kPullStageBytes = 32 * 1024;  // default pipeline stage of the pull kernels
constexpr int kMaxLanes = 4;
constexpr int64_t kCeWireAlign = 64;  // elements: wire offsets keep 16-B (and 256-B) alignment
constexpr int kCeFlagKinds = 4;       // stream-memop flags per bucket: ready, consumed, gathered, bitmap

struct EmuGroup;  // peer emulation (core/emulation.cpp)

struct Bucket {
  int64_t numel = 0;
  std::vector<int32_t> params;  // slot -> param, scan (reverse registration) order
  std::vector<int64_t> off;     // slot offsets, n+1 entries
  std::vector<void*> grads;     // slot -> gradient pointer supplied this pass
  int64_t byte_off = 0;         // inside the symmetric storage
  int64_t alt_off = 0;          // pull kernels: second buffer (pass parity), inside the storage
  uint32_t p2p_count = 0;       // fused launches of this bucket so far (pass parity)
  bool pull = false;            // fused bucket run by the pull kernels (kernels/pull.cu)
  int algo = DDP_ALGO_NCCL;
  int ctas = 1;
  int64_t shard = 0, chunk = 0, sub = 0;
  int32_t stages = 0;
  // copy-engine algorithm: W slots at ce_off + q * ce_stride (wire layout: direct
  // gradients, then the gathered small ones from ce_small0); passes launched so far
  int64_t ce_off = 0, ce_stride = 0, ce_small0 = 0, ce_wire_numel = 0;
  std::vector<int64_t> ce_wire;     // per slot: element offset in a slot
  std::vector<uint8_t> ce_direct;   // per slot: copied by the copy engine straight from .grad
  uint32_t ce_count = 0;
};

enum class State { CREATED, IDLE, IN_PASS };

struct ProfRec {
  int kind;
  cudaEvent_t a, b;
  int ready;  // index into ddp_ctx::prof_ready (producer-stream event at launch time)
};

}  // namespace b200ddp

using namespace b200ddp;

struct ddp_ctx {
  // configuration
  int32_t world = 1, rank = 0, dtype = 0, esize = 4;
  int64_t cap = 0;
  std::vector<int64_t> numel;
  std::vector<int32_t> scan;  // bucketing scan order (default: reverse registration)
  std::vector<Bucket> buckets;
  std::vector<int32_t> p_bucket, p_slot;
  std::vector<int64_t> p_off;
  // options
  // oneshot_max < 0: automatic (<= 1 MiB at every world size)
  int64_t overlap = 1, oneshot_max = -1, twoshot_max = INT64_MAX,
          comm_ctas = 32,  // x 4 lanes: measured best exposed time at W=4 (profiles/r01_n4.md)
          dry_run = 0, profile = 0, algo = DDP_ALGO_AUTO,
          pack_ctas = 148 * 32,  // many small CTAs balance best on HBM-bound copies (tools/local_probe.cu)
          stage_bytes = 0,
          find_unused = 0, multicast = 0, ce_streams = 1, nccl_comms = 1,
          // CE: gradients of at least this many bytes travel straight from .grad (one
          // cudaMemcpyAsync per peer, a few us of host + copy-engine fixed cost each);
          // smaller ones are gathered into one region first (2x their bytes of HBM)
          ce_direct = 16 << 20,
          wire_bf16 = 0,  // N-3: fp32 gradients travel as bf16 (CE exchange)
          // P2P / NVLS kernels of consecutive buckets run on `lanes` streams (bucket b on
          // lane b mod lanes), each with its own barrier flags, sequence and staging, so
          // bucket b+1's local phases overlap bucket b's NVLink phase
          lanes = 4,
          low_priority = 1;  // library streams at the lowest priority: backward's kernels first
                             // (measured: exposed 3.1 -> 2.8% at W=2, 9.3 -> 9.0% at W=4)
  int64_t prefer_overlap = 0;  // policy for buckets synced under a running backward (see resolve_algo)
  int64_t grad_view = 0;       // N-3 zero-copy: gradients live in their bucket slots (NCCL in place)
  int64_t p2p_timeout_ms = 30000;   // bound of every P2P / NVLS barrier spin (%globaltimer)
  int64_t wait_timeout_ms = 60000;  // bound of a host wait for a peer's issue (peer emulation) and
                                    // of a finalized pass's completion (ddp_check_device_errors)
  int64_t emu_dead_rank = -1;       // test support (cooperative emulation): this rank never signals
  int64_t p2p_pull = 1;             // fused kernels: 0 push everywhere, 1 pull for the last bucket, 2 pull everywhere
  int64_t p2p_signal = 0;           // pull kernels: flag publication mode (DDP_OPT_P2P_SIGNAL)
  int64_t p2p_debug = 0;            // measurement only: skip data phases (DDP_OPT_P2P_DEBUG)
  int64_t last_on_producer = 1;     // the pass's last fused bucket runs on its producer stream
  // symmetric storage layout (bytes)
  int64_t flags_off = 0, buckets_off = 0, stage2_off = 0, stage2_stride = 0, stage1_off = 0,
          stage1_stride = 0, ce_flags_off = 0, bitmap_off = 0, bitmap_stride = 0, global_off = 0,
          scratch_off = 0, storage_bytes = 0;
  // find_unused: local participation since the last
  // synced pass, this pass's locally-unused parameters and their destinations
  std::vector<uint8_t> used_local;
  std::vector<int32_t> un_param;
  std::vector<void*> un_dst;
  std::vector<const void*> un_src;
  std::vector<int64_t> un_numel;
  int32_t* bitmap_host = nullptr;   // pinned: local bitmap (H2D source)
  int32_t* global_host = nullptr;   // pinned: summed bitmap (D2H target)
  cudaEvent_t bitmap_done = nullptr;
  bool bitmap_valid = false;
  uint32_t un_count = 0;            // synced find_unused passes (bitmap exchange flag value)
  // copy-engine path: reduce stream, events, driver stream-memory-op entry points
  cudaStream_t ce_red = nullptr, ce_pack = nullptr;
  cudaStream_t ce_ag = nullptr, ce_up = nullptr;  // CE2: all-gather copies, unpack
  std::vector<cudaEvent_t> ce_reduced;             // CE2, per bucket: own shard reduced
  std::vector<cudaStream_t> ce2_rs, ce2_ag;        // CE2: one reduce-scatter / all-gather stream per peer
  std::vector<cudaEvent_t> ce2_done;               // CE2: joins those streams at finalize
  bool ce2_used = false;
  std::vector<cudaEvent_t> ce_packed;  // per bucket: small gradients gathered (pack -> comm stream)
  std::vector<cudaEvent_t> ce_copied;  // per bucket: copies issued (comm -> reduce stream)
  std::vector<void*> ce_grad;          // scratch argument arrays
  std::vector<int64_t> ce_wire, ce_numel;
  cudaEvent_t ce_red_done = nullptr;
  void* fn_write32 = nullptr;
  void* fn_wait32 = nullptr;
  bool ce_used = false;  // a CE bucket was launched in the open pass
  // protocol state
  State state = State::CREATED;
  bool bound = false, emulated = false, poisoned = false;
  // peer emulation: this context is ONE of `world` contexts (one per rank) in one
  // process on one device, each driven by its own host thread (core/emulation.cpp)
  bool peer_emu = false;
  EmuGroup* emu = nullptr;
  cudaEvent_t emu_pre[kMaxLanes] = {};
  bool no_sync = false, pass_no_sync = false;
  bool pass_launched = false;    // a device launch happened in the open pass
  bool comm_done_valid = false;  // comm_done recorded by an earlier finalize
  bool watch = false;            // comm_done not yet seen complete by ddp_check_device_errors
  std::chrono::steady_clock::time_point done_since;  // finalize of the oldest pass not seen complete
  std::vector<uint8_t> ready;
  std::vector<int32_t> pending;
  int32_t cursor = 0, n_ready = 0;
  std::vector<std::pair<int32_t, int32_t>> trace, last_trace;
  std::vector<int32_t> order, last_order;  // ready-signal order of the open / last finished pass
  // device state
  int device = -1;
  cudaStream_t comm = nullptr;
  ncclComm_t nccl = nullptr;
  // round-robin process groups: NCCL bucket b runs on communicator
  // b mod k and its own stream (index 0 = the main communicator / comm stream)
  std::vector<ncclComm_t> rr_comm;
  std::vector<cudaStream_t> rr_stream;
  std::vector<cudaEvent_t> rr_done;
  std::vector<uint8_t> rr_used;
  void* storage[kMaxWorld] = {};
  void* mc = nullptr;  // NVLS multicast address of the storage base
  int64_t grad_rank_stride = 0;
  std::vector<cudaStream_t> unwaited;  // producer streams since the last event wait
  cudaStream_t producer = nullptr;     // stream of the most recent ready signal
  bool from_signal = false;            // device work issued from a ready signal (not finalize)
  cudaStream_t last_on = nullptr;      // the pass's last bucket ran on this producer stream
  cudaStream_t done_stream = nullptr;  // stream comm_done was last recorded on
  bool lone_last = false;              // this pass's only device work: the last bucket on its producer
  std::vector<cudaEvent_t> join_ev;    // joins of library streams into last_on
  std::vector<std::pair<cudaStream_t, cudaEvent_t>> stream_events;
  cudaEvent_t comm_done = nullptr;
  uint32_t p2p_seq[kMaxLanes] = {1, 1, 1, 1};
  uint64_t p2p_launches[kMaxLanes] = {};
  cudaStream_t lane_stream[kMaxLanes] = {};  // [0] = comm
  cudaEvent_t lane_done[kMaxLanes] = {};
  bool lane_used[kMaxLanes] = {};
  uint32_t* err_host = nullptr;
  uint32_t* err_dev = nullptr;
  std::vector<ProfRec> prof;
  std::vector<cudaEvent_t> prof_ready;
  std::vector<cudaEvent_t> event_pool;
  // scratch for world-1 group launches
  std::vector<int64_t> g_off, g_dst;
  std::vector<void*> g_grad;
  // batched ready signals: device launches deferred to the end of the batch
  bool defer = false;
  int32_t defer_b0 = 0, defer_b1 = 0;
};

namespace b200ddp {

// Lanes run spinning P2P kernels side by side: all of them must fit on the SMs at
// once (one CTA per SM guaranteed), else a lane could wait for a peer lane that
// cannot be scheduled.  Same options on every rank -> same choice everywhere.
inline int lanes_in_use(const ddp_ctx* c) {
  return c->lanes * std::min<int64_t>(c->comm_ctas, kMaxCtas) <= 148 ? (int)c->lanes : 1;
}

// error paths: record the message, poison the context (CUDA / NCCL failures are fatal)
ddp_status_t cuda_fail(ddp_ctx* c, cudaError_t e, const char* what);
ddp_status_t nccl_fail(ddp_ctx* c, ncclResult_t r, const char* what);
#define CUDA_TRY(c, expr)                                   \
  do {                                                      \
    cudaError_t _e = (expr);                                \
    if (_e != cudaSuccess) return cuda_fail((c), _e, #expr); \
  } while (0)
#define NCCL_TRY(c, expr)                                   \
  do {                                                      \
    ncclResult_t _r = (expr);                               \
    if (_r != ncclSuccess) return nccl_fail((c), _r, #expr); \
  } while (0)

// ---- core/exchange.cpp ----------------------------------------------------------
cudaEvent_t pool_event(ddp_ctx* c);
void prof_begin(ddp_ctx* c, int kind, cudaStream_t s = nullptr);
void prof_end(ddp_ctx* c, cudaStream_t s = nullptr);
// device work of buckets [b0, b1), in order (a3/a4/a6), after the producer streams (a5)
ddp_status_t device_range(ddp_ctx* c, int b0, int b1);
// find_unused, end of a synced pass: bitmap allreduce + write-back (N-1)
ddp_status_t finish_unused(ddp_ctx* c);
// library side streams, events and stream-memop entry points (both bind paths)
ddp_status_t create_side_streams(ddp_ctx* c);

// ---- core/emulation.cpp (peer emulation: W contexts, one device, one host thread each) ----
// join / leave the group of contexts sharing storages[0]; join blocks until every
// rank has joined (the bind-time barrier of the multi-process path)
ddp_status_t emu_join(ddp_ctx* c);
void emu_leave(ddp_ctx* c);
// a stream write of value v to addr has been issued (enqueued) by this host thread
void emu_issued(ddp_ctx* c, const uint32_t* addr, uint32_t v);
// block the host until some thread has issued a write of >= v to addr (bounded)
ddp_status_t emu_await_issue(ddp_ctx* c, const uint32_t* addr, uint32_t v);
// fused P2P kernels (they spin on peers' flags): the W ranks meet on the host and
// ONE cooperative kernel runs all of them, ordered after / before each rank's lane stream
ddp_status_t emu_p2p_launch(ddp_ctx* c, int algo, const SlotView& sv, const P2PLaunch& a, cudaStream_t ls,
                            int lane);
uint32_t emu_error_word(const ddp_ctx* c);

}  // namespace b200ddp
