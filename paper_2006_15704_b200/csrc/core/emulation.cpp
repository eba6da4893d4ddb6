// emulation.cpp — peer emulation (test support, include/b200ddp_emu.h): the W
// ranks of a data-parallel job as W contexts in ONE process on ONE device, each
// driven by its own host thread exactly as a rank's process drives its context
// (one process per replica; here one thread per replica).  Every
// context runs the product code unchanged — assignment, ready tracking, launch
// order, the copy-engine exchanges with their stream-memory-operation flags,
// find_unused's bitmap exchange — over peer storages that all live on this
// device.  Two things differ from the multi-process path, both because the
// ranks now share one GPU:
//
//  * Issue order of stream waits.  A cuStreamWaitValue32 is invisible to the
//    CUDA scheduler, and streams may share a hardware queue.  In a rank's own
//    process every flag it waits for is written by ANOTHER GPU, so a blocked
//    wait can only hold back that rank's own later work.  With all ranks on one
//    GPU, a wait issued before the peer's matching write could sit ahead of that
//    write in a shared queue forever.  So the host holds each wait back until
//    some thread has issued (enqueued) the write it waits for (emu_await_issue):
//    every operation then depends only on operations issued before it, and
//    nothing can deadlock.  A peer that never issues the write makes the wait
//    fail after DDP_OPT_WAIT_TIMEOUT_MS with DDP_ERR_TIMEOUT (poisoned context).
//  * Kernels that spin on peers' flags (the fused one-shot / two-shot P2P
//    kernels) must never run as separate launches on one GPU: nothing makes them
//    co-resident.  The W ranks instead meet on the host at each such launch
//    (same lane, same sequence on every rank), and the last to arrive
//    runs ONE cooperative kernel over all ranks (blockIdx.y = rank, as
//    ddp_bind_emulated does), ordered after every rank's lane stream and before
//    every rank's next work on it.
//
// The bind-time barrier of the multi-process path (an NCCL allreduce) is a host
// barrier here: every rank has zeroed its flags before any rank issues work.
#include <chrono>
#include <condition_variable>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "ctx.h"

namespace b200ddp {

struct EmuDep {
  P2PLaunch a;
  SlotView sv;
  int algo;
  cudaEvent_t pre;
};

struct EmuRdv {
  uint64_t gen = 0;
  int arrived = 0;
  ddp_status_t status = DDP_OK;
  std::string msg;
  EmuDep dep[kMaxWorld];
};

struct EmuGroup {
  void* key = nullptr;  // storages[0]
  int world = 0, device = -1;
  int refs = 0, joined = 0;
  bool dead = false;  // a member timed out waiting for a peer: everyone fails fast
  std::mutex mu;
  std::condition_variable cv;
  std::unordered_map<uintptr_t, uint32_t> issued;  // flag address -> largest value issued
  EmuRdv rdv[kMaxLanes];
  cudaStream_t lane[kMaxLanes] = {};
  cudaEvent_t done[kMaxLanes] = {};
  uint32_t* err_host = nullptr;
  uint32_t* err_dev = nullptr;
};

namespace {
std::mutex g_groups_mu;
std::vector<EmuGroup*> g_groups;

std::chrono::milliseconds timeout_of(const ddp_ctx* c) { return std::chrono::milliseconds(c->wait_timeout_ms); }

// "kind k of bucket b from src" for a CE flag address in this rank's storage
std::string describe_flag(const ddp_ctx* c, const uint32_t* addr) {
  const uint32_t* base = reinterpret_cast<const uint32_t*>(static_cast<const char*>(c->storage[c->rank]) +
                                                           c->ce_flags_off);
  const int64_t idx = addr - base, nb = (int64_t)c->buckets.size();
  static const char* kinds[kCeFlagKinds] = {"ready", "consumed", "gathered", "bitmap"};
  const int64_t kind = idx / (kMaxWorld * nb), b = (idx / kMaxWorld) % nb, src = idx % kMaxWorld;
  if (idx < 0 || kind >= kCeFlagKinds) return "flag";
  return std::string(kinds[kind]) + " flag of bucket " + std::to_string(b) + " from rank " + std::to_string(src);
}
}  // namespace

ddp_status_t emu_join(ddp_ctx* c) {
  EmuGroup* g = nullptr;
  {
    std::lock_guard<std::mutex> lk(g_groups_mu);
    for (EmuGroup* x : g_groups)
      if (x->key == c->storage[0] && x->world == c->world && x->joined < x->world && !x->dead) g = x;
    if (!g) {
      g = new EmuGroup();
      g->key = c->storage[0];
      g->world = c->world;
      g->device = c->device;
      g_groups.push_back(g);
    }
    g->refs++;
  }
  c->emu = g;
  std::unique_lock<std::mutex> lk(g->mu);
  if (!g->err_host) {  // first member: the group's lanes for the cooperative P2P launches
    CUDA_TRY(c, cudaHostAlloc(reinterpret_cast<void**>(&g->err_host), sizeof(uint32_t), cudaHostAllocMapped));
    *g->err_host = 0;
    CUDA_TRY(c, cudaHostGetDevicePointer(reinterpret_cast<void**>(&g->err_dev), g->err_host, 0));
    for (int k = 0; k < kMaxLanes; ++k) {
      CUDA_TRY(c, cudaStreamCreateWithFlags(&g->lane[k], cudaStreamNonBlocking));
      CUDA_TRY(c, cudaEventCreateWithFlags(&g->done[k], cudaEventDisableTiming));
    }
  }
  g->joined++;
  g->cv.notify_all();
  if (!g->cv.wait_for(lk, timeout_of(c), [&] { return g->joined == g->world || g->dead; }) || g->dead) {
    g->dead = true;
    g->cv.notify_all();
    c->poisoned = true;
    return fail(DDP_ERR_TIMEOUT, "peer emulation: not every rank bound its context (bind barrier timed out)");
  }
  return DDP_OK;
}

void emu_leave(ddp_ctx* c) {
  EmuGroup* g = c->emu;
  if (!g) return;
  c->emu = nullptr;
  std::lock_guard<std::mutex> lk(g_groups_mu);
  if (--g->refs > 0) return;
  for (int k = 0; k < kMaxLanes; ++k) {
    if (g->lane[k]) {
      if (!g->dead) cudaStreamSynchronize(g->lane[k]);
      cudaStreamDestroy(g->lane[k]);
    }
    if (g->done[k]) cudaEventDestroy(g->done[k]);
  }
  if (g->err_host) cudaFreeHost(g->err_host);
  for (size_t i = 0; i < g_groups.size(); ++i)
    if (g_groups[i] == g) {
      g_groups.erase(g_groups.begin() + (long)i);
      break;
    }
  delete g;
}

void emu_issued(ddp_ctx* c, const uint32_t* addr, uint32_t v) {
  EmuGroup* g = c->emu;
  std::lock_guard<std::mutex> lk(g->mu);
  uint32_t& x = g->issued[reinterpret_cast<uintptr_t>(addr)];
  if ((int32_t)(v - x) > 0) x = v;
  g->cv.notify_all();
}

ddp_status_t emu_await_issue(ddp_ctx* c, const uint32_t* addr, uint32_t v) {
  EmuGroup* g = c->emu;
  std::unique_lock<std::mutex> lk(g->mu);
  auto ok = [&] {
    auto it = g->issued.find(reinterpret_cast<uintptr_t>(addr));
    return it != g->issued.end() && (int32_t)(it->second - v) >= 0;
  };
  if (!g->cv.wait_for(lk, timeout_of(c), [&] { return ok() || g->dead; }) || (g->dead && !ok())) {
    g->dead = true;
    g->cv.notify_all();
    c->poisoned = true;
    return fail(DDP_ERR_TIMEOUT, "peer emulation: the " + describe_flag(c, addr) + " (pass " + std::to_string(v) +
                                     ") was never issued: a peer never reached this step");
  }
  return DDP_OK;
}

// The last rank to arrive launches the cooperative kernel for all of them.
// Called with g->mu held.
static ddp_status_t launch_all(ddp_ctx* c, EmuGroup* g, EmuRdv& R, int lane, std::string& msg) {
  const int W = g->world;
  const EmuDep& d0 = R.dep[0];
  const int64_t stride = (const char*)R.dep[1].sv.grad[0] - (const char*)d0.sv.grad[0];
  for (int r = 0; r < W; ++r) {
    const EmuDep& d = R.dep[r];
    bool same = d.algo == d0.algo && d.sv.n == d0.sv.n && d.a.numel == d0.a.numel && d.a.ctas == d0.a.ctas &&
                d.a.seq == d0.a.seq && d.a.stage_byte_off == d0.a.stage_byte_off &&
                d.a.bucket_byte_off == d0.a.bucket_byte_off;
    for (int k = 0; same && !d.a.view && k < d.sv.n; ++k)  // the in-place form uses no slot table
      same = (const char*)d.sv.grad[k] - (const char*)d0.sv.grad[k] == (int64_t)r * stride &&
             d.sv.off[k] == d0.sv.off[k];
    if (!same) {
      msg = "peer emulation runs the fused P2P kernels as ONE cooperative launch: every rank must launch the "
            "same bucket with its gradients at a fixed byte stride from rank 0's (rank " + std::to_string(r) + ")";
      return DDP_ERR_UNSUPPORTED;
    }
  }
  cudaError_t e = cudaSuccess;
  for (int r = 0; r < W && e == cudaSuccess; ++r) e = cudaStreamWaitEvent(g->lane[lane], R.dep[r].pre, 0);
  P2PLaunch a = d0.a;
  a.emulated = 1;
  a.grad_rank_stride = stride;
  a.err = g->err_dev;
  if (e == cudaSuccess) e = launch_p2p(d0.algo, c->dtype, d0.sv, a, g->lane[lane]);
  if (e == cudaSuccess) e = cudaEventRecord(g->done[lane], g->lane[lane]);
  if (e != cudaSuccess) {
    msg = std::string("peer emulation cooperative launch: ") + cudaGetErrorString(e);
    return DDP_ERR_CUDA;
  }
  return DDP_OK;
}

ddp_status_t emu_p2p_launch(ddp_ctx* c, int algo, const SlotView& sv, const P2PLaunch& a, cudaStream_t ls,
                            int lane) {
  EmuGroup* g = c->emu;
  CUDA_TRY(c, cudaEventRecord(c->emu_pre[lane], ls));
  ddp_status_t st = DDP_OK;
  std::string msg;
  {
    std::unique_lock<std::mutex> lk(g->mu);
    EmuRdv& R = g->rdv[lane];
    const uint64_t gen = R.gen;
    R.dep[c->rank] = EmuDep{a, sv, algo, c->emu_pre[lane]};
    if (++R.arrived == g->world) {
      R.status = launch_all(c, g, R, lane, R.msg);
      R.arrived = 0;
      R.gen++;
      g->cv.notify_all();
    } else if (!g->cv.wait_for(lk, timeout_of(c), [&] { return R.gen != gen || g->dead; }) || R.gen == gen) {
      g->dead = true;
      g->cv.notify_all();
      c->poisoned = true;
      return fail(DDP_ERR_TIMEOUT, "peer emulation: a peer never reached the P2P launch on lane " +
                                       std::to_string(lane) + " (sequence " + std::to_string(a.seq) + ")");
    }
    st = R.status;
    msg = R.msg;
  }
  if (st != DDP_OK) {
    c->poisoned = true;
    return fail(st, msg);
  }
  CUDA_TRY(c, cudaStreamWaitEvent(ls, g->done[lane], 0));
  return DDP_OK;
}

uint32_t emu_error_word(const ddp_ctx* c) {
  return c->emu && c->emu->err_host ? *reinterpret_cast<volatile uint32_t*>(c->emu->err_host) : 0u;
}

}  // namespace b200ddp
