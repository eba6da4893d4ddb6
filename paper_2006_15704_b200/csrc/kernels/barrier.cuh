// barrier.cuh — cross-GPU barrier helpers of the P2P / NVLS kernels:
// per-CTA-index monotonic flags in every rank's symmetric storage, written
// with a system-scope release after a CTA barrier, polled with system-scope
// acquire loads under a bounded spin (a peer that never arrives sets the
// mapped error word instead of hanging the GPU).
#pragma once

#include "common.cuh"

namespace b200ddp {

namespace {

__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// flags: uint32 [2][kMaxCtas][kMaxWorld]; kind 0 = "pushed (reduce-scatter /
// one-shot data) through stage k", kind 1 = "all-gather pushed through stage k".
__device__ __forceinline__ uint32_t* flag_ptr(void* storage, int64_t flags_off, int kind, int cta, int src) {
  return reinterpret_cast<uint32_t*>(static_cast<char*>(storage) + flags_off + kind * kFlagArrayBytes) +
         cta * kMaxWorld + src;
}

// Publish "this CTA's stores up to here are done" to the same CTA index of every
// peer.  bar.sync orders every thread's stores before the signalling threads
// (CTA-scope synchronization, cumulative); each signalling thread then fences
// at system scope and writes the monotonic value with release semantics.  Only
// W-1 threads of warp 0 fence: a MEMBAR.SYS per warp of the CTA would serialize.
template <int W>
__device__ __forceinline__ void p2p_signal(const P2PLaunch& a, int r, int kind, uint32_t val) {
  if (W == 1) return;
  __syncthreads();
  const int t = threadIdx.x;
  if (t < W && t != r) {
    __threadfence_system();
    uint32_t* f = flag_ptr(a.storage[t], a.flags_byte_off, kind, blockIdx.x, r);
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(f), "r"(val) : "memory");
  }
}

// Wait until every peer's same-index CTA has published >= val (bounded spin).
template <int W>
__device__ __forceinline__ void p2p_wait(const P2PLaunch& a, int r, int kind, uint32_t val) {
  const int t = threadIdx.x;
  if (W > 1 && t < W && t != r) {
    const uint32_t* mine = flag_ptr(a.storage[r], a.flags_byte_off, kind, blockIdx.x, t);
    const uint64_t t0 = globaltimer();
    while (true) {
      uint32_t v;
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(mine) : "memory");
      if ((int32_t)(v - val) >= 0) break;
      if (globaltimer() - t0 > a.timeout_ns) {
        atomicExch(a.err, 1u);
        break;
      }
    }
  }
  __syncthreads();
}

template <typename T>
__device__ __forceinline__ T* at(void* base, int64_t byte_off) {
  return reinterpret_cast<T*>(static_cast<char*>(base) + byte_off);
}

}  // namespace

}  // namespace b200ddp
