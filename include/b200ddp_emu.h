/*
 * b200ddp_emu.h — single-GPU emulation of `world` ranks (test support).
 * Two modes: ddp_bind_emulated (one context, every rank of each fused P2P launch
 * in one cooperative kernel) and ddp_bind_peer_emulated (one context per rank,
 * one host thread per rank; every algorithm except NCCL / NVLS).
 *
 * The P2P allreduce kernels wait on flags written by the other ranks, so two
 * ranks must never be run as separate launches on one GPU (nothing makes them
 * co-resident).  Emulation instead runs ALL ranks of one bucket launch as ONE
 * cooperative kernel (gridDim.y = world, blockIdx.y = rank), over `world`
 * storages that all live on `device`.  The arithmetic, memory layout, barrier
 * protocol and grid shape per rank are exactly those of the multi-process
 * path; only the peer addresses differ.  Used by tests/test_gpu_parity.py to
 * check the P2P kernels against the oracle at W = 2, 3, 4, 8 on one B200.
 *
 * ddp_bind_emulated: ctx must be CREATED with rank 0 and the emulated world.
 *   storages[world]: device pointers (ddp_storage_bytes each) on `device`.
 *   Rank r's gradient of param p is at (char*)grad_p + r * grad_rank_stride_bytes,
 *   where grad_p is the pointer given to ddp_grad_ready (rank 0's).
 *   Buckets that would use NCCL use the two-shot kernel instead.
 * Errors: DDP_ERR_STATE, DDP_ERR_INVALID_ARG, DDP_ERR_CUDA,
 * DDP_ERR_UNSUPPORTED (grid larger than what is co-resident).
 */
#ifndef B200DDP_EMU_H
#define B200DDP_EMU_H

#include "b200ddp.h"

#ifdef __cplusplus
extern "C" {
#endif

ddp_status_t ddp_bind_emulated(ddp_ctx_t* ctx, int32_t device, void* comm_stream,
                               void* const* storages, int64_t grad_rank_stride_bytes);

/*
 * ddp_bind_peer_emulated — peer emulation: `world` contexts in ONE process on ONE
 * device stand for the `world` ranks, each created with its own rank and driven by
 * its OWN host thread, exactly as each rank's process drives its context (one
 * replica per process).  The whole product path runs per rank —
 * ready tracking and launch order, the copy-engine exchanges (CE, PUSH, CE2,
 * bf16 wire, gradient-as-bucket-view) with their stream-memory-operation flags,
 * the lanes, the last-bucket drain, no_sync, find_unused with its bitmap exchange —
 * over peer storages that all live on `device`.  What differs (ranks share a GPU):
 *   - a stream wait on a peer's flag is issued only once some thread has issued
 *     the matching write (the host blocks, bounded by DDP_OPT_WAIT_TIMEOUT_MS,
 *     then DDP_ERR_TIMEOUT and a poisoned context): waits invisible to the CUDA
 *     scheduler can then never sit ahead of their write in a shared queue;
 *   - the fused one-shot / two-shot kernels, which spin on peers' flags, never run
 *     as separate launches on one GPU: the ranks meet on the host and ONE
 *     cooperative kernel runs all of them (as ddp_bind_emulated), which needs every
 *     rank's gradients of a bucket at one fixed byte stride from rank 0's
 *     (else DDP_ERR_UNSUPPORTED);
 *   - no NCCL communicator: buckets that resolve to NCCL (or NVLS) are refused at
 *     bind (DDP_ERR_UNSUPPORTED); ddp_broadcast is unavailable.
 *   storages[world]: every rank's storage (ddp_storage_bytes each, 256-B aligned)
 *   on `device`; every rank passes the same array.  comm_stream: this rank's.
 * Collective: blocks until all `world` contexts sharing storages[0] are bound (the
 * bind-time barrier of ddp_bind_device), so call it from the ranks' threads.
 * Errors: DDP_ERR_STATE, DDP_ERR_INVALID_ARG, DDP_ERR_UNSUPPORTED, DDP_ERR_CUDA,
 * DDP_ERR_TIMEOUT.
 */
ddp_status_t ddp_bind_peer_emulated(ddp_ctx_t* ctx, int32_t device, void* comm_stream, void* const* storages);

#ifdef __cplusplus
}
#endif
#endif /* B200DDP_EMU_H */
