/*
 * b200ddp_emu.h — single-GPU emulation of `world` ranks (test support).
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

#ifdef __cplusplus
}
#endif
#endif /* B200DDP_EMU_H */
