/*
 * b200ddp.h — C ABI of the B200-native DDP Reducer gradient synchronization.
 *
 * Implements the hot path of Li et al., "PyTorch Distributed: Experiences on
 * Accelerating Data Parallel Training" (arXiv 2006.15704), §3.2-§4.2
 * and Algorithm 1 (L205-L244):
 *   - bucket assignment in reverse registration order under a byte cap
 *     (P:L217, L304, L308, L415);
 *   - one ready signal per gradient (the autograd hook) with a
 *     pending count per bucket and in-order bucket launch;
 *   - pack + scale by 1/world into the flat bucket;
 *   - bucket allreduce on a communication stream overlapping backward
 *      — hand-written sm_100a kernels over NVLink peer
 *     memory (fused one-shot / two-shot in push or pull form, NVLS), copy-engine
 *     exchanges ordered by stream memory operations, or NCCL;
 *   - unpack of the averaged values into the gradients;
 *   - no_sync accumulation.
 *
 * Conventions (all functions):
 *   - Every call returns a ddp_status_t; no C++ exception crosses the ABI.
 *     ddp_last_error() returns a thread-local message for the last failure.
 *   - A context is single-threaded: calls come from the one autograd device
 *     thread (or a bench loop).
 *   - "stream" arguments are cudaStream_t values passed as void* (NULL = the
 *     legacy default stream).  Device pointers are plain CUDA device
 *     addresses on the bound device.
 *   - Ownership: param_numel is copied at create.  Gradient buffers passed to
 *     ddp_grad_ready are BORROWED and must stay valid (and must not be written
 *     by the caller) until the consumer stream passes the wait enqueued by
 *     ddp_finalize_backward; they are re-supplied every pass because .grad may
 *     be reallocated between iterations.  Symmetric storage passed to
 *     ddp_bind_device is caller-allocated and must outlive the context.  The
 *     library owns its NCCL communicator, CUDA events and tables.
 *   - Ordering: a launched bucket's device work follows everything the
 *     producer stream(s) of its ready signals had enqueued; the first launch of
 *     a pass follows the previous pass's end (the event finalize recorded), so
 *     the library's staging and flags are never reused early.
 *   - State machine: CREATED -> (bind) -> IDLE <-> IN_PASS.  The first
 *     ddp_grad_ready of a pass opens it; ddp_finalize_backward closes it.
 *     A CUDA or NCCL failure, a peer timeout or DDP_ERR_INCOMPLETE poisons
 *     the context: every later call returns DDP_ERR_POISONED.
 */
#ifndef B200DDP_H
#define B200DDP_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ddp_ctx ddp_ctx_t; /* opaque, library-owned */

typedef enum { DDP_FP32 = 0, DDP_BF16 = 1 } ddp_dtype_t;

typedef enum {
  DDP_OK = 0,
  DDP_ERR_INVALID_ARG = 1, /* bad argument; context unchanged */
  DDP_ERR_STATE = 2,       /* call not legal in the current state (e.g. nested no_sync) */
  DDP_ERR_DUPLICATE = 3,   /* param marked ready twice in one pass */
  DDP_ERR_INCOMPLETE = 4,  /* finalize with params never ready (P:L199 hang) — poisons */
  DDP_ERR_CUDA = 5,        /* CUDA runtime error — poisons */
  DDP_ERR_NCCL = 6,        /* NCCL error — poisons */
  DDP_ERR_NOMEM = 7,       /* host allocation failed */
  DDP_ERR_POISONED = 8,    /* context poisoned by an earlier fatal error */
  DDP_ERR_TIMEOUT = 9,     /* a peer never reached a P2P barrier — poisons */
  DDP_ERR_UNSUPPORTED = 10 /* feature not available in this build / state */
} ddp_status_t;

/* Option keys for ddp_set_option / ddp_get_option (legal in CREATED or IDLE;
 * every rank must use identical values, because the algorithm choice and the
 * P2P grid shape must agree across ranks). */
enum {
  DDP_OPT_OVERLAP = 1,          /* 1 (default): launch buckets from the hooks; 0: launch all at
                                   finalize — the non-overlapped baseline of P:L164-L175 / L399 */
  DDP_OPT_P2P_ONESHOT_MAX = 2,  /* buckets <= this many bytes use the one-shot P2P kernel (default
                                   -1 = automatic: 1 MiB; settable >= 0); larger ones the
                                   world-dependent default (world 2: one-shot with the pull kernels
                                   (CE with the push kernels), world > 2: two-shot) */
  DDP_OPT_P2P_TWOSHOT_MAX = 3,  /* buckets larger than this many bytes use NCCL (default INT64_MAX:
                                   none) */
  DDP_OPT_COMM_CTAS = 4,        /* max CTAs of a P2P kernel when world > 1 (1..148, default 32);
                                   the last bucket of a pass always runs on 148 */
  DDP_OPT_DRY_RUN = 5,          /* 1: protocol only, no device work (host tests; CREATED only) */
  DDP_OPT_PROFILE = 6,          /* 1: time every device launch with CUDA events */
  DDP_OPT_ALGO = 7,             /* force the bucket allreduce: 0 auto, 1 NCCL, 2 one-shot, 3 two-shot,
                                   4 copy-engine one-shot (world > 1), 5 NVLS (needs MULTICAST),
                                   6 SM push + stream-ordered reduce, 7 copy-engine two-shot */
  DDP_OPT_PACK_CTAS = 8,        /* max CTAs of the HBM-bound kernels (pack, unpack, CE gather /
                                   reduce, world-1 fused kernel); 1..9472, default 4736 */
  DDP_OPT_P2P_STAGE_BYTES = 9,  /* 0 (default): one pipeline stage per CTA chunk; else split each
                                   CTA chunk into stages of this many bytes (one sync per stage) */
  DDP_OPT_FIND_UNUSED = 10,     /* 1: globally-unused-parameter detection:
                                   enables ddp_mark_unused, a participation bitmap and one extra
                                   allreduce per synced pass (the bitmaps travel by copy engine, one
                                   transfer per peer ordered by stream memory operations, and are
                                   summed on the comm stream); CREATED only (storage grows by one
                                   bucket-region-sized scratch + 2W+1 bitmaps) */
  DDP_OPT_MULTICAST = 11,       /* 1: the caller will pass a multicast (NVLS) address of the storage
                                   to ddp_bind_device, enabling DDP_ALGO_NVLS; CREATED only.  Every
                                   rank must agree.  Never increases ddp_storage_bytes */
  DDP_OPT_CE_STREAMS = 12,      /* CE2: number of streams its peer copies are spread over (1..16,
                                   default 1; more measured slower).  CE copies use the comm stream.
                                   Before binding */
  DDP_OPT_NCCL_COMMS = 13,      /* round-robin process groups (Fig. 12 "rrx"): NCCL
                                   bucket b runs on communicator b mod k (split off the first with
                                   ncclCommSplit) and its own stream; 1..8, default 1; before binding */
  DDP_OPT_CE_DIRECT_BYTES = 14, /* CE algorithm: gradients >= this many bytes are copied straight
                                   from .grad (one copy per peer); smaller ones are gathered into
                                   one region first.  Default 16 MiB; layout key */
  DDP_OPT_WIRE_BF16 = 15,       /* compressed wire (§8(f) N-3): fp32 gradients travel
                                   as bf16 through the CE exchange (every bucket uses DDP_ALGO_CE at
                                   world > 1): s_q = RNE_bf16(g_q * fl(1/W)), fp32 rank-order sum,
                                   fp32 result (oracle O-8).  fp32 contexts only; layout key */
  DDP_OPT_LANES = 16,           /* P2P / NVLS kernels of bucket b run on stream (lane) b mod LANES,
                                   each lane with its own barrier flags, sequence and staging, so
                                   consecutive buckets' kernels overlap.  1..4, default 4; layout key.
                                   Lanes are used only while LANES x COMM_CTAS <= 148 (all lanes'
                                   spinning kernels must fit on the SMs at once) */
  DDP_OPT_LOW_PRIORITY = 17,    /* 1 (default): the library's own streams (lanes, copy-engine,
                                   round-robin) are created at the lowest priority, so queued backward
                                   kernels are scheduled first; 0: highest.  Before binding only */
  DDP_OPT_PREFER_OVERLAP = 18,  /* automatic policy for gradients produced by a running backward
                                   (the front end's DistributedDataParallel sets it).  0 (default):
                                   the policy that is fastest when all buckets are ready at once.
                                   1 (copy engines; chosen for fp32): every bucket but the last uses
                                   an SM-free copy-engine exchange (CE at world 2, CE2 wider), the
                                   last one the fastest fused kernel on every SM.  2 (SM kernels;
                                   chosen for bf16): at world 2 the one-shot kernel everywhere.
                                   Layout key */
  DDP_OPT_GRAD_VIEW = 19,       /* gradient-as-bucket-view (§8(f) N-3, zero-copy variant; the
                                   paper's buckets hold copies, Alg. 1 L231-L232 / L246): 1 = the
                                   caller places each gradient AT its bucket slot in this rank's
                                   storage (ddp_param_storage_offset), so a3 and a6 vanish and every
                                   bucket is averaged in place: by the fused two-shot in place
                                   (kernels/pull.cu pull_view_twoshot_kernel: each rank reads its
                                   peers' raw gradients, scales every operand by fl(1/W), sums its
                                   own shard in rank order in place, then reads the peers' sums;
                                   O-3b, bit-exact), except beside a running backward under
                                   PREFER_OVERLAP=1, where the copy-engine exchanges run in place (CE
                                   at world 2: the region as one transfer per peer; CE2 wider).
                                   DDP_OPT_ALGO = CE / CE2 force those; NCCL (or world 1): an
                                   in-place ncclAllReduce with ncclAvg (each operand x fl(1/W), then
                                   the sum — O-3b up to NCCL's summation order).  A gradient passed
                                   at any other address is still correct: it is copied raw into its
                                   slot before and back after the exchange.  Not combinable with
                                   FIND_UNUSED or WIRE_BF16 (DDP_ERR_UNSUPPORTED), nor with
                                   ddp_bind_emulated (use ddp_bind_peer_emulated).  Default 0; layout
                                   key */
  DDP_OPT_P2P_TIMEOUT_MS = 20,  /* bound of every barrier spin inside the fused P2P / NVLS kernels
                                   (%globaltimer); a peer that never arrives makes the waiting CTAs
                                   give up, set the error word and exit -> DDP_ERR_TIMEOUT from
                                   ddp_check_device_errors (poisons).  Default 30000; any time */
  DDP_OPT_WAIT_TIMEOUT_MS = 21, /* bound of a host wait for a peer's step under peer emulation
                                   (b200ddp_emu.h), and the host watchdog's bound: a finalized pass not
                                   complete this long after ddp_finalize_backward is reported by
                                   ddp_check_device_errors (default 60000); any time */
  DDP_OPT_EMU_DEAD_RANK = 22,   /* test support, cooperative emulation only (ddp_bind_emulated):
                                   this rank's CTAs return at once and never signal, so the others
                                   must time out (DDP_OPT_P2P_TIMEOUT_MS).  -1 (default) = none */
  DDP_OPT_P2P_PULL = 23,        /* which fused ONESHOT / TWOSHOT buckets (world > 1) run the pull form
                                   (kernels/pull.cu): each rank packs into its own bucket buffer (two
                                   per bucket, alternating by pass) and reads its peers' buffers; the
                                   release before each flag drains local stores only and .grad is
                                   written by the reads (no unpack pass, no closing barrier).  The
                                   others run the push form (remote stores into per-lane staging,
                                   round 1), whose stores need ~3x fewer SMs for the same NVLink rate.
                                   1 (default): pull for the LAST bucket (every SM) and, at world 2
                                   under the throughput policy (PREFER_OVERLAP 0), for every bucket;
                                   push for the buckets that run beside backward on COMM_CTAS CTAs;
                                   2: pull for every fused bucket; 0: push everywhere.  Layout key */
  DDP_OPT_P2P_SIGNAL = 24,      /* pull kernels: how a group publishes "my (local) stores are done"
                                   after its named barrier.  0 (default): fence.acq_rel.gpu +
                                   st.relaxed.sys of the flag into each peer (reading A-1);
                                   1: fence.sc.sys + st.release.sys (the formal system-scope release,
                                   5-8 us per publish); 2: st.release.sys alone; 3: st.release.gpu of
                                   a flag in the OWN storage, polled by the peers over NVLink
                                   (ld.acquire.sys).  Any time */
  DDP_OPT_P2P_DEBUG = 25,       /* measurement only: bit 0 skips the pull kernels' data reads and
                                   bit 1 their pack (syncs kept; wrong results!); bit 2 records a
                                   %globaltimer trace per CTA into the lane's flag-region scratch
                                   (kernels/pull.cu trace_point).  Default 0 */
  DDP_OPT_LAST_ON_PRODUCER = 26 /* 1 (default): the pass's last bucket, when fused and launched from
                                   a ready signal, runs on that signal's producer stream after every
                                   library stream is joined into it (the pass then ends there);
                                   0: on its lane like the others.  Any time */
};

/* Algorithm codes reported by ddp_bucket_algo / used by DDP_OPT_ALGO.
 * Failure behaviour: the fused kernels (ONESHOT, TWOSHOT, NVLS) bound every wait
 * for a peer (DDP_OPT_P2P_TIMEOUT_MS) and report DDP_ERR_TIMEOUT.  The copy-engine
 * exchanges (CE, PUSH, CE2) and the find_unused bitmap exchange wait with
 * cuStreamWaitValue32, which has no timeout: a peer that dies mid-pass leaves this
 * rank's library streams (and every stream ordered after them) blocked, exactly
 * as a dead peer leaves an NCCL collective blocked ("the backward pass
 * could hang").  The host watchdog in ddp_check_device_errors reports such a pass
 * (DDP_ERR_TIMEOUT, poisoned) once it is DDP_OPT_WAIT_TIMEOUT_MS past its
 * finalize.  Recovery is process-level: destroy the context (it does not wait for
 * its streams when poisoned; the NCCL communicator is aborted) and exit.
 *
 *   NCCL:    pack kernel -> ncclAllReduce(sum) -> unpack kernel (DDP_OPT_GRAD_VIEW: in-place
 *            ncclAllReduce(avg) on the slots the gradients live in; no pack / unpack)
 *   ONESHOT: one fused sm_100a kernel: pack, push to every peer, rank-order reduce into .grad
 *   TWOSHOT: one fused sm_100a kernel: pack + reduce-scatter push, reduce, all-gather push, unpack
 *   CE:      pack kernel -> copy-engine pushes (cudaMemcpyAsync over NVLink) ordered by stream
 *            memory operations (no SM waits) -> rank-order reduce kernel into .grad on a second
 *            stream.  Frees the SMs for the overlapped backward.
 *   NVLS:    one fused sm_100a kernel: pack -> multimem.ld_reduce / multimem.st through the
 *            NVSwitch multicast address ((1+1/W) S NVLink bytes per direction) -> unpack.
 *            Needs DDP_OPT_MULTICAST; otherwise resolves to TWOSHOT.
 *   PUSH:    as CE, but the transfer is one sm_100a kernel per bucket that reads every gradient
 *            once and stores it into every peer's slot (no waiting inside kernels; the ready /
 *            consumed flags are stream memory operations), so bucket b+1's push overlaps bucket
 *            b's reduction on the second stream.
 *   CE2:     copy-engine two-shot: pack kernel -> reduce-scatter copies of shards -> rank-order
 *            shard reduce kernel -> all-gather copies -> unpack kernel, five streams ordered by
 *            stream memory operations; 2(W-1)/W S NVLink bytes per direction, no SM waits. */
enum { DDP_ALGO_AUTO = 0, DDP_ALGO_NCCL = 1, DDP_ALGO_ONESHOT = 2, DDP_ALGO_TWOSHOT = 3, DDP_ALGO_CE = 4,
       DDP_ALGO_NVLS = 5, DDP_ALGO_PUSH = 6, DDP_ALGO_CE2 = 7 };

/* ---- construction (host only, deterministic, touches no GPU) -------------
 * Bucket assignment (Alg. 1 "allocate parameters to buckets in the
 * reverse order of net.parameters()"; P:L308 cap; P:L415 cap 0 = one bucket
 * per gradient; reading C-1: a bucket is closed before the parameter that
 * would push it over bucket_cap_bytes, an oversized parameter sits alone;
 * C-6: tight packing, offset = running element count).
 *   param_numel[n_params]: element counts in registration order, each >= 1.
 *   dtype: DDP_FP32 or DDP_BF16 (one dtype per context, C-11).
 *   bucket_cap_bytes >= 0.  world >= 1 (<= 8), 0 <= rank < world.
 * Errors: DDP_ERR_INVALID_ARG, DDP_ERR_NOMEM.  *out untouched on error. */
ddp_status_t ddp_create(const int64_t* param_numel, int32_t n_params, int32_t dtype,
                        int64_t bucket_cap_bytes, int32_t world, int32_t rank, ddp_ctx_t** out);
void ddp_destroy(ddp_ctx_t* ctx); /* NULL-safe; aborts the NCCL comm if poisoned */
/* ddp_create_ordered: as ddp_create, but the bucketing scan visits the
 * parameters in scan_order[n_params] (a permutation) instead of reverse
 * registration order — the "gradient order prediction" of PAPER.md §6.2.1
 * (L563-L565): trace the backward order (ddp_ready_order) and rebuild the
 * parameter-to-bucket map, rarely, with one order agreed by every rank (e.g.
 * rank 0's, broadcast).  NULL = reverse registration order (= ddp_create).
 * Errors: as ddp_create; DDP_ERR_INVALID_ARG if scan_order is not a permutation. */
ddp_status_t ddp_create_ordered(const int64_t* param_numel, int32_t n_params, const int32_t* scan_order,
                                int32_t dtype, int64_t bucket_cap_bytes, int32_t world, int32_t rank,
                                ddp_ctx_t** out);

/* ---- introspection: the bit-exact mapping contract ---------------------- */
int32_t ddp_num_buckets(const ddp_ctx_t* ctx); /* -1 if ctx is NULL */
ddp_status_t ddp_bucket_info(const ddp_ctx_t* ctx, int32_t b, int64_t* numel, int32_t* n_slots);
/* slot s of bucket b, in scan (reverse registration) order */
ddp_status_t ddp_bucket_slot(const ddp_ctx_t* ctx, int32_t b, int32_t s, int32_t* param, int64_t* offset);
ddp_status_t ddp_param_location(const ddp_ctx_t* ctx, int32_t p, int32_t* bucket, int64_t* offset);
/* Bytes of symmetric storage each rank must allocate (peer-mapped) and pass to
 * ddp_bind_device; depends on options, so query after ddp_set_option. */
ddp_status_t ddp_storage_bytes(const ddp_ctx_t* ctx, int64_t* bytes);
/* Allreduce algorithm chosen for bucket b (DDP_ALGO_*), given current options. */
ddp_status_t ddp_bucket_algo(const ddp_ctx_t* ctx, int32_t b, int32_t* algo);
/* Byte offset, inside this rank's storage, of parameter p's bucket slot — the
 * view `b_i.narrow(offset, var.size())` of Alg. 1: its
 * gradient (param_numel[p] elements of the context dtype, contiguous) lives
 * there under DDP_OPT_GRAD_VIEW (§8(f) N-3, zero-copy).  The caller owns the
 * storage (ddp_bind_device's peer_storage[rank]); the library only reads and
 * writes it inside launched buckets.  Depends on options: query after
 * ddp_set_option.  Errors: DDP_ERR_INVALID_ARG (NULL / bad index). */
ddp_status_t ddp_param_storage_offset(const ddp_ctx_t* ctx, int32_t p, int64_t* byte_offset);

/* ---- device binding (once; collective across ranks) ---------------------
 * ddp_get_nccl_id: rank 0 creates the NCCL unique id (128 bytes); the caller
 * broadcasts it to all ranks (PAPER.md L278 rendezvous).
 * ddp_bind_device: creates the NCCL communicator (blocking, collective),
 * zeroes this rank's barrier flags and synchronizes all ranks once.
 *   device: CUDA ordinal.  comm_stream: caller-owned stream that carries all
 *   of the library's device work ("dedicated set of CUDA streams").
 *   peer_storage[world]: device addresses, valid on `device`, of every rank's
 *   storage (ddp_storage_bytes each, 256-B aligned, peer-mapped, e.g. torch
 *   symmetric memory); peer_storage[rank] is this rank's own.
 *   multicast_ptr: multicast (NVLS) address of this rank's storage base, i.e. the
 *   address whose loads/stores reach the same offset of every rank's storage;
 *   required iff DDP_OPT_MULTICAST is set, else ignored (may be NULL).
 * Errors: DDP_ERR_STATE (already bound), DDP_ERR_INVALID_ARG, DDP_ERR_CUDA,
 * DDP_ERR_NCCL. */
ddp_status_t ddp_get_nccl_id(uint8_t out[128]);
ddp_status_t ddp_bind_device(ddp_ctx_t* ctx, int32_t device, const uint8_t nccl_id[128],
                             void* comm_stream, void* const* peer_storage, void* multicast_ptr);

/* ---- per-iteration hot path -----------------------------------------------
 * ddp_grad_ready: the autograd hook.  Marks param_idx
 * ready for this pass; `grad` is its gradient (param_numel elements of the
 * context dtype, contiguous, any alignment) produced on `producer_stream`.
 * When the lowest unlaunched bucket(s) become complete, they are launched in
 * bucket order on the comm stream after an event wait on the producer
 * stream(s): pack (x 1/world) -> allreduce -> unpack into the gradients.
 * Inside no_sync (C-9: sampled at pass open) the call only records readiness.
 * Errors: DDP_ERR_INVALID_ARG (index / NULL grad), DDP_ERR_DUPLICATE,
 * DDP_ERR_STATE (not bound and not dry-run), DDP_ERR_CUDA / _NCCL. */
ddp_status_t ddp_grad_ready(ddp_ctx_t* ctx, int32_t param_idx, void* grad, void* producer_stream);
/* Batched form: equivalent to n successive ddp_grad_ready calls in array order. */
ddp_status_t ddp_grads_ready(ddp_ctx_t* ctx, int32_t n, const int32_t* param_idx,
                             void* const* grads, void* producer_stream);
/* ddp_mark_unused: Alg. 1 forward (L224-L225) "traverse autograd graph from out
 * and mark unused parameters as ready": param_idx will get no gradient in this
 * pass.  Counts as its ready signal (buckets holding it can launch without
 * waiting).  Requires DDP_OPT_FIND_UNUSED.
 *   grad: param_idx's current gradient buffer, or NULL if it has none.  If the
 *   parameter got a gradient in an earlier no_sync pass since the last synced
 *   pass (so it participates), grad must be that accumulated gradient
 *   and it is synchronized like any other.  Otherwise its local contribution is
 *   zero (P:L310 local bitmap); after the pass's extra bitmap allreduce the
 *   average is written into grad (if non-NULL) only when some rank used the
 *   parameter; a parameter unused on every rank keeps its gradient intact
 *   ("DDP should only touch gradients that are indeed involved").
 *   producer_stream: orders the library's zero-fill of the local contribution.
 * Errors: as ddp_grad_ready; DDP_ERR_STATE if FIND_UNUSED is off;
 * DDP_ERR_INVALID_ARG if grad is NULL for a participating parameter. */
ddp_status_t ddp_mark_unused(ddp_ctx_t* ctx, int32_t param_idx, void* grad, void* producer_stream);
/* ddp_global_unused: after the finalize of a synced pass with FIND_UNUSED, blocks
 * the host until that pass's bitmap allreduce has completed and writes
 * out[p] = 1 if parameter p was unused on every rank (its gradient was left
 * untouched), else 0, for p < n (n <= number of parameters).
 * Errors: DDP_ERR_STATE if no synced FIND_UNUSED pass has finished. */
ddp_status_t ddp_global_unused(ddp_ctx_t* ctx, uint8_t* out, int32_t n);
/* ddp_finalize_backward: closes the pass ("block waiting for all
 * AllReduce ops", done asynchronously: the consumer stream waits on the comm
 * stream, no host block).  Launches any deferred buckets (OVERLAP=0) and
 * replenishes the pending counts.  Returns DDP_ERR_INCOMPLETE (and
 * poisons) if some parameter was never ready; DDP_ERR_STATE if no pass is
 * open.  After it returns, gradients read on consumer_stream hold the
 * averages. */
ddp_status_t ddp_finalize_backward(ddp_ctx_t* ctx, void* consumer_stream);
/* no_sync: legal only between passes; nesting / end without
 * begin -> DDP_ERR_STATE.  Passes opened inside the scope do no device work;
 * the caller keeps accumulating .grad, and the first pass after
 * ddp_no_sync_end synchronizes the accumulated gradients. */
ddp_status_t ddp_no_sync_begin(ddp_ctx_t* ctx);
ddp_status_t ddp_no_sync_end(ddp_ctx_t* ctx);

/* ---- measurement / test knobs --------------------------------------------- */
ddp_status_t ddp_set_option(ddp_ctx_t* ctx, int32_t key, int64_t value);
ddp_status_t ddp_get_option(const ddp_ctx_t* ctx, int32_t key, int64_t* value);
/* Launch trace of the most recent pass: bucket indices in launch order and,
 * for each, the 0-based index (within the pass) of the ready signal that
 * triggered it (= number of ready signals in the pass if launched at
 * finalize).  *n receives the count; at most `cap` entries are written. */
ddp_status_t ddp_launch_trace(const ddp_ctx_t* ctx, int32_t* buckets, int32_t* triggers,
                              int32_t cap, int32_t* n);
/* With DDP_OPT_PROFILE=1: synchronizes the recorded events and returns the
 * summed device milliseconds and launch counts since the last read, per kind
 * [0]=pack (CE: gather of small gradients) [1]=NCCL allreduce [2]=unpack [3]=fused P2P / NVLS
 * kernel (incl. world-1 group) [4]=CE / PUSH transfer (copy engines or the push kernel)
 * [5]=CE / PUSH reduce kernel; then clears. */
ddp_status_t ddp_profile_read(ddp_ctx_t* ctx, double ms[6], int64_t launches[6]);
/* With DDP_OPT_PROFILE=1: per device launch since the last read (in launch
 * order), its kind (as above), the time its bucket(s) became ready on the
 * producer stream, and its start / end on the comm stream, in ms relative to
 * the first recorded ready point (the Fig. 2(c)-style ready/launch/done
 * timeline).  *n receives the count; at most cap entries are written; clears. */
ddp_status_t ddp_profile_timeline(ddp_ctx_t* ctx, int32_t cap, int32_t* kinds, double* ready_ms,
                                  double* start_ms, double* end_ms, int32_t* n);
/* Parameter indices in the order their ready signals (ddp_grad_ready /
 * ddp_mark_unused) arrived in the most recent finished pass (the open one if a
 * pass is open) — the trace for ddp_create_ordered.  *n receives the count. */
ddp_status_t ddp_ready_order(const ddp_ctx_t* ctx, int32_t* out, int32_t cap, int32_t* n);
/* Alg. 1 constructor (L214-L215): "broadcast net states to other processes".
 * Broadcasts n device buffers (bytes[i] bytes each, in place) from rank root over
 * the library's communicator, as one NCCL group on `stream`.  Collective: every
 * rank calls it with the same sizes.  Legal between passes on a bound context.
 * Errors: DDP_ERR_STATE, DDP_ERR_INVALID_ARG, DDP_ERR_NCCL. */
ddp_status_t ddp_broadcast(ddp_ctx_t* ctx, void* const* bufs, const int64_t* bytes, int32_t n, int32_t root,
                           void* stream);
/* Non-blocking health check; call it from the host between steps.  Reports, in
 * this order: the device-side error word (a fused kernel's peer wait timed out,
 * DDP_OPT_P2P_TIMEOUT_MS), an NCCL asynchronous error, and the host watchdog: the
 * last finalized pass not complete DDP_OPT_WAIT_TIMEOUT_MS after its finalize (a
 * copy-engine flag wait or a collective stuck on a dead peer).  Each poisons the
 * context and returns DDP_ERR_TIMEOUT (DDP_ERR_NCCL for the NCCL error). */
ddp_status_t ddp_check_device_errors(ddp_ctx_t* ctx);
const char* ddp_last_error(void);
/* Library version string. */
const char* ddp_version(void);

#ifdef __cplusplus
}
#endif
#endif /* B200DDP_H */
