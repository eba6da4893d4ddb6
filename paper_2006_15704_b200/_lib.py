"""Thin ctypes binding over the C ABI (include/b200ddp.h, include/b200ddp_emu.h).

Argument marshalling only: every step of the hot path runs in the native
library.  Function names are the C names.  Each wrapper raises ``DDPError``
(with ``ddp_last_error()``) on a non-OK status.  The library is built in-tree
(``paper_2006_15704_b200/lib/libb200ddp.so``); if it is missing this module
fails loudly — there is no fallback implementation.
"""

from __future__ import annotations

import ctypes as C
import os
from typing import List, Optional, Sequence, Tuple

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libb200ddp.so")

# ddp_status_t
OK, ERR_INVALID_ARG, ERR_STATE, ERR_DUPLICATE, ERR_INCOMPLETE, ERR_CUDA, ERR_NCCL, ERR_NOMEM, \
    ERR_POISONED, ERR_TIMEOUT, ERR_UNSUPPORTED = range(11)
STATUS_NAMES = ["OK", "INVALID_ARG", "STATE", "DUPLICATE", "INCOMPLETE", "CUDA", "NCCL", "NOMEM",
                "POISONED", "TIMEOUT", "UNSUPPORTED"]
FP32, BF16 = 0, 1
OPT_OVERLAP, OPT_P2P_ONESHOT_MAX, OPT_P2P_TWOSHOT_MAX, OPT_COMM_CTAS, OPT_DRY_RUN, OPT_PROFILE, \
    OPT_ALGO, OPT_PACK_CTAS, OPT_P2P_STAGE_BYTES, OPT_FIND_UNUSED, OPT_MULTICAST, OPT_CE_STREAMS, \
    OPT_NCCL_COMMS, OPT_CE_DIRECT_BYTES, OPT_WIRE_BF16, OPT_LANES, OPT_LOW_PRIORITY, \
    OPT_PREFER_OVERLAP, OPT_GRAD_VIEW, OPT_P2P_TIMEOUT_MS, OPT_WAIT_TIMEOUT_MS, OPT_EMU_DEAD_RANK, \
    OPT_P2P_PULL, OPT_P2P_SIGNAL, OPT_P2P_DEBUG, OPT_LAST_ON_PRODUCER = range(1, 27)
ALGO_AUTO, ALGO_NCCL, ALGO_ONESHOT, ALGO_TWOSHOT, ALGO_CE, ALGO_NVLS, ALGO_PUSH, ALGO_CE2 = range(8)
ALGO_NAMES = {ALGO_NCCL: "nccl", ALGO_ONESHOT: "oneshot", ALGO_TWOSHOT: "twoshot", ALGO_CE: "ce",
              ALGO_NVLS: "nvls", ALGO_PUSH: "push", ALGO_CE2: "ce2"}
PROFILE_KINDS = ("pack", "nccl_allreduce", "unpack", "p2p_fused", "ce_copy", "ce_reduce")


class DDPError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES[status] if 0 <= status < len(STATUS_NAMES) else status}: {msg}")
        self.status = status


_lib: Optional[C.CDLL] = None

_P = C.c_void_p
_SIGS = {
    "ddp_create": (C.c_int, [C.POINTER(C.c_int64), C.c_int32, C.c_int32, C.c_int64, C.c_int32, C.c_int32,
                             C.POINTER(_P)]),
    "ddp_destroy": (None, [_P]),
    "ddp_create_ordered": (C.c_int, [C.POINTER(C.c_int64), C.c_int32, C.POINTER(C.c_int32), C.c_int32, C.c_int64,
                                     C.c_int32, C.c_int32, C.POINTER(_P)]),
    "ddp_ready_order": (C.c_int, [_P, C.POINTER(C.c_int32), C.c_int32, C.POINTER(C.c_int32)]),
    "ddp_broadcast": (C.c_int, [_P, C.POINTER(_P), C.POINTER(C.c_int64), C.c_int32, C.c_int32, _P]),
    "ddp_num_buckets": (C.c_int32, [_P]),
    "ddp_bucket_info": (C.c_int, [_P, C.c_int32, C.POINTER(C.c_int64), C.POINTER(C.c_int32)]),
    "ddp_bucket_slot": (C.c_int, [_P, C.c_int32, C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_int64)]),
    "ddp_param_location": (C.c_int, [_P, C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_int64)]),
    "ddp_storage_bytes": (C.c_int, [_P, C.POINTER(C.c_int64)]),
    "ddp_param_storage_offset": (C.c_int, [_P, C.c_int32, C.POINTER(C.c_int64)]),
    "ddp_bucket_algo": (C.c_int, [_P, C.c_int32, C.POINTER(C.c_int32)]),
    "ddp_get_nccl_id": (C.c_int, [C.c_char_p]),
    "ddp_bind_device": (C.c_int, [_P, C.c_int32, C.c_char_p, _P, C.POINTER(_P), _P]),
    "ddp_bind_emulated": (C.c_int, [_P, C.c_int32, _P, C.POINTER(_P), C.c_int64]),
    "ddp_bind_peer_emulated": (C.c_int, [_P, C.c_int32, _P, C.POINTER(_P)]),
    "ddp_grad_ready": (C.c_int, [_P, C.c_int32, _P, _P]),
    "ddp_grads_ready": (C.c_int, [_P, C.c_int32, C.POINTER(C.c_int32), C.POINTER(_P), _P]),
    "ddp_finalize_backward": (C.c_int, [_P, _P]),
    "ddp_mark_unused": (C.c_int, [_P, C.c_int32, _P, _P]),
    "ddp_global_unused": (C.c_int, [_P, C.POINTER(C.c_uint8), C.c_int32]),
    "ddp_no_sync_begin": (C.c_int, [_P]),
    "ddp_no_sync_end": (C.c_int, [_P]),
    "ddp_set_option": (C.c_int, [_P, C.c_int32, C.c_int64]),
    "ddp_get_option": (C.c_int, [_P, C.c_int32, C.POINTER(C.c_int64)]),
    "ddp_launch_trace": (C.c_int, [_P, C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.c_int32,
                                   C.POINTER(C.c_int32)]),
    "ddp_profile_read": (C.c_int, [_P, C.POINTER(C.c_double), C.POINTER(C.c_int64)]),
    "ddp_profile_timeline": (C.c_int, [_P, C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_double),
                                       C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_int32)]),
    "ddp_check_device_errors": (C.c_int, [_P]),
    "ddp_last_error": (C.c_char_p, []),
    "ddp_version": (C.c_char_p, []),
}


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"native library missing: {LIB_PATH} "
                              "(build it with `python -m paper_2006_15704_b200.build`); no fallback exists")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _check(st: int) -> None:
    if st != OK:
        raise DDPError(st, lib().ddp_last_error().decode(errors="replace"))


# ---- same-name wrappers --------------------------------------------------------

def ddp_create(param_numel: Sequence[int], dtype: int, bucket_cap_bytes: int, world: int, rank: int) -> int:
    arr = (C.c_int64 * len(param_numel))(*[int(x) for x in param_numel])
    out = _P()
    _check(lib().ddp_create(arr, len(param_numel), dtype, int(bucket_cap_bytes), world, rank, C.byref(out)))
    return out.value


def ddp_create_ordered(param_numel: Sequence[int], scan_order: Optional[Sequence[int]], dtype: int,
                       bucket_cap_bytes: int, world: int, rank: int) -> int:
    arr = (C.c_int64 * len(param_numel))(*[int(x) for x in param_numel])
    order = None if scan_order is None else (C.c_int32 * len(scan_order))(*[int(x) for x in scan_order])
    out = _P()
    _check(lib().ddp_create_ordered(arr, len(param_numel), order, dtype, int(bucket_cap_bytes), world, rank,
                                    C.byref(out)))
    return out.value


def ddp_ready_order(ctx: int) -> List[int]:
    n = C.c_int32()
    _check(lib().ddp_ready_order(ctx, None, 0, C.byref(n)))
    buf = (C.c_int32 * max(1, n.value))()
    _check(lib().ddp_ready_order(ctx, buf, n.value, C.byref(n)))
    return [buf[i] for i in range(n.value)]


def ddp_broadcast(ctx: int, ptrs: Sequence[int], nbytes: Sequence[int], root: int, stream: int) -> None:
    p = (_P * max(1, len(ptrs)))(*ptrs)
    b = (C.c_int64 * max(1, len(nbytes)))(*[int(x) for x in nbytes])
    _check(lib().ddp_broadcast(ctx, p, b, len(ptrs), root, stream))


def ddp_destroy(ctx: int) -> None:
    lib().ddp_destroy(ctx)


def ddp_num_buckets(ctx: int) -> int:
    return lib().ddp_num_buckets(ctx)


def ddp_bucket_info(ctx: int, b: int) -> Tuple[int, int]:
    n, s = C.c_int64(), C.c_int32()
    _check(lib().ddp_bucket_info(ctx, b, C.byref(n), C.byref(s)))
    return n.value, s.value


def ddp_bucket_slot(ctx: int, b: int, s: int) -> Tuple[int, int]:
    p, o = C.c_int32(), C.c_int64()
    _check(lib().ddp_bucket_slot(ctx, b, s, C.byref(p), C.byref(o)))
    return p.value, o.value


def ddp_param_location(ctx: int, p: int) -> Tuple[int, int]:
    b, o = C.c_int32(), C.c_int64()
    _check(lib().ddp_param_location(ctx, p, C.byref(b), C.byref(o)))
    return b.value, o.value


def ddp_param_storage_offset(ctx: int, p: int) -> int:
    v = C.c_int64()
    _check(lib().ddp_param_storage_offset(ctx, p, C.byref(v)))
    return v.value


def ddp_storage_bytes(ctx: int) -> int:
    v = C.c_int64()
    _check(lib().ddp_storage_bytes(ctx, C.byref(v)))
    return v.value


def ddp_bucket_algo(ctx: int, b: int) -> int:
    v = C.c_int32()
    _check(lib().ddp_bucket_algo(ctx, b, C.byref(v)))
    return v.value


def ddp_get_nccl_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(lib().ddp_get_nccl_id(buf))
    return buf.raw


def ddp_bind_device(ctx: int, device: int, nccl_id: bytes, comm_stream: int,
                    peer_storage: Sequence[int], multicast_ptr: int = 0) -> None:
    ptrs = (_P * len(peer_storage))(*peer_storage)
    _check(lib().ddp_bind_device(ctx, device, nccl_id, comm_stream, ptrs, multicast_ptr or None))


def ddp_bind_emulated(ctx: int, device: int, comm_stream: int, storages: Sequence[int],
                      grad_rank_stride_bytes: int) -> None:
    ptrs = (_P * len(storages))(*storages)
    _check(lib().ddp_bind_emulated(ctx, device, comm_stream, ptrs, grad_rank_stride_bytes))


def ddp_bind_peer_emulated(ctx: int, device: int, comm_stream: int, storages: Sequence[int]) -> None:
    ptrs = (_P * len(storages))(*storages)
    _check(lib().ddp_bind_peer_emulated(ctx, device, comm_stream, ptrs))


def ddp_grad_ready(ctx: int, param_idx: int, grad_ptr: int, producer_stream: int) -> None:
    _check(lib().ddp_grad_ready(ctx, param_idx, grad_ptr, producer_stream))


class ReadyBatch:
    """Pre-marshalled argument arrays for ddp_grads_ready (reused every pass)."""

    def __init__(self, params: Sequence[int], grad_ptrs: Sequence[int]):
        self.n = len(params)
        self.params = (C.c_int32 * self.n)(*params)
        self.grads = (_P * self.n)(*grad_ptrs)


def ddp_grads_ready(ctx: int, batch: ReadyBatch, producer_stream: int) -> None:
    _check(lib().ddp_grads_ready(ctx, batch.n, batch.params, batch.grads, producer_stream))


def ddp_finalize_backward(ctx: int, consumer_stream: int) -> None:
    _check(lib().ddp_finalize_backward(ctx, consumer_stream))


def ddp_mark_unused(ctx: int, param_idx: int, grad_ptr: int, producer_stream: int) -> None:
    _check(lib().ddp_mark_unused(ctx, param_idx, grad_ptr or None, producer_stream))


def ddp_global_unused(ctx: int, n: int) -> List[bool]:
    out = (C.c_uint8 * max(1, n))()
    _check(lib().ddp_global_unused(ctx, out, n))
    return [bool(out[i]) for i in range(n)]


def ddp_no_sync_begin(ctx: int) -> None:
    _check(lib().ddp_no_sync_begin(ctx))


def ddp_no_sync_end(ctx: int) -> None:
    _check(lib().ddp_no_sync_end(ctx))


def ddp_set_option(ctx: int, key: int, value: int) -> None:
    _check(lib().ddp_set_option(ctx, key, int(value)))


def ddp_get_option(ctx: int, key: int) -> int:
    v = C.c_int64()
    _check(lib().ddp_get_option(ctx, key, C.byref(v)))
    return v.value


def ddp_launch_trace(ctx: int) -> List[Tuple[int, int]]:
    n = C.c_int32()
    _check(lib().ddp_launch_trace(ctx, None, None, 0, C.byref(n)))
    b = (C.c_int32 * max(1, n.value))()
    t = (C.c_int32 * max(1, n.value))()
    _check(lib().ddp_launch_trace(ctx, b, t, n.value, C.byref(n)))
    return [(b[i], t[i]) for i in range(n.value)]


def ddp_profile_read(ctx: int):
    ms = (C.c_double * 6)()
    cnt = (C.c_int64 * 6)()
    _check(lib().ddp_profile_read(ctx, ms, cnt))
    return {k: (ms[i], cnt[i]) for i, k in enumerate(PROFILE_KINDS)}


def ddp_profile_timeline(ctx: int, cap: int = 4096):
    """[(kind, ready_ms, start_ms, end_ms)] per device launch since the last read."""
    k = (C.c_int32 * cap)()
    r, s, e = (C.c_double * cap)(), (C.c_double * cap)(), (C.c_double * cap)()
    n = C.c_int32()
    _check(lib().ddp_profile_timeline(ctx, cap, k, r, s, e, C.byref(n)))
    return [(PROFILE_KINDS[k[i]], r[i], s[i], e[i]) for i in range(min(cap, n.value))]


def ddp_check_device_errors(ctx: int) -> None:
    _check(lib().ddp_check_device_errors(ctx))


def ddp_last_error() -> str:
    return lib().ddp_last_error().decode(errors="replace")


def ddp_version() -> str:
    return lib().ddp_version().decode()
