"""Helpers for the -m gpu parity tests (drive the C ABI; compare with oracle/)."""

from __future__ import annotations

from typing import List, Sequence

import numpy as np
import torch

from paper_2006_15704_b200 import _lib as L
from synth import device as sdev

TDT = {"fp32": torch.float32, "bf16": torch.bfloat16}
LDT = {"fp32": L.FP32, "bf16": L.BF16}
ESZ = {"fp32": 4, "bf16": 2}
GUARD = 4096          # guard band bytes around each emulated rank's storage
SENTINEL = -1234.5    # exactly representable in fp32 and bf16


def to_np(t: torch.Tensor, dtype: str) -> np.ndarray:
    t = t.detach().contiguous().cpu()
    if dtype == "fp32":
        return t.numpy().copy()
    return t.view(torch.int16).numpy().view(np.uint16).copy()


def flat_layout(numels: Sequence[int], misalign: bool):
    """Element offsets of each param inside one per-rank flat buffer.  With
    misalign, every param starts at an odd element offset (exercises the
    scalar / head-tail paths of the kernels)."""
    offs, pos = [], 0
    for n in numels:
        if misalign:
            pos += 1
        offs.append(pos)
        pos += n
        if not misalign:
            pos = (pos + 63) // 64 * 64
    return offs, (pos + 63) // 64 * 64


def run_emulated(numels: Sequence[int], dtype: str, cap: int, W: int, algo: int, *, seed=15704,
                 dist="normal", iters=1, misalign=False, options=None, order=None):
    """Runs `iters` synced passes of W emulated ranks on one GPU through the C ABI.
    Returns (inputs[it] as [W, total] cpu tensors, outputs[it], offs)."""
    dev = torch.cuda.current_device()
    offs, total = flat_layout(numels, misalign)
    big = torch.full((W, total), SENTINEL, dtype=TDT[dtype], device="cuda")   # gaps keep the sentinel
    ctx = L.ddp_create(numels, LDT[dtype], cap, W, 0)
    ins, outs = [], []
    try:
        L.ddp_set_option(ctx, L.OPT_ALGO, algo)
        for k, v in (options or {}).items():
            L.ddp_set_option(ctx, k, v)
        sb = L.ddp_storage_bytes(ctx)
        raw = [torch.full((sb + 2 * GUARD,), 0xA5, dtype=torch.uint8, device="cuda") for _ in range(W)]
        stor = [x[GUARD:GUARD + sb] for x in raw]
        comm = torch.cuda.Stream()
        L.ddp_bind_emulated(ctx, dev, comm.cuda_stream, [s.data_ptr() for s in stor], total * ESZ[dtype])
        ptrs = [big[0, o:].data_ptr() for o in offs]
        order = list(range(len(numels) - 1, -1, -1)) if order is None else order
        batch = L.ReadyBatch(order, [ptrs[p] for p in order])
        cur = torch.cuda.current_stream()
        for it in range(iters):
            for r in range(W):
                for p, (o, n) in enumerate(zip(offs, numels)):
                    sdev.fill(big[r, o:o + n], seed, r, it, p, dist, dtype, cur.cuda_stream)
            ins.append(big.cpu())
            L.ddp_grads_ready(ctx, batch, cur.cuda_stream)
            L.ddp_finalize_backward(ctx, cur.cuda_stream)
            outs.append(big.cpu())
        torch.cuda.synchronize()
        L.ddp_check_device_errors(ctx)
        check_bounds(raw, big, offs, numels)
    finally:
        L.ddp_destroy(ctx)
    return ins, outs, offs


def check_bounds(raw, big, offs, numels):
    """No kernel wrote outside a storage (guard bands) or between the gradients
    (sentinels): the bounds check this pool offers in place of compute-sanitizer."""
    torch.cuda.synchronize()
    for r, x in enumerate(raw):
        assert bool((x[:GUARD] == 0xA5).all()) and bool((x[-GUARD:] == 0xA5).all()), f"storage guard of rank {r}"
    mask = torch.ones(big.shape[1], dtype=torch.bool, device=big.device)
    for o, n in zip(offs, numels):
        mask[o:o + n] = False
    assert bool((big[:, mask] == SENTINEL).all()), "a write landed between gradients"


def param_slices(t: torch.Tensor, offs, numels, dtype) -> List[List[np.ndarray]]:
    """[rank][param] numpy views of a [W, total] tensor."""
    a = to_np(t, dtype)
    return [[a[r, o:o + n] for o, n in zip(offs, numels)] for r in range(a.shape[0])]


# ---- peer emulation: one context + one host thread per rank (ddp_bind_peer_emulated) ----

def run_threads(W: int, fn) -> None:
    """fn(rank) on W host threads (the ranks' "processes"); re-raises the first error."""
    import threading
    dev = torch.cuda.current_device()
    errs = [None] * W

    def body(r):
        try:
            torch.cuda.set_device(dev)
            fn(r)
        except BaseException as e:  # noqa: BLE001 - reported to the caller
            errs[r] = e
    ts = [threading.Thread(target=body, args=(r,), daemon=True) for r in range(W)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for r, e in enumerate(errs):
        if e is not None:
            raise RuntimeError(f"rank {r}: {e!r}") from e


class PeerEmu:
    """W ranks as W native contexts on one GPU, each bound with
    ddp_bind_peer_emulated and driven from its own host thread (the product
    path per rank; include/b200ddp_emu.h).  Gradients: rank r's param p at
    ``big[r, offs[p]:offs[p]+n]`` (a fixed stride between ranks), or, with
    ``grad_view``, its bucket slot in rank r's storage (N-3 zero-copy)."""

    def __init__(self, numels: Sequence[int], dtype: str, cap: int, W: int, algo: int = L.ALGO_AUTO,
                 options=None, misalign=False, grad_view=False, elsewhere=()):
        self.ns, self.dtype, self.W = list(numels), dtype, W
        self.offs, self.total = flat_layout(self.ns, misalign)
        self.ctx = []
        try:
            for r in range(W):
                c = L.ddp_create(self.ns, LDT[dtype], cap, W, r)
                self.ctx.append(c)
                L.ddp_set_option(c, L.OPT_ALGO, algo)
                if grad_view:
                    L.ddp_set_option(c, L.OPT_GRAD_VIEW, 1)
                for k, v in (options or {}).items():
                    L.ddp_set_option(c, k, v)
            sb = L.ddp_storage_bytes(self.ctx[0])
            # each storage sits between two guard bands (a fixed byte pattern) that no
            # kernel or copy may touch: checked by check_guards() (out-of-bounds writes)
            self._raw = [torch.full((sb + 2 * GUARD,), 0xA5, dtype=torch.uint8, device="cuda") for _ in range(W)]
            self.stor = [x[GUARD:GUARD + sb] for x in self._raw]
            self.comm = [torch.cuda.Stream() for _ in range(W)]
            self.prod = [torch.cuda.Stream() for _ in range(W)]
            ptrs = [s.data_ptr() for s in self.stor]
            dev = torch.cuda.current_device()
            torch.cuda.synchronize()
            run_threads(W, lambda r: L.ddp_bind_peer_emulated(self.ctx[r], dev, self.comm[r].cuda_stream, ptrs))
        except Exception:
            self.close()
            raise
        # gaps between (and after) the parameters hold a sentinel that must survive every pass
        self.big = torch.full((W, self.total), SENTINEL, dtype=TDT[dtype], device="cuda")
        es = ESZ[dtype]
        if grad_view:
            so = [L.ddp_param_storage_offset(self.ctx[0], p) for p in range(len(self.ns))]
            # `elsewhere`: gradients handed over at another address than their slot
            # (copied raw into the slot and back, exchange.cpp alias_runs)
            self.grads = [[self.big[r, self.offs[p]:self.offs[p] + n] if p in elsewhere
                           else self.stor[r][o:o + n * es].view(TDT[dtype])
                           for p, (o, n) in enumerate(zip(so, self.ns))] for r in range(W)]
        else:
            self.grads = [[self.big[r, o:o + n] for o, n in zip(self.offs, self.ns)] for r in range(W)]

    def fill(self, seed, it, dist="normal", stream=None):
        s = (stream or torch.cuda.current_stream()).cuda_stream
        for r in range(self.W):
            for p, g in enumerate(self.grads[r]):
                sdev.fill(g, seed, r, it, p, dist, self.dtype, s)

    def snapshot(self) -> torch.Tensor:
        """[W, total] cpu copy of every rank's gradients (flat layout)."""
        out = torch.zeros(self.W, self.total, dtype=TDT[self.dtype], device="cuda")
        for r in range(self.W):
            for o, g in zip(self.offs, self.grads[r]):
                out[r, o:o + g.numel()].copy_(g)
        torch.cuda.synchronize()
        return out.cpu()

    def sync_pass(self, orders=None, unused=None, no_sync=False, late_fill=None):
        """One backward pass on every rank's thread: ready signals in orders[r]
        (default reverse registration), unused[r] = params marked unused
        (ddp_mark_unused with the current gradient buffer), then finalize.
        late_fill = (seed, it, dist): each rank's thread first stalls its producer
        stream (~2 ms GPU sleep) and only then generates its gradients ON that
        stream, right before the ready signals — the library must order its device
        work after the producer stream, or it reads stale gradients."""
        torch.cuda.synchronize()
        n = len(self.ns)

        def rank(r):
            c, s = self.ctx[r], self.prod[r].cuda_stream
            if late_fill is not None:
                seed, it, dist = late_fill
                with torch.cuda.stream(self.prod[r]):
                    torch.cuda._sleep(4_000_000)
                for p, g in enumerate(self.grads[r]):
                    sdev.fill(g, seed, r, it, p, dist, self.dtype, s)
            if no_sync:
                L.ddp_no_sync_begin(c)
            un = set((unused or {}).get(r, ()))
            for p in sorted(un, reverse=True):
                L.ddp_mark_unused(c, p, self.grads[r][p].data_ptr(), s)
            order = [p for p in (orders[r] if orders else range(n - 1, -1, -1)) if p not in un]
            L.ddp_grads_ready(c, L.ReadyBatch(order, [self.grads[r][p].data_ptr() for p in order]), s)
            L.ddp_finalize_backward(c, s)
            if no_sync:
                L.ddp_no_sync_end(c)
        run_threads(self.W, rank)
        torch.cuda.synchronize()
        for c in self.ctx:
            L.ddp_check_device_errors(c)

    def check_guards(self):
        """No write outside a storage or between the gradients (bounds check in
        place of compute-sanitizer, which this pool does not offer)."""
        check_bounds(self._raw, self.big, self.offs, self.ns)

    def algos(self):
        return [L.ALGO_NAMES[L.ddp_bucket_algo(self.ctx[0], b)] for b in range(L.ddp_num_buckets(self.ctx[0]))]

    def close(self):
        torch.cuda.synchronize()
        for c in self.ctx:
            L.ddp_destroy(c)
        self.ctx = []


def run_peer_emulated(numels: Sequence[int], dtype: str, cap: int, W: int, algo: int, *, seed=15704,
                      dist="normal", iters=1, misalign=False, options=None, orders=None, grad_view=False,
                      elsewhere=()):
    """`iters` synced passes of W peer-emulated ranks.  Returns (inputs[it],
    outputs[it], offs) as [W, total] cpu tensors in the flat layout."""
    pe = PeerEmu(numels, dtype, cap, W, algo, options=options, misalign=misalign, grad_view=grad_view,
                 elsewhere=elsewhere)
    ins, outs = [], []
    try:
        for it in range(iters):
            pe.fill(seed, it, dist)
            ins.append(pe.snapshot())
            pe.sync_pass(orders)
            outs.append(pe.snapshot())
        pe.check_guards()
    finally:
        pe.close()
    return ins, outs, pe.offs
