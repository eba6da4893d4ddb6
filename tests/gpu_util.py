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
    big = torch.zeros(W, total, dtype=TDT[dtype], device="cuda")
    ctx = L.ddp_create(numels, LDT[dtype], cap, W, 0)
    ins, outs = [], []
    try:
        L.ddp_set_option(ctx, L.OPT_ALGO, algo)
        for k, v in (options or {}).items():
            L.ddp_set_option(ctx, k, v)
        sb = L.ddp_storage_bytes(ctx)
        stor = [torch.empty(sb, dtype=torch.uint8, device="cuda") for _ in range(W)]
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
    finally:
        L.ddp_destroy(ctx)
    return ins, outs, offs


def param_slices(t: torch.Tensor, offs, numels, dtype) -> List[List[np.ndarray]]:
    """[rank][param] numpy views of a [W, total] tensor."""
    a = to_np(t, dtype)
    return [[a[r, o:o + n] for o, n in zip(offs, numels)] for r in range(a.shape[0])]
