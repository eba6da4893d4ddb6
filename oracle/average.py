"""O-3 / O-3b: the averaged gradient, and a full pack -> allreduce -> unpack
simulation of W replicas.  TEST INFRASTRUCTURE (see oracle/__init__).

Paper:
* PAPER.md L166 (§3.2.1): the hook "uses the AllReduce collective
  communication call to calculate the average gradients on each parameter
  across all processes, and writes the result back to the gradient tensor".
* "DDP always computes the average of all gradients".
* PAPER.md L68 / L278: AllReduce gives every participant the elementwise sum
  of equally-sized tensors; "returns the same result tensor to each
  participant".
* PAPER.md L231-L232 (Alg. 1): pack ``view.copy_(var.grad)`` into the bucket;
  L246 / L304: averaged values "copied back" into the gradients.

Readings: C-2 the 1/W scale is applied while packing (SPEC.md
L276/L309); C-3 one fixed summation order for the bit-faithful mode; C-4
fp32 accumulation for bf16 buckets, one final rounding; C-12 W=1 is the
identity.

Two definitions are provided:

``average_fp64``  (O-3): ref = RNE_dtype( (sum_r g_r) / W ) with the sum in
    fp64 over the exact input values; also den = (sum_r |g_r|) / W, the
    tolerance denominator (|y - ref| <= rtol * den per element).

``average_bitfaithful`` (O-3b): the arithmetic the B200 P2P kernels are
    specified to perform, written out step by step:
        s_r  = RNE_dtype( fp32(g_r) *fp32 fp32(1/W) )        (pack + scale)
        acc  = s_0 ;  acc = acc +fp32 s_r  for r = 1..W-1       (rank order)
        y    = RNE_dtype(acc)                                  (one rounding)
"""

from __future__ import annotations

from typing import List, Sequence, Tuple

import numpy as np

from .assignment import Assignment


# ---- dtype helpers (bf16 is carried as uint16 bit patterns) -------------------

def to_fp32(x: np.ndarray, dtype: str) -> np.ndarray:
    if dtype == "fp32":
        return np.asarray(x, dtype=np.float32)
    if dtype == "bf16":
        return (np.asarray(x, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32)
    raise ValueError(dtype)


def round_fp32_to(x: np.ndarray, dtype: str) -> np.ndarray:
    """RNE of fp32 values to the storage dtype (fp32: identity)."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    if dtype == "fp32":
        return x
    if dtype == "bf16":
        b = x.view(np.uint32)
        lsb = (b >> np.uint32(16)) & np.uint32(1)
        out = ((b + np.uint32(0x7FFF) + lsb) >> np.uint32(16)).astype(np.uint16)
        nan = np.isnan(x)
        if nan.any():
            out[nan] = ((b[nan] >> np.uint32(16)) | np.uint32(0x40)).astype(np.uint16)
        return out
    raise ValueError(dtype)


def round_fp64_to(x: np.ndarray, dtype: str) -> np.ndarray:
    """Single RNE of fp64 values to the storage dtype.

    fp32: numpy's float64->float32 cast is IEEE RNE.  bf16: fp64 -> bf16 done
    directly on the fp64 bit pattern (bf16 keeps 8 significant bits; fp64
    has 53) so there is no intermediate fp32 double-rounding."""
    x = np.asarray(x, dtype=np.float64)
    if dtype == "fp32":
        return x.astype(np.float32)
    if dtype == "bf16":
        # Exactly round to 8 significant bits with RNE, then convert (exact).
        m, e = np.frexp(x)                      # x = m * 2^e, 0.5 <= |m| < 1
        scaled = np.ldexp(m, 8)                 # 8 significant bits before the point
        r = np.rint(scaled)                     # numpy rint = round half to even
        y = np.ldexp(r, e - 8)
        return round_fp32_to(y.astype(np.float32), "bf16")   # exact: y has <= 8 bits
    raise ValueError(dtype)


# ---- O-3 ----------------------------------------------------------------------

def average_fp64(grads: Sequence[np.ndarray], dtype: str) -> Tuple[np.ndarray, np.ndarray]:
    """grads[r] = rank r's gradient (same shape).  Returns (ref, den) where
    ref is in the storage dtype and den is fp64."""
    W = len(grads)
    xs = [to_fp32(g, dtype).astype(np.float64) for g in grads]
    tot = np.zeros_like(xs[0])
    absum = np.zeros_like(xs[0])
    for x in xs:
        tot += x          # exact enough: fp64 over <= 8 fp32 values
        absum += np.abs(x)
    return round_fp64_to(tot / W, dtype), absum / W


# ---- O-3b ---------------------------------------------------------------------

def average_bitfaithful(grads: Sequence[np.ndarray], dtype: str) -> np.ndarray:
    W = len(grads)
    s = np.float32(1.0 / W)
    acc = None
    for r in range(W):
        scaled = round_fp32_to(to_fp32(grads[r], dtype) * s, dtype)   # pack + scale
        v = to_fp32(scaled, dtype)
        acc = v.copy() if acc is None else (acc + v).astype(np.float32)
    return round_fp32_to(acc, dtype)


# ---- full simulation: pack -> allreduce -> unpack, W replicas ------------------

def _empty(n: int, dtype: str) -> np.ndarray:
    return np.zeros(n, dtype=np.float32 if dtype == "fp32" else np.uint16)


def pack(a: Assignment, grads: Sequence[np.ndarray], W: int, dtype: str) -> List[np.ndarray]:
    """Alg. 1: view <- b_i.narrow(offset, numel); view.copy_(grad),
    with the 1/W scale applied here (C-2)."""
    s = np.float32(1.0 / W)
    buckets = [_empty(n, dtype) for n in a.bucket_numel]
    for b, slots in enumerate(a.buckets):
        for p, off in slots:
            g = grads[p]
            buckets[b][off:off + g.size] = round_fp32_to(to_fp32(g, dtype) * s, dtype)
    return buckets


def allreduce_sum(per_rank: Sequence[np.ndarray], dtype: str) -> np.ndarray:
    """Elementwise sum over ranks in rank order 0..W-1, fp32 accumulation,
    one rounding to the bucket dtype (C-3, C-4)."""
    acc = None
    for x in per_rank:
        v = to_fp32(x, dtype)
        acc = v.copy() if acc is None else (acc + v).astype(np.float32)
    return round_fp32_to(acc, dtype)


def unpack(a: Assignment, bucket_results: Sequence[np.ndarray], numel: Sequence[int]) -> List[np.ndarray]:
    """L246 / L304: averaged gradients are copied back into the .grad tensors."""
    out = []
    for p, n in enumerate(numel):
        b, off = a.param_bucket[p], a.param_offset[p]
        out.append(bucket_results[b][off:off + n].copy())
    return out


def simulate_ddp_sync(a: Assignment, grads_per_rank: Sequence[Sequence[np.ndarray]], dtype: str
                      ) -> List[List[np.ndarray]]:
    """Every rank packs, the buckets are allreduced (in bucket order), every
    rank unpacks.  Returns per-rank lists of averaged gradients (identical on
    all ranks)."""
    W = len(grads_per_rank)
    numel = [g.size for g in grads_per_rank[0]]
    packed = [pack(a, grads_per_rank[r], W, dtype) for r in range(W)]
    reduced = [allreduce_sum([packed[r][b] for r in range(W)], dtype) for b in range(a.num_buckets)]
    return [unpack(a, reduced, numel) for _ in range(W)]
