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

import math
from fractions import Fraction
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

def _round_fraction(x: Fraction, dtype: str) -> float:
    """Exact RNE of a rational to the storage dtype's precision (fp32: 24
    significant bits, bf16: 8), normal range; ties to the even significand."""
    if x == 0:
        return 0.0
    bits = 24 if dtype == "fp32" else 8
    _, e = math.frexp(float(abs(x)))
    # pick e so that 2^(e-1) <= |x| < 2^e exactly (the float estimate may be off by one)
    while Fraction(2) ** (e - 1) > abs(x):
        e -= 1
    while Fraction(2) ** e <= abs(x):
        e += 1
    q = Fraction(2) ** (e - bits)                 # spacing of the target grid in [2^(e-1), 2^e)
    lo = (abs(x) / q).__floor__()
    rem = abs(x) / q - lo
    up = rem > Fraction(1, 2) or (rem == Fraction(1, 2) and lo % 2 == 1)
    v = float((lo + (1 if up else 0)) * q)
    return v if x > 0 else -v


def average_fp64(grads: Sequence[np.ndarray], dtype: str) -> Tuple[np.ndarray, np.ndarray]:
    """grads[r] = rank r's gradient (same shape).  Returns (ref, den) where
    ref = RNE_dtype( (sum_r g_r) / W ) rounded ONCE from the exact rational
    value, and den = (sum_r |g_r|) / W in fp64.

    The sum runs in fp64 with an error-free transformation (TwoSum) per add, so
    every element knows whether its fp64 sum is exact.  A value computed in fp64
    rounds to the target like the exact value unless it sits exactly on a
    target rounding midpoint (midpoints are fp64 numbers, and rounding is
    monotonic); only elements that are on a midpoint AND whose fp64 sum or
    quotient was inexact are recomputed with exact rationals."""
    W = len(grads)
    xs = [to_fp32(g, dtype).astype(np.float64) for g in grads]
    tot = np.zeros_like(xs[0])
    absum = np.zeros_like(xs[0])
    inexact = np.zeros(tot.shape, dtype=bool)
    for x in xs:
        s = tot + x
        bb = s - tot
        err = (tot - (s - bb)) + (x - bb)      # TwoSum: tot + x == s + err exactly
        inexact |= err != 0
        tot = s
        absum += np.abs(x)
    q = tot / W
    if W & (W - 1):                            # W not a power of two: the quotient may be rounded
        inexact[...] = True
    ref = round_fp64_to(q, dtype)
    m, _ = np.frexp(q)
    scaled = np.ldexp(m, 24 if dtype == "fp32" else 8)
    midpoint = (scaled - np.floor(scaled)) == 0.5
    redo = np.nonzero(np.ravel(midpoint & inexact))[0]
    if redo.size:
        flat_ref = ref.reshape(-1)
        flat = [np.ravel(x) for x in xs]
        for i in redo:
            exact = sum((Fraction(float(x[i])) for x in flat), Fraction(0)) / W
            v = np.array([_round_fraction(exact, dtype)], dtype=np.float64)
            flat_ref[i] = round_fp64_to(v, dtype)[0]   # exact: v has <= 24 (8) significant bits
    return ref, absum / W


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
