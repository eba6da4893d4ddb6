"""Seeded synthetic gradients, host implementation.

This module holds NO arithmetic of the method (no bucketing, no scaling, no
reduction).  It only turns (seed, rank, iter, param, element) into a gradient
value.  The device implementation of the same counter-based generator lives in
``synth/csrc/synth.cu`` (library ``libb200synth.so``); both follow the recipe
below and are cross-checked bit-for-bit by ``tests/test_gpu_synth.py``.

Recipe:

* per-parameter key  k_p = F(F(F(F(seed) ^ rank) ^ iter) ^ p)   (host only)
  with F(x) = fmix64(x + GOLDEN)  (splitmix64 step)
* per-element hash   h_i = fmix64(k_p + (i + 1) * GOLDEN)  mod 2^64
* dist "grid"  (exact sums):  g = k * 2^-e_p,  k = (h mod (2K+1)) - K,
  e_p = 10 + (p mod 11);  K = 2^16 (fp32) or 3 (bf16).  Any sum of <= 64 such
  terms (times any power of two) is exactly representable.
* dist "normal" (realistic):  z = ((u0 + u1) + (u2 + u3)) - 2 with
  u_j = ((h >> 16 j) & 0xFFFF) * 2^-16   (exact in fp32; Irwin-Hall n=4,
  bell-shaped, var 1/3), g = fp32(z * sigma_p) (one IEEE RNE multiply),
  sigma_p = fp32(10^(-4 + 3 u_p)), u_p = (F(k_p) >> 11) * 2^-53
  (log-uniform in [1e-4, 1e-1] per tensor).
* bf16 runs round the fp32 value to bf16 with round-to-nearest-even.

bf16 tensors are carried on the host as uint16 bit patterns (numpy has no bf16).
"""

from __future__ import annotations

from typing import List, Sequence

import numpy as np

SEED = 15704
GOLDEN = 0x9E3779B97F4A7C15
_M1 = 0xBF58476D1CE4E5B9
_M2 = 0x94D049BB133111EB
_MASK = (1 << 64) - 1

DISTS = ("grid", "normal")


def _fmix_int(z: int) -> int:
    z &= _MASK
    z = ((z ^ (z >> 30)) * _M1) & _MASK
    z = ((z ^ (z >> 27)) * _M2) & _MASK
    return z ^ (z >> 31)


def _F(x: int) -> int:
    return _fmix_int((x + GOLDEN) & _MASK)


def param_key(seed: int, rank: int, it: int, p: int) -> int:
    return _F(_F(_F(_F(seed) ^ rank) ^ it) ^ p)


def param_sigma(key: int) -> np.float32:
    u = (_F(key) >> 11) * (2.0 ** -53)
    return np.float32(10.0 ** (-4.0 + 3.0 * u))


def param_exp(p: int) -> int:
    return 10 + (p % 11)


def grid_K(dtype: str) -> int:
    return (1 << 16) if dtype == "fp32" else 3


def _fmix_vec(z: np.ndarray) -> np.ndarray:
    z = z ^ (z >> np.uint64(30))
    z = z * np.uint64(_M1)
    z = z ^ (z >> np.uint64(27))
    z = z * np.uint64(_M2)
    return z ^ (z >> np.uint64(31))


def element_hashes(key: int, idx: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = np.uint64(key) + (idx.astype(np.uint64) + np.uint64(1)) * np.uint64(GOLDEN)
        return _fmix_vec(z)


def fp32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """fp32 -> bf16 bit pattern, round-to-nearest-even (NaN kept quiet)."""
    b = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    rounding = ((b >> np.uint32(16)) & np.uint32(1)) + np.uint32(0x7FFF)
    out = ((b + rounding) >> np.uint32(16)).astype(np.uint16)
    nan = np.isnan(x)
    if nan.any():
        out[nan] = ((b[nan] >> np.uint32(16)) | np.uint32(0x40)).astype(np.uint16)
    return out


def bf16_bits_to_fp32(b: np.ndarray) -> np.ndarray:
    return (np.asarray(b, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32)


def gen_values(seed: int, rank: int, it: int, p: int, idx: np.ndarray, dist: str,
               dtype: str) -> np.ndarray:
    """Values of param p's gradient at element indices ``idx``.

    Returns float32 for dtype 'fp32' and uint16 bf16 bits for 'bf16'."""
    key = param_key(seed, rank, it, p)
    h = element_hashes(key, idx)
    if dist == "grid":
        K = grid_K(dtype)
        k = (h % np.uint64(2 * K + 1)).astype(np.int64) - K
        v = (k.astype(np.float64) * (2.0 ** -param_exp(p))).astype(np.float32)
    elif dist == "normal":
        u = [((h >> np.uint64(16 * j)) & np.uint64(0xFFFF)).astype(np.float32) * np.float32(2.0 ** -16)
             for j in range(4)]
        z = ((u[0] + u[1]) + (u[2] + u[3])) - np.float32(2.0)
        v = (z * param_sigma(key)).astype(np.float32)
    else:
        raise ValueError(f"unknown dist {dist!r}")
    if dtype == "bf16":
        return fp32_to_bf16_bits(v)
    if dtype != "fp32":
        raise ValueError(f"unknown dtype {dtype!r}")
    return v


def gen_grad(seed: int, rank: int, it: int, p: int, numel: int, dist: str, dtype: str) -> np.ndarray:
    return gen_values(seed, rank, it, p, np.arange(numel, dtype=np.int64), dist, dtype)


def gen_grads(numels: Sequence[int], seed: int, rank: int, it: int, dist: str, dtype: str) -> List[np.ndarray]:
    return [gen_grad(seed, rank, it, p, n, dist, dtype) for p, n in enumerate(numels)]


def device_params(numels: Sequence[int], seed: int, rank: int, it: int):
    """Per-parameter (key, sigma, exp) tables handed to the device generator."""
    keys = [param_key(seed, rank, it, p) for p in range(len(numels))]
    sig = [float(param_sigma(k)) for k in keys]
    exps = [param_exp(p) for p in range(len(numels))]
    return keys, sig, exps
