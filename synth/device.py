"""Device-side synthetic gradients (same recipe as synth/gen.py), via
``synth/lib/libb200synth.so``.  Input generation only."""

from __future__ import annotations

import ctypes as C
import os
from typing import Sequence

from .gen import DISTS, grid_K, param_exp, param_key, param_sigma

_LIB = os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib", "libb200synth.so")
_lib = None


def _l():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB):
            raise ImportError(f"{_LIB} missing; run `python -m paper_2006_15704_b200.build`")
        _lib = C.CDLL(_LIB)
        _lib.synth_fill.restype = C.c_int
        _lib.synth_fill.argtypes = [C.c_void_p, C.c_int64, C.c_int, C.c_int, C.c_uint64, C.c_float, C.c_int,
                                    C.c_int64, C.c_void_p]
    return _lib


def fill(t, seed: int, rank: int, it: int, p: int, dist: str, dtype: str, stream: int = 0) -> None:
    """Fill tensor ``t`` (contiguous, fp32 or bf16, on a CUDA device) with param
    p's synthetic gradient for (seed, rank, it)."""
    key = param_key(seed, rank, it, p)
    st = _l().synth_fill(C.c_void_p(t.data_ptr()), t.numel(), 0 if dtype == "fp32" else 1,
                         DISTS.index(dist), key, float(param_sigma(key)), param_exp(p), grid_K(dtype),
                         C.c_void_p(stream))
    if st != 0:
        raise RuntimeError(f"synth_fill failed with cudaError {st}")


def fill_all(tensors: Sequence, seed: int, rank: int, it: int, dist: str, dtype: str, stream: int = 0) -> None:
    for p, t in enumerate(tensors):
        fill(t, seed, rank, it, p, dist, dtype, stream)
