"""O-8: compressed wire (§8(f) N-3).  TEST INFRASTRUCTURE (see oracle/__init__).

Paper: PAPER.md L571-L573 (§6.2.3 "Gradient Compression"): "DDP would
benefit from adaptive compression levels by only communicating gradients with
the necessary precision" — the parameter (and gradient) type need not be the
wire type.

Reading (C-14): fp32 gradients travel as bf16.  Each rank's packed
value is rounded once to the wire type, the sum is accumulated in fp32 in rank
order, and the fp32 result is written back (no second rounding):
    s_q = RNE_bf16( fp32(g_q) *fp32 fl(1/W) )          (pack: scale + compress)
    acc = fp32(s_0) ;  acc = acc +fp32 fp32(s_q),  q = 1..W-1
    y   = acc                                          (fp32 gradient)
"""

from __future__ import annotations

from typing import Sequence

import numpy as np

from .average import round_fp32_to, to_fp32


def average_bf16_wire(grads: Sequence[np.ndarray]) -> np.ndarray:
    """grads[q]: rank q's fp32 gradient.  Returns the fp32 result on every rank."""
    W = len(grads)
    s = np.float32(1.0 / W)
    acc = None
    for q in range(W):
        scaled = (np.asarray(grads[q], dtype=np.float32) * s).astype(np.float32)
        v = to_fp32(round_fp32_to(scaled, "bf16"), "bf16")
        acc = v.copy() if acc is None else (acc + v).astype(np.float32)
    return acc
