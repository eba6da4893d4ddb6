"""O-5: no_sync gradient accumulation.  TEST INFRASTRUCTURE (see oracle/__init__).

Paper:
* "the application can conduct n local training iterations
  before synchronizing gradients globally ... this should produce the same
  results as if all data in the large batch is processed in one shot, as
  gradients will simply be accumulated to the same tensor."
* "In no_sync mode, all DDP hooks are disabled, and the first
  backward pass out of the context will synchronize the accumulated gradients
  altogether."

The caller (autograd) accumulates ``.grad += g_t`` in the gradient dtype, in
micro-step order t = 1..n; the synced pass then averages the accumulated
tensors across ranks.  ``accumulate`` replays that accumulation exactly
(fp32 adds for fp32; for bf16, each add is done in fp32 and rounded back to
bf16, as a bf16 ``.grad += g`` does), and ``nosync_average`` applies O-3 /
O-3b to the accumulated tensors.
"""

from __future__ import annotations

from typing import Sequence, Tuple

import numpy as np

from .average import average_bitfaithful, average_fp64, round_fp32_to, to_fp32


def accumulate(micro: Sequence[np.ndarray], dtype: str) -> np.ndarray:
    acc = to_fp32(micro[0], dtype).copy()
    acc = to_fp32(round_fp32_to(acc, dtype), dtype)
    for g in micro[1:]:
        acc = to_fp32(round_fp32_to((acc + to_fp32(g, dtype)).astype(np.float32), dtype), dtype)
    return round_fp32_to(acc, dtype)


def nosync_average(micro_per_rank: Sequence[Sequence[np.ndarray]], dtype: str
                   ) -> Tuple[np.ndarray, np.ndarray, np.ndarray]:
    """micro_per_rank[r][t] = rank r's micro-step-t gradient of one parameter.
    Returns (bitfaithful, ref_fp64, den) of the accumulated gradients."""
    accs = [accumulate(m, dtype) for m in micro_per_rank]
    ref, den = average_fp64(accs, dtype)
    return average_bitfaithful(accs, dtype), ref, den
