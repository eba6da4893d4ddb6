"""O-7: globally unused parameters (find_unused_parameters).  TEST
INFRASTRUCTURE (see oracle/__init__).

Paper:
* PAPER.md L199-L201 (§3.2.3, second caveat): a pass may use only a
  sub-graph; DDP "traverses the autograd graph from the output tensors of the
  forward pass to find all participating parameters" and marks the others
  ready at the end of the forward pass (Alg. 1).
* "DDP should only touch gradients that are indeed involved in
  the backward pass ... locally absent gradients might still be involved in
  the forward/backward pass in a peer DDP process.  Therefore, DDP uses a
  bitmap to keep track of local parameter participants and launches one
  additional AllReduce to collect globally unused parameters."
* one bitmap shared by all parameters, allreduced once.

What the synced pass computes, per parameter p (the plain definition):
  used_r(p)   = rank r produced a gradient for p since the last synced pass
                (no_sync passes accumulate participation)
  c_r(p)      = rank r's gradient of p if used_r(p), else 0 (its bucket slot
                holds zeros: the bucket is averaged as a whole)
  global(p)   = OR_r used_r(p)                        (the bitmap allreduce)
  out_r(p)    = average over r of c_r(p)   if global(p)   (O-3b arithmetic)
              = rank r's gradient untouched otherwise (may be "none")
"""

from __future__ import annotations

from typing import List, Optional, Sequence

import numpy as np

from .average import _empty, average_bitfaithful


def global_used(used: Sequence[Sequence[bool]]) -> List[bool]:
    """used[r][p] -> global participation (the summed bitmap is > 0)."""
    W, n = len(used), len(used[0])
    return [sum(int(used[r][p]) for r in range(W)) > 0 for p in range(n)]


def find_unused_sync(grads: Sequence[Sequence[Optional[np.ndarray]]], used: Sequence[Sequence[bool]],
                     numel: Sequence[int], dtype: str) -> List[List[Optional[np.ndarray]]]:
    """grads[r][p]: rank r's gradient buffer of p before the sync (None = no
    buffer); used[r][p]: participation.  A used parameter must have a buffer.
    Returns out[r][p] per the module docstring; for a globally used parameter
    with no buffer on rank r the average has nowhere to go locally (None)."""
    W = len(grads)
    g = global_used(used)
    out: List[List[Optional[np.ndarray]]] = [[None] * len(numel) for _ in range(W)]
    for p, n in enumerate(numel):
        if not g[p]:
            for r in range(W):
                out[r][p] = None if grads[r][p] is None else grads[r][p].copy()
            continue
        contrib = []
        for r in range(W):
            if used[r][p]:
                assert grads[r][p] is not None, "a participating parameter has a gradient"
                contrib.append(grads[r][p])
            else:
                contrib.append(_empty(n, dtype))       # zeros in the bucket slot
        avg = average_bitfaithful(contrib, dtype)
        for r in range(W):
            out[r][p] = None if grads[r][p] is None else avg.copy()
    return out
