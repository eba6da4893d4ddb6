"""O-4: mathematical equivalence on the toy MLP (BASELINE.json configs[0]).
TEST INFRASTRUCTURE (see oracle/__init__).

Paper:
* PAPER.md L25 / L71: distributed data parallel training and local training
  "must be mathematically equivalent"; DDP keeps replicas identical by
  (1) the same initial state and (2) the same (averaged) gradients (L166).
* Reading C-10: equality holds for equal shard sizes and a
  per-rank *mean* loss: mean_r grad(L_r) == grad(L_global).

Model: widths [64,100,37,10], Linear -> ReLU -> Linear -> ReLU -> Linear,
MSE loss averaged over all (batch x output) elements.  Parameters are
ordered like torch's ``nn.Sequential`` registration: fc0.weight (out,in),
fc0.bias, fc1.weight, fc1.bias, fc2.weight, fc2.bias.  All arithmetic fp64;
matmul is numpy's (a library primitive, per the task rules).
"""

from __future__ import annotations

from typing import List, Sequence

import numpy as np

WIDTHS = (64, 100, 37, 10)


def init_params(rng: np.random.Generator, widths=WIDTHS) -> List[np.ndarray]:
    ps = []
    for i in range(len(widths) - 1):
        ps.append(rng.uniform(-0.1, 0.1, size=(widths[i + 1], widths[i])))
        ps.append(rng.uniform(-0.1, 0.1, size=(widths[i + 1],)))
    return ps


def loss(params: Sequence[np.ndarray], x: np.ndarray, y: np.ndarray) -> float:
    h = x
    nl = len(params) // 2
    for i in range(nl):
        h = h @ params[2 * i].T + params[2 * i + 1]
        if i < nl - 1:
            h = np.maximum(h, 0.0)
    return float(np.mean((h - y) ** 2))


def grads(params: Sequence[np.ndarray], x: np.ndarray, y: np.ndarray) -> List[np.ndarray]:
    """Reverse-mode gradient of ``loss`` written out layer by layer."""
    nl = len(params) // 2
    acts = [x]          # inputs to each linear layer
    pre = []            # pre-activations
    h = x
    for i in range(nl):
        z = h @ params[2 * i].T + params[2 * i + 1]
        pre.append(z)
        h = np.maximum(z, 0.0) if i < nl - 1 else z
        if i < nl - 1:
            acts.append(h)
    out = h
    d = 2.0 * (out - y) / out.size                    # dL/dout for the mean
    g: List[np.ndarray] = [None] * len(params)        # type: ignore[list-item]
    for i in range(nl - 1, -1, -1):
        g[2 * i] = d.T @ acts[i]                       # dL/dW_i  (out, in)
        g[2 * i + 1] = d.sum(axis=0)                   # dL/db_i
        if i > 0:
            d = (d @ params[2 * i]) * (pre[i - 1] > 0)  # through ReLU of layer i-1
    return g


def shard_average(params, x, y, W: int) -> List[np.ndarray]:
    """mean over W equal shards of each shard's gradient (what DDP computes)."""
    B = x.shape[0]
    if B % W:
        raise ValueError("equal shards required (reading C-10)")
    s = B // W
    per = [grads(params, x[r * s:(r + 1) * s], y[r * s:(r + 1) * s]) for r in range(W)]
    return [sum(per[r][k] for r in range(W)) / W for k in range(len(params))]
