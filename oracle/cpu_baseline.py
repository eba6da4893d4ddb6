"""O-6: CPU baseline timing of the oracle AS IT STANDS (never tuned).
TEST INFRASTRUCTURE (see oracle/__init__); called only by bench.py's
``cpu_baseline`` leg and ``bench.py --impl reference``.

Times ``average.simulate_ddp_sync`` (pack with 1/W -> rank-order fp32
allreduce -> unpack, for W in-memory replicas) on seeded synthetic gradients
of the bench workload.  Input generation is outside the timed region.  numpy
elementwise kernels are single-threaded, so ``cores`` = 1.
"""

from __future__ import annotations

import time
from typing import Dict, Sequence

import numpy as np

from .assignment import assign_buckets
from .average import simulate_ddp_sync


def time_sync(numel: Sequence[int], dtype: str, cap_bytes: int, W: int, *, seed: int,
              gen_grads, max_iters: int = 3, budget_s: float = 20.0, warmup: int = 0) -> Dict:
    """Returns a dict with per-iteration seconds (median), iterations timed and
    the sample description.  ``gen_grads(numel, seed, rank, it, dist, dtype)``
    is the shared synthetic generator (synth.gen.gen_grads).  ``warmup``
    untimed iterations run first (stopped early past half the budget); then up
    to ``max_iters`` timed ones within ``budget_s``."""
    esize = 4 if dtype == "fp32" else 2
    t0 = time.perf_counter()
    a = assign_buckets(numel, esize, cap_bytes)
    t_assign = time.perf_counter() - t0
    grads = [gen_grads(numel, seed, r, 0, "normal", dtype) for r in range(W)]
    start = time.perf_counter()
    done_warmup = 0
    for _ in range(warmup):
        simulate_ddp_sync(a, grads, dtype)
        done_warmup += 1
        if time.perf_counter() - start > budget_s / 2:
            break
    times = []
    start = time.perf_counter()
    for _ in range(max(1, max_iters)):
        t0 = time.perf_counter()
        out = simulate_ddp_sync(a, grads, dtype)
        times.append(time.perf_counter() - t0)
        del out
        if time.perf_counter() - start > budget_s:
            break
    return {
        "sec_per_iter": float(np.median(times)),
        "iters": len(times),
        "warmup": done_warmup,
        "assign_s": t_assign,
        "params": int(sum(numel)),
        "W": W,
        "cores": 1,
    }
