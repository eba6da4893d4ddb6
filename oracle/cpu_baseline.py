"""O-6: CPU baseline timing of the oracle AS IT STANDS (never tuned).
TEST INFRASTRUCTURE (see oracle/__init__); called only by bench.py's
``cpu_baseline`` leg and ``bench.py --impl reference``.

Times ``average.simulate_ddp_sync`` (pack with 1/W -> rank-order fp32
allreduce -> unpack, for W in-memory replicas) on seeded synthetic gradients
of the bench workload.  Input generation is outside the timed region.  numpy
elementwise kernels are single-threaded, so one call uses one core.

SURVEY §8(c) O-6 also times T threads, each owning an element range: every
gradient is cut into T contiguous pieces (numpy views, no copy), thread t runs
the SAME ``simulate_ddp_sync`` on piece t of every gradient (its own bucket
assignment of the pieces, made outside the timed region).  The arithmetic is
elementwise, so the pieces' results are the whole problem's results; numpy
releases the GIL inside its loops, so the threads run on separate cores.
"""

from __future__ import annotations

import os
import time
from concurrent.futures import ThreadPoolExecutor
from typing import Dict, Sequence

import numpy as np

from .assignment import assign_buckets
from .average import simulate_ddp_sync


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def time_sync_threads(numel: Sequence[int], dtype: str, cap_bytes: int, W: int, *, seed: int, gen_grads,
                      threads: int = 0, max_iters: int = 3, budget_s: float = 20.0) -> Dict:
    """O-6 all-core mode (module docstring): T = threads or os.cpu_count()."""
    T = threads or os.cpu_count() or 1
    esize = 4 if dtype == "fp32" else 2
    grads = [gen_grads(numel, seed, r, 0, "normal", dtype) for r in range(W)]

    def cut(n, t):
        return (n * t) // T, (n * (t + 1)) // T
    pieces, assigns = [], []
    for t in range(T):
        keep = [p for p, n in enumerate(numel) if cut(n, t)[1] > cut(n, t)[0]]
        pieces.append([[grads[r][p][slice(*cut(numel[p], t))] for p in keep] for r in range(W)])
        assigns.append(assign_buckets([cut(numel[p], t)[1] - cut(numel[p], t)[0] for p in keep], esize, cap_bytes)
                       if keep else None)
    times = []
    start = time.perf_counter()
    with ThreadPoolExecutor(max_workers=T) as ex:
        for _ in range(max(1, max_iters)):
            t0 = time.perf_counter()
            list(ex.map(lambda t: simulate_ddp_sync(assigns[t], pieces[t], dtype) if assigns[t] else None, range(T)))
            times.append(time.perf_counter() - t0)
            if time.perf_counter() - start > budget_s:
                break
    return {"sec_per_iter": float(np.median(times)), "iters": len(times), "threads": T, "W": W}


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
