"""O-2: per-gradient ready tracking and in-order bucket launch, replayed on a
given ready order.  TEST INFRASTRUCTURE (see oracle/__init__).

Paper:
* PAPER.md L186 (§3.2.3): one hook per gradient accumulator; "If hooks of all
  gradients in the same buckets have fired, the last hook will trigger an
  asynchronous AllReduce on that bucket."
* "no process can launch AllReduce on bucket i+1 before
  embarking bucket i".
* PAPER.md L233-L236 (Algorithm 1): "if all grads in b_i are ready, mark b_i as
  ready ... launch AllReduce on ready buckets in order".
* PAPER.md L306 (§4.2): "each bucket keeps a count of pending gradients. Each
  post-hook function decrements the count ... DDP replenishes the pending
  gradient count for every bucket."
* PAPER.md L275 (§3.2.4): in no_sync mode "all DDP hooks are disabled".

Readings: C-7 every consecutive ready bucket from the cursor is
launched within the triggering call; C-8 duplicate -> error, missing ->
error at finalize; C-9 no_sync sampled at pass open.  ``overlap=False`` is
the non-overlapped baseline of PAPER.md L164-L175 / L399 (all launches at
finalize, still in bucket order).
"""

from __future__ import annotations

from typing import List, Sequence, Tuple

from .assignment import Assignment


class ProtocolError(Exception):
    pass


class DuplicateReady(ProtocolError):
    pass


class Incomplete(ProtocolError):
    pass


def replay(a: Assignment, ready_order: Sequence[int], *, no_sync: bool = False,
           overlap: bool = True) -> List[Tuple[int, int]]:
    """Return launches as (bucket, t) where t is the index in ``ready_order`` of
    the grad_ready call that triggered the launch (t = len(order) means the
    launch happened at finalize)."""
    nb = a.num_buckets
    n = len(a.param_bucket)
    pending = [len(s) for s in a.buckets]          # replenished per pass (L306)
    ready = [False] * n
    cursor = 0
    launches: List[Tuple[int, int]] = []
    for t, p in enumerate(ready_order):
        if not (0 <= p < n):
            raise ProtocolError(f"bad param {p}")
        if ready[p]:
            raise DuplicateReady(f"param {p} ready twice")
        ready[p] = True
        b = a.param_bucket[p]
        pending[b] -= 1
        if no_sync or not overlap:
            continue
        while cursor < nb and pending[cursor] == 0:
            launches.append((cursor, t))
            cursor += 1
    if not all(ready):
        raise Incomplete(f"{ready.count(False)} params never became ready")
    if not no_sync:
        while cursor < nb:
            launches.append((cursor, len(ready_order)))
            cursor += 1
    return launches
