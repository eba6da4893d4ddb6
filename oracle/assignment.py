"""O-1: parameter-to-bucket assignment.  TEST INFRASTRUCTURE (see oracle/__init__).

Paper:
* PAPER.md L217 (Algorithm 1, constructor): "init buckets, allocate parameters
  to buckets in the reverse order of net.parameters()".
* PAPER.md L304 (§4.2): "DDP launches AllReduce in the reverse order of
  model.parameters()".
* PAPER.md L308 (§4.2): "By default, each bucket is 25MB in size."
* PAPER.md L415 (§5.2): "zero bucket size means each gradient will be
  communicated on its own".
* PAPER.md L231 (Algorithm 1): ``view <- b_i.narrow(offset, var.size())`` —
  a parameter occupies a contiguous slot [offset, offset+numel) of its bucket.

Readings: C-1 close-before-overflow ("start a new
bucket when adding the next parameter would exceed cap (unless bucket empty)");
an oversized parameter sits alone.  C-5 "MB" = MiB.  C-6 tight packing
(offset = running sum of numel, no padding).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional, Sequence, Tuple

MIB = 1 << 20


@dataclass
class Assignment:
    buckets: List[List[Tuple[int, int]]]   # per bucket: [(param, offset), ...] in scan order
    bucket_numel: List[int]
    param_bucket: List[int]                # param -> bucket
    param_offset: List[int]                # param -> element offset in its bucket

    @property
    def num_buckets(self) -> int:
        return len(self.buckets)


def assign_buckets(numel: Sequence[int], elem_size: int, cap_bytes: int,
                   order: Optional[Sequence[int]] = None) -> Assignment:
    """Greedy scan p = n-1 ... 0 (reverse registration order, Alg. 1), or
    over ``order`` when given (the traced backward order of PAPER.md L563-L565,
    "gradient order prediction": the map is rebuilt from the observed order).

    A bucket is closed before the parameter that would push its byte size over
    ``cap_bytes`` (unless the bucket is empty); each parameter is appended at
    offset = current bucket numel.  Bucket indices increase along the scan."""
    n = len(numel)
    if n < 1:
        raise ValueError("need at least one parameter")
    if cap_bytes < 0 or elem_size <= 0 or any(int(x) < 1 for x in numel):
        raise ValueError("invalid arguments")
    scan = list(range(n - 1, -1, -1)) if order is None else [int(p) for p in order]
    if sorted(scan) != list(range(n)):
        raise ValueError("order must be a permutation of the parameters")
    buckets: List[List[Tuple[int, int]]] = []
    sizes: List[int] = []
    cur: List[Tuple[int, int]] = []
    cur_numel = 0
    for p in scan:
        if cur and (cur_numel + numel[p]) * elem_size > cap_bytes:
            buckets.append(cur)
            sizes.append(cur_numel)
            cur, cur_numel = [], 0
        cur.append((p, cur_numel))
        cur_numel += int(numel[p])
    buckets.append(cur)
    sizes.append(cur_numel)

    pb = [-1] * n
    po = [-1] * n
    for b, slots in enumerate(buckets):
        for p, off in slots:
            pb[p] = b
            po[p] = off
    return Assignment(buckets, sizes, pb, po)
