"""Pins for oracle O-2 (ready tracking + in-order launch), PAPER.md L186,
L197, L233-L236, L306 and SPEC.md L279-L281, L304."""

import itertools
import random

import pytest

from oracle.assignment import assign_buckets
from oracle.protocol import DuplicateReady, Incomplete, replay
from synth.shapes import numels


def _closed_form(a, order):
    """Bucket b launches at the first call t by which every param of buckets
    0..b has been seen: t_b = max_{b' <= b} max_{p in b'} pos(p)."""
    pos = {p: t for t, p in enumerate(order)}
    out, run = [], -1
    for b, slots in enumerate(a.buckets):
        run = max(run, max(pos[p] for p, _ in slots))
        out.append((b, run))
    return out


def test_spec_L279_reverse_order_launches_mid_backward():
    # 2 buckets of a 4-param chain; hooks fire p_last .. p_first.
    a = assign_buckets([4, 4, 4, 4], 8, 64)
    launches = replay(a, [3, 2, 1, 0])
    assert launches == [(0, 1), (1, 3)]           # b0 launched after the 2nd hook
    assert launches[0][1] < 2                       # before b1's grads exist


def test_spec_L280_deferred_launch():
    a = assign_buckets([4, 4, 4, 4], 8, 64)        # b0={p3,p2}, b1={p1,p0}
    launches = replay(a, [1, 0, 3, 2])               # b1 complete first
    assert [b for b, _ in launches] == [0, 1]
    assert launches == [(0, 3), (1, 3)]              # b1 deferred to b0's launch


def test_spec_L281_no_sync_no_launch():
    a = assign_buckets([4, 4, 4, 4], 8, 64)
    assert replay(a, [3, 2, 1, 0], no_sync=True) == []


def test_all_toy_permutations_closed_form():
    a = assign_buckets(numels("toy"), 4, 4096)
    for order in itertools.permutations(range(6)):
        launches = replay(a, order)
        assert [b for b, _ in launches] == list(range(a.num_buckets))
        assert launches == _closed_form(a, order)


def test_random_orders_real_model():
    rng = random.Random(7)
    a = assign_buckets(numels("resnet50"), 4, 5 << 20)
    for _ in range(50):
        order = list(range(161))
        rng.shuffle(order)
        assert replay(a, order) == _closed_form(a, order)


def test_no_overlap_launches_at_finalize():
    a = assign_buckets(numels("toy"), 4, 4096)
    order = [5, 4, 3, 2, 1, 0]
    assert replay(a, order, overlap=False) == [(b, 6) for b in range(4)]


def test_errors():
    a = assign_buckets(numels("toy"), 4, 4096)
    with pytest.raises(DuplicateReady):
        replay(a, [5, 5])
    with pytest.raises(Incomplete):
        replay(a, [5, 4, 3])
