"""Pins for oracle O-7 (globally unused parameters, PAPER.md L199-L201, L259,
L310), independent of the oracle's own averaging code where possible:
exact rational arithmetic on grid inputs, the all-used / all-unused
reductions, and the W=2 one-rank-absent closed form."""

from fractions import Fraction

import numpy as np
import pytest

from oracle.average import average_bitfaithful, to_fp32
from oracle.unused import find_unused_sync, global_used
from synth.gen import gen_grad


def _grads(W, numel, dtype, dist="grid", it=0):
    return [[gen_grad(15704, r, it, p, n, dist, dtype) for p, n in enumerate(numel)] for r in range(W)]


def test_bitmap_or():
    used = [[True, False, False], [False, False, True]]
    assert global_used(used) == [True, False, True]


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
@pytest.mark.parametrize("W", [1, 2, 4, 8])
def test_all_used_is_plain_average(dtype, W):
    numel = [7, 100, 33]
    g = _grads(W, numel, dtype, "normal")
    out = find_unused_sync(g, [[True] * 3] * W, numel, dtype)
    for p in range(3):
        want = average_bitfaithful([g[r][p] for r in range(W)], dtype)
        for r in range(W):
            assert np.array_equal(out[r][p], want)


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
def test_globally_unused_untouched(dtype):
    numel = [50, 9]
    g = _grads(3, numel, dtype, "normal")
    g[1][1] = None                                   # rank 1 has no buffer for p1
    used = [[True, False], [True, False], [True, False]]
    out = find_unused_sync(g, used, numel, dtype)
    assert out[1][1] is None
    for r in (0, 2):
        assert np.array_equal(out[r][1], g[r][1])    # not touched
        assert out[r][1] is not g[r][1]


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
@pytest.mark.parametrize("W", [2, 4, 8])
def test_grid_exact_rational(dtype, W):
    """Grid inputs: every partial sum is exact, so the result equals the exact
    rational (sum over participating ranks) / W — zeros for absent ranks."""
    numel = [64, 31]
    g = _grads(W, numel, dtype)
    rng = np.random.default_rng(W)
    used = [[bool(rng.integers(0, 2)) for _ in numel] for _ in range(W)]
    used[0][0] = True
    out = find_unused_sync(g, used, numel, dtype)
    for p, n in enumerate(numel):
        if not any(used[r][p] for r in range(W)):
            continue
        for i in range(n):
            q = sum(Fraction(float(to_fp32(g[r][p], dtype)[i])) for r in range(W) if used[r][p]) / W
            for r in range(W):
                assert Fraction(float(to_fp32(out[r][p], dtype)[i])) == q


def test_w2_one_rank_absent_is_half():
    """W=2, p used only on rank 0: out = g0 * 1/2 on both ranks (the halving is
    exact in fp32 outside the subnormal range)."""
    g = _grads(2, [1000], "fp32", "normal")
    out = find_unused_sync(g, [[True], [False]], [1000], "fp32")
    want = (g[0][0].astype(np.float64) / 2).astype(np.float32)
    assert np.array_equal(out[0][0], want) and np.array_equal(out[1][0], want)
