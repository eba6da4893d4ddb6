"""Pins for oracle O-8 (bf16 wire for fp32 gradients):
torch's own bf16 rounding as an independent implementation (W=1), exact
rationals on bf16-representable grid inputs, and the error bound that follows
from one bf16 rounding per operand plus an fp32 sum of W terms."""

from fractions import Fraction

import numpy as np
import pytest
import torch

from oracle.average import average_fp64, to_fp32
from oracle.compress import average_bf16_wire
from synth.gen import gen_grad


def test_w1_is_torch_bf16_roundtrip():
    g = gen_grad(15704, 0, 0, 5, 100_000, "normal", "fp32")
    want = torch.from_numpy(g).to(torch.bfloat16).to(torch.float32).numpy()
    assert np.array_equal(average_bf16_wire([g]), want)


@pytest.mark.parametrize("W", [2, 4, 8])
def test_grid_bf16_exact(W):
    """bf16-grid inputs (K=3, so k*2^-e is exact in bf16 and every partial sum is
    exact in fp32): the result is the exact rational average."""
    gs = [to_fp32(gen_grad(15704, r, 0, 7, 513, "grid", "bf16"), "bf16") for r in range(W)]
    y = average_bf16_wire(gs)
    for i in range(513):
        q = sum(Fraction(float(g[i])) for g in gs) / W
        assert Fraction(float(y[i])) == q


@pytest.mark.parametrize("W", [2, 3, 4, 8])
def test_error_bound(W):
    """|y - avg| <= (u8 (1 + 2u) + (W-1) u24 (1 + u8)) den with u8 = 2^-8 (bf16 has 8
    significant bits: one RNE costs at most 2^-8 relative), u24 = 2^-24: each
    operand is scaled (exact or one fp32 rounding, plus fl(1/W)) and rounded
    once to bf16, then the fp32 sum adds at most (W-1) u24."""
    gs = [gen_grad(15704, r, 0, 3, 200_000, "normal", "fp32") for r in range(W)]
    y = average_bf16_wire(gs).astype(np.float64)
    xs = [g.astype(np.float64) for g in gs]
    ref = sum(xs) / W
    den = sum(np.abs(x) for x in xs) / W
    u, e = 2.0 ** -8, 2.0 ** -24
    bound = (u * (1 + 2 * e) + 2 * e + (W - 1) * e * (1 + u)) * den
    assert np.all(np.abs(y - ref) <= bound + 1e-45)
    # and it is not the fp32 average: compression is visible
    r32, _ = average_fp64(gs, "fp32")
    assert not np.array_equal(y.astype(np.float32), r32)
