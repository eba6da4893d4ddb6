"""Pins for oracle O-3 / O-3b / the full pack->allreduce->unpack simulation.

Pins: SPEC worked examples (golden), exact rational arithmetic on small
inputs (brute force), exact-grid inputs, Higham's summation bound, the W=1
identity, layout independence (knobs never change values),
and torch's own bf16 rounding as an independent implementation."""

from fractions import Fraction

import numpy as np
import pytest
import torch

from oracle.assignment import assign_buckets
from oracle.average import (allreduce_sum, average_bitfaithful, average_fp64, round_fp32_to,
                            round_fp64_to, simulate_ddp_sync, to_fp32)
from synth.gen import gen_grad, gen_grads
from synth.shapes import numels
from tests.conftest import load_golden


def test_spec_allreduce_examples():
    for ex in load_golden("paper_examples.json")["allreduce"]:
        xs = [np.array(v, dtype=np.float32) for v in ex["inputs"]]
        assert allreduce_sum(xs, "fp32").tolist() == ex["sum"], ex["cite"]
        ref, _ = average_fp64(xs, "fp32")
        assert ref.tolist() == [s / len(xs) for s in ex["sum"]]


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
def test_spec_L288_g_and_3g_give_2g(dtype):
    g = gen_grad(15704, 0, 0, 3, 4096, "grid", dtype)
    g32 = to_fp32(g, dtype)
    g3 = round_fp32_to(g32 * np.float32(3), dtype)
    assert np.array_equal(to_fp32(g3, dtype), g32 * 3)          # grid: 3g exact
    want = round_fp32_to(g32 * np.float32(2), dtype)
    ref, _ = average_fp64([g, g3], dtype)
    assert np.array_equal(ref, want)
    assert np.array_equal(average_bitfaithful([g, g3], dtype), want)


def _exact_rne(q: Fraction, bits: int) -> Fraction:
    """Round a rational to `bits` significant bits, ties to even (normal range)."""
    if q == 0:
        return q
    sign = -1 if q < 0 else 1
    q = abs(q)
    e = 0
    while q >= 2 ** bits:
        q /= 2
        e += 1
    while q < 2 ** (bits - 1):
        q *= 2
        e -= 1
    fl = q.numerator // q.denominator
    rem = q - fl
    if rem > Fraction(1, 2) or (rem == Fraction(1, 2) and fl % 2 == 1):
        fl += 1
    return sign * Fraction(fl) * Fraction(2) ** e


@pytest.mark.parametrize("dtype,bits", [("fp32", 24), ("bf16", 8)])
@pytest.mark.parametrize("W", [1, 2, 3, 4, 8])
def test_o3_equals_exact_rational_rounding(dtype, bits, W):
    rng = np.random.default_rng(W)
    xs = []
    for r in range(W):
        v = (rng.standard_normal(64) * 10.0 ** rng.uniform(-4, 1)).astype(np.float32)
        xs.append(round_fp32_to(v, dtype))
    ref, den = average_fp64(xs, dtype)
    ref32 = to_fp32(ref, dtype)
    for i in range(64):
        vals = [Fraction(float(to_fp32(xs[r], dtype)[i])) for r in range(W)]
        exact = sum(vals) / W
        assert Fraction(float(ref32[i])) == _exact_rne(exact, bits), (i, W)
        assert den[i] == pytest.approx(float(sum(abs(v) for v in vals) / W), rel=1e-15)


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
@pytest.mark.parametrize("W", [1, 2, 4, 8])
def test_grid_inputs_bit_exact(dtype, W):
    n = 5000
    xs = [gen_grad(15704, r, 0, 7, n, "grid", dtype) for r in range(W)]
    ref, _ = average_fp64(xs, dtype)
    assert np.array_equal(average_bitfaithful(xs, dtype), ref)


@pytest.mark.parametrize("W", [2, 3, 4, 8])
def test_higham_bound_fp32(W):
    n = 200_000
    xs = [gen_grad(1, r, 0, 2, n, "normal", "fp32") for r in range(W)]
    ref, den = average_fp64(xs, "fp32")
    y = average_bitfaithful(xs, "fp32").astype(np.float64)
    err = np.abs(y - ref.astype(np.float64))
    u = 2.0 ** -24
    # (W-1)u from the rank-order fp32 sum, u from the final RNE of ref, and for
    # non-power-of-two W another 2u from fl(1/W) and the pre-scale multiply.
    k = W if (W & (W - 1)) == 0 else W + 2
    assert np.all(err <= k * u * den + 1e-45)
    assert np.all(err <= 1e-6 * den + 1e-45)          # north_star fp32 tolerance


@pytest.mark.parametrize("W", [2, 4, 8])
def test_bf16_tolerance(W):
    n = 200_000
    xs = [gen_grad(1, r, 0, 2, n, "normal", "bf16") for r in range(W)]
    ref, den = average_fp64(xs, "bf16")
    y = to_fp32(average_bitfaithful(xs, "bf16"), "bf16").astype(np.float64)
    r64 = to_fp32(ref, "bf16").astype(np.float64)
    err = np.abs(y - r64)
    assert np.all(err <= 2.0 ** -8 * den + 1e-45)
    assert np.all(err <= 1e-2 * den + 1e-45)           # north_star bf16 tolerance


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
def test_w1_identity(dtype):
    g = gen_grad(3, 0, 0, 1, 9999, "normal", dtype)
    assert np.array_equal(average_bitfaithful([g], dtype), g)
    ref, _ = average_fp64([g], dtype)
    assert np.array_equal(ref, g)
    ns = numels("toy")
    a = assign_buckets(ns, 4 if dtype == "fp32" else 2, 4096)
    gs = gen_grads(ns, 3, 0, 0, "normal", dtype)
    out = simulate_ddp_sync(a, [gs], dtype)[0]
    assert all(np.array_equal(o, g) for o, g in zip(out, gs))


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
@pytest.mark.parametrize("W", [2, 3, 4])
def test_layout_independence_and_replica_consistency(dtype, W):
    ns = numels("toy")
    esize = 4 if dtype == "fp32" else 2
    grads = [gen_grads(ns, 11, r, 0, "normal", dtype) for r in range(W)]
    want = [average_bitfaithful([grads[r][p] for r in range(W)], dtype) for p in range(len(ns))]
    for cap in (0, 1000, 4096, 1 << 30):
        a = assign_buckets(ns, esize, cap)
        out = simulate_ddp_sync(a, grads, dtype)
        for r in range(W):
            for p in range(len(ns)):
                assert np.array_equal(out[r][p], want[p]), (cap, r, p)


def test_bf16_rounding_matches_torch():
    rng = np.random.default_rng(0)
    x = np.concatenate([
        (rng.standard_normal(100_000) * 10.0 ** rng.uniform(-6, 3, 100_000)).astype(np.float32),
        # exact ties: low 16 bits == 0x8000 with even / odd kept LSB
        (np.arange(1000, dtype=np.uint32) << np.uint32(17) | np.uint32(0x3F808000)).view(np.float32),
        (np.arange(1000, dtype=np.uint32) << np.uint32(17) | np.uint32(0x3F818000)).view(np.float32),
    ])
    ours = round_fp32_to(x, "bf16")
    theirs = torch.from_numpy(x).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(ours, theirs)


def test_round_fp64_to_bf16_single_rounding():
    # a value just above a bf16 tie in fp64 that an fp32 intermediate would round onto the tie
    x = np.array([1.0 + 2.0 ** -8 + 2.0 ** -30], dtype=np.float64)
    assert to_fp32(round_fp64_to(x, "bf16"), "bf16")[0] == np.float32(1.0 + 2.0 ** -7)
    rng = np.random.default_rng(5)
    v = rng.standard_normal(2000) * 3
    got = to_fp32(round_fp64_to(v, "bf16"), "bf16")
    for a, b in zip(v, got):
        assert Fraction(float(b)) == _exact_rne(Fraction(float(a)), 8)


def _f32(*vs):
    return [np.array([v], dtype=np.float32) for v in vs]


def test_o3_single_rounding_when_the_fp64_sum_is_inexact():
    """O-3 rounds the EXACT average once.  Hand-derived closed forms where a
    double rounding (fp64 sum, then the target) lands on a target midpoint and
    ties the wrong way:
      W=4: (2 + 2^-23 + 2^-80 + 0)/4 = 0.5 + 2^-25 + 2^-82 -> above the fp32
           midpoint 0.5 + 2^-25 -> 0.5 + 2^-24  (fp64 drops 2^-80: tie -> 0.5);
      W=3: (3 + 3*2^-24 + 2^-60)/3 = 1 + 2^-24 + 2^-60/3 -> 1 + 2^-23
           (fp64: exactly the midpoint 1 + 2^-24 -> 1.0);
      bf16, W=4: (2 + 2^-7 + 2^-80 + 0)/4 -> 0.5 + 2^-8 (bf16 spacing 2^-8)."""
    ref, _ = average_fp64(_f32(2.0, 2.0 ** -23, 2.0 ** -80, 0.0), "fp32")
    assert ref[0] == np.float32(0.5 + 2.0 ** -24)
    ref, _ = average_fp64(_f32(3.0, 3 * 2.0 ** -24, 2.0 ** -60), "fp32")
    assert ref[0] == np.float32(1 + 2.0 ** -23)
    b = [round_fp32_to(x, "bf16") for x in _f32(2.0, 2.0 ** -7, 2.0 ** -80, 0.0)]
    ref, _ = average_fp64(b, "bf16")
    assert to_fp32(ref, "bf16")[0] == np.float32(0.5 + 2.0 ** -8)
    # and a negative mirror image: the sign is carried through
    ref, _ = average_fp64(_f32(-2.0, -(2.0 ** -23), -(2.0 ** -80), 0.0), "fp32")
    assert ref[0] == np.float32(-(0.5 + 2.0 ** -24))
