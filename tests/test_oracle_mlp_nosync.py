"""Pins for O-4 (mathematical equivalence) and O-5 (no_sync,
PAPER.md L264/L275).

The manual backprop in oracle/mlp.py is pinned by central finite differences
(brute force) and by torch.autograd in fp64 (an independent implementation)."""

import numpy as np
import pytest
import torch

from oracle import mlp
from oracle.assignment import assign_buckets
from oracle.average import average_fp64, simulate_ddp_sync, to_fp32
from oracle.nosync import accumulate, nosync_average
from oracle.protocol import replay
from synth.gen import gen_grad
from synth.shapes import numels


def _data(rng, B, widths=mlp.WIDTHS):
    x = rng.uniform(-1, 1, size=(B, widths[0]))
    y = rng.uniform(-1, 1, size=(B, widths[-1]))
    return x, y


def test_grads_match_finite_differences():
    rng = np.random.default_rng(1)
    widths = (5, 4, 3, 2)
    ps = mlp.init_params(rng, widths)
    ps = [p * 5 for p in ps]                        # keep ReLUs away from kinks
    x, y = _data(rng, 3, widths)
    g = mlp.grads(ps, x, y)
    h = 1e-6
    for k, p in enumerate(ps):
        for idx in np.ndindex(p.shape):
            old = p[idx]
            p[idx] = old + h
            lp = mlp.loss(ps, x, y)
            p[idx] = old - h
            lm = mlp.loss(ps, x, y)
            p[idx] = old
            fd = (lp - lm) / (2 * h)
            assert abs(fd - g[k][idx]) <= 1e-7 * max(1.0, abs(fd)), (k, idx)


def test_grads_match_torch_autograd_fp64():
    rng = np.random.default_rng(15704)
    ps = mlp.init_params(rng)
    x, y = _data(rng, 16)
    g = mlp.grads(ps, x, y)
    tp = [torch.tensor(p, dtype=torch.float64, requires_grad=True) for p in ps]
    h = torch.tensor(x)
    for i in range(3):
        h = h @ tp[2 * i].T + tp[2 * i + 1]
        if i < 2:
            h = torch.relu(h)
    torch.mean((h - torch.tensor(y)) ** 2).backward()
    for a, b in zip(g, tp):
        np.testing.assert_allclose(a, b.grad.numpy(), rtol=1e-13, atol=1e-16)


@pytest.mark.parametrize("W", [1, 2, 4, 8])
def test_shard_average_equals_full_batch(W):
    rng = np.random.default_rng(15704)
    ps = mlp.init_params(rng)
    x, y = _data(rng, 16)
    full = mlp.grads(ps, x, y)
    avg = mlp.shard_average(ps, x, y, W)
    for a, b in zip(avg, full):
        assert np.max(np.abs(a - b)) <= 1e-12 * max(1e-300, np.max(np.abs(b)))
    if W > 1:   # the collective must AVERAGE, a plain sum is W x off
        s = [a * W for a in avg]
        assert not np.allclose(s[0], full[0])


def test_toy_shapes_match_oracle_mlp():
    rng = np.random.default_rng(0)
    assert [p.size for p in mlp.init_params(rng)] == numels("toy")


def test_ddp_pipeline_on_mlp_grads_fp64_equivalence():
    """Bucketed pack -> allreduce -> unpack (fp32, W=2) of the shard grads is the
    full-batch gradient within fp32 rounding (equivalence through the whole path)."""
    rng = np.random.default_rng(15704)
    ps = mlp.init_params(rng)
    x, y = _data(rng, 16)
    W = 2
    full = mlp.grads(ps, x, y)
    shards = [[g.astype(np.float32).ravel() for g in mlp.grads(ps, x[r * 8:(r + 1) * 8], y[r * 8:(r + 1) * 8])]
              for r in range(W)]
    a = assign_buckets(numels("toy"), 4, 4096)
    out = simulate_ddp_sync(a, shards, "fp32")
    for r in range(W):
        for o, f in zip(out[r], full):
            np.testing.assert_allclose(o.astype(np.float64), f.ravel(), rtol=0, atol=1e-7 * np.max(np.abs(f)))


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
def test_accumulate_grid_exact(dtype):
    micro = [gen_grad(15704, 0, t, 4, 3000, "grid", dtype) for t in range(8)]
    exact = sum(to_fp32(m, dtype).astype(np.float64) for m in micro)
    assert np.array_equal(to_fp32(accumulate(micro, dtype), dtype).astype(np.float64), exact)


def test_spec_L297_three_in_scope_one_outside():
    """3 micro-batches inside no_sync + 1 synced, W=2 -> equals (4x) the one-shot
    large-batch gradient within 1e-12 (fp64 path)."""
    rng = np.random.default_rng(15704)
    ps = mlp.init_params(rng)
    W, n, b = 2, 4, 4
    x, y = _data(rng, W * n * b)
    # rank r, micro-step t consumes rows [(r*n + t)*b, +b)
    per_rank = []
    for r in range(W):
        acc = None
        for t in range(n):
            sl = slice((r * n + t) * b, (r * n + t + 1) * b)
            g = mlp.grads(ps, x[sl], y[sl])
            acc = g if acc is None else [a + c for a, c in zip(acc, g)]
        per_rank.append(acc)
    synced = [(per_rank[0][k] + per_rank[1][k]) / W for k in range(len(ps))]
    full = mlp.grads(ps, x, y)
    for s, f in zip(synced, full):
        assert np.max(np.abs(s - n * f)) <= 1e-12 * np.max(np.abs(n * f))


def test_nosync_average_fp32_tolerance():
    W, n = 4, 4
    micro = [[gen_grad(9, r, t, 1, 20000, "normal", "fp32") for t in range(n)] for r in range(W)]
    bf, ref, den = nosync_average(micro, "fp32")
    # fp64 closed form (1/W) sum_r sum_t g, vs the replayed accumulation
    closed = sum(to_fp32(micro[r][t], "fp32").astype(np.float64) for r in range(W) for t in range(n)) / W
    acc_err = n * 2.0 ** -24 * den + 1e-45          # accumulation rounding (caller's adds)
    assert np.all(np.abs(ref.astype(np.float64) - closed) <= acc_err + 2.0 ** -24 * np.abs(closed))
    assert np.all(np.abs(bf.astype(np.float64) - ref.astype(np.float64)) <= 1e-6 * den + 1e-45)


def test_empty_scope_is_normal_sync_and_scope_has_no_launches():
    a = assign_buckets(numels("toy"), 4, 4096)
    order = [5, 4, 3, 2, 1, 0]
    assert replay(a, order, no_sync=True) == []
    assert [b for b, _ in replay(a, order)] == [0, 1, 2, 3]


def test_accumulate_bf16_rounds_every_add():
    """A bf16 ``.grad += g`` rounds after EVERY add (gradients are
    accumulated into the same tensor).  1 + 2^-8 is the bf16 midpoint between 1
    and 1 + 2^-7 and ties to the even 1, twice: sequential bf16 adds give 1.0,
    while one rounding of the fp32 sum would give 1 + 2^-7."""
    from oracle.average import round_fp32_to, to_fp32
    micro = [round_fp32_to(np.array([v], dtype=np.float32), "bf16") for v in (1.0, 2.0 ** -8, 2.0 ** -8)]
    assert to_fp32(accumulate(micro, "bf16"), "bf16")[0] == 1.0
    micro = [round_fp32_to(np.array([v], dtype=np.float32), "bf16") for v in (2.0 ** -8, 2.0 ** -8, 1.0)]
    assert to_fp32(accumulate(micro, "bf16"), "bf16")[0] == np.float32(1 + 2.0 ** -7)   # order matters
