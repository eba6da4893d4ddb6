"""Input structure pins: workload shapes vs the real model libraries, and the
synthetic generator's documented properties (DESIGN.md input recipe)."""

import numpy as np
import pytest

from synth.gen import (bf16_bits_to_fp32, gen_grad, grid_K, param_exp, param_key, param_sigma)
from synth.shapes import bert_large_shapes, numels, resnet50_shapes


def test_resnet50_matches_torchvision():
    tv = pytest.importorskip("torchvision")
    import torch
    with torch.device("meta"):
        m = tv.models.resnet50()
    theirs = [(n, tuple(p.shape)) for n, p in m.named_parameters()]
    assert theirs == resnet50_shapes()
    assert sum(numels("resnet50")) == 25_557_032 and len(theirs) == 161


def test_bert_large_matches_transformers():
    tr = pytest.importorskip("transformers")
    import torch
    cfg = tr.BertConfig(hidden_size=1024, num_hidden_layers=24, num_attention_heads=16,
                        intermediate_size=4096)
    with torch.device("meta"):
        m = tr.BertModel(cfg)
    theirs = [(n, tuple(p.shape)) for n, p in m.named_parameters()]
    assert theirs == bert_large_shapes()
    assert sum(numels("bert_large")) == 335_141_888 and len(theirs) == 391


def test_toy_total():
    assert sum(numels("toy")) == 10_617 and len(numels("toy")) == 6


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
def test_grid_values_on_grid(dtype):
    p = 5
    v = gen_grad(1, 0, 0, p, 100_000, "grid", dtype)
    x = v if dtype == "fp32" else bf16_bits_to_fp32(v)
    k = x.astype(np.float64) * 2.0 ** param_exp(p)
    assert np.array_equal(k, np.round(k))
    assert np.max(np.abs(k)) <= grid_K(dtype)
    assert len(np.unique(k)) == 2 * grid_K(dtype) + 1 if dtype == "bf16" else len(np.unique(k)) > 50_000


def test_normal_moments_and_sigma_range():
    for p in range(20):
        key = param_key(15704, 0, 0, p)
        s = float(param_sigma(key))
        assert 1e-4 <= s <= 1e-1
    v = gen_grad(15704, 0, 0, 0, 1_000_000, "normal", "fp32").astype(np.float64)
    s = float(param_sigma(param_key(15704, 0, 0, 0)))
    assert abs(v.mean()) < 3e-3 * s
    assert v.var() / s ** 2 == pytest.approx(1 / 3, rel=1e-2)
    assert np.max(np.abs(v)) <= 2 * s


def test_streams_differ_across_rank_iter_param():
    a = gen_grad(1, 0, 0, 0, 64, "normal", "fp32")
    for args in ((1, 1, 0, 0), (1, 0, 1, 0), (1, 0, 0, 1), (2, 0, 0, 0)):
        assert not np.array_equal(a, gen_grad(*args, 64, "normal", "fp32"))
