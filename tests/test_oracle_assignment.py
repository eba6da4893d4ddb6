"""Pins for oracle O-1 (bucket assignment) against what the paper/SPEC fix.

Each pin is independent of oracle/assignment.py's code: hand-worked examples
(tests/golden, cited), degenerate caps, the survey's independently derived
Appendix A table, invariants, and a brute-force alternative formulation."""

import itertools
import random

import pytest

from oracle.assignment import MIB, assign_buckets
from synth.shapes import numels
from tests.conftest import load_golden


def _params_per_bucket(a):
    return [[p for p, _ in slots] for slots in a.buckets]


@pytest.mark.parametrize("case", load_golden("spec_assignment.json")["cases"], ids=lambda c: c["cite"][:40])
def test_spec_examples(case):
    a = assign_buckets(case["numel"], case["elem_size"], case["cap_bytes"])
    assert _params_per_bucket(a) == case["buckets"], case["cite"]


def test_toy_worked_example():
    g = load_golden("toy_buckets.json")
    assert g["numel"] == numels("toy")
    a = assign_buckets(g["numel"], g["elem_size"], g["cap_bytes"])
    assert a.num_buckets == len(g["buckets"])
    for b, exp in enumerate(g["buckets"]):
        assert [list(s) for s in a.buckets[b]] == exp["slots"]
        assert a.bucket_numel[b] == exp["numel"]
        assert a.bucket_numel[b] * 4 == exp["bytes"]


def test_close_after_rule_is_rejected_by_toy():
    # The PyTorch close-after rule gives {p5,p4,p3,p2},{p1,p0} (SURVEY C-1).
    a = assign_buckets(numels("toy"), 4, 4096)
    assert _params_per_bucket(a) != [[5, 4, 3, 2], [1, 0]]


@pytest.mark.parametrize("model", ["resnet50", "bert_large"])
@pytest.mark.parametrize("dtype,esize", [("fp32", 4), ("bf16", 2)])
def test_appendix_a_counts(model, dtype, esize):
    g = load_golden("appendix_a_counts.json")
    ns = numels(model)
    for cap_mib, (nb, last_mib) in zip(g["caps_mib"], g[model][dtype]):
        a = assign_buckets(ns, esize, cap_mib * MIB)
        assert a.num_buckets == nb, (model, dtype, cap_mib)
        nd = 3 if model == "resnet50" else 1
        assert round(a.bucket_numel[-1] * esize / MIB, nd) == pytest.approx(last_mib), (model, dtype, cap_mib)


def test_resnet50_fp32_25mib_membership():
    g = load_golden("appendix_a_counts.json")["resnet50_fp32_25mib_membership"]
    a = assign_buckets(numels("resnet50"), 4, 25 * MIB)
    for b, ((hi, lo), mib) in enumerate(zip(g["param_ranges"], g["mib"])):
        assert _params_per_bucket(a)[b] == list(range(hi, lo - 1, -1))
        assert round(a.bucket_numel[b] * 4 / MIB, 3) == pytest.approx(mib)


def _check_invariants(ns, esize, cap, a):
    # slot tiling: every param in exactly one slot; slots tile [0, numel)
    seen = sorted(p for slots in a.buckets for p, _ in slots)
    assert seen == list(range(len(ns)))
    for b, slots in enumerate(a.buckets):
        off = 0
        for p, o in slots:
            assert o == off
            off += ns[p]
        assert off == a.bucket_numel[b]
        # cap respected unless singleton
        assert len(slots) == 1 or a.bucket_numel[b] * esize <= cap
    # reverse registration order along the scan
    flat = [p for slots in a.buckets for p, _ in slots]
    assert flat == list(range(len(ns) - 1, -1, -1))
    # maximality: the next bucket's first param would have overflowed (greedy)
    for b in range(a.num_buckets - 1):
        nxt = a.buckets[b + 1][0][0]
        assert (a.bucket_numel[b] + ns[nxt]) * esize > cap


def _brute_force(ns, esize, cap):
    """Alternative formulation: repeatedly take the LONGEST prefix of the
    remaining reversed list whose bytes fit in cap (at least one element)."""
    rev = list(range(len(ns) - 1, -1, -1))
    out = []
    while rev:
        best = 1
        for k in range(1, len(rev) + 1):
            if sum(ns[p] for p in rev[:k]) * esize <= cap:
                best = k
        out.append(rev[:best])
        rev = rev[best:]
    return out


def test_brute_force_and_invariants_random():
    rng = random.Random(15704)
    for _ in range(400):
        n = rng.randint(1, 9)
        ns = [rng.randint(1, 50) for _ in range(n)]
        esize = rng.choice([1, 2, 4, 8])
        cap = rng.choice([0, 1, rng.randint(1, 400), 10 ** 9])
        a = assign_buckets(ns, esize, cap)
        _check_invariants(ns, esize, cap, a)
        assert _params_per_bucket(a) == _brute_force(ns, esize, cap)


def test_degenerate_caps_real_models():
    for model in ("resnet50", "bert_large", "toy"):
        ns = numels(model)
        assert assign_buckets(ns, 4, 0).num_buckets == len(ns)
        one = assign_buckets(ns, 4, 1 << 62)
        assert one.num_buckets == 1 and one.bucket_numel[0] == sum(ns)


def test_invalid_args():
    for bad in ([], [0], [3, -1]):
        with pytest.raises(ValueError):
            assign_buckets(bad, 4, 10)
    with pytest.raises(ValueError):
        assign_buckets([3], 4, -1)


def _brute_force_order(ns, esize, cap, order):
    """Longest-prefix formulation over an explicit scan order."""
    rest, out = list(order), []
    while rest:
        best = 1
        for k in range(1, len(rest) + 1):
            if sum(ns[p] for p in rest[:k]) * esize <= cap:
                best = k
        out.append(rest[:best])
        rest = rest[best:]
    return out


def test_explicit_order_brute_force_and_invariants():
    """O-1 with a traced scan order: same greedy rule, scan order
    preserved along the buckets; reverse registration order = the default."""
    rng = random.Random(563)
    for _ in range(300):
        n = rng.randint(1, 9)
        ns = [rng.randint(1, 50) for _ in range(n)]
        esize = rng.choice([1, 2, 4])
        cap = rng.choice([0, rng.randint(1, 300), 10 ** 9])
        order = list(range(n))
        rng.shuffle(order)
        a = assign_buckets(ns, esize, cap, order)
        assert _params_per_bucket(a) == _brute_force_order(ns, esize, cap, order)
        assert [p for slots in a.buckets for p, _ in slots] == order
        d = assign_buckets(ns, esize, cap, list(range(n - 1, -1, -1)))
        assert _params_per_bucket(d) == _params_per_bucket(assign_buckets(ns, esize, cap))
    with pytest.raises(ValueError):
        assign_buckets([1, 2, 3], 4, 10, [0, 0, 1])


try:
    from hypothesis import given, settings
    from hypothesis import strategies as st
except ImportError:  # pragma: no cover
    given = None

if given is not None:
    @settings(max_examples=300, deadline=None)
    @given(ns=st.lists(st.integers(1, 64), min_size=1, max_size=10),
           esize=st.sampled_from([1, 2, 4]), cap=st.integers(0, 400), seed=st.integers(0, 10 ** 6))
    def test_property_assignment_matches_longest_prefix(ns, esize, cap, seed):
        """Property: for any sizes, cap and scan order, the greedy map equals the
        longest-prefix formulation and tiles every bucket exactly."""
        order = list(range(len(ns)))
        random.Random(seed).shuffle(order)
        a = assign_buckets(ns, esize, cap, order)
        assert _params_per_bucket(a) == _brute_force_order(ns, esize, cap, order)
        for b, slots in enumerate(a.buckets):
            assert [o for _, o in slots] == list(itertools.accumulate([0] + [ns[p] for p, _ in slots[:-1]]))
            assert a.bucket_numel[b] == sum(ns[p] for p, _ in slots)
