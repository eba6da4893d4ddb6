"""Host-side tests of the C ABI (no GPU): the library loads, exports every
symbol the headers declare, and its integer logic (bucket mapping, ready
tracking, launch order, state machine) equals the oracle bit-for-bit.

Device work is never issued here: protocol tests use DDP_OPT_DRY_RUN, which
runs the same tracking code and records the launch trace only."""

import itertools
import os
import random
import re

import pytest

from oracle.assignment import MIB, assign_buckets
from oracle.protocol import replay
from paper_2006_15704_b200 import _lib as L
from synth.shapes import numels

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    syms = set()
    for h in ("b200ddp.h", "b200ddp_emu.h"):
        txt = open(os.path.join(ROOT, "include", h)).read()
        txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
        syms |= set(re.findall(r"\b(ddp_[a-z_]+)\s*\(", txt))
    return syms


def test_library_exports_every_declared_symbol():
    lib = L.lib()
    syms = _declared_symbols()
    assert syms == set(L._SIGS)          # the binding covers exactly the declared ABI
    for s in sorted(syms):
        assert hasattr(lib, s), s
    assert L.ddp_version().startswith("b200ddp")


def _mapping(ctx):
    out = []
    for b in range(L.ddp_num_buckets(ctx)):
        n, ns = L.ddp_bucket_info(ctx, b)
        out.append((n, [L.ddp_bucket_slot(ctx, b, s) for s in range(ns)]))
    return out


def _oracle_mapping(a):
    return [(a.bucket_numel[b], [(p, o) for p, o in a.buckets[b]]) for b in range(a.num_buckets)]


CASES = [("toy", 4, 4096)] + [(m, e, c * MIB) for m in ("resnet50", "bert_large") for e in (4, 2)
                               for c in (0, 1, 5, 25, 200)]


@pytest.mark.parametrize("model,esize,cap", CASES)
def test_mapping_bit_exact_vs_oracle(model, esize, cap):
    ns = numels(model)
    ctx = L.ddp_create(ns, L.FP32 if esize == 4 else L.BF16, cap, 1, 0)
    try:
        a = assign_buckets(ns, esize, cap)
        assert L.ddp_num_buckets(ctx) == a.num_buckets
        assert _mapping(ctx) == _oracle_mapping(a)
        for p in range(len(ns)):
            assert L.ddp_param_location(ctx, p) == (a.param_bucket[p], a.param_offset[p])
    finally:
        L.ddp_destroy(ctx)


def test_mapping_random_small():
    rng = random.Random(3)
    for _ in range(300):
        ns = [rng.randint(1, 40) for _ in range(rng.randint(1, 10))]
        esize = rng.choice([4, 2])
        cap = rng.choice([0, rng.randint(1, 200), 1 << 40])
        ctx = L.ddp_create(ns, L.FP32 if esize == 4 else L.BF16, cap, 1, 0)
        try:
            assert _mapping(ctx) == _oracle_mapping(assign_buckets(ns, esize, cap))
        finally:
            L.ddp_destroy(ctx)


def _dry_ctx(ns, cap, esize=4, world=1, rank=0):
    ctx = L.ddp_create(ns, L.FP32 if esize == 4 else L.BF16, cap, world, rank)
    L.ddp_set_option(ctx, L.OPT_DRY_RUN, 1)
    return ctx


def _run_pass(ctx, order, batched=False):
    if batched:
        L.ddp_grads_ready(ctx, L.ReadyBatch(order, [0] * len(order)), 0)
    else:
        for p in order:
            L.ddp_grad_ready(ctx, p, 0, 0)
    L.ddp_finalize_backward(ctx, 0)
    return L.ddp_launch_trace(ctx)


def test_launch_trace_all_toy_permutations():
    ns = numels("toy")
    a = assign_buckets(ns, 4, 4096)
    ctx = _dry_ctx(ns, 4096)
    try:
        for order in itertools.permutations(range(6)):   # 720 passes on one context
            assert _run_pass(ctx, list(order)) == replay(a, order)
    finally:
        L.ddp_destroy(ctx)


@pytest.mark.parametrize("model,cap", [("resnet50", 25 * MIB), ("resnet50", 1 * MIB), ("bert_large", 25 * MIB)])
def test_launch_trace_random_orders(model, cap):
    ns = numels(model)
    a = assign_buckets(ns, 4, cap)
    ctx = _dry_ctx(ns, cap)
    rng = random.Random(11)
    try:
        rev = list(range(len(ns) - 1, -1, -1))
        assert _run_pass(ctx, rev) == replay(a, rev)
        assert _run_pass(ctx, rev, batched=True) == replay(a, rev)
        for _ in range(20):
            order = list(range(len(ns)))
            rng.shuffle(order)
            assert _run_pass(ctx, order) == replay(a, order)
    finally:
        L.ddp_destroy(ctx)


def test_overlap_off_launches_at_finalize():
    ns = numels("toy")
    a = assign_buckets(ns, 4, 4096)
    ctx = _dry_ctx(ns, 4096)
    L.ddp_set_option(ctx, L.OPT_OVERLAP, 0)
    try:
        assert _run_pass(ctx, [5, 4, 3, 2, 1, 0]) == replay(a, [5, 4, 3, 2, 1, 0], overlap=False)
    finally:
        L.ddp_destroy(ctx)


def test_no_sync_state_machine():
    ns = numels("toy")
    ctx = _dry_ctx(ns, 4096)
    try:
        L.ddp_no_sync_begin(ctx)
        with pytest.raises(L.DDPError) as e:
            L.ddp_no_sync_begin(ctx)                     # nested
        assert e.value.status == L.ERR_STATE
        assert _run_pass(ctx, [5, 4, 3, 2, 1, 0]) == []   # no launches
        L.ddp_grad_ready(ctx, 5, 0, 0)
        with pytest.raises(L.DDPError) as e:
            L.ddp_no_sync_end(ctx)                       # toggle mid-pass (C-9)
        assert e.value.status == L.ERR_STATE
        for p in [4, 3, 2, 1, 0]:
            L.ddp_grad_ready(ctx, p, 0, 0)
        L.ddp_finalize_backward(ctx, 0)
        L.ddp_no_sync_end(ctx)
        with pytest.raises(L.DDPError) as e:
            L.ddp_no_sync_end(ctx)                       # end without begin
        assert e.value.status == L.ERR_STATE
        assert [b for b, _ in _run_pass(ctx, [5, 4, 3, 2, 1, 0])] == [0, 1, 2, 3]
        L.ddp_no_sync_begin(ctx)                         # empty scope
        L.ddp_no_sync_end(ctx)
        assert [b for b, _ in _run_pass(ctx, [5, 4, 3, 2, 1, 0])] == [0, 1, 2, 3]
    finally:
        L.ddp_destroy(ctx)


def test_duplicate_and_incomplete():
    ns = numels("toy")
    ctx = _dry_ctx(ns, 4096)
    try:
        L.ddp_grad_ready(ctx, 5, 0, 0)
        with pytest.raises(L.DDPError) as e:
            L.ddp_grad_ready(ctx, 5, 0, 0)
        assert e.value.status == L.ERR_DUPLICATE
        with pytest.raises(L.DDPError) as e:
            L.ddp_finalize_backward(ctx, 0)
        assert e.value.status == L.ERR_INCOMPLETE
        with pytest.raises(L.DDPError) as e:
            L.ddp_grad_ready(ctx, 4, 0, 0)
        assert e.value.status == L.ERR_POISONED
    finally:
        L.ddp_destroy(ctx)


def test_argument_and_state_errors():
    with pytest.raises(L.DDPError) as e:
        L.ddp_create([3, 0], L.FP32, 10, 1, 0)
    assert e.value.status == L.ERR_INVALID_ARG
    for bad in (dict(world=0, rank=0), dict(world=2, rank=2), dict(world=9, rank=0)):
        with pytest.raises(L.DDPError):
            L.ddp_create([3], L.FP32, 10, **bad)
    with pytest.raises(L.DDPError):
        L.ddp_create([3], 7, 10, 1, 0)
    ctx = L.ddp_create([3, 4], L.FP32, 10, 1, 0)
    try:
        with pytest.raises(L.DDPError) as e:
            L.ddp_grad_ready(ctx, 0, 0, 0)               # not bound, not dry-run
        assert e.value.status == L.ERR_STATE
        with pytest.raises(L.DDPError) as e:
            L.ddp_finalize_backward(ctx, 0)
        assert e.value.status == L.ERR_STATE
        with pytest.raises(L.DDPError):
            L.ddp_set_option(ctx, 999, 1)
        with pytest.raises(L.DDPError):
            L.ddp_set_option(ctx, L.OPT_COMM_CTAS, 0)
        L.ddp_set_option(ctx, L.OPT_DRY_RUN, 1)
        with pytest.raises(L.DDPError) as e:
            L.ddp_grad_ready(ctx, 2, 0, 0)
        assert e.value.status == L.ERR_INVALID_ARG
        with pytest.raises(L.DDPError) as e:
            L.ddp_bind_device(ctx, 0, b"\0" * 128, 0, [0])
        assert e.value.status == L.ERR_STATE
    finally:
        L.ddp_destroy(ctx)
    L.ddp_destroy(0)   # NULL-safe


def test_algorithm_selection_and_storage_layout():
    ns = numels("resnet50")
    ctx = L.ddp_create(ns, L.FP32, 25 * MIB, 4, 1)
    try:
        L.ddp_set_option(ctx, L.OPT_P2P_ONESHOT_MAX, 9 * MIB)
        L.ddp_set_option(ctx, L.OPT_P2P_TWOSHOT_MAX, 20 * MIB)
        sizes = [L.ddp_bucket_info(ctx, b)[0] * 4 for b in range(L.ddp_num_buckets(ctx))]
        want = [L.ALGO_ONESHOT if s <= 9 * MIB else L.ALGO_TWOSHOT if s <= 20 * MIB else L.ALGO_NCCL
                for s in sizes]
        assert [L.ddp_bucket_algo(ctx, b) for b in range(len(sizes))] == want
        total = L.ddp_storage_bytes(ctx)
        assert total >= sum(sizes) + 64 * 1024
        L.ddp_set_option(ctx, L.OPT_ALGO, L.ALGO_NCCL)
        assert {L.ddp_bucket_algo(ctx, b) for b in range(len(sizes))} == {L.ALGO_NCCL}
        assert L.ddp_get_option(ctx, L.OPT_ALGO) == L.ALGO_NCCL
    finally:
        L.ddp_destroy(ctx)
    one = L.ddp_create(ns, L.FP32, 25 * MIB, 1, 0)   # world 1: everything one-shot
    try:
        assert {L.ddp_bucket_algo(one, b) for b in range(L.ddp_num_buckets(one))} == {L.ALGO_ONESHOT}
    finally:
        L.ddp_destroy(one)


def _algos(ctx):
    return [L.ALGO_NAMES[L.ddp_bucket_algo(ctx, b)] for b in range(L.ddp_num_buckets(ctx))]


@pytest.mark.parametrize("world", [2, 3, 4, 8])
def test_policies_per_world(world):
    """the default (throughput) policy — W=2: the fused one-shot at
    every size (pull kernels), CE with the round-1 push kernels; W>2: one-shot up
    to 1 MiB, two-shot above — and PREFER_OVERLAP=1 (the front end's fp32
    policy): copy engines for every bucket but the last (CE at W=2, CE2 wider),
    the fused kernel for the last; PREFER_OVERLAP=2: fused everywhere."""
    ns = numels("resnet50")
    fused = "oneshot" if world == 2 else "twoshot"
    ctx = L.ddp_create(ns, L.FP32, 25 * MIB, world, 0)
    try:
        sizes = [L.ddp_bucket_info(ctx, b)[0] * 4 for b in range(L.ddp_num_buckets(ctx))]
        assert _algos(ctx) == ["oneshot" if world == 2 or s <= MIB else "twoshot" for s in sizes]
        L.ddp_set_option(ctx, L.OPT_PREFER_OVERLAP, 1)
        a = _algos(ctx)
        assert a[:-1] == ["ce" if world == 2 else "ce2"] * (len(a) - 1) and a[-1] == fused
        L.ddp_set_option(ctx, L.OPT_PREFER_OVERLAP, 2)
        assert set(_algos(ctx)) == {fused}
        L.ddp_set_option(ctx, L.OPT_PREFER_OVERLAP, 0)
        L.ddp_set_option(ctx, L.OPT_P2P_PULL, 0)
        if world == 2:
            assert set(_algos(ctx)) == {"ce"}
    finally:
        L.ddp_destroy(ctx)


def test_pull_kernels_double_buffer_fused_buckets():
    """Pull kernels: a fused bucket run by them gets a second buffer (pass
    parity) instead of per-lane staging.  P2P_PULL=2: every fused bucket;
    1 (default): only the last one, the others keep the push form's per-lane
    two-shot staging (LANES x W slots of the largest shard)."""
    ns = numels("resnet50")
    W, lanes = 4, 4
    ctx = L.ddp_create(ns, L.FP32, 25 * MIB, W, 0)
    try:
        L.ddp_set_option(ctx, L.OPT_ALGO, L.ALGO_NCCL)              # no fused bucket: no second buffers
        base = L.ddp_storage_bytes(ctx)
        sizes = [L.ddp_bucket_info(ctx, b)[0] * 4 for b in range(L.ddp_num_buckets(ctx))]
        a256 = lambda x: (x + 255) // 256 * 256
        L.ddp_set_option(ctx, L.OPT_ALGO, L.ALGO_TWOSHOT)
        L.ddp_set_option(ctx, L.OPT_P2P_PULL, 2)
        assert L.ddp_storage_bytes(ctx) - base == sum(a256(s) for s in sizes)
        L.ddp_set_option(ctx, L.OPT_P2P_PULL, 1)
        shard = max(((s // 4 + W - 1) // W + 255) // 256 * 256 for s in sizes[:-1])
        assert L.ddp_storage_bytes(ctx) - base == a256(sizes[-1]) + lanes * W * a256(shard * 4)
    finally:
        L.ddp_destroy(ctx)


def test_peer_emulated_bind_checks_before_any_device_call():
    """ddp_bind_peer_emulated refuses what it cannot emulate before touching a
    GPU: world 1, missing storages, buckets that need NCCL (> 1024 slots)."""
    c1 = L.ddp_create(numels("toy"), L.FP32, 4096, 1, 0)
    try:
        with pytest.raises(L.DDPError) as e:
            L.ddp_bind_peer_emulated(c1, 0, 0, [256])
        assert e.value.status == L.ERR_INVALID_ARG
    finally:
        L.ddp_destroy(c1)
    big = L.ddp_create([1] * 2000, L.FP32, 1 << 30, 2, 1)           # one bucket of 2000 slots -> NCCL
    try:
        with pytest.raises(L.DDPError) as e:
            L.ddp_bind_peer_emulated(big, 0, 0, [256, 512])
        assert e.value.status == L.ERR_UNSUPPORTED and "NCCL" in str(e.value)
    finally:
        L.ddp_destroy(big)


def test_mark_unused_protocol():
    """ddp_mark_unused is a ready signal (Alg. 1 forward L224-L225): buckets
    holding unused params launch without their hooks, in order (O-2 replay of
    the combined signal sequence); it needs FIND_UNUSED; duplicates are errors;
    FIND_UNUSED adds the bitmap + scratch to the storage."""
    ns = numels("toy")
    ctx = L.ddp_create(ns, L.FP32, 4096, 2, 0)
    try:
        base = L.ddp_storage_bytes(ctx)
        L.ddp_set_option(ctx, L.OPT_DRY_RUN, 1)
        with pytest.raises(L.DDPError) as e:
            L.ddp_mark_unused(ctx, 0, 0, 0)
        assert e.value.status == L.ERR_STATE
        L.ddp_set_option(ctx, L.OPT_FIND_UNUSED, 1)
        assert L.ddp_storage_bytes(ctx) >= base + sum(ns) * 4 + len(ns) * 4
        a = assign_buckets(ns, 4, 4096)
        rng = random.Random(7)
        for _ in range(20):
            unused = [p for p in range(len(ns)) if rng.random() < 0.4]
            order = unused + [p for p in range(len(ns) - 1, -1, -1) if p not in unused]
            for p in order:
                if p in unused:
                    L.ddp_mark_unused(ctx, p, 0, 0)
                else:
                    L.ddp_grad_ready(ctx, p, 0, 0)
            L.ddp_finalize_backward(ctx, 0)
            assert L.ddp_launch_trace(ctx) == replay(a, order)
        L.ddp_mark_unused(ctx, 2, 0, 0)
        for bad in (lambda: L.ddp_mark_unused(ctx, 2, 0, 0), lambda: L.ddp_grad_ready(ctx, 2, 0, 0)):
            with pytest.raises(L.DDPError) as e:
                bad()
            assert e.value.status == L.ERR_DUPLICATE
        with pytest.raises(L.DDPError) as e:
            L.ddp_global_unused(ctx, len(ns))
        assert e.value.status == L.ERR_STATE      # dry run: no bitmap allreduce ever ran
    finally:
        L.ddp_destroy(ctx)


def test_mark_unused_accumulated_grad_required():
    """A param that got a gradient in a no_sync pass participates in the next
    synced pass: marking it unused then needs its accumulated grad."""
    ns = numels("toy")
    ctx = L.ddp_create(ns, L.FP32, 4096, 2, 0)
    try:
        L.ddp_set_option(ctx, L.OPT_DRY_RUN, 1)
        L.ddp_set_option(ctx, L.OPT_FIND_UNUSED, 1)
        L.ddp_no_sync_begin(ctx)
        for p in range(len(ns)):
            L.ddp_grad_ready(ctx, p, 0, 0)
        L.ddp_finalize_backward(ctx, 0)
        L.ddp_no_sync_end(ctx)
        L.ddp_set_option(ctx, L.OPT_DRY_RUN, 1)
        L.ddp_mark_unused(ctx, 0, 0, 0)   # dry run: pointers are not checked
        for p in range(1, len(ns)):
            L.ddp_grad_ready(ctx, p, 0, 0)
        L.ddp_finalize_backward(ctx, 0)
    finally:
        L.ddp_destroy(ctx)


def test_create_ordered_mapping_vs_oracle():
    """ddp_create_ordered (gradient order prediction): the map built
    from an explicit scan order equals the oracle's, bit-exactly; the reverse
    registration order reproduces ddp_create; non-permutations are rejected."""
    rng = random.Random(11)
    for model, cap in [("toy", 4096), ("resnet50", 5 * MIB), ("bert_large", 25 * MIB)]:
        ns = numels(model)
        order = list(range(len(ns)))
        rng.shuffle(order)
        ctx = L.ddp_create_ordered(ns, order, L.FP32, cap, 1, 0)
        try:
            assert _mapping(ctx) == _oracle_mapping(assign_buckets(ns, 4, cap, order))
        finally:
            L.ddp_destroy(ctx)
        rev = list(range(len(ns) - 1, -1, -1))
        c1, c2 = L.ddp_create_ordered(ns, rev, L.FP32, cap, 1, 0), L.ddp_create(ns, L.FP32, cap, 1, 0)
        try:
            assert _mapping(c1) == _mapping(c2)
        finally:
            L.ddp_destroy(c1)
            L.ddp_destroy(c2)
    for bad in ([0, 0, 1, 2, 3, 4], [0, 1, 2, 3, 4, 6], [0, 1, 2]):
        with pytest.raises(L.DDPError) as e:
            L.ddp_create_ordered(numels("toy"), bad + [0] * (6 - len(bad)) if len(bad) < 6 else bad,
                                 L.FP32, 4096, 1, 0)
        assert e.value.status == L.ERR_INVALID_ARG


def test_rebuild_from_traced_order_launches_without_deferral():
    """Trace a pass whose hooks fire in a non-reverse order (ddp_ready_order),
    rebuild the map from it: every bucket then launches exactly at the signal
    of its last slot — no bucket waits behind an earlier one (P:L197 caveat),
    which the replay oracle O-2 confirms."""
    ns = numels("resnet50")
    rng = random.Random(5)
    order = list(range(len(ns)))
    rng.shuffle(order)
    ctx = L.ddp_create(ns, L.FP32, 5 * MIB, 1, 0)
    try:
        L.ddp_set_option(ctx, L.OPT_DRY_RUN, 1)
        for p in order:
            L.ddp_grad_ready(ctx, p, 0, 0)
        L.ddp_finalize_backward(ctx, 0)
        assert L.ddp_ready_order(ctx) == order
    finally:
        L.ddp_destroy(ctx)
    ctx = L.ddp_create_ordered(ns, order, L.FP32, 5 * MIB, 1, 0)
    try:
        L.ddp_set_option(ctx, L.OPT_DRY_RUN, 1)
        for p in order:
            L.ddp_grad_ready(ctx, p, 0, 0)
        L.ddp_finalize_backward(ctx, 0)
        tr = L.ddp_launch_trace(ctx)
        a = assign_buckets(ns, 4, 5 * MIB, order)
        assert tr == replay(a, order)
        ends = list(itertools.accumulate(len(s) for s in a.buckets))
        assert [t for _, t in tr] == [e - 1 for e in ends]
    finally:
        L.ddp_destroy(ctx)


def test_option_and_algo_constants_match_header():
    """The binding's OPT_* / ALGO_* constants equal the header's enum values, and
    every option round-trips through ddp_set_option / ddp_get_option."""
    txt = open(os.path.join(ROOT, "include", "b200ddp.h")).read()
    opts = dict((k, int(v)) for k, v in re.findall(r"^\s*DDP_OPT_([A-Z0-9_]+)\s*=\s*(\d+)\s*,?", txt, re.M))
    algos = dict((k, int(v)) for k, v in re.findall(r"\bDDP_ALGO_([A-Z0-9_]+)\s*=\s*(\d+)\s*[,}]", txt))
    for k, v in opts.items():
        assert getattr(L, "OPT_" + k) == v, k
    for k, v in algos.items():
        assert getattr(L, "ALGO_" + k) == v, k
    ctx = L.ddp_create(numels("toy"), L.FP32, 4096, 2, 0)
    try:
        for k, v in opts.items():
            L.ddp_get_option(ctx, v)                 # every key is known to the library
        for a in algos.values():
            L.ddp_set_option(ctx, L.OPT_ALGO, a)
            assert L.ddp_get_option(ctx, L.OPT_ALGO) == a
    finally:
        L.ddp_destroy(ctx)


@pytest.mark.parametrize("model,esize", [("resnet50", 4), ("bert_large", 2), ("toy", 4)])
def test_grad_view_layout(model, esize):
    """DDP_OPT_GRAD_VIEW (N-3 zero-copy): every bucket is averaged in place (the
    fused two-shot; CE / CE2 when forced or beside a backward under the overlap
    policy; NCCL when forced or at world 1); each parameter's slot (ddp_param_storage_offset) sits at its bucket's
    base + its element offset (O-1 mapping), inside the storage, slots disjoint
    and in the same order as the oracle's buckets."""
    ns = numels(model)
    cap = 25 * MIB
    ctx = L.ddp_create(ns, L.FP32 if esize == 4 else L.BF16, cap, 4, 1)
    try:
        L.ddp_set_option(ctx, L.OPT_ALGO, L.ALGO_CE2)
        L.ddp_set_option(ctx, L.OPT_GRAD_VIEW, 1)
        assert L.ddp_get_option(ctx, L.OPT_GRAD_VIEW) == 1
        nb = L.ddp_num_buckets(ctx)
        assert {L.ddp_bucket_algo(ctx, b) for b in range(nb)} == {L.ALGO_CE2}   # forced: CE2 in place
        L.ddp_set_option(ctx, L.OPT_ALGO, L.ALGO_AUTO)
        assert {L.ddp_bucket_algo(ctx, b) for b in range(nb)} == {L.ALGO_TWOSHOT}  # fused two-shot in place
        L.ddp_set_option(ctx, L.OPT_ALGO, L.ALGO_NCCL)
        assert {L.ddp_bucket_algo(ctx, b) for b in range(nb)} == {L.ALGO_NCCL}
        L.ddp_set_option(ctx, L.OPT_ALGO, L.ALGO_TWOSHOT)
        total = L.ddp_storage_bytes(ctx)
        a = assign_buckets(ns, esize, cap)
        spans = []
        for b, slots in enumerate(a.buckets):
            base = None
            for p, off in slots:
                o = L.ddp_param_storage_offset(ctx, p)
                bb, eo = L.ddp_param_location(ctx, p)
                assert bb == b and eo == off
                base = o - eo * esize if base is None else base
                assert o == base + off * esize and base % 256 == 0
                assert 0 <= o and o + ns[p] * esize <= total
                spans.append((o, o + ns[p] * esize))
        spans.sort()
        assert all(x[1] <= y[0] for x, y in zip(spans, spans[1:]))
        # not combinable with the options that need their own copies
        with pytest.raises(L.DDPError) as e:
            L.ddp_set_option(ctx, L.OPT_FIND_UNUSED, 1)
        assert e.value.status == L.ERR_UNSUPPORTED
        if esize == 4:
            with pytest.raises(L.DDPError) as e:
                L.ddp_set_option(ctx, L.OPT_WIRE_BF16, 1)
            assert e.value.status == L.ERR_UNSUPPORTED
        with pytest.raises(L.DDPError):
            L.ddp_param_storage_offset(ctx, len(ns))
        L.ddp_set_option(ctx, L.OPT_GRAD_VIEW, 0)
        assert {L.ddp_bucket_algo(ctx, b) for b in range(nb)} == {L.ALGO_TWOSHOT}
        # world 2: the fused two-shot in place (no second buffer, no staging); under the
        # overlap policy the copy engines beside backward, the fused kernel for the last
        # bucket; NCCL when forced
        two = L.ddp_create(ns, L.FP32 if esize == 4 else L.BF16, cap, 2, 0)
        try:
            L.ddp_set_option(two, L.OPT_GRAD_VIEW, 1)
            assert {L.ddp_bucket_algo(two, b) for b in range(nb)} == {L.ALGO_TWOSHOT}
            in_place = L.ddp_storage_bytes(two)
            L.ddp_set_option(two, L.OPT_ALGO, L.ALGO_CE)
            assert L.ddp_storage_bytes(two) >= in_place + 2 * sum(ns) * esize   # CE adds W receive slots
            L.ddp_set_option(two, L.OPT_ALGO, L.ALGO_AUTO)
            L.ddp_set_option(two, L.OPT_PREFER_OVERLAP, 1)
            al = [L.ddp_bucket_algo(two, b) for b in range(nb)]
            assert al[-1] == L.ALGO_TWOSHOT and set(al[:-1]) <= {L.ALGO_CE}
            L.ddp_set_option(two, L.OPT_PREFER_OVERLAP, 0)
            L.ddp_set_option(two, L.OPT_ALGO, L.ALGO_NCCL)
            assert {L.ddp_bucket_algo(two, b) for b in range(nb)} == {L.ALGO_NCCL}
        finally:
            L.ddp_destroy(two)
        L.ddp_set_option(ctx, L.OPT_FIND_UNUSED, 1)
        with pytest.raises(L.DDPError) as e:
            L.ddp_set_option(ctx, L.OPT_GRAD_VIEW, 1)
        assert e.value.status == L.ERR_UNSUPPORTED
    finally:
        L.ddp_destroy(ctx)


@pytest.mark.parametrize("world", [1, 2, 4])
def test_grad_view_protocol_unchanged(world):
    """GRAD_VIEW changes only what a launched bucket does on the device, not the
    protocol: the launch trace of random ready orders (dry run) is the oracle
    replay O-2 of the O-1 map, as without the option (Alg. 1)."""
    ns = numels("resnet50")
    a = assign_buckets(ns, 4, 5 * MIB)
    ctx = L.ddp_create(ns, L.FP32, 5 * MIB, world, world - 1)
    L.ddp_set_option(ctx, L.OPT_GRAD_VIEW, 1)
    L.ddp_set_option(ctx, L.OPT_DRY_RUN, 1)
    rng = random.Random(29 + world)
    try:
        want = {1: L.ALGO_NCCL, 2: L.ALGO_TWOSHOT, 4: L.ALGO_TWOSHOT}[world]
        assert {L.ddp_bucket_algo(ctx, b) for b in range(L.ddp_num_buckets(ctx))} == {want}
        for _ in range(10):
            order = list(range(len(ns)))
            rng.shuffle(order)
            assert _run_pass(ctx, order) == replay(a, order)
    finally:
        L.ddp_destroy(ctx)


# Defaults as include/b200ddp.h documents them, and the accepted range of every
# bounded option (one below / the bounds / one above).
_DEFAULTS = {
    "OVERLAP": 1, "P2P_ONESHOT_MAX": -1, "P2P_TWOSHOT_MAX": 2**63 - 1, "COMM_CTAS": 32, "DRY_RUN": 0,
    "PROFILE": 0, "ALGO": 0, "PACK_CTAS": 4736, "P2P_STAGE_BYTES": 0, "FIND_UNUSED": 0, "MULTICAST": 0,
    "CE_STREAMS": 1, "NCCL_COMMS": 1, "CE_DIRECT_BYTES": 16 * MIB, "WIRE_BF16": 0, "LANES": 4,
    "LOW_PRIORITY": 1, "PREFER_OVERLAP": 0, "GRAD_VIEW": 0, "P2P_TIMEOUT_MS": 30000, "WAIT_TIMEOUT_MS": 60000,
    "EMU_DEAD_RANK": -1, "P2P_PULL": 1, "P2P_SIGNAL": 0, "P2P_DEBUG": 0, "LAST_ON_PRODUCER": 1,
}
_RANGES = {  # name: (lowest legal, highest legal or None = unbounded)
    "ALGO": (0, 7), "PREFER_OVERLAP": (0, 2), "LANES": (1, 4), "CE_STREAMS": (1, 16), "NCCL_COMMS": (1, 8),
    "COMM_CTAS": (1, 148), "PACK_CTAS": (1, 148 * 64), "P2P_PULL": (0, 2), "P2P_SIGNAL": (0, 3),
    "P2P_DEBUG": (0, 7), "EMU_DEAD_RANK": (-1, 1), "P2P_ONESHOT_MAX": (0, None), "P2P_TWOSHOT_MAX": (0, None),
    "CE_DIRECT_BYTES": (0, None), "P2P_STAGE_BYTES": (0, None), "P2P_TIMEOUT_MS": (1, None),
    "WAIT_TIMEOUT_MS": (1, None),
}
_BOOLEANS = ("OVERLAP", "PROFILE", "DRY_RUN", "FIND_UNUSED", "MULTICAST", "WIRE_BF16", "LOW_PRIORITY",
             "GRAD_VIEW", "LAST_ON_PRODUCER")


def test_option_defaults_ranges_and_booleans():
    keys = {n[4:]: getattr(L, n) for n in dir(L) if n.startswith("OPT_")}
    assert set(keys) == set(_DEFAULTS)
    ctx = L.ddp_create([3, 4], L.FP32, 10, 2, 0)
    try:
        for name, want in _DEFAULTS.items():
            assert L.ddp_get_option(ctx, keys[name]) == want, name
    finally:
        L.ddp_destroy(ctx)

    def accepted(name, v):
        c = L.ddp_create([3, 4], L.FP32, 10, 2, 0)
        try:
            L.ddp_set_option(c, keys[name], v)
            return L.ddp_get_option(c, keys[name])
        except L.DDPError as e:
            assert e.status == L.ERR_INVALID_ARG, (name, v)
            return None
        finally:
            L.ddp_destroy(c)

    for name, (lo, hi) in _RANGES.items():
        assert accepted(name, lo - 1) is None, name
        assert accepted(name, lo) == lo, name
        if hi is not None:
            assert accepted(name, hi) == hi, name
            assert accepted(name, hi + 1) is None, name
    for name in _BOOLEANS:                       # any non-zero value reads back as 1
        assert accepted(name, 2) == 1 and accepted(name, 0) == 0, name


def test_product_path_has_no_fallback(monkeypatch):
    """The product path fails loudly without its native library (no CPU or
    oracle fallback), and nothing in the package or the C/CUDA sources refers to
    oracle/ (the oracle is test infrastructure only)."""
    monkeypatch.setattr(L, "_lib", None)
    monkeypatch.setattr(L, "LIB_PATH", os.path.join(ROOT, "no-such-dir", "libb200ddp.so"))
    with pytest.raises(ImportError, match="no fallback"):
        L.ddp_version()
    pkg = os.path.join(ROOT, "paper_2006_15704_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                txt = open(os.path.join(dirpath, f), errors="replace").read()
                assert not re.search(r"^\s*(from|import)\s+oracle\b|#include\s*[<\"][^>\"]*oracle", txt, re.M), f
