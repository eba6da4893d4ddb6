"""GPU parity of every W >= 2 exchange on ONE B200 through peer emulation
(include/b200ddp_emu.h ``ddp_bind_peer_emulated``): W native contexts, one
per rank, each driven from its own host thread, over W storages on one device
— the product code per rank (ready tracking, launch order, lanes, the
copy-engine exchanges and their stream-memory-operation flags, the fused P2P
kernels as one cooperative launch per bucket, find_unused's bitmap exchange).

Bars: every path here sums in rank order in fp32 and rounds
once, so outputs equal oracle O-3b (oracle/average.py) BIT FOR BIT, on every
rank (replica consistency); the bf16 wire equals O-8
(oracle/compress.py); find_unused equals O-7 (oracle/unused.py).  Every run
also checks guard bands around each storage and sentinels between the
gradients (no out-of-bounds write).  Inputs are the seeded synthetic
gradients of synth/ (DESIGN.md §4)."""

import numpy as np
import pytest
import torch

from oracle.assignment import MIB
from oracle.average import average_bitfaithful
from oracle.compress import average_bf16_wire
from oracle.nosync import accumulate
from oracle.unused import find_unused_sync, global_used
from paper_2006_15704_b200 import _lib as L
from synth import device as sdev
from synth.gen import gen_values
from synth.shapes import numels
from tests.gpu_util import PeerEmu, flat_layout, param_slices, run_peer_emulated, to_np

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)


def _orders(n, W, seed):
    """Per-rank ready orders: rank 0 reverse registration, the others permuted."""
    rng = np.random.default_rng(seed)
    return [list(range(n - 1, -1, -1))] + [list(rng.permutation(n)) for _ in range(W - 1)]


def _check(ins, outs, offs, ns, dtype, W, ref=average_bitfaithful):
    for it in range(len(ins)):
        gi = param_slices(ins[it], offs, ns, dtype)
        go = param_slices(outs[it], offs, ns, dtype)
        for p in range(len(ns)):
            want = ref([gi[r][p] for r in range(W)], dtype) if ref is average_bitfaithful else \
                ref([gi[r][p] for r in range(W)])
            for r in range(W):
                assert np.array_equal(go[r][p], want), (it, p, r)


# ---- toy: every algorithm, every world, misaligned slots, 3 passes (slot reuse) ----

ALGOS = [L.ALGO_CE, L.ALGO_CE2, L.ALGO_PUSH, L.ALGO_ONESHOT, L.ALGO_TWOSHOT, L.ALGO_AUTO]


@pytest.mark.parametrize("W", [2, 3, 4, 8])
@pytest.mark.parametrize("algo", ALGOS)
@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
@pytest.mark.parametrize("misalign", [False, True])
def test_toy_every_algo(W, algo, dtype, misalign):
    ns = numels("toy")
    ins, outs, offs = run_peer_emulated(ns, dtype, 4096, W, algo, iters=3, misalign=misalign,
                                        orders=_orders(len(ns), W, W * 10 + algo))
    _check(ins, outs, offs, ns, dtype, W)


def test_edge_sizes_ce_family():
    ns = [1, 2, 3, 5, 7, 255, 256, 257, 4095, 4097, 65537, 1, 3]
    for W in (2, 3):
        for algo in (L.ALGO_CE, L.ALGO_CE2, L.ALGO_PUSH):
            for cap in (0, 64, 1 << 30):
                ins, outs, offs = run_peer_emulated(ns, "bf16", cap, W, algo, misalign=True, iters=2)
                _check(ins, outs, offs, ns, "bf16", W)


# ---- full ResNet-50 (25.6M params, 161 tensors), element by element -----------------

RESNET = [  # (W, algo, options, dtype): the shipped policies and every forced exchange
    (2, L.ALGO_AUTO, {}, "fp32"),                                  # one-shot <= 1 MiB, CE above
    (2, L.ALGO_AUTO, {L.OPT_PREFER_OVERLAP: 2}, "bf16"),           # front end's bf16 policy
    (2, L.ALGO_CE, {L.OPT_CE_DIRECT_BYTES: 4 * MIB}, "fp32"),      # direct copies + gathered region
    (3, L.ALGO_CE2, {}, "fp32"),
    (3, L.ALGO_AUTO, {}, "bf16"),
    (4, L.ALGO_AUTO, {}, "fp32"),                                  # two-shot, lanes, last on all CTAs
    (4, L.ALGO_AUTO, {L.OPT_PREFER_OVERLAP: 1}, "fp32"),           # front end's fp32 policy: CE2 + last two-shot
    (4, L.ALGO_PUSH, {}, "bf16"),
    (4, L.ALGO_CE2, {L.OPT_CE_STREAMS: 3}, "fp32"),
    (8, L.ALGO_AUTO, {}, "fp32"),
    (8, L.ALGO_AUTO, {L.OPT_PREFER_OVERLAP: 1}, "fp32"),
    (8, L.ALGO_CE, {}, "bf16"),
    (4, L.ALGO_AUTO, {L.OPT_P2P_PULL: 2}, "fp32"),                  # pull kernels for every bucket
    (2, L.ALGO_AUTO, {L.OPT_P2P_PULL: 0}, "bf16"),                  # push kernels only (round 1)
    (8, L.ALGO_TWOSHOT, {L.OPT_P2P_PULL: 2}, "bf16"),
]


@pytest.mark.parametrize("W,algo,opts,dtype", RESNET)
def test_resnet50_full(W, algo, opts, dtype):
    ns = numels("resnet50")
    ins, outs, offs = run_peer_emulated(ns, dtype, 25 * MIB, W, algo, options=opts, iters=2,
                                        orders=_orders(len(ns), W, 7))
    _check(ins, outs, offs, ns, dtype, W)


@pytest.mark.parametrize("W", [2, 4])
def test_single_bucket_passes(W):
    """A model in ONE bucket: every pass's only device work is the last bucket,
    run on its producer stream with no cross-stream hop (exchange.cpp lone_last);
    three passes alternate the pull buffers and follow each other only through
    the producer stream."""
    ns = numels("resnet50")
    ins, outs, offs = run_peer_emulated(ns, "fp32", 1 << 30, W, L.ALGO_AUTO, iters=3)
    _check(ins, outs, offs, ns, "fp32", W)


@pytest.mark.parametrize("W,cap,algo", [(2, 1 << 30, L.ALGO_AUTO), (4, 1 << 30, L.ALGO_AUTO),
                                         (2, 4096, L.ALGO_AUTO), (4, 4096, L.ALGO_AUTO),
                                         (2, 4096, L.ALGO_CE), (4, 4096, L.ALGO_CE2), (3, 4096, L.ALGO_PUSH)])
def test_device_work_follows_the_producer_stream(W, cap, algo):
    """P:L184-L186 / a5: every bucket's device work is ordered after the hooks'
    producer stream.  Each rank stalls its producer stream, generates its
    gradients on it and only then signals: any launch not ordered after the
    producer would read the previous pass's gradients and miss O-3b."""
    ns = numels("toy")
    pe = PeerEmu(ns, "fp32", cap, W, algo)
    try:
        for it in range(3):
            pe.sync_pass(late_fill=(77, it, "normal"))
            out = param_slices(pe.snapshot(), pe.offs, ns, "fp32")
            for p, n in enumerate(ns):
                want = average_bitfaithful([gen_values(77, r, it, p, np.arange(n), "normal", "fp32")
                                            for r in range(W)], "fp32")
                for r in range(W):
                    assert np.array_equal(out[r][p], want), (it, p, r)
        pe.check_guards()
    finally:
        pe.close()


def test_knobs_never_change_values():
    """cap, exchange, streams and CTA counts change time, never bits."""
    ns = numels("resnet50")[:60]
    W, base = 4, None
    for cap, algo, opts in [(25 * MIB, L.ALGO_CE2, {}), (1 * MIB, L.ALGO_CE, {L.OPT_CE_DIRECT_BYTES: 1 << 16}),
                            (0, L.ALGO_PUSH, {L.OPT_COMM_CTAS: 7}), (5 * MIB, L.ALGO_TWOSHOT, {L.OPT_LANES: 1}),
                            (2 * MIB, L.ALGO_ONESHOT, {L.OPT_COMM_CTAS: 16}),
                            (5 * MIB, L.ALGO_AUTO, {L.OPT_PREFER_OVERLAP: 1, L.OPT_PACK_CTAS: 300})]:
        ins, outs, offs = run_peer_emulated(ns, "fp32", cap, W, algo, options=opts)
        if base is None:
            base = outs[0]
            _check(ins, outs, offs, ns, "fp32", W)
        else:
            assert torch.equal(outs[0], base), (cap, algo, opts)


# ---- N-3: compressed wire (vs O-8) and gradient-as-bucket-view (vs O-3b) ------------

@pytest.mark.parametrize("model,W", [("toy", 3), ("resnet50", 2), ("resnet50", 4), ("resnet50", 8)])
def test_bf16_wire_vs_o8(model, W):
    ns = numels(model)
    ins, outs, offs = run_peer_emulated(ns, "fp32", 4096 if model == "toy" else 25 * MIB, W, L.ALGO_AUTO,
                                        options={L.OPT_WIRE_BF16: 1}, iters=2, misalign=model == "toy")
    _check(ins, outs, offs, ns, "fp32", W, ref=average_bf16_wire)


@pytest.mark.parametrize("model,W,dtype,algo", [("toy", 3, "bf16", L.ALGO_AUTO), ("resnet50", 2, "fp32", L.ALGO_AUTO),
                                                ("resnet50", 4, "fp32", L.ALGO_AUTO),
                                                ("resnet50", 8, "bf16", L.ALGO_AUTO),
                                                ("resnet50", 4, "bf16", L.ALGO_CE)])
def test_grad_view_in_place(model, W, dtype, algo):
    """Gradients ARE their bucket slots (CE in place at W=2, CE2 wider): no pack
    / unpack, each operand x fl(1/W) inside the reduce = O-3b."""
    ns = numels(model)
    cap = 4096 if model == "toy" else 25 * MIB
    ins, outs, offs = run_peer_emulated(ns, dtype, cap, W, algo, grad_view=True, iters=2)
    _check(ins, outs, offs, ns, dtype, W)


def test_grad_view_with_gradients_elsewhere():
    """Some gradients handed over at another address than their slot: copied raw
    in and back (alias runs), still O-3b on every rank."""
    ns = numels("resnet50")
    for W in (2, 4):
        ins, outs, offs = run_peer_emulated(ns, "fp32", 25 * MIB, W, L.ALGO_AUTO, grad_view=True, iters=2,
                                            elsewhere={0, 1, 2, 50, 51, 159, 160})
        _check(ins, outs, offs, ns, "fp32", W)


# ---- N-1: find_unused with rank-specific unused sets (vs O-7) -----------------------

@pytest.mark.parametrize("W,algo", [(2, L.ALGO_CE), (3, L.ALGO_CE2), (4, L.ALGO_PUSH), (4, L.ALGO_CE2),
                                    (8, L.ALGO_CE)])
def test_find_unused_vs_o7(W, algo):
    """p1 unused on every rank (untouched, reported globally unused); p3 used on
    rank 0 only (averaged with zero contributions); p4 unused on odd ranks.  Two
    synced passes (the bitmap slots alternate by pass parity)."""
    ns = numels("toy")
    unused = {r: {1, 3} | ({4} if r % 2 else set()) for r in range(W)}
    unused[0] = {1} | ({4} if 0 % 2 else set())
    pe = PeerEmu(ns, "fp32", 4096, W, algo, options={L.OPT_FIND_UNUSED: 1}, misalign=True)
    try:
        for it in range(2):
            pe.fill(15704, it, "normal")
            before = param_slices(pe.snapshot(), pe.offs, ns, "fp32")
            pe.sync_pass(unused=unused)
            after = param_slices(pe.snapshot(), pe.offs, ns, "fp32")
            used = [[p not in unused[r] for p in range(len(ns))] for r in range(W)]
            want = find_unused_sync(before, used, ns, "fp32")
            gu = [not x for x in global_used(used)]
            for r in range(W):
                assert L.ddp_global_unused(pe.ctx[r], len(ns)) == gu
                for p in range(len(ns)):
                    assert np.array_equal(after[r][p], want[r][p]), (it, r, p)
        pe.check_guards()
    finally:
        pe.close()


def test_find_unused_no_sync_participation():
    """a parameter used in a no_sync pass participates in the next synced
    pass even if that pass does not use it (its accumulated gradient is synced)."""
    ns = numels("toy")
    W = 2
    pe = PeerEmu(ns, "fp32", 4096, W, L.ALGO_CE, options={L.OPT_FIND_UNUSED: 1})
    try:
        pe.fill(3, 0, "normal")
        pe.sync_pass(no_sync=True)                         # every param used, nothing synced
        g0 = param_slices(pe.snapshot(), pe.offs, ns, "fp32")
        pe.sync_pass(unused={0: {2}, 1: {2}})              # p2 unused in the synced pass itself
        out = param_slices(pe.snapshot(), pe.offs, ns, "fp32")
        for r in range(W):
            assert L.ddp_global_unused(pe.ctx[r], len(ns)) == [False] * len(ns)
            for p in range(len(ns)):
                assert np.array_equal(out[r][p], average_bitfaithful([g0[q][p] for q in range(W)], "fp32")), (r, p)
        pe.check_guards()
    finally:
        pe.close()


# ---- a7: no_sync accumulation through the copy-engine exchanges (vs O-5) -----------

@pytest.mark.parametrize("W,algo,dtype", [(2, L.ALGO_AUTO, "bf16"), (4, L.ALGO_CE2, "fp32"),
                                          (4, L.ALGO_AUTO, "fp32")])
def test_no_sync_accumulation(W, algo, dtype):
    """3 passes inside no_sync (the caller accumulates .grad += g_t) + 1 synced
    pass, vs O-5: accumulate in the gradient dtype, then O-3b."""
    ns = numels("toy")
    pe = PeerEmu(ns, dtype, 4096, W, algo)
    try:
        acc_host = [[[] for _ in ns] for _ in range(W)]
        for r in range(W):
            for g in pe.grads[r]:
                g.zero_()
        for t in range(4):
            for r in range(W):
                for p, g in enumerate(pe.grads[r]):
                    m = torch.empty_like(g)
                    sdev.fill(m, 11, r, t, p, "normal", dtype)
                    g += m                                   # the caller's .grad += g_t
                    acc_host[r][p].append(to_np(m, dtype))
            pe.sync_pass(no_sync=t < 3)
        out = param_slices(pe.snapshot(), pe.offs, ns, dtype)
        for p in range(len(ns)):
            want = average_bitfaithful([accumulate(acc_host[r][p], dtype) for r in range(W)], dtype)
            for r in range(W):
                assert np.array_equal(out[r][p], want), (r, p)
    finally:
        pe.close()


# ---- BERT-large (335M params; 119 MiB word-embedding bucket) -------------------------

@pytest.mark.parametrize("W,dtype,opts", [(2, "fp32", {}), (4, "fp32", {L.OPT_PREFER_OVERLAP: 1}),
                                          (4, "bf16", {}), (8, "bf16", {})])
def test_bert_large_word_embedding_whole(W, dtype, opts):
    """The default / overlap policies on BERT-large-shaped gradients (50 fp32 /
    26 bf16 buckets at 25 MiB).  The word embedding (param 0, 31.3M elements,
    the last bucket alone) is compared WHOLE against O-3b; 12 other tensors on
    sampled indices."""
    ns = numels("bert_large")
    pe = PeerEmu(ns, dtype, 25 * MIB, W, L.ALGO_AUTO, options=opts)
    try:
        pe.fill(15704, 0, "normal")
        torch.cuda.synchronize()
        emb_in = [to_np(pe.grads[r][0], dtype) for r in range(W)]
        pe.sync_pass(orders=_orders(len(ns), W, 3))
        want = average_bitfaithful(emb_in, dtype)
        for r in range(W):
            assert np.array_equal(to_np(pe.grads[r][0], dtype), want), r
        rng = np.random.default_rng(0)
        for p in [1, 2, 5, 16, 100, 200, 201, 300, 383, 388, 389, 390]:
            n = ns[p]
            idx = np.unique(np.concatenate([rng.integers(0, n, 500), [0, n - 1]]))
            want = average_bitfaithful([gen_values(15704, r, 0, p, idx, "normal", dtype) for r in range(W)], dtype)
            ti = torch.from_numpy(idx).cuda()
            for r in range(W):
                assert np.array_equal(to_np(pe.grads[r][p][ti], dtype), want), (p, r)
        pe.check_guards()
    finally:
        pe.close()


# ---- failure path: a peer that never arrives ----------------------------------------

def test_dead_peer_copy_engine_times_out():
    """W=2 CE: rank 1 stops after one pass.  Rank 0's wait for rank 1's ready
    flag gives up after DDP_OPT_WAIT_TIMEOUT_MS with DDP_ERR_TIMEOUT and the
    context is poisoned (every later call fails fast)."""
    ns = numels("toy")
    pe = PeerEmu(ns, "fp32", 4096, 2, L.ALGO_CE, options={L.OPT_WAIT_TIMEOUT_MS: 300})
    try:
        pe.fill(1, 0)
        pe.sync_pass()
        order = list(range(len(ns) - 1, -1, -1))
        batch = L.ReadyBatch(order, [pe.grads[0][p].data_ptr() for p in order])
        with pytest.raises(L.DDPError) as e:
            L.ddp_grads_ready(pe.ctx[0], batch, pe.prod[0].cuda_stream)
        assert e.value.status == L.ERR_TIMEOUT and "rank 1" in str(e.value)
        with pytest.raises(L.DDPError) as e:
            L.ddp_finalize_backward(pe.ctx[0], pe.prod[0].cuda_stream)
        assert e.value.status == L.ERR_POISONED
    finally:
        pe.close()


def test_dead_peer_fused_kernel_rendezvous_times_out():
    """W=2, one-shot buckets: rank 1 never reaches the launch -> DDP_ERR_TIMEOUT."""
    ns = numels("toy")
    pe = PeerEmu(ns, "fp32", 4096, 2, L.ALGO_ONESHOT, options={L.OPT_WAIT_TIMEOUT_MS: 300})
    try:
        order = list(range(len(ns) - 1, -1, -1))
        with pytest.raises(L.DDPError) as e:
            L.ddp_grads_ready(pe.ctx[0], L.ReadyBatch(order, [pe.grads[0][p].data_ptr() for p in order]),
                              pe.prod[0].cuda_stream)
        assert e.value.status == L.ERR_TIMEOUT
    finally:
        pe.close()


def test_watchdog_reports_a_pass_that_never_completes():
    """ddp_check_device_errors' host watchdog over the waits with no device-side
    bound (copy-engine flags, NCCL): a finalized pass whose end has not completed
    DDP_OPT_WAIT_TIMEOUT_MS later -> DDP_ERR_TIMEOUT, context poisoned.  Stand-in
    for a peer that never raises a flag: a ~1.5 s GPU spin ahead of the pass on
    the producer stream.  A pass that completes in time is never reported."""
    import time
    from paper_2006_15704_b200.ddp import GradReducer
    ns = numels("toy")
    red = GradReducer(ns, "fp32", 4096, options={L.OPT_WAIT_TIMEOUT_MS: 200})
    try:
        grads = [torch.ones(n, device="cuda") for n in ns]
        for p in range(len(ns) - 1, -1, -1):   # a pass that completes: no report
            red.grad_ready(p, grads[p])
        red.finalize()
        red.check_errors()
        torch.cuda.synchronize()
        time.sleep(0.3)
        red.check_errors()
        torch.cuda._sleep(3_000_000_000)        # holds the producer stream ~1.5 s
        for p in range(len(ns) - 1, -1, -1):
            red.grad_ready(p, grads[p])
        red.finalize()
        red.check_errors()                      # within the bound
        time.sleep(0.5)
        with pytest.raises(L.DDPError) as e:
            red.check_errors()
        assert e.value.status == L.ERR_TIMEOUT and "has not completed" in str(e.value)
        torch.cuda.synchronize()
        with pytest.raises(L.DDPError) as e:
            red.grad_ready(0, grads[0])
        assert e.value.status == L.ERR_POISONED
    finally:
        red.close()


@pytest.mark.parametrize("algo", [L.ALGO_ONESHOT, L.ALGO_TWOSHOT])
def test_dead_peer_in_kernel_barrier_times_out(algo):
    """Cooperative emulation with rank 1's CTAs absent (DDP_OPT_EMU_DEAD_RANK):
    rank 0's CTAs give up after DDP_OPT_P2P_TIMEOUT_MS instead of hanging the
    GPU, set the error word, and ddp_check_device_errors reports DDP_ERR_TIMEOUT
    and poisons the context."""
    ns = numels("toy")
    offs, total = flat_layout(ns, False)
    big = torch.zeros(2, total, device="cuda")
    ctx = L.ddp_create(ns, L.FP32, 4096, 2, 0)
    try:
        L.ddp_set_option(ctx, L.OPT_ALGO, algo)
        L.ddp_set_option(ctx, L.OPT_P2P_TIMEOUT_MS, 50)
        L.ddp_set_option(ctx, L.OPT_EMU_DEAD_RANK, 1)
        stor = [torch.zeros(L.ddp_storage_bytes(ctx), dtype=torch.uint8, device="cuda") for _ in range(2)]
        comm = torch.cuda.Stream()
        L.ddp_bind_emulated(ctx, torch.cuda.current_device(), comm.cuda_stream, [s.data_ptr() for s in stor],
                            total * 4)
        order = list(range(len(ns) - 1, -1, -1))
        cur = torch.cuda.current_stream().cuda_stream
        L.ddp_grads_ready(ctx, L.ReadyBatch(order, [big[0, offs[p]:].data_ptr() for p in order]), cur)
        L.ddp_finalize_backward(ctx, cur)
        torch.cuda.synchronize()
        with pytest.raises(L.DDPError) as e:
            L.ddp_check_device_errors(ctx)
        assert e.value.status == L.ERR_TIMEOUT
        with pytest.raises(L.DDPError) as e:
            L.ddp_grads_ready(ctx, L.ReadyBatch(order, [big[0, offs[p]:].data_ptr() for p in order]), cur)
        assert e.value.status == L.ERR_POISONED
    finally:
        L.ddp_destroy(ctx)
