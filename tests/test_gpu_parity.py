"""GPU parity: the CUDA path (through the C ABI) vs the oracle, element by element.

Bars: P2P kernels bit-exact vs O-3b on any inputs; every path
bit-exact on exact-grid inputs; NCCL path fp32 |y-ref| <= 1e-6 den, bf16
normwise <= 1e-2; W=1 output == input bit-for-bit (C-12).  Multi-rank
arithmetic is exercised on one GPU by emulation (all ranks in one cooperative
launch, include/b200ddp_emu.h); real multi-process runs are in
tests/test_gpu_multigpu.py."""

import numpy as np
import pytest
import torch

from oracle.assignment import MIB
from oracle.average import average_bitfaithful, average_fp64, to_fp32
from oracle.nosync import accumulate
from paper_2006_15704_b200 import _lib as L
from synth import device as sdev
from synth.gen import gen_grad, gen_values
from synth.shapes import numels
from tests.gpu_util import ESZ, LDT, TDT, param_slices, run_emulated, to_np

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)


# ---- inputs: device generator == host generator ------------------------------

@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
@pytest.mark.parametrize("dist", ["grid", "normal"])
def test_device_generator_bit_exact(dtype, dist):
    for p, n in [(0, 1), (3, 1000), (160, 100_003)]:
        t = torch.empty(n, dtype=TDT[dtype], device="cuda")
        sdev.fill(t, 15704, 2, 1, p, dist, dtype)
        torch.cuda.synchronize()
        assert np.array_equal(to_np(t, dtype), gen_grad(15704, 2, 1, p, n, dist, dtype))


# ---- emulated W ranks: P2P kernels bit-exact vs O-3b -------------------------

def _check_bitfaithful(ins, outs, offs, ns, dtype, W):
    for it in range(len(ins)):
        gi = param_slices(ins[it], offs, ns, dtype)
        go = param_slices(outs[it], offs, ns, dtype)
        for p in range(len(ns)):
            want = average_bitfaithful([gi[r][p] for r in range(W)], dtype)
            for r in range(W):                          # replica consistency too
                assert np.array_equal(go[r][p], want), (it, p, r)


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
@pytest.mark.parametrize("W", [2, 3, 4, 8])
@pytest.mark.parametrize("algo", [L.ALGO_ONESHOT, L.ALGO_TWOSHOT])
@pytest.mark.parametrize("misalign", [False, True])
def test_toy_emulated_bitfaithful(dtype, W, algo, misalign):
    ns = numels("toy")
    ins, outs, offs = run_emulated(ns, dtype, 4096, W, algo, iters=2, misalign=misalign)
    _check_bitfaithful(ins, outs, offs, ns, dtype, W)


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
@pytest.mark.parametrize("W,algo,cap", [(2, L.ALGO_TWOSHOT, 25 * MIB), (4, L.ALGO_TWOSHOT, 5 * MIB),
                                        (8, L.ALGO_TWOSHOT, 25 * MIB), (4, L.ALGO_ONESHOT, 1 * MIB)])
def test_resnet50_emulated_bitfaithful(dtype, W, algo, cap):
    ns = numels("resnet50")
    ins, outs, offs = run_emulated(ns, dtype, cap, W, algo, iters=1)
    _check_bitfaithful(ins, outs, offs, ns, dtype, W)


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
def test_grid_inputs_exact_vs_fp64(dtype):
    ns = numels("toy")
    W = 4
    ins, outs, offs = run_emulated(ns, dtype, 4096, W, L.ALGO_TWOSHOT, dist="grid")
    gi = param_slices(ins[0], offs, ns, dtype)
    go = param_slices(outs[0], offs, ns, dtype)
    for p in range(len(ns)):
        ref, _ = average_fp64([gi[r][p] for r in range(W)], dtype)
        assert np.array_equal(go[0][p], ref)


def test_knobs_never_change_values():
    """cap, algorithm and CTA count change time, never bits."""
    ns = numels("resnet50")[:40]
    W = 4
    base = None
    for cap, algo, ctas, stage in [(1 * MIB, L.ALGO_TWOSHOT, 32, 0), (0, L.ALGO_ONESHOT, 8, 0),
                                   (1 << 40, L.ALGO_TWOSHOT, 3, 0), (4 * MIB, L.ALGO_ONESHOT, 64, 0),
                                   (1 << 40, L.ALGO_TWOSHOT, 5, 16 << 10), (2 * MIB, L.ALGO_ONESHOT, 7, 8 << 10)]:
        ins, outs, offs = run_emulated(ns, "fp32", cap, W, algo,
                                       options={L.OPT_COMM_CTAS: ctas, L.OPT_P2P_STAGE_BYTES: stage})
        if base is None:
            base = outs[0]
            _check_bitfaithful(ins, outs, offs, ns, "fp32", W)
        else:
            assert torch.equal(outs[0], base)


def test_edge_sizes_emulated():
    ns = [1, 2, 3, 5, 7, 255, 256, 257, 4095, 4097, 65537, 1, 3]
    for algo in (L.ALGO_ONESHOT, L.ALGO_TWOSHOT):
        for cap in (0, 64, 1 << 30):
            ins, outs, offs = run_emulated(ns, "bf16", cap, 3, algo, misalign=True)
            _check_bitfaithful(ins, outs, offs, ns, "bf16", 3)


def test_ready_order_permutation_same_result():
    ns = numels("toy")
    rng = np.random.default_rng(1)
    a = run_emulated(ns, "fp32", 4096, 2, L.ALGO_TWOSHOT)[1][0]
    for _ in range(3):
        order = list(rng.permutation(len(ns)))
        assert torch.equal(run_emulated(ns, "fp32", 4096, 2, L.ALGO_TWOSHOT, order=order)[1][0], a)


# ---- real single-process path (W = 1, NCCL communicator of one rank) ----------

def _bind_single(ns, dtype, cap, options=None):
    from paper_2006_15704_b200.ddp import GradReducer
    return GradReducer(ns, dtype, cap, options=options)


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
@pytest.mark.parametrize("algo", [L.ALGO_AUTO, L.ALGO_NCCL, L.ALGO_TWOSHOT])
@pytest.mark.parametrize("model,cap", [("toy", 4096), ("resnet50", 25 * MIB)])
def test_world1_identity(dtype, algo, model, cap):
    ns = numels(model)
    red = _bind_single(ns, dtype, cap, {L.OPT_ALGO: algo})
    grads = [torch.empty(n, dtype=TDT[dtype], device="cuda") for n in ns]
    for it in range(2):
        sdev.fill_all(grads, 7, 0, it, "normal", dtype)
        ref = [g.clone() for g in grads]
        order = list(range(len(ns) - 1, -1, -1))
        for p in order:
            red.grad_ready(p, grads[p])
        red.finalize()
        torch.cuda.synchronize()
        for g, r in zip(grads, ref):
            assert torch.equal(g, r)
    red.check_errors()
    red.close()


def test_world1_many_slots_nccl_split_launch():
    ns = [1 + (i % 7) for i in range(2500)]       # > 1024 slots in one bucket
    red = _bind_single(ns, "fp32", 1 << 40)
    assert red.bucket_algos() == ["nccl"]
    grads = [torch.randn(n, device="cuda") for n in ns]
    ref = [g.clone() for g in grads]
    batch = L.ReadyBatch(list(range(len(ns))), [g.data_ptr() for g in grads])
    red.grads_ready(batch)
    red.finalize()
    torch.cuda.synchronize()
    assert all(torch.equal(a, b) for a, b in zip(grads, ref))
    red.close()


# ---- no_sync (O-5) -------------------------------------------------------------

@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
def test_nosync_accumulation_emulated(dtype):
    """3 passes inside no_sync (the caller accumulates .grad) + 1 synced pass,
    W=2, vs O-5: accumulate in the grad dtype then O-3b."""
    ns = numels("toy")
    W, n_micro = 2, 4
    from tests.gpu_util import flat_layout
    offs, total = flat_layout(ns, False)
    big = torch.zeros(W, total, dtype=TDT[dtype], device="cuda")
    micro = torch.zeros_like(big)
    ctx = L.ddp_create(ns, LDT[dtype], 4096, W, 0)
    L.ddp_set_option(ctx, L.OPT_ALGO, L.ALGO_TWOSHOT)
    sb = L.ddp_storage_bytes(ctx)
    stor = [torch.empty(sb, dtype=torch.uint8, device="cuda") for _ in range(W)]
    comm = torch.cuda.Stream()
    L.ddp_bind_emulated(ctx, torch.cuda.current_device(), comm.cuda_stream, [s.data_ptr() for s in stor],
                        total * ESZ[dtype])
    cur = torch.cuda.current_stream().cuda_stream
    order = list(range(len(ns) - 1, -1, -1))
    batch = L.ReadyBatch(order, [big[0, offs[p]:].data_ptr() for p in order])
    host_micro = [[[] for _ in ns] for _ in range(W)]
    for t in range(n_micro):
        for r in range(W):
            for p, (o, n) in enumerate(zip(offs, ns)):
                sdev.fill(micro[r, o:o + n], 3, r, t, p, "normal", dtype, cur)
        big += micro                                   # caller's .grad += g_t
        for r in range(W):
            for p, (o, n) in enumerate(zip(offs, ns)):
                host_micro[r][p].append(to_np(micro[r, o:o + n], dtype))
        if t < n_micro - 1:
            L.ddp_no_sync_begin(ctx)
            L.ddp_grads_ready(ctx, batch, cur)
            L.ddp_finalize_backward(ctx, cur)
            L.ddp_no_sync_end(ctx)
            assert L.ddp_launch_trace(ctx) == []
        else:
            L.ddp_grads_ready(ctx, batch, cur)
            L.ddp_finalize_backward(ctx, cur)
    torch.cuda.synchronize()
    L.ddp_destroy(ctx)
    out = param_slices(big.cpu(), offs, ns, dtype)
    for p in range(len(ns)):
        accs = [accumulate(host_micro[r][p], dtype) for r in range(W)]
        want = average_bitfaithful(accs, dtype)
        for r in range(W):
            assert np.array_equal(out[r][p], want), p


# ---- full BASELINE sizes: sampled outputs ---------------------------------------

@pytest.mark.parametrize("W,dtype", [(4, "fp32"), (8, "bf16")])
def test_bert_large_emulated_sampled(W, dtype):
    """BERT-large-shaped gradients (335M params, 50/26 buckets at 25 MiB incl.
    the 119 MiB word-embedding bucket) through the two-shot kernel; sampled
    elements vs O-3b computed one by one from the host generator."""
    ns = numels("bert_large")
    ins, outs, offs = None, None, None
    from tests.gpu_util import flat_layout
    offs, total = flat_layout(ns, False)
    if W * total * ESZ[dtype] > 16 * (1 << 30):
        pytest.skip("too large")
    dev = torch.cuda.current_device()
    big = torch.empty(W, total, dtype=TDT[dtype], device="cuda")
    cur = torch.cuda.current_stream().cuda_stream
    for r in range(W):
        for p, (o, n) in enumerate(zip(offs, ns)):
            sdev.fill(big[r, o:o + n], 15704, r, 0, p, "normal", dtype, cur)
    ctx = L.ddp_create(ns, LDT[dtype], 25 * MIB, W, 0)
    L.ddp_set_option(ctx, L.OPT_ALGO, L.ALGO_TWOSHOT)
    stor = [torch.empty(L.ddp_storage_bytes(ctx), dtype=torch.uint8, device="cuda") for _ in range(W)]
    comm = torch.cuda.Stream()
    L.ddp_bind_emulated(ctx, dev, comm.cuda_stream, [s.data_ptr() for s in stor], total * ESZ[dtype])
    order = list(range(len(ns) - 1, -1, -1))
    L.ddp_grads_ready(ctx, L.ReadyBatch(order, [big[0, offs[p]:].data_ptr() for p in order]), cur)
    L.ddp_finalize_backward(ctx, cur)
    torch.cuda.synchronize()
    L.ddp_check_device_errors(ctx)
    L.ddp_destroy(ctx)
    rng = np.random.default_rng(0)
    for p in [0, 1, 2, 5, 100, 200, 390]:
        n = ns[p]
        idx = np.unique(np.concatenate([rng.integers(0, n, 300), [0, n - 1]]))
        want = average_bitfaithful([gen_values(15704, r, 0, p, idx, "normal", dtype) for r in range(W)], dtype)
        got = to_np(big[:, offs[p]:offs[p] + n][:, torch.from_numpy(idx).cuda()], dtype)
        for r in range(W):
            assert np.array_equal(got[r], want), p


@pytest.mark.parametrize("W", [2, 3, 4])
@pytest.mark.parametrize("algo", [L.ALGO_ONESHOT, L.ALGO_TWOSHOT])
def test_pull_and_push_kernels_every_signal_mode(W, algo):
    """The fused kernels in both forms (pull, push, and the default mix: pull for the last bucket),
    every flag-publication mode of the pull form and pipelined stages: bit-exact
    vs O-3b over 3 passes (the pull form alternates two buffers per bucket)."""
    ns = numels("resnet50")[:50]
    for opts in ([{L.OPT_P2P_PULL: 0}, {L.OPT_P2P_PULL: 0, L.OPT_P2P_STAGE_BYTES: 16 << 10}, {L.OPT_P2P_PULL: 1}]
                 + [{L.OPT_P2P_PULL: 2, L.OPT_P2P_SIGNAL: m, L.OPT_P2P_STAGE_BYTES: st}
                    for m in range(4) for st in (0, 16 << 10)]):
        ins, outs, offs = run_emulated(ns, "fp32", 2 * MIB, W, algo, iters=3, misalign=True, options=opts)
        _check_bitfaithful(ins, outs, offs, ns, "fp32", W)
