"""GPU tests of gradient-as-bucket-view (§8(f) N-3, zero-copy variant;
DDP_OPT_GRAD_VIEW) through the front end and the C ABI: after the first synced
backward every ``.grad`` is its bucket slot in the library's storage, the
buckets are averaged in place (no pack / unpack launches) and the result is
the average of the ranks' local gradients — oracle O-3 (Alg. 1
L231-L238): bit-exact O-3b with the copy-engine exchange (world 2 default),
within the NCCL tolerance of test_gpu_multigpu when NCCL is forced, identity
at world 1 (C-12)."""

import os
import tempfile

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from oracle.average import average_bitfaithful, average_fp64

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

NGPU = torch.cuda.device_count()


class _Mlp(torch.nn.Module):
    def __init__(self):
        super().__init__()
        self.a = torch.nn.Linear(32, 64)
        self.b = torch.nn.Linear(64, 64)
        self.c = torch.nn.Linear(64, 8)

    def forward(self, x):
        return self.c(torch.tanh(self.b(torch.tanh(self.a(x)))))


def _in_storage(t: torch.Tensor, st: torch.Tensor) -> bool:
    lo = st.data_ptr()
    return lo <= t.data_ptr() and t.data_ptr() + t.numel() * t.element_size() <= lo + st.numel()


def _passes(ddp, m, local, x, L):
    """Three synced passes: .grad re-created (set_to_none -> copy path), then
    zeroed in place twice (aliased -> zero-copy path).  Returns per pass
    (synced grads, local grads, pack launches, unpack launches, all views)."""
    outs = []
    for it in range(3):
        for p in list(m.parameters()) + list(local.parameters()):
            if it == 0 or p.grad is None:
                p.grad = None
            else:
                p.grad.zero_()
        ddp(x).pow(2).mean().backward()
        local(x).pow(2).mean().backward()
        torch.cuda.synchronize()
        prof = ddp.reducer.profile_read()
        views = all(_in_storage(p.grad, ddp.reducer._storage) for p in m.parameters())
        outs.append(([p.grad.cpu().numpy().copy() for p in m.parameters()],
                     [p.grad.cpu().numpy().copy() for p in local.parameters()],
                     prof["pack"][1], prof["unpack"][1], views))
    return outs


def test_world1_grad_view():
    from paper_2006_15704_b200 import _lib as L
    from paper_2006_15704_b200.ddp import DistributedDataParallel
    torch.manual_seed(3)
    m = _Mlp().cuda()
    local = _Mlp().cuda()
    local.load_state_dict(m.state_dict())
    ddp = DistributedDataParallel(m, bucket_cap_mb=64 * 64 * 4 / 2 ** 20, gradient_as_bucket_view=True,
                                  options={L.OPT_PROFILE: 1})
    try:
        assert set(ddp.reducer.bucket_algos()) == {"nccl"} and ddp.reducer.num_buckets > 1
        outs = _passes(ddp, m, local, torch.randn(16, 32, device="cuda"), L)
        for it, (got, ref, npack, nunpack, views) in enumerate(outs):
            for g, r in zip(got, ref):
                assert np.array_equal(g, r), it                 # world 1: identity (C-12)
            assert views, it                                    # .grad are the slots after every pass
            if it == 0:
                assert npack > 0 and nunpack > 0                # fresh .grad: copied in and back
            else:
                assert npack == 0 and nunpack == 0, (it, npack, nunpack)   # zero-copy
    finally:
        ddp.close()


def _worker(rank, world, init_file, q, opts=None):
    torch.cuda.set_device(rank)
    import torch.distributed as dist
    dist.init_process_group("nccl", init_method=f"file://{init_file}", rank=rank, world_size=world,
                            device_id=torch.device("cuda", rank))
    try:
        from paper_2006_15704_b200 import _lib as L
        from paper_2006_15704_b200.ddp import DistributedDataParallel
        torch.manual_seed(11)
        m = _Mlp().cuda()
        ddp = DistributedDataParallel(m, bucket_cap_mb=0.01, gradient_as_bucket_view=True,
                                      options={L.OPT_PROFILE: 1, **(opts or {})})
        local = _Mlp().cuda()
        local.load_state_dict(m.state_dict())
        torch.manual_seed(50 + rank)                    # different data on every rank
        outs = _passes(ddp, m, local, torch.randn(8, 32, device="cuda"), L)
        algos = ddp.reducer.bucket_algos()
        ddp.close()
        q.put((rank, outs, algos, None))
    except Exception as e:
        q.put((rank, None, None, repr(e)))
    finally:
        dist.destroy_process_group()


def _run2(opts=None, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    fd, init_file = tempfile.mkstemp(prefix="b200ddp_gv_")
    os.close(fd)
    os.unlink(init_file)
    ps = [ctx.Process(target=_worker, args=(r, world, init_file, q, opts)) for r in range(world)]
    for p in ps:
        p.start()
    try:
        res = sorted([q.get(timeout=300) for _ in range(world)], key=lambda x: x[0])
    finally:
        for p in ps:
            p.join(timeout=60)
            if p.is_alive():
                p.kill()
    for r, _, _, err in res:
        assert err is None, f"rank {r}: {err}"
    return res


def _check_views(res, world=2):
    for r in range(world):
        for it in range(3):
            _, _, npack, nunpack, views = res[r][1][it]
            assert views
            assert (npack > 0) if it == 0 else (npack == 0 and nunpack == 0), (it, r, npack, nunpack)


@pytest.mark.multigpu
@pytest.mark.skipif(NGPU < 2, reason="needs >= 2 GPUs")
def test_world2_grad_view_ce():
    world = 2
    res = _run2()
    _check_views(res)
    # the front end's fp32 overlap policy: copy engines in place beside backward, the
    # fused two-shot in place for the last bucket
    assert set(res[0][2][:-1]) == {"ce"} and res[0][2][-1] == "twoshot" and len(res[0][2]) > 1
    for it in range(3):
        for k in range(len(res[0][1][it][0])):
            want = average_bitfaithful([res[r][1][it][1][k].ravel() for r in range(world)], "fp32")
            for r in range(world):
                assert np.array_equal(res[r][1][it][0][k].ravel(), want), (it, k, r)   # O-3b, bit-exact


@pytest.mark.multigpu
@pytest.mark.skipif(NGPU < 2, reason="needs >= 2 GPUs")
def test_world2_grad_view_nccl():
    from paper_2006_15704_b200 import _lib as L
    world = 2
    res = _run2({L.OPT_ALGO: L.ALGO_NCCL})
    _check_views(res)
    assert set(res[0][2]) == {"nccl"}
    for it in range(3):
        for k in range(len(res[0][1][it][0])):
            ref, den = average_fp64([res[r][1][it][1][k].ravel() for r in range(world)], "fp32")
            for r in range(world):
                got = res[r][1][it][0][k].ravel()
                assert np.array_equal(got, res[0][1][it][0][k].ravel())     # replicas identical
                y = got.astype(np.float64)
                assert np.all(np.abs(y - ref.astype(np.float64)) <= 1e-6 * den + 1e-45), (it, k, r)


@pytest.mark.multigpu
@pytest.mark.skipif(NGPU < 4, reason="needs >= 4 GPUs")
def test_world4_grad_view_ce2():
    """World 4: the copy-engine two-shot in place (CE2), bit-exact vs O-3b,
    front end (MLP) and C ABI at full ResNet-50 size (sampled outputs)."""
    world = 4
    res = _run2(world=world)
    _check_views(res, world)
    assert set(res[0][2][:-1]) == {"ce2"} and res[0][2][-1] == "twoshot" and len(res[0][2]) > 1
    for it in range(3):
        for k in range(len(res[0][1][it][0])):
            want = average_bitfaithful([res[r][1][it][1][k].ravel() for r in range(world)], "fp32")
            for r in range(world):
                assert np.array_equal(res[r][1][it][0][k].ravel(), want), (it, k, r)
    from oracle.assignment import MIB
    from paper_2006_15704_b200 import _lib as L
    from synth.gen import gen_values
    from synth.shapes import numels
    from tests.test_gpu_multigpu import _run, _sample_idx
    cfgs = [("resnet50", "fp32", 25 * MIB, L.ALGO_AUTO, 2, {L.OPT_GRAD_VIEW: 1}),
            ("toy", "bf16", 4096, L.ALGO_AUTO, 2, {L.OPT_GRAD_VIEW: 1})]
    outs = _run(world, cfgs)
    for ci, (model, dtype, cap, algo, iters, _) in enumerate(cfgs):
        ns = numels(model)
        assert set(outs[0][ci][1]) == {"twoshot"}   # GradReducer, throughput policy: fused in place
        for it in range(iters):
            for p in range(len(ns)):
                assert len({outs[r][ci][0][it][0][p] for r in range(world)}) == 1, (model, p)
                idx = _sample_idx(p, ns[p])
                xs = [gen_values(15704, r, it, p, idx, "normal", dtype) for r in range(world)]
                assert np.array_equal(outs[0][ci][0][it][1][p], average_bitfaithful(xs, dtype)), (model, it, p)
