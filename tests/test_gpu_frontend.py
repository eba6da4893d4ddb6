"""GPU tests of the front end's construction-side rows (§8(f) N-4) through the
C ABI: the constructor's parameter broadcast (Alg. 1) and the
rebuild of the parameter-to-bucket map from the traced backward order
("gradient order prediction"), checked against oracle O-1
(assignment with an explicit order) and O-2 (launch replay), and gradients
against a plain local backward (world 1) / oracle O-3b (world 2)."""

import itertools
import os
import tempfile

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from oracle.assignment import assign_buckets
from oracle.average import average_bitfaithful
from oracle.protocol import replay

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

NGPU = torch.cuda.device_count()


class _Mlp(torch.nn.Module):
    """Registration order a, b, c; the forward uses them in the order c(b(a))."""

    def __init__(self):
        super().__init__()
        self.a = torch.nn.Linear(32, 64)
        self.b = torch.nn.Linear(64, 64)
        self.c = torch.nn.Linear(64, 8)

    def forward(self, x):
        return self.c(torch.tanh(self.b(torch.tanh(self.a(x)))))


class _Shuffled(torch.nn.Module):
    """Registered a, b, c but used a -> c -> b, so backward's hooks fire b, c, a:
    not the reverse registration order the default map assumes."""

    def __init__(self):
        super().__init__()
        self.a = torch.nn.Linear(32, 64)
        self.b = torch.nn.Linear(64, 8)
        self.c = torch.nn.Linear(64, 64)

    def forward(self, x):
        return self.b(torch.tanh(self.c(torch.tanh(self.a(x)))))


def test_world1_rebuild_from_traced_order():
    from paper_2006_15704_b200 import _lib as L
    from paper_2006_15704_b200.ddp import DistributedDataParallel
    torch.manual_seed(1)
    m = _Shuffled().cuda()
    ref = _Shuffled().cuda()
    ref.load_state_dict(m.state_dict())
    ddp = DistributedDataParallel(m, bucket_cap_mb=64 * 64 * 4 / 2 ** 20, rebuild_buckets=True)
    try:
        x = torch.randn(16, 32, device="cuda")
        ns = [p.numel() for p in ddp.params]
        for it in range(3):
            for p in list(m.parameters()) + list(ref.parameters()):
                p.grad = None
            ddp(x).pow(2).mean().backward()
            ref(x).pow(2).mean().backward()
            torch.cuda.synchronize()
            for pm, pr in zip(m.parameters(), ref.parameters()):
                assert torch.equal(pm.grad, pr.grad)            # world 1: identity (C-12)
            traced = L.ddp_ready_order(ddp.reducer.ctx)
            trace = L.ddp_launch_trace(ddp.reducer.ctx)
            if it == 0:
                first_order = traced
                # default map (reverse registration) vs the real hook order: O-2 replay
                assert trace == replay(assign_buckets(ns, 4, int(ddp.bucket_cap_mb * 2 ** 20)), traced)
            else:
                # rebuilt from the first pass's order: map = O-1 over that order, and
                # every bucket launches at the signal of its last slot (no deferral)
                a = assign_buckets(ns, 4, int(ddp.bucket_cap_mb * 2 ** 20), first_order)
                assert trace == replay(a, traced)
                if traced == first_order:
                    ends = list(itertools.accumulate(len(s) for s in a.buckets))
                    assert [t for _, t in trace] == [e - 1 for e in ends]
    finally:
        ddp.close()


def _worker(rank, world, init_file, q):
    torch.cuda.set_device(rank)
    import torch.distributed as dist
    dist.init_process_group("nccl", init_method=f"file://{init_file}", rank=rank, world_size=world,
                            device_id=torch.device("cuda", rank))
    try:
        from paper_2006_15704_b200.ddp import DistributedDataParallel
        torch.manual_seed(100 + rank)                  # different init on every rank
        m = _Mlp().cuda()
        ddp = DistributedDataParallel(m, bucket_cap_mb=0.01, rebuild_buckets=True)
        params = [p.detach().cpu().numpy().copy() for p in m.parameters()]
        torch.manual_seed(7 + rank)
        x = torch.randn(8, 32, device="cuda")
        outs = []
        for it in range(2):
            for p in m.parameters():
                p.grad = None
            loss = ddp(x).pow(2).mean()
            # local gradient of this rank (same params, autograd on a copy)
            local = _Mlp().cuda()
            local.load_state_dict(m.state_dict())
            local(x).pow(2).mean().backward()
            loss.backward()
            torch.cuda.synchronize()
            outs.append(([p.grad.cpu().numpy().copy() for p in m.parameters()],
                         [p.grad.cpu().numpy().copy() for p in local.parameters()]))
        ddp.close()
        q.put((rank, params, outs, None))
    except Exception as e:
        q.put((rank, None, None, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.multigpu
@pytest.mark.skipif(NGPU < 2, reason="needs >= 2 GPUs")
def test_world2_broadcast_and_rebuild():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    fd, init_file = tempfile.mkstemp(prefix="b200ddp_fe_")
    os.close(fd)
    os.unlink(init_file)
    ps = [ctx.Process(target=_worker, args=(r, world, init_file, q)) for r in range(world)]
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
    # Alg. 1: after construction every rank holds rank 0's parameters
    for a, b in zip(res[0][1], res[1][1]):
        assert np.array_equal(a, b)
    # every iteration (before and after the rebuild): .grad = O-3b average of the
    # ranks' local gradients, bit-exact (world 2: P2P / CE paths)
    for it in range(2):
        for k in range(len(res[0][2][it][0])):
            want = average_bitfaithful([res[r][2][it][1][k].ravel() for r in range(world)], "fp32")
            for r in range(world):
                assert np.array_equal(res[r][2][it][0][k].ravel(), want), (it, k, r)


class _Conv(torch.nn.Module):
    def __init__(self):
        super().__init__()
        self.c1 = torch.nn.Conv2d(3, 16, 3, padding=1)
        self.c2 = torch.nn.Conv2d(16, 8, 3, padding=1)

    def forward(self, x):
        return self.c2(torch.relu(self.c1(x)))


def test_world1_channels_last_gradients():
    """A channels_last model: its weight gradients are dense but not contiguous.
    The hook synchronizes them as flat arrays (the average is elementwise and
    every replica has the same layout): world 1 leaves them bit-for-bit equal to
    a plain local backward."""
    from paper_2006_15704_b200.ddp import DistributedDataParallel
    torch.manual_seed(0)
    m = _Conv().cuda().to(memory_format=torch.channels_last)
    ref = _Conv().cuda().to(memory_format=torch.channels_last)
    ref.load_state_dict(m.state_dict())
    ddp = DistributedDataParallel(m, bucket_cap_mb=0.001)
    try:
        x = torch.randn(4, 3, 16, 16, device="cuda").to(memory_format=torch.channels_last)
        ddp(x).square().mean().backward()
        ref(x).square().mean().backward()
        torch.cuda.synchronize()
        assert not m.c1.weight.grad.is_contiguous()          # really exercised the dense path
        for pm, pr in zip(m.parameters(), ref.parameters()):
            assert torch.equal(pm.grad, pr.grad)
    finally:
        ddp.close()
