"""GPU tests of find_unused_parameters (§8(f) N-1; PAPER.md L199-L201, L259,
L310) through the C ABI, against oracle O-7 (oracle/unused.py).

* world 1 (real binding): locally unused = globally unused -> the gradient
  buffer stays bit-for-bit intact; used params follow the identity (C-12);
  participation accumulated in a no_sync pass makes the param take part in
  the next synced pass;
* the front end's autograd-graph traversal (Alg. 1 forward) on a module whose
  forward skips a branch: skipped params keep .grad None;
* world 2 (one process per GPU): rank-specific unused sets vs O-7 — a param
  unused on every rank is untouched, a param used on one rank averages with a
  zero contribution, bit-exact (P2P / CE paths, rank-order fp32)."""

import os
import tempfile

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from oracle.unused import find_unused_sync
from synth.gen import gen_grad
from synth.shapes import numels

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

NGPU = torch.cuda.device_count()


def _np(t):
    return t.detach().cpu().numpy().copy()


def test_world1_unused_untouched_and_accumulated_participation():
    from paper_2006_15704_b200 import _lib as L
    from paper_2006_15704_b200.ddp import GradReducer
    from synth import device as sdev
    ns = numels("toy")
    red = GradReducer(ns, "fp32", 4096, options={L.OPT_FIND_UNUSED: 1})
    try:
        grads = [torch.empty(n, device="cuda") for n in ns]
        sdev.fill_all(grads, 15704, 0, 0, "normal", "fp32")
        before = [_np(g) for g in grads]
        sentinel = torch.full((ns[2],), 7.25, device="cuda")
        red.mark_unused(2, sentinel)          # unused everywhere (world 1)
        red.mark_unused(4, None)              # no buffer at all
        for p in (5, 3, 1, 0):
            red.grad_ready(p, grads[p])
        red.finalize()
        torch.cuda.synchronize()
        assert red.global_unused() == [False, False, True, False, True, False]
        assert torch.all(sentinel == 7.25)
        for p in (5, 3, 1, 0):
            assert np.array_equal(_np(grads[p]), before[p])
        # no_sync pass uses p2; the synced pass marks it unused with its accumulated grad
        with red.no_sync():
            for p in range(len(ns) - 1, -1, -1):
                red.grad_ready(p, grads[p])
            red.finalize()
        red.mark_unused(2, grads[2])
        for p in (5, 4, 3, 1, 0):
            red.grad_ready(p, grads[p])
        red.finalize()
        torch.cuda.synchronize()
        assert red.global_unused() == [False] * len(ns)
        for p in range(len(ns)):
            assert np.array_equal(_np(grads[p]), before[p])
        red.check_errors()
    finally:
        red.close()


class _Branchy(torch.nn.Module):
    def __init__(self):
        super().__init__()
        self.a = torch.nn.Linear(16, 8)
        self.b = torch.nn.Linear(16, 8)     # skipped when use_b is False
        self.c = torch.nn.Linear(8, 4)
        self.use_b = False

    def forward(self, x):
        h = self.a(x) + (self.b(x) if self.use_b else 0)
        return self.c(torch.relu(h))


def test_front_end_graph_traversal_world1():
    from paper_2006_15704_b200.ddp import DistributedDataParallel
    torch.manual_seed(0)
    m = _Branchy().cuda()
    ref = _Branchy().cuda()
    ref.load_state_dict(m.state_dict())
    ddp = DistributedDataParallel(m, bucket_cap_mb=0.0001, find_unused_parameters=True)
    try:
        x = torch.randn(5, 16, device="cuda")
        ddp(x).pow(2).sum().backward()
        ref(x).pow(2).sum().backward()
        torch.cuda.synchronize()
        assert m.b.weight.grad is None and m.b.bias.grad is None      # untouched
        for pm, pr in zip(m.parameters(), ref.parameters()):
            if pr.grad is not None:
                assert torch.equal(pm.grad, pr.grad)
        m.use_b = ref.use_b = True                                    # now b participates
        for p in list(m.parameters()) + list(ref.parameters()):
            p.grad = None
        ddp(x).sum().backward()
        ref(x).sum().backward()
        torch.cuda.synchronize()
        for pm, pr in zip(m.parameters(), ref.parameters()):
            assert torch.equal(pm.grad, pr.grad)
    finally:
        ddp.close()


# ---- world 2 -------------------------------------------------------------------------

UNUSED = {0: {1}, 1: {1, 3}}     # p1 unused everywhere; p3 used on rank 0 only


def _worker(rank, world, init_file, algo, q):
    torch.cuda.set_device(rank)
    import torch.distributed as dist
    dist.init_process_group("nccl", init_method=f"file://{init_file}", rank=rank, world_size=world,
                            device_id=torch.device("cuda", rank))
    try:
        from paper_2006_15704_b200 import _lib as L
        from paper_2006_15704_b200.ddp import GradReducer
        from synth import device as sdev
        ns = numels("toy")
        red = GradReducer(ns, "fp32", 4096, options={L.OPT_FIND_UNUSED: 1, L.OPT_ALGO: algo})
        grads = [torch.empty(n, device="cuda") for n in ns]
        sdev.fill_all(grads, 15704, rank, 0, "normal", "fp32")
        for p in range(len(ns) - 1, -1, -1):
            if p in UNUSED[rank]:
                red.mark_unused(p, grads[p])     # buffer holds stale values (must be replaced or kept)
            else:
                red.grad_ready(p, grads[p])
        red.finalize()
        torch.cuda.synchronize()
        gu = red.global_unused()
        red.check_errors()
        red.close()
        q.put((rank, [_np(g) for g in grads], gu, None))
    except Exception as e:
        q.put((rank, None, None, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.multigpu
@pytest.mark.skipif(NGPU < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("algo", [2, 3, 4, 6, 7, 1])   # one-shot, two-shot, CE, push, CE2, NCCL
def test_world2_unused_vs_oracle(algo):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    fd, init_file = tempfile.mkstemp(prefix="b200ddp_unused_")
    os.close(fd)
    os.unlink(init_file)
    ps = [ctx.Process(target=_worker, args=(r, world, init_file, algo, q)) for r in range(world)]
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
    ns = numels("toy")
    ins = [[gen_grad(15704, r, 0, p, n, "normal", "fp32") for p, n in enumerate(ns)] for r in range(world)]
    used = [[p not in UNUSED[r] for p in range(len(ns))] for r in range(world)]
    want = find_unused_sync(ins, used, ns, "fp32")
    for r in range(world):
        assert res[r][2] == [p == 1 for p in range(len(ns))]
        for p in range(len(ns)):
            if algo == 1:      # NCCL: tolerance (its own summation order); W=2 sums are exact anyway
                assert np.allclose(res[r][1][p], want[r][p], rtol=1e-6, atol=0), (r, p)
            else:
                assert np.array_equal(res[r][1][p], want[r][p]), (algo, r, p)
