"""Real multi-process, multi-GPU parity (one process per GPU, NCCL bootstrap,
torch symmetric memory for the peer-mapped storage).  Skipped with < 2 GPUs.

Each rank fills rank-specific synthetic gradients on its own GPU, runs synced
passes through ``ddp.GradReducer`` (the C ABI), and returns its outputs; the
parent compares them with the oracle: P2P paths bit-exact vs O-3b and
identical across ranks; NCCL path within the fp32/bf16 tolerances."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from oracle.assignment import MIB
from oracle.average import average_bitfaithful, average_fp64, to_fp32
from synth.gen import gen_grads
from synth.shapes import numels

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]

NGPU = torch.cuda.device_count() if torch.cuda.is_available() else 0
if NGPU < 2:
    pytest.skip("needs >= 2 GPUs", allow_module_level=True)


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cfgs, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    import torch.distributed as dist
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    from paper_2006_15704_b200 import _lib as L
    from paper_2006_15704_b200.ddp import GradReducer
    from synth import device as sdev
    from tests.gpu_util import TDT, to_np
    out = []
    try:
        for (model, dtype, cap, algo, iters) in cfgs:
            ns = numels(model)
            red = GradReducer(ns, dtype, cap, options={L.OPT_ALGO: algo})
            grads = [torch.empty(n, dtype=TDT[dtype], device="cuda") for n in ns]
            res = []
            for it in range(iters):
                sdev.fill_all(grads, 15704, rank, it, "normal", dtype)
                for p in range(len(ns) - 1, -1, -1):
                    red.grad_ready(p, grads[p])
                red.finalize()
                torch.cuda.synchronize()
                res.append([to_np(g, dtype) for g in grads])
            red.check_errors()
            red.close()
            out.append(res)
        q.put((rank, out, None))
    except Exception as e:  # report instead of hanging the parent
        q.put((rank, None, repr(e)))
    finally:
        dist.destroy_process_group()


def _run(world, cfgs):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, cfgs, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = sorted([q.get(timeout=600) for _ in range(world)], key=lambda x: x[0])
    for p in ps:
        p.join(timeout=120)
    for r, _, err in res:
        assert err is None, f"rank {r}: {err}"
    return [x[1] for x in res]


@pytest.mark.parametrize("world", sorted({2, min(4, NGPU)}))
def test_multigpu_parity(world):
    from paper_2006_15704_b200 import _lib as L
    cfgs = [("toy", "fp32", 4096, L.ALGO_ONESHOT, 2), ("toy", "bf16", 4096, L.ALGO_TWOSHOT, 2),
            ("toy", "fp32", 4096, L.ALGO_NCCL, 1), ("resnet50", "fp32", 25 * MIB, L.ALGO_AUTO, 2),
            ("resnet50", "bf16", 25 * MIB, L.ALGO_NCCL, 1)]
    outs = _run(world, cfgs)
    for ci, (model, dtype, cap, algo, iters) in enumerate(cfgs):
        ns = numels(model)
        for it in range(iters):
            ins = [gen_grads(ns, 15704, r, it, "normal", dtype) for r in range(world)]
            for p in range(len(ns)):
                got = [outs[r][ci][it][p] for r in range(world)]
                for r in range(1, world):                 # replica consistency
                    assert np.array_equal(got[r], got[0]), (model, p)
                xs = [ins[r][p] for r in range(world)]
                if algo == L.ALGO_NCCL:
                    ref, den = average_fp64(xs, dtype)
                    y = to_fp32(got[0], dtype).astype(np.float64)
                    r64 = to_fp32(ref, dtype).astype(np.float64)
                    if dtype == "fp32":
                        assert np.all(np.abs(y - r64) <= 1e-6 * den + 1e-45), (model, p)
                    else:
                        assert np.linalg.norm(y - r64) <= 1e-2 * np.linalg.norm(r64) + 1e-30, (model, p)
                else:
                    assert np.array_equal(got[0], average_bitfaithful(xs, dtype)), (model, dtype, algo, p)
