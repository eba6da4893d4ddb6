"""World-size-2 multi-process tests on CPU (gloo): the host-side N>1 logic.

* every rank runs the native library's protocol (dry-run) on a DIFFERENT
  gradient ready order and the bucket launch sequences still agree
  ("all processes must use the same bucketing order");
* the NCCL unique id is created by rank 0 and reaches every rank through
  the torch process group (PAPER.md L278 rendezvous), as ddp.GradReducer
  does before ddp_bind_device.
"""

import os
import random
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2006_15704_b200 import _lib as L
        from paper_2006_15704_b200.ddp import _broadcast_id
        from synth.shapes import numels
        ns = numels("resnet50")
        ctx = L.ddp_create(ns, L.FP32, 5 << 20, world, rank)
        L.ddp_set_option(ctx, L.OPT_DRY_RUN, 1)
        rng = random.Random(100 + rank)          # rank-specific ready orders
        seqs = []
        for _ in range(5):
            order = list(range(len(ns)))
            rng.shuffle(order)
            for p in order:
                L.ddp_grad_ready(ctx, p, 0, 0)
            L.ddp_finalize_backward(ctx, 0)
            seqs.append([b for b, _ in L.ddp_launch_trace(ctx)])
        L.ddp_destroy(ctx)
        gathered = [None] * world
        dist.all_gather_object(gathered, seqs)
        nid = L.ddp_get_nccl_id() if rank == 0 else None
        got = _broadcast_id(nid, rank, None, torch.device("cpu"))
        ids = [None] * world
        dist.all_gather_object(ids, got)
        q.put((rank, gathered, ids, nid))
    finally:
        dist.destroy_process_group()


def test_two_ranks_agree_on_launch_order_and_nccl_id():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    gathered = res[0][1]
    nb = len(gathered[0][0])
    for r in range(world):
        for seq in gathered[r]:
            assert seq == list(range(nb))         # 0,1,2,... on every rank, every pass
    ids = res[0][2]
    assert ids[0] == ids[1] == res[0][3] and len(ids[0]) == 128
