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
        # gradient-as-bucket-view: the copy engines write a peer's slot at THIS
        # rank's offsets, so every rank must derive the same slot layout
        vctx = L.ddp_create(ns, L.FP32, 5 << 20, world, rank)
        L.ddp_set_option(vctx, L.OPT_GRAD_VIEW, 1)
        layout = ([L.ddp_param_storage_offset(vctx, p) for p in range(len(ns))], L.ddp_storage_bytes(vctx),
                  [L.ddp_bucket_algo(vctx, b) for b in range(L.ddp_num_buckets(vctx))])
        L.ddp_destroy(vctx)
        layouts = [None] * world
        dist.all_gather_object(layouts, layout)
        nid = L.ddp_get_nccl_id() if rank == 0 else None
        got = _broadcast_id(nid, rank, None, torch.device("cpu"))
        ids = [None] * world
        dist.all_gather_object(ids, got)
        q.put((rank, gathered, ids, nid, layouts))
    finally:
        dist.destroy_process_group()


def test_two_ranks_agree_on_launch_order_nccl_id_and_view_layout():
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
    layouts = res[0][4]
    assert all(lay == layouts[0] for lay in layouts)          # identical slot layout on every rank
    offs, total, algos = layouts[0]
    from paper_2006_15704_b200 import _lib as L
    assert set(algos) == {L.ALGO_TWOSHOT}                    # world 2: the fused two-shot in place
    assert len(set(offs)) == len(offs) and max(offs) < total


def _worker_unused(rank, world, port, q):
    """Each rank: rank-specific unused sets (marked at 'forward end', Alg. 1
    L224-L225) and rank-specific hook orders, traced order-rebuilt maps (rank
    0's order broadcast through the process group, as the front end does)."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2006_15704_b200 import _lib as L
        from synth.shapes import numels
        ns = numels("resnet50")
        rng = random.Random(7 + rank)
        ctx = L.ddp_create(ns, L.FP32, 5 << 20, world, rank)
        L.ddp_set_option(ctx, L.OPT_DRY_RUN, 1)
        L.ddp_set_option(ctx, L.OPT_FIND_UNUSED, 1)
        seqs = []
        for _ in range(4):
            unused = set(rng.sample(range(len(ns)), 20))
            for p in sorted(unused):
                L.ddp_mark_unused(ctx, p, 0, 0)
            order = [p for p in range(len(ns)) if p not in unused]
            rng.shuffle(order)
            for p in order:
                L.ddp_grad_ready(ctx, p, 0, 0)
            L.ddp_finalize_backward(ctx, 0)
            seqs.append([b for b, _ in L.ddp_launch_trace(ctx)])
        traced = L.ddp_ready_order(ctx)
        L.ddp_destroy(ctx)
        t = torch.tensor(traced, dtype=torch.int32)
        dist.broadcast(t, src=0)                     # the agreed order (rank 0's)
        c2 = L.ddp_create_ordered(ns, t.tolist(), L.FP32, 5 << 20, world, rank)
        mapping = [(L.ddp_bucket_info(c2, b)[0],
                    [L.ddp_bucket_slot(c2, b, s) for s in range(L.ddp_bucket_info(c2, b)[1])])
                   for b in range(L.ddp_num_buckets(c2))]
        L.ddp_destroy(c2)
        gathered = [None] * world
        dist.all_gather_object(gathered, (seqs, mapping))
        q.put((rank, gathered))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_ranks_unused_and_rebuilt_map_agree(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_unused, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    gathered = res[0][1]
    nb = len(gathered[0][0][0])
    for seqs, _ in gathered:
        assert all(seq == list(range(nb)) for seq in seqs)   # same launch sequence on every rank
    assert all(m == gathered[0][1] for _, m in gathered)      # same rebuilt map on every rank
