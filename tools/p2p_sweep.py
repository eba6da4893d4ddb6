"""Measurement sweep of the fused P2P kernels on one 25 MiB bucket (run under
torchrun, one process per GPU):

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \
        --master-port 29513 tools/p2p_sweep.py [--mib 25] [--dtype fp32]

For each option set: whole sync (producer-stream events around grad_ready ->
finalize, L2 flushed between reps, median of 50) and the fused kernel alone
(profile events), max over ranks, as busBW = (S/t) 2(W-1)/W.  Rank 0 prints one
JSON line per option set."""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

MIB = 1 << 20


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mib", type=float, default=25)
    ap.add_argument("--dtype", default="fp32")
    ap.add_argument("--reps", type=int, default=50)
    ap.add_argument("--sets", default="default")
    a = ap.parse_args()
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    from paper_2006_15704_b200 import _lib as L
    from paper_2006_15704_b200.ddp import GradReducer
    from synth import device as sdev

    esize = 4 if a.dtype == "fp32" else 2
    tdt = torch.float32 if a.dtype == "fp32" else torch.bfloat16
    S = int(a.mib * MIB) // 256 * 256
    n = S // esize
    g = torch.empty(n, dtype=tdt, device=dev)
    sdev.fill(g, 15704, rank, 0, 0, "normal", a.dtype)
    flush = torch.zeros(256 * MIB // 8, dtype=torch.int64, device=dev)
    stream = torch.cuda.current_stream(dev)
    O, A = L, L
    sets = {
        "default": [
            ("oneshot push", {O.OPT_ALGO: A.ALGO_ONESHOT, O.OPT_P2P_PULL: 0}),
            ("twoshot push", {O.OPT_ALGO: A.ALGO_TWOSHOT, O.OPT_P2P_PULL: 0}),
        ] + [(f"{alg} pull sig{m} stage{st}", {O.OPT_ALGO: getattr(A, "ALGO_" + alg.upper()), O.OPT_P2P_SIGNAL: m,
                                               O.OPT_P2P_STAGE_BYTES: st << 10})
             for alg in ("oneshot", "twoshot") for m in (0, 1, 3) for st in (16, 32, 64, 1 << 20)]
        + [(f"{alg} pull debug{d}", {O.OPT_ALGO: getattr(A, "ALGO_" + alg.upper()), O.OPT_P2P_DEBUG: d})
           for alg in ("oneshot", "twoshot") for d in (1, 2, 3)]
        + [("ce", {O.OPT_ALGO: A.ALGO_CE}), ("ce2", {O.OPT_ALGO: A.ALGO_CE2}), ("nccl", {O.OPT_ALGO: A.ALGO_NCCL})],
        "quick": [(f"{alg} pull", {O.OPT_ALGO: getattr(A, "ALGO_" + alg.upper())}) for alg in ("oneshot", "twoshot")]
        + [("ce", {O.OPT_ALGO: A.ALGO_CE}), ("ce2", {O.OPT_ALGO: A.ALGO_CE2}), ("nccl", {O.OPT_ALGO: A.ALGO_NCCL})],
    }[a.sets]

    def tmax(x):
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for name, opts in sets:
        red = GradReducer([n], a.dtype, S, options=opts)

        def one():
            red.grad_ready(0, g, stream)
            red.finalize(stream)
        for _ in range(10):
            one()
        L.ddp_set_option(red.ctx, L.OPT_PROFILE, 1)
        L.ddp_profile_timeline(red.ctx)
        dist.barrier(device_ids=[local])
        torch.cuda.synchronize(dev)
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.reps)]
        for i in range(a.reps):
            flush.add_(1)
            evs[i][0].record(stream)
            one()
            evs[i][1].record(stream)
        torch.cuda.synchronize(dev)
        tl = L.ddp_profile_timeline(red.ctx, cap=64 * a.reps)
        whole = tmax(statistics.median(s.elapsed_time(e) for s, e in evs))
        ks = [e_ - s_ for k, _, s_, e_ in tl if k == "p2p_fused"]
        kern = tmax(statistics.median(ks)) if ks else 0.0
        red.check_errors()
        red.close()
        bw = (lambda t: S / (t * 1e-3) * 2 * (world - 1) / world / 1e9 if t else None)
        if rank == 0:
            print(json.dumps({"set": name, "W": world, "bytes": S, "whole_ms": whole, "whole_busbw": bw(whole),
                              "kernel_ms": kern, "kernel_busbw": bw(kern)}), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
