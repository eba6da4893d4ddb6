"""In-kernel timeline of one synthetic ResNet-50 step (all gradients ready at
once, the bench's step) at W ranks under torchrun: with DDP_OPT_P2P_DEBUG bit 2
every fused kernel records per-CTA %globaltimer points in its lane's flag
region; after the last step this prints, per lane, the span of its last kernel
(first CTA entry, median / last CTA end) relative to the earliest entry."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

MIB = 1 << 20


def main():
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    from paper_2006_15704_b200 import _lib as L
    from paper_2006_15704_b200.ddp import GradReducer
    from synth import device as sdev
    from synth.shapes import numels
    ns = numels(sys.argv[1] if len(sys.argv) > 1 else "resnet50")
    extra = json.loads(sys.argv[2]) if len(sys.argv) > 2 else {}
    red = GradReducer(ns, "fp32", 25 * MIB, options={L.OPT_P2P_DEBUG: 4, **{int(k): v for k, v in extra.items()}})
    grads = [torch.empty(n, device=dev) for n in ns]
    sdev.fill_all(grads, 15704, rank, 0, "normal", "fp32")
    order = list(range(len(ns) - 1, -1, -1))
    batch = L.ReadyBatch(order, [grads[p].data_ptr() for p in order])
    flush = torch.zeros(256 * MIB // 8, dtype=torch.int64, device=dev)
    stream = torch.cuda.current_stream(dev)
    for _ in range(10):
        flush.add_(1)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        red.grads_ready(batch, stream)
        red.finalize(stream)
        e.record(stream)
    torch.cuda.synchronize(dev)
    step_ms = s.elapsed_time(e)
    lanes = int(L.ddp_get_option(red.ctx, L.OPT_LANES))
    out = {"rank": rank, "step_ms": step_ms, "algos": red.bucket_algos(), "lanes": {}}
    t0 = None
    rows_all = {}
    for ln in range(lanes):
        base = ln * 64 * 1024 + 40 * 1024
        tr = red._storage[base:base + 256 * 64].view(torch.int64).view(256, 8).cpu().tolist()
        rows = [r for r in tr if r[0] > 0]
        if rows:
            rows_all[ln] = rows
            m = min(r[0] for r in rows)
            t0 = m if t0 is None else min(t0, m)
    for ln, rows in rows_all.items():
        ends = sorted(r[6] for r in rows if r[6] > 0)
        ent = sorted(r[0] for r in rows)
        out["lanes"][ln] = {"ctas": len(rows), "entry_us": round((ent[0] - t0) / 1e3, 1),
                            "entry_last_us": round((ent[-1] - t0) / 1e3, 1),
                            "end_med_us": round((ends[len(ends) // 2] - t0) / 1e3, 1) if ends else None,
                            "end_max_us": round((ends[-1] - t0) / 1e3, 1) if ends else None}
    red.close()
    lines = [None] * world
    dist.all_gather_object(lines, out)
    if rank == 0:
        for x in lines:
            print(json.dumps(x), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
