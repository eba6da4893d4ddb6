"""In-kernel timeline of the fused pull kernels (DDP_OPT_P2P_DEBUG bit 2): per
CTA, %globaltimer at entry / packed / published / peers seen / reads done / end,
on one 25 MiB bucket, under torchrun (one process per GPU).  Prints, per rank,
the spread over CTAs of each phase (min / median / max, microseconds) for the
last of `reps` launches."""
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
    S = 25 * MIB
    n = S // 4
    g = torch.empty(n, device=dev)
    sdev.fill(g, 15704, rank, 0, 0, "normal", "fp32")
    flush = torch.zeros(256 * MIB // 8, dtype=torch.int64, device=dev)
    stream = torch.cuda.current_stream(dev)
    for algo in (L.ALGO_ONESHOT, L.ALGO_TWOSHOT):
        for sig in (0,):
            for dbg in (4, 7):
                red = GradReducer([n], "fp32", S, options={L.OPT_ALGO: algo, L.OPT_P2P_SIGNAL: sig,
                                                           L.OPT_P2P_DEBUG: dbg})
                for i in range(20):
                    flush.add_(1)
                    red.grad_ready(0, g, stream)
                    red.finalize(stream)
                torch.cuda.synchronize(dev)
                ctas = red.bucket_algos() and L.ddp_get_option(red.ctx, L.OPT_COMM_CTAS)
                tr = red._storage[40 * 1024:40 * 1024 + 256 * 64].view(torch.int64).view(256, 8).cpu()
                red.close()
                rows = [r for r in tr.tolist() if r[0] > 0][:148]
                t0 = min(r[0] for r in rows)
                out = {"algo": L.ALGO_NAMES[algo], "sig": sig, "debug": dbg, "rank": rank, "ctas": len(rows)}
                names = ["entry", "packed0", "published0", "seen0", "read0", "reads_done", "end"]
                for i, nm in enumerate(names):
                    v = sorted((r[i] - t0) / 1000 for r in rows if r[i] > 0)
                    if v:
                        out[nm] = [round(v[0], 1), round(v[len(v) // 2], 1), round(v[-1], 1)]
                out["t0_abs_us"] = t0 / 1000
                lines = [None] * world
                dist.all_gather_object(lines, out)
                if rank == 0:
                    for x in lines:
                        print(json.dumps(x), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
