"""torch.distributed (NCCL) all_reduce bus bandwidth reference, torchrun N ranks."""
import os, torch, torch.distributed as dist
r, w = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(r)
dist.init_process_group("nccl", device_id=torch.device("cuda", r))
for mib in (1, 8, 25, 64, 256, 1024):
    x = torch.ones(mib * (1 << 20) // 4, device="cuda")
    for _ in range(5):
        dist.all_reduce(x)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    n = 20
    for _ in range(n):
        dist.all_reduce(x)
    b.record()
    torch.cuda.synchronize()
    t = a.elapsed_time(b) / n
    if r == 0:
        print(f"nccl all_reduce {mib} MiB: {t*1e3:.1f} us busbw {mib*(1<<20)/(t*1e-3)*2*(w-1)/w/1e9:.1f} GB/s", flush=True)
dist.destroy_process_group()
