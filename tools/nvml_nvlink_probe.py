"""Which NVML NVLink counters does this driver expose?  Prints the raw field
values (per link and aggregate) and the legacy utilization counters, before
and after a 256 MiB peer copy between GPU 0 and 1 (needs 2 GPUs)."""
import pynvml as N
import torch

N.nvmlInit()
h = N.nvmlDeviceGetHandleByIndex(0)


def fields(scope):
    out = {}
    for name in ("NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX", "NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX",
                 "NVML_FI_DEV_NVLINK_THROUGHPUT_RAW_TX", "NVML_FI_DEV_NVLINK_THROUGHPUT_RAW_RX"):
        try:
            v = N.nvmlDeviceGetFieldValues(h, [(getattr(N, name), scope)])[0]
            out[name[-7:]] = (v.nvmlReturn, v.valueType, int(v.value.ullVal))
        except Exception as e:  # noqa: BLE001
            out[name[-7:]] = repr(e)
    return out


def snap():
    s = {"all": fields(0xFFFFFFFF)}
    for l in range(18):
        s[l] = fields(l)
    return s


a = snap()
x = torch.ones(64 << 20, device="cuda:0")
y = torch.empty(64 << 20, device="cuda:1")
for _ in range(4):
    y.copy_(x)
torch.cuda.synchronize(0)
torch.cuda.synchronize(1)
b = snap()
print("after 4 x 256 MiB GPU0 -> GPU1")
for k in a:
    print(k, {n: (a[k][n], b[k][n]) for n in a[k]})
