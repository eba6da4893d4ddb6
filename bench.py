#!/usr/bin/env python
"""Benchmark of the DDP Reducer gradient-sync hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload resnet50|bert_large] [--dtype fp32|bf16] [--cap-mib 25]

Metric (BASELINE.json): "exposed grad-sync ms/iter and bucket allreduce bus
GB/s at 1/2/4/8 B200".  One step = one pass of the whole hot path (§8(a)
rows a1-a7) over one batch of synthetic gradients already resident in HBM:
all gradients of the workload become ready in reverse registration order (one
batched ddp_grads_ready call: the hooks of a backward whose compute takes no
time), buckets are launched in order (pack x 1/W -> allreduce -> unpack), and
ddp_finalize_backward closes the pass.  With no backward compute to hide
behind, the whole sync is exposed: `value` = device ms per step (CUDA events
on the producer stream, max over ranks), lower is better.  `busbw` reports the
bucket allreduce bus bandwidth of a 25 MiB bucket (N > 1).  L2 (126 MB) is
flushed between timed steps (256 MiB written then read) outside the per-step events.

For N > 1 launch with torchrun (one process per GPU); rank 0 prints ONE JSON
line.  `--impl reference` times the oracle (oracle/, numpy on host cores) on
a bounded sample of the same workload (the reference arm of this tier).
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "exposed grad-sync ms/iter and bucket allreduce bus GB/s at 1/2/4/8 B200"
MIB = 1 << 20


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="resnet50", choices=["resnet50", "bert_large"])
    ap.add_argument("--dtype", default="fp32", choices=["fp32", "bf16"])
    ap.add_argument("--cap-mib", type=float, default=25)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--algo", type=int, default=0, help="force DDP_OPT_ALGO (0 auto)")
    ap.add_argument("--comm-ctas", type=int, default=0)
    ap.add_argument("--pack-ctas", type=int, default=0)
    ap.add_argument("--stage-kib", type=int, default=0)
    ap.add_argument("--ce-streams", type=int, default=0)
    ap.add_argument("--throughput-policy", action="store_true",
                    help="exposed-time runs: DDP without the overlap policy (PREFER_OVERLAP=0)")
    ap.add_argument("--overlap-policy", type=int, default=-1,
                    help="force PREFER_OVERLAP (1 copy engines, 2 SM kernels) for the DDP / exposed runs")
    ap.add_argument("--high-priority", action="store_true",
                    help="communication streams at the highest priority (default: lowest)")
    ap.add_argument("--lanes", type=int, default=0, help="P2P/NVLS kernel lanes (streams)")
    ap.add_argument("--p2p-push", action="store_true", help="push kernels for every fused bucket (DDP_OPT_P2P_PULL=0)")
    ap.add_argument("--p2p-pull-all", action="store_true", help="pull kernels for every fused bucket (DDP_OPT_P2P_PULL=2)")
    ap.add_argument("--last-on-lane", action="store_true", help="DDP_OPT_LAST_ON_PRODUCER=0")
    ap.add_argument("--wire-bf16", action="store_true", help="N-3: fp32 gradients travel as bf16 (CE exchange)")
    ap.add_argument("--grad-view", action="store_true",
                    help="N-3 zero-copy: gradients live in their bucket slots (in-place NCCL, no pack/unpack)")
    ap.add_argument("--ce-direct-mib", type=float, default=-1, help="CE: copy gradients >= this straight from .grad")
    ap.add_argument("--nccl-comms", type=int, default=0, help="round-robin NCCL communicators (P:L535)")
    ap.add_argument("--exposed-model", default="resnet50", choices=["none", "resnet50", "bert_large"],
                    help="real-model backward for the exposed-time measurement")
    ap.add_argument("--exposed-batch", type=int, default=0)
    ap.add_argument("--exposed-iters", type=int, default=50)
    ap.add_argument("--timeline-detail", action="store_true", help="include per-launch timeline in the JSON")
    ap.add_argument("--oneshot-max", type=int, default=-1)
    ap.add_argument("--twoshot-max", type=int, default=-1)
    ap.add_argument("--mode", default="step", choices=["step", "cap-sweep", "nosync", "allreduce-sweep"],
                    help="step: the contract line (default).  cap-sweep: BASELINE config 4 (exposed time vs "
                         "bucket cap, real model).  nosync: config 5 (sync every 1/2/4/8).  allreduce-sweep: "
                         "M-3 per-size busBW per algorithm + the paper's fixed-total split (Fig. 2 method)")
    ap.add_argument("--exposed-seq", type=int, default=0, help="BERT sequence length (default 512)")
    ap.add_argument("--caps", default="0,1,5,10,25,50,100,200", help="cap-sweep caps in MiB")
    return ap.parse_args()


def env_rank():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def workload_name(a):
    return f"{a.workload}_grads_{a.dtype}_cap{a.cap_mib:g}MiB"


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d.get("hbm_gbs", 6541.5), "measured"
    return 6650.0, "fallback"


def ncu_traffic(workload, world, kind):
    """DRAM bytes per launch of the dominant kernel from a committed ncu --set full
    capture (profiles/traffic.json), or (None, None) when none matches."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(p) as f:
            e = json.load(f).get(f"{workload}|W{world}|{kind}")
    except (OSError, ValueError):
        e = None
    return (e["bytes"], e["source"]) if e else (None, None)


class ClockSampler:
    """SM clocks + throttle reasons sampled DURING the timed region: NVML polled
    every ~2 ms from a thread (nvidia-smi as a fallback when NVML is missing)."""

    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index: int):
        self.index, self.samples, self._stop = index, [], threading.Event()
        self.t = threading.Thread(target=self._run, daemon=True)
        self.src = "nvml"

    def _run(self):
        try:
            import pynvml as N
            N.nvmlInit()
            h = N.nvmlDeviceGetHandleByIndex(self.index)
            bits = [N.nvmlClocksEventReasonHwSlowdown, N.nvmlClocksEventReasonHwThermalSlowdown,
                    N.nvmlClocksEventReasonSwThermalSlowdown, N.nvmlClocksEventReasonSwPowerCap]
            mx = N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)
            while not self._stop.is_set():
                sm = N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)
                rs = N.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.samples.append([sm, mx] + [bool(rs & b) for b in bits])
                self._stop.wait(0.002)
            return
        except Exception:
            self.src = "nvidia-smi"
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                x = [v.strip() for v in out.split(",")]
                self.samples.append([float(x[0]), float(x[1])] + [v == "Active" for v in x[2:6]])
            except Exception:
                pass
            self._stop.wait(0.05)

    def __enter__(self):
        self.t.start()
        time.sleep(0.01)
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self.t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        import statistics
        reasons = sorted({self.NAMES[i] for s in self.samples for i in range(4) if s[2 + i]})
        return {"sm_mhz": statistics.median(s[0] for s in self.samples),
                "sm_max_mhz": max(s[1] for s in self.samples), "reasons": reasons,
                "samples": len(self.samples), "source": self.src}


# ---------------------------------------------------------------------------------
def run_reference(a):
    """Reference arm: the oracle as it stands, on host cores, rank 0 only."""
    rank, world, _ = env_rank()
    if rank != 0:
        return
    from oracle.cpu_baseline import time_sync
    from synth.gen import gen_grads
    from synth.shapes import numels
    ns = numels(a.workload)
    W = max(1, world)
    r = time_sync(ns, a.dtype, int(a.cap_mib * MIB), W, seed=15704, gen_grads=gen_grads,
                  max_iters=a.steps, budget_s=120.0, warmup=a.warmup)
    ms = r["sec_per_iter"] * 1e3
    line = {
        "impl": "reference", "metric": METRIC, "value": ms, "unit": "ms/iter", "n_gpus": W,
        "steps": r["iters"], "warmup": r["warmup"], "ms_per_step": ms, "higher_is_better": False, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32" if a.dtype == "fp32" else "bf16", "data": "synthetic",
        "config": {"workload": workload_name(a), "params": r["params"], "world_simulated": W},
        "cpu_baseline": {"value": ms, "unit": "ms/iter", "cores": r["cores"], "kind": "oracle",
                         "sample": f"{r['warmup']} untimed + {r['iters']} timed full iterations (median; at most "
                                   f"--steps, within a 120 s budget) of oracle.average.simulate_ddp_sync "
                                   f"(pack x1/W, rank-order fp32 allreduce, unpack) over {W} in-memory replicas"},
        "e2e": {"value": ms, "unit": "ms/iter", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------------
def run_ours(a):
    import torch
    import torch.distributed as dist

    rank, world, local = env_rank()
    if world != a.gpus:
        raise SystemExit(f"--gpus {a.gpus} but WORLD_SIZE={world}; launch N>1 with torchrun")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)

    from paper_2006_15704_b200 import _lib as L
    from paper_2006_15704_b200.ddp import GradReducer
    from synth import device as sdev
    from synth.shapes import numels

    ns = numels(a.workload)
    esize = 4 if a.dtype == "fp32" else 2
    tdt = torch.float32 if a.dtype == "fp32" else torch.bfloat16
    cap = int(a.cap_mib * MIB)
    opts = {}
    if a.algo:
        opts[L.OPT_ALGO] = a.algo
    if a.comm_ctas:
        opts[L.OPT_COMM_CTAS] = a.comm_ctas
    if a.pack_ctas:
        opts[L.OPT_PACK_CTAS] = a.pack_ctas
    if a.stage_kib:
        opts[L.OPT_P2P_STAGE_BYTES] = a.stage_kib * 1024
    if a.ce_streams:
        opts[L.OPT_CE_STREAMS] = a.ce_streams
    if a.throughput_policy:
        opts[L.OPT_PREFER_OVERLAP] = 0
    if a.overlap_policy >= 0:
        opts[L.OPT_PREFER_OVERLAP] = a.overlap_policy
    if a.high_priority:
        opts[L.OPT_LOW_PRIORITY] = 0
    if a.lanes:
        opts[L.OPT_LANES] = a.lanes
    if a.p2p_push:
        opts[L.OPT_P2P_PULL] = 0
    if a.p2p_pull_all:
        opts[L.OPT_P2P_PULL] = 2
    if a.last_on_lane:
        opts[L.OPT_LAST_ON_PRODUCER] = 0
    if a.wire_bf16:
        opts[L.OPT_WIRE_BF16] = 1
    if a.grad_view:
        opts[L.OPT_GRAD_VIEW] = 1
    if a.ce_direct_mib >= 0:
        opts[L.OPT_CE_DIRECT_BYTES] = int(a.ce_direct_mib * MIB)
    if a.nccl_comms:
        opts[L.OPT_NCCL_COMMS] = a.nccl_comms
    if a.oneshot_max >= 0:
        opts[L.OPT_P2P_ONESHOT_MAX] = a.oneshot_max
    if a.twoshot_max >= 0:
        opts[L.OPT_P2P_TWOSHOT_MAX] = a.twoshot_max
    red = GradReducer(ns, a.dtype, cap, options=opts)

    # gradients: views into one flat buffer (256-B aligned params), synthetic, rank-specific
    offs, pos = [], 0
    for n in ns:
        offs.append(pos)
        pos += (n * esize + 255) // 256 * 256 // esize
    flat = torch.empty(pos, dtype=tdt, device=dev)
    grads = [flat[o:o + n] for o, n in zip(offs, ns)]
    if a.grad_view:  # each gradient IS its bucket slot (ddp_param_storage_offset)
        grads = [red._storage[o:o + n * esize].view(tdt)
                 for o, n in ((L.ddp_param_storage_offset(red.ctx, p), n) for p, n in enumerate(ns))]
    sdev.fill_all(grads, 15704, rank, 0, "normal", a.dtype)
    order = list(range(len(ns) - 1, -1, -1))
    batch = L.ReadyBatch(order, [grads[p].data_ptr() for p in order])
    flush = torch.zeros(256 * MIB // 8, dtype=torch.int64, device=dev)

    def flush_l2():
        # write then read 256 MiB (> 126 MB L2): evicts the step's data and leaves
        # clean lines, so no dirty write-back is charged to the next step
        flush.add_(1)
        flush.sum()
    stream = torch.cuda.current_stream(dev)

    def step():
        red.grads_ready(batch, stream)
        red.finalize(stream)

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local])
        torch.cuda.synchronize(dev)

    def timed(fn, k, pre=None):
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(k)]
        for i in range(k):
            flush_l2()
            if pre:
                pre()
            evs[i][0].record(stream)
            fn()
            evs[i][1].record(stream)
        torch.cuda.synchronize(dev)
        return [s.elapsed_time(e) for s, e in evs]

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- main timed region -------------------------------------------------------
    for _ in range(a.warmup):
        step()
    barrier()
    with ClockSampler(local) as clk:
        barrier()
        times = timed(step, a.steps)
        barrier()
    ms = max_over_ranks(sum(times) / len(times))
    # host cost of issuing one step (ready signals + finalize), no device sync inside:
    # if it approaches the device time the step is host-bound
    torch.cuda.synchronize(dev)
    hs = []
    for _ in range(5):
        t0 = time.perf_counter()
        step()
        hs.append((time.perf_counter() - t0) * 1e3)
        torch.cuda.synchronize(dev)
    host_ms = max_over_ranks(sorted(hs)[len(hs) // 2])

    # ---- per-kernel device time (profile events on the comm stream) -----------------
    L.ddp_set_option(red.ctx, L.OPT_PROFILE, 1)
    L.ddp_profile_timeline(red.ctx)
    kprof_steps = min(10, a.steps)
    timed(step, kprof_steps)
    tl = L.ddp_profile_timeline(red.ctx, cap=1 << 20)
    L.ddp_set_option(red.ctx, L.OPT_PROFILE, 0)
    # per kind: (summed launch ms, launches, union ms of the launch intervals) — with
    # lanes several launches of one kind run at once; the union is the time the kind
    # was active, the honest denominator for "bytes per launch / launch duration"
    prof = {}
    for k in L.PROFILE_KINDS:
        iv = sorted((s_, e_) for kk, _, s_, e_ in tl if kk == k)
        union, cur_s, cur_e = 0.0, None, None
        for s_, e_ in iv:
            if cur_e is None or s_ > cur_e:
                if cur_e is not None:
                    union += cur_e - cur_s
                cur_s, cur_e = s_, e_
            else:
                cur_e = max(cur_e, e_)
        if cur_e is not None:
            union += cur_e - cur_s
        prof[k] = (sum(e_ - s_ for s_, e_ in iv), len(iv), union)
    algos = red.bucket_algos()
    bnumel = red.bucket_numels()
    S_tot = sum(bnumel) * esize
    # our kernel launches per step (NCCL's own kernels excluded)
    launches_per_step = sum(prof[k][1] for k in ("pack", "unpack", "p2p_fused", "ce_reduce")) / kprof_steps
    if "push" in red.bucket_algos():   # the push kernels are ours too (copy-engine transfers are not kernels)
        launches_per_step += prof["ce_copy"][1] / kprof_steps

    # dominant kernel roofline: algorithmic bytes per launch / measured launch time
    peak_hbm, peak_src = measured_peaks()
    kinds = {k: v for k, v in prof.items() if v[1] > 0}
    # the dominant KERNEL of ours (copy-engine transfers and NCCL's kernels are reported
    # in roofline.all_kinds but are not our kernels; the push transfer is)
    ours = [k for k in kinds if k in ("pack", "unpack", "p2p_fused", "ce_reduce")
            or (k == "ce_copy" and "push" in algos)]
    dom = max(ours or list(kinds), key=lambda k: kinds[k][2]) if kinds else None
    small = 0   # CE buckets: bytes of the gradients gathered by the pack kernel (< CE_DIRECT_BYTES each)
    for b, x in enumerate(algos):
        if x == "ce":
            for s_ in range(L.ddp_bucket_info(red.ctx, b)[1]):
                p, _ = L.ddp_bucket_slot(red.ctx, b, s_)
                small += ns[p] * esize if ns[p] * esize < L.ddp_get_option(red.ctx, L.OPT_CE_DIRECT_BYTES) else 0
    by = {x: sum(n * esize for n, y in zip(bnumel, algos) if y == x) for x in ("nccl", "oneshot", "twoshot", "ce", "nvls", "push", "ce2")}

    def kind_bytes(kind):
        """(algorithmic bytes per step, bound, rule) of one profile kind."""
        if kind == "p2p_fused" and world == 1:
            return 3 * (by["oneshot"] + by["twoshot"]), "hbm", "3 x bucket bytes (read g, write bucket, write g)"
        if kind == "pack":
            if a.wire_bf16:
                return 1.5 * by["ce"], "hbm", "fp32 read + bf16 write of every gradient (compressed wire)"
            return (2 * (by["nccl"] + small + by["ce2"]), "hbm",
                    "2 x bytes packed (NCCL and CE2 buckets; CE small gradients)")
        if kind == "unpack":
            return 2 * (by["nccl"] + by["ce2"]), "hbm", "2 x bucket bytes"
        if kind == "p2p_fused":
            return (by["oneshot"] * (world - 1) + by["twoshot"] * 2 * (world - 1) / world
                    + by["nvls"] * (1 + 1 / world), "nvlink",
                    "NVLink bytes per direction: one-shot (W-1)S, two-shot 2(W-1)/W S, NVLS (1+1/W)S")
        if kind == "ce_copy":
            wf = 0.5 if a.wire_bf16 else 1.0   # the compressed wire carries bf16
            return ((by["ce"] * wf + by["push"]) * (world - 1) + by["ce2"] * 2 * (world - 1) / world, "nvlink",
                    "NVLink bytes per direction: CE/PUSH (W-1)S_wire, CE2 2(W-1)/W S (copy engines / push kernel)")
        if kind == "ce_reduce":
            if a.wire_bf16:
                return (by["ce"] * (2 + (world - 1) / 2), "hbm",
                        "own fp32 read + (W-1) bf16 slots + fp32 .grad write")
            return ((by["ce"] + by["push"]) * (world + 1) + by["ce2"] * (world + 1) / world, "hbm",
                    "(W+1) x bucket bytes (W operands read, .grad written); CE2 (W+1)/W S (one shard)")
        return 2 * (world - 1) / world * by["nccl"], "nvlink", "ring 2(W-1)/W x bucket bytes"

    def roof_of(kind):
        tot_ms, cnt, union_ms = kinds[kind]
        avg_ms = union_ms / cnt   # = summed duration / cnt when launches do not overlap
        step_bytes, bound, per = kind_bytes(kind)
        byts = step_bytes / (cnt / kprof_steps)
        peak = peak_hbm if bound == "hbm" else 770.0
        r_ = {"bound": bound, "achieved": byts / (avg_ms * 1e-3) / 1e9, "peak": peak, "unit": "GB/s"}
        r_["frac"] = r_["achieved"] / peak
        r_["traffic"], r_["traffic_source"] = ncu_traffic(workload_name(a), world, kind)
        r_.update(kernel=kind, algorithmic_bytes_per_launch=byts, bytes_rule=per, avg_launch_ms=avg_ms,
                  launch_duration=("union of the launch intervals / launches (lanes overlap launches)"
                                   if union_ms < tot_ms * 0.999 else "CUDA events around each launch"),
                  peak_source=(f"MEASURED_PEAKS.json hbm_gbs ({peak_src})" if bound == "hbm"
                               else "B200_PROFILING.md measured peer copy 770 GB/s per direction"))
        return r_
    roof = None
    if dom is not None:
        roof = roof_of(dom)
        roof["all_kinds"] = {k: {"achieved": round(x["achieved"], 1), "frac": round(x["frac"], 3),
                                 "bound": x["bound"], "active_ms_per_step": kinds[k][2] / kprof_steps}
                             for k in kinds for x in [roof_of(k)]}

    # ---- bucket allreduce bus bandwidth on a 25 MiB bucket (N > 1), every algorithm ----
    busbw = None
    if world > 1:
        busbw = busbw_suite(a, world, local, dev, opts, stream, flush_l2, barrier, max_over_ranks)

    # ---- e2e through the public API with host buffers --------------------------------
    # Every step: its gradients copied in from pinned host memory, the whole sync
    # (grads_ready -> finalize), its averaged gradients copied back out.  Pipelined
    # like a training loop that prefetches: two gradient buffers, the copy-in of step
    # k+1 (own stream) and the copy-out of step k (own stream) overlap the sync; a
    # buffer is refilled only after its copy-out finished.  `serial_ms`: the same
    # three stages back to back on one stream.
    e2e = None
    if not a.no_e2e:
        host = torch.empty(flat.numel(), dtype=tdt, pin_memory=True)
        host.copy_(flat)
        outs_h = [torch.empty_like(host, pin_memory=True) for _ in range(2)]

        def e2e_step():
            flat.copy_(host, non_blocking=True)
            step()
            outs_h[0].copy_(flat, non_blocking=True)
        for _ in range(2):
            e2e_step()
        barrier()
        et = timed(e2e_step, max(3, min(a.steps, 20)))
        serial = max_over_ranks(sum(et) / len(et))
        e2e = {"value": serial, "unit": "ms/iter",
               "h2d_bytes_per_step": flat.numel() * esize, "d2h_bytes_per_step": flat.numel() * esize,
               "serial_ms": serial, "pipelined": False}
        if not a.grad_view:   # (with the view, the gradients are the library's slots, not `flat`)
            flat2 = torch.empty_like(flat)
            g2 = [flat2[o:o + n] for o, n in zip(offs, ns)]
            bufs = [(flat, batch), (flat2, L.ReadyBatch(order, [g2[p].data_ptr() for p in order]))]
            s_in, s_out = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
            ev = {k: [torch.cuda.Event() for _ in range(2)] for k in ("in", "done", "free")}

            def pipelined(K):
                t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                t0.record(stream)
                s_in.wait_event(t0)
                s_out.wait_event(t0)
                for k in range(K):
                    b = k % 2
                    f, bt = bufs[b]
                    if k >= 2:
                        s_in.wait_event(ev["free"][b])
                    with torch.cuda.stream(s_in):
                        f.copy_(host, non_blocking=True)
                    ev["in"][b].record(s_in)
                    stream.wait_event(ev["in"][b])
                    red.grads_ready(bt, stream)
                    red.finalize(stream)
                    ev["done"][b].record(stream)
                    s_out.wait_event(ev["done"][b])
                    with torch.cuda.stream(s_out):
                        outs_h[b].copy_(f, non_blocking=True)
                    ev["free"][b].record(s_out)
                for b in range(min(2, K)):
                    stream.wait_event(ev["free"][b])
                t1.record(stream)
                torch.cuda.synchronize(dev)
                return t0.elapsed_time(t1) / K
            pipelined(4)
            barrier()
            pm = max_over_ranks(pipelined(max(8, min(a.steps, 40))))
            e2e.update(value=pm, pipelined=True)
    # ---- host overhead of the per-gradient hook call ----------------------------------
    t0 = time.perf_counter()
    for p in order:
        red.grad_ready(p, grads[p], stream)
    t1 = time.perf_counter()
    red.finalize(stream)
    torch.cuda.synchronize(dev)
    host_us = (t1 - t0) / len(order) * 1e6

    red.check_errors()
    red.close()
    exposed = None
    if a.exposed_model != "none":
        exposed = measure_exposed(a, rank, world, local, dev, opts)
    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        from oracle.cpu_baseline import cpu_model, time_sync, time_sync_threads
        from synth.gen import gen_grads
        r = time_sync(ns, a.dtype, cap, 1, seed=15704, gen_grads=gen_grads, max_iters=3, budget_s=30)
        rt = time_sync_threads(ns, a.dtype, cap, 1, seed=15704, gen_grads=gen_grads, max_iters=3, budget_s=30)
        cpu = {"value": r["sec_per_iter"] * 1e3, "unit": "ms/iter", "cores": r["cores"], "kind": "oracle",
               "sample": f"{r['iters']} full iterations of oracle simulate_ddp_sync on the same workload (W=1)",
               "all_core": {"value": rt["sec_per_iter"] * 1e3, "unit": "ms/iter", "cores": rt["threads"],
                            "sample": f"{rt['iters']} full iterations, {rt['threads']} threads each owning an "
                                      "element range of every gradient (oracle.cpu_baseline.time_sync_threads)"},
               "assign_ms": r["assign_s"] * 1e3, "cpu_model": cpu_model(), "os_cpu_count": os.cpu_count()}

    if rank == 0:
        line = {
            "metric": METRIC, "value": ms, "unit": "ms/iter", "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": False, "scaling": "weak",
            "vs_baseline": None, "dtype": ("f32 (bf16 wire)" if a.wire_bf16 else "f32") if a.dtype == "fp32" else "bf16",
            "data": "synthetic (seeded splitmix64 gradients shaped like the workload; no model compute)",
            "config": {"workload": workload_name(a), "params": sum(ns), "tensors": len(ns),
                       "buckets": len(bnumel), "bucket_algos": algos, "bucket_cap_mib": a.cap_mib,
                       "grad_bytes_per_step": S_tot, "l2": "flushed between steps (256 MiB write + read, outside the per-step events)",
                       "ready_order": "reverse registration, one batched ddp_grads_ready per step",
                       "parallelism": f"dp{world}"},
            "busbw": busbw,
            "exposed": exposed,
            "roofline": roof,
            "kernel_ms_per_step": {k: v[0] / kprof_steps for k, v in prof.items() if v[1]},
            "kernel_active_ms_per_step": {k: v[2] / kprof_steps for k, v in prof.items() if v[1]},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(round(launches_per_step * a.steps)),
            "host_us_per_grad_ready": host_us,
            "host_ms_to_issue_step": host_ms,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


class NvlinkCounter:
    """Cumulative NVLink data bytes (TX, RX) of one GPU, summed over its links
    (NVML field values NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX / _RX, KiB; payload
    only, no protocol overhead).  read() -> (tx_bytes, rx_bytes) or None."""

    def __init__(self, index: int):
        self.h = None
        try:
            import pynvml as N
            N.nvmlInit()
            self.N, self.h = N, N.nvmlDeviceGetHandleByIndex(index)
            self.fields = [(N.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX, 0xFFFFFFFF),
                           (N.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX, 0xFFFFFFFF)]
            if self.read() is None:
                self.h = None
        except Exception:
            self.h = None

    def read(self):
        if self.h is None:
            return None
        try:
            v = self.N.nvmlDeviceGetFieldValues(self.h, self.fields)
        except Exception:
            return None
        if any(x.nvmlReturn != 0 for x in v):
            return None
        return tuple(int(x.value.ullVal) * 1024 for x in v)


def busbw_suite(a, world, local, dev, opts, stream, flush_l2, barrier, max_over_ranks, reps=100):
    """SURVEY §8(d) M-2 bucket busBW, per algorithm, on one 25 MiB bucket:
    t = the WHOLE sync as the caller sees it — a CUDA event on the producer stream
    before ddp_grad_ready and one after ddp_finalize_backward (which makes that
    stream wait for every library stream) — median over `reps` reps, L2 flushed
    between reps outside the events, max over ranks; busBW = (S/t) 2(W-1)/W.
    'default' is the library's choice for this bucket as the LAST bucket of a pass
    (fused kernels on all 148 SMs); 'nonlast' times the same bucket as bucket 0 of a
    two-bucket pass (COMM_CTAS CTAs per lane) from the profile events around its
    fused kernel.  'grad_view' runs the allreduce alone (gradient-as-bucket-view:
    no pack / unpack).  NVLink TX / RX data bytes per rep from NVML counters."""
    import statistics

    import torch
    from paper_2006_15704_b200 import _lib as L
    from paper_2006_15704_b200.ddp import GradReducer
    from synth import device as sdev

    esize = 4 if a.dtype == "fp32" else 2
    tdt = torch.float32 if a.dtype == "fp32" else torch.bfloat16
    S = 25 * MIB
    n25 = S // esize
    nv = NvlinkCounter(local)
    cfgs = [("default", {})] + [(L.ALGO_NAMES[x], {L.OPT_ALGO: x}) for x in
                                (L.ALGO_ONESHOT, L.ALGO_TWOSHOT, L.ALGO_CE, L.ALGO_CE2, L.ALGO_PUSH, L.ALGO_NCCL,
                                 L.ALGO_NVLS)]
    cfgs.append(("grad_view", {L.OPT_GRAD_VIEW: 1}))
    out = {"bucket_mib": 25, "reps": reps, "l2": "flushed between reps (outside the events)",
           "timing": "producer-stream events around grad_ready -> finalize (whole sync), median, max over ranks",
           "algorithmic_nvlink_bytes_per_direction": {
               "oneshot/ce/push": (world - 1) * S, "twoshot/ce2/nccl(ring)": 2 * (world - 1) * S // world,
               "nvls": S + S // world},
           "per_algo": {}}
    base = dict(opts)
    base.pop(L.OPT_ALGO, None)
    base.pop(L.OPT_GRAD_VIEW, None)
    for name, extra in cfgs:
        o = {**base, **extra}
        red = GradReducer([n25], a.dtype, S, options=o)
        algo = red.bucket_algos()[0]
        if name == "nvls" and algo != "nvls":
            red.close()
            continue
        if extra.get(L.OPT_GRAD_VIEW):
            g = red._storage[L.ddp_param_storage_offset(red.ctx, 0):][:S].view(tdt)
        else:
            g = torch.empty(n25, dtype=tdt, device=dev)
        sdev.fill(g, 15704, int(os.environ.get("RANK", 0)), 0, 0, "normal", a.dtype)

        def one():
            red.grad_ready(0, g, stream)
            red.finalize(stream)
        for _ in range(10):
            one()
        barrier()
        c0 = nv.read()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
        for i in range(reps):
            flush_l2()
            evs[i][0].record(stream)
            one()
            evs[i][1].record(stream)
        torch.cuda.synchronize(dev)
        c1 = nv.read()
        ts = sorted(x.elapsed_time(y) for x, y in evs)
        med = max_over_ranks(statistics.median(ts))
        p10, p90 = max_over_ranks(ts[len(ts) // 10]), max_over_ranks(ts[(9 * len(ts)) // 10])
        r = {"algo": algo, "ms": med, "ms_p10": p10, "ms_p90": p90,
             "busbw_gbs": S / (med * 1e-3) * 2 * (world - 1) / world / 1e9,
             "includes": "allreduce only (gradients are the bucket)" if extra.get(L.OPT_GRAD_VIEW)
             else "pack x1/W + allreduce + unpack"}
        if c0 is not None and c1 is not None:
            # read after the warm-up reps; the L2 flushes are local HBM traffic only
            r["nvlink_tx_bytes_per_rep"] = (c1[0] - c0[0]) / reps
            r["nvlink_rx_bytes_per_rep"] = (c1[1] - c0[1]) / reps
        red.close()
        del g
        if algo in ("oneshot", "twoshot", "nvls"):   # the same bucket as a NON-last bucket
            red2 = GradReducer([1024, n25], a.dtype, S, options=o)
            g2 = torch.empty(n25, dtype=tdt, device=dev)
            gt = torch.empty(1024, dtype=tdt, device=dev)
            sdev.fill(g2, 15704, 0, 0, 1, "normal", a.dtype)
            sdev.fill(gt, 15704, 0, 0, 0, "normal", a.dtype)
            L.ddp_set_option(red2.ctx, L.OPT_PROFILE, 1)

            def two():
                red2.grad_ready(1, g2, stream)
                red2.grad_ready(0, gt, stream)
                red2.finalize(stream)
            for _ in range(5):
                two()
            L.ddp_profile_timeline(red2.ctx)
            barrier()
            for _ in range(reps // 2):
                flush_l2()
                two()
            tl = L.ddp_profile_timeline(red2.ctx, cap=4 * reps)
            fused = [e_ - s_ for k, _, s_, e_ in tl if k == "p2p_fused"]
            first = fused[0::2]   # per pass: bucket 0's fused kernel, then the small last bucket's
            if first:
                t2 = max_over_ranks(statistics.median(first))
                r["nonlast"] = {"ms": t2, "busbw_gbs": S / (t2 * 1e-3) * 2 * (world - 1) / world / 1e9,
                                "ctas_per_rank": int(L.ddp_get_option(red2.ctx, L.OPT_COMM_CTAS)),
                                "timing": "profile events around the fused kernel of bucket 0 (median)"}
            red2.close()
        out["per_algo"][name] = r
    d = out["per_algo"].get("default")
    if d:
        out.update(value=d["busbw_gbs"], unit="GB/s", algo=d["algo"], ms=d["ms"],
                   frac_of_nominal_900=d["busbw_gbs"] / 900.0, frac_of_measured_770=d["busbw_gbs"] / 770.0)
    return out


def build_model(name, dtype, batch, seq, rank, dev):
    """A randomly initialised model of the paper's families on synthetic data:
    torchvision ResNet-50 (224x224 images, CrossEntropy as in P:L329) or HF
    BertModel-large (random token ids).  Returns (model, loss_fn, description)."""
    import torch

    torch.backends.cudnn.benchmark = True
    torch.backends.cuda.matmul.allow_tf32 = True
    torch.backends.cudnn.allow_tf32 = True
    g = torch.Generator(device=dev).manual_seed(15704 + rank)
    if name == "resnet50":
        import torchvision
        model = torchvision.models.resnet50().to(dev)
        B = batch or 64
        x = torch.randn(B, 3, 224, 224, device=dev, generator=g)
        y = torch.randint(0, 1000, (B,), device=dev, generator=g)
        if dtype == "bf16":
            model, x = model.to(torch.bfloat16), x.to(torch.bfloat16)
        lossf = torch.nn.CrossEntropyLoss()

        def fwd(m):
            return lossf(m(x), y)
        return model, fwd, f"torchvision resnet50, batch {B}/GPU, 224x224, CrossEntropy"
    import transformers
    cfg = transformers.BertConfig(hidden_size=1024, num_hidden_layers=24, num_attention_heads=16,
                                  intermediate_size=4096)
    model = transformers.BertModel(cfg).to(dev)
    if dtype == "bf16":
        model = model.to(torch.bfloat16)
    B, S = (batch or 8), (seq or 512)
    ids = torch.randint(0, cfg.vocab_size, (B, S), device=dev, generator=g)

    def fwd(m):  # touches every parameter (pooler included): no unused parameters
        o = m(input_ids=ids)
        return o.last_hidden_state.float().pow(2).mean() + o.pooler_output.float().pow(2).mean()
    return model, fwd, f"HF BertModel-large, {B}x{S} tokens/GPU, mean-square loss on hidden states + pooler"


def exposed_for(model, fwd, desc, cap_mib, opts, iters, rank, world, local, dev, dtype,
                timeline_detail=False, nosync_every=(), no_overlap=True):
    """Exposed (non-overlapped) sync time with a REAL backward:
    the DDP front end's post-accumulate hooks drive the library during
    loss.backward().  T_sync: event before backward() -> event after it returns
    (the finalize callback has made the stream wait for the comm stream).
    T_bwd: the same window inside no_sync (hooks still fire and return early).
    Interleaved; exposed = median(T_sync) - median(T_bwd), max over ranks.
    nosync_every: for each n, groups of n-1 no_sync passes + 1 synced pass
    (config 5): amortized ms/iter of the group and exposed/iter."""
    import statistics

    import torch
    import torch.distributed as dist
    from paper_2006_15704_b200 import _lib as L
    from paper_2006_15704_b200.ddp import DistributedDataParallel

    ddp = DistributedDataParallel(model, bucket_cap_mb=cap_mib, options=opts)
    stream = torch.cuda.current_stream(dev)

    def clear_grads():
        for p in ddp.params:
            if ddp.gradient_as_bucket_view and p.grad is not None:
                p.grad.zero_()          # keeps the bucket views (zero_grad(set_to_none=False))
            else:
                p.grad = None

    def one(sync: bool) -> float:
        clear_grads()
        loss = fwd(ddp)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if sync:
            s.record(stream)
            loss.backward()
            e.record(stream)
        else:
            with ddp.no_sync():
                s.record(stream)
                loss.backward()
                e.record(stream)
        torch.cuda.synchronize(dev)
        return s.elapsed_time(e)

    def group(n: int, sync_last: bool = True) -> float:
        """n-1 accumulating no_sync backward passes + 1 synced one (sync_last) or n
        no_sync ones (the baseline with the same .grad accumulation): summed backward ms."""
        clear_grads()
        tot = 0.0
        for k in range(n):
            loss = fwd(ddp)
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            if k < n - 1 or not sync_last:
                with ddp.no_sync():
                    s.record(stream)
                    loss.backward()
                    e.record(stream)
            else:
                s.record(stream)
                loss.backward()
                e.record(stream)
            torch.cuda.synchronize(dev)
            tot += s.elapsed_time(e)
        return tot

    for _ in range(10):
        one(True)
        one(False)
    if world > 1:
        dist.barrier(device_ids=[local])
    ts, tb, tn = [], [], []
    for _ in range(iters):
        ts.append(one(True))
        tb.append(one(False))
        if no_overlap:
            ddp.reducer.set_option(L.OPT_OVERLAP, 0)   # paper's non-overlapped baseline
            tn.append(one(True))
            ddp.reducer.set_option(L.OPT_OVERLAP, 1)
    ns_res, ns_base, ns_spread = {}, {}, {}
    for n in nosync_every:
        group(n)
        group(n, False)
        gt, gb = [], []
        for _ in range(max(2, iters // 2)):
            gt.append(group(n))
            gb.append(group(n, False))
        ns_res[n], ns_base[n] = statistics.median(gt), statistics.median(gb)
        dd = sorted(x - y for x, y in zip(gt, gb))
        ns_spread[n] = (dd[len(dd) // 10], dd[(9 * len(dd)) // 10])
    # one profiled synced pass: Fig. 2(c)-style ready / start / end timeline of the comm launches
    ddp.reducer.set_option(L.OPT_PROFILE, 1)
    L.ddp_profile_timeline(ddp.reducer.ctx)
    one(True)
    tl = L.ddp_profile_timeline(ddp.reducer.ctx)
    ddp.reducer.set_option(L.OPT_PROFILE, 0)
    timeline = None
    if tl:
        timeline = {"launches": len(tl), "last_ready_ms": max(r for _, r, _, _ in tl),
                    "last_end_ms": max(e for _, _, _, e in tl),
                    "tail_ms": max(e for _, _, _, e in tl) - max(r for _, r, _, _ in tl),
                    "max_queue_delay_ms": max(s - r for _, r, s, _ in tl),
                    "comm_busy_ms": sum(e - s for _, _, s, e in tl),
                    "per_launch": [[k, round(r, 4), round(s, 4), round(e, 4)] for k, r, s, e in tl]
                    if timeline_detail else None}
    ddp.reducer.check_errors()
    # sanity floor: the last bucket holds the first-registered
    # params, so its whole sync cannot start before backward ends: exposed >= the
    # sync time of that bucket alone (same algorithm, measured in isolation)
    from paper_2006_15704_b200.ddp import GradReducer
    last = ddp.reducer.bucket_numels()[-1]
    o2 = dict(opts)
    o2[L.OPT_ALGO] = L.ddp_bucket_algo(ddp.reducer.ctx, ddp.reducer.num_buckets - 1)
    solo = GradReducer([last], dtype, last * (4 if dtype == "fp32" else 2), options=o2)
    gl = torch.empty(last, dtype=torch.float32 if dtype == "fp32" else torch.bfloat16, device=dev)
    gl.normal_()
    fl = []
    for i in range(8):
        s0, e0 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        solo.grad_ready(0, gl, stream)
        solo.finalize(stream)
        e0.record(stream)
        torch.cuda.synchronize(dev)
        if i >= 3:
            fl.append(s0.elapsed_time(e0))
    solo.close()
    vals = [statistics.median(ts), statistics.median(tb), statistics.median(tn) if tn else 0.0]
    vals += [ns_res[n] for n in nosync_every] + [ns_base[n] for n in nosync_every]
    vals.append(statistics.median(fl))
    # spread: paired differences of the interleaved (synced, no_sync) passes
    dif = sorted(x - y for x, y in zip(ts, tb))

    def pct(v, q):
        return v[min(len(v) - 1, int(q * (len(v) - 1) + 0.5))]
    spread = [pct(dif, 0.1), pct(dif, 0.5), pct(dif, 0.9), pct(sorted(tb), 0.1), pct(sorted(tb), 0.9)]
    vals += spread
    vt = torch.tensor(vals, dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(vt, op=dist.ReduceOp.MAX)
    t_sync, t_bwd, t_noov = float(vt[0]), float(vt[1]), float(vt[2])
    d10, d50, d90, b10, b90 = (float(x) for x in vt[-5:])
    vt = vt[:-5]
    res = {"model": desc, "dtype": dtype, "bucket_cap_mib": cap_mib,
           "buckets": ddp.reducer.num_buckets, "bucket_algos": ddp.reducer.bucket_algos(),
           "t_bwd_ms": t_bwd, "t_bwd_plus_sync_ms": t_sync, "exposed_ms": t_sync - t_bwd,
           "exposed_pct_of_bwd": 100.0 * (t_sync - t_bwd) / t_bwd,
           "iters": iters, "warmup": 10, "timing": "median of interleaved passes, max over ranks",
           "exposed_paired_ms": {"p10": d10, "p50": d50, "p90": d90},
           "exposed_paired_pct_of_bwd": {"p10": 100 * d10 / t_bwd, "p50": 100 * d50 / t_bwd, "p90": 100 * d90 / t_bwd},
           "t_bwd_ms_p10_p90": [b10, b90],
           "spread_doc": "percentiles of the per-pair difference (synced pass - the no_sync pass right after it), "
                         "each percentile max over ranks",
           "floor_ms": float(vt[-1]),
           "floor_ok": bool(t_sync - t_bwd >= float(vt[-1]) * 0.9),
           "floor_doc": "whole sync of the last bucket alone (it cannot start before backward ends)",
           "timeline_rank0": timeline if rank == 0 else None}
    if no_overlap:
        res["t_bwd_plus_sync_no_overlap_ms"] = t_noov
        res["exposed_no_overlap_ms"] = t_noov - t_bwd
    if nosync_every:
        k = len(nosync_every)
        sp = torch.tensor([x for n in nosync_every for x in ns_spread[n]], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(sp, op=dist.ReduceOp.MAX)
        res["nosync"] = {str(n): {"ms_per_iter": float(vt[3 + i]) / n,
                                  "no_sync_baseline_ms_per_iter": float(vt[3 + k + i]) / n,
                                  "exposed_ms_per_iter": (float(vt[3 + i]) - float(vt[3 + k + i])) / n,
                                  "exposed_ms_per_iter_p10_p90": [float(sp[2 * i]) / n, float(sp[2 * i + 1]) / n],
                                  "groups": max(2, iters // 2)}
                         for i, n in enumerate(nosync_every)}
        res["nosync_doc"] = ("group of n backward passes with .grad accumulation: n-1 inside no_sync + 1 synced "
                             "(ms_per_iter) vs all n inside no_sync (baseline); exposed = difference / n")
    ddp.close()
    return res


def measure_exposed(a, rank, world, local, dev, opts):
    import torch
    model, fwd, desc = build_model(a.exposed_model, a.dtype, a.exposed_batch, 0, rank, dev)
    res = exposed_for(model, fwd, desc, a.cap_mib, opts, a.exposed_iters, rank, world, local, dev, a.dtype,
                      a.timeline_detail)
    del model
    torch.cuda.empty_cache()
    return res


def _init_dist(a):
    import torch
    import torch.distributed as dist
    rank, world, local = env_rank()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    return rank, world, local, dev


def _opts(a):
    from paper_2006_15704_b200 import _lib as L
    o = {}
    for key, v in ((L.OPT_ALGO, a.algo), (L.OPT_COMM_CTAS, a.comm_ctas), (L.OPT_PACK_CTAS, a.pack_ctas)):
        if v:
            o[key] = v
    if a.stage_kib:
        o[L.OPT_P2P_STAGE_BYTES] = a.stage_kib * 1024
    if a.ce_streams:
        o[L.OPT_CE_STREAMS] = a.ce_streams
    if a.throughput_policy:
        o[L.OPT_PREFER_OVERLAP] = 0
    if a.overlap_policy >= 0:
        o[L.OPT_PREFER_OVERLAP] = a.overlap_policy
    if a.high_priority:
        o[L.OPT_LOW_PRIORITY] = 0
    if a.lanes:
        o[L.OPT_LANES] = a.lanes
    if a.p2p_push:
        o[L.OPT_P2P_PULL] = 0
    if a.p2p_pull_all:
        o[L.OPT_P2P_PULL] = 2
    if a.last_on_lane:
        o[L.OPT_LAST_ON_PRODUCER] = 0
    if a.wire_bf16:
        o[L.OPT_WIRE_BF16] = 1
    if a.grad_view:
        o[L.OPT_GRAD_VIEW] = 1
    if a.ce_direct_mib >= 0:
        o[L.OPT_CE_DIRECT_BYTES] = int(a.ce_direct_mib * MIB)
    if a.nccl_comms:
        o[L.OPT_NCCL_COMMS] = a.nccl_comms
    if a.oneshot_max >= 0:
        o[L.OPT_P2P_ONESHOT_MAX] = a.oneshot_max
    if a.twoshot_max >= 0:
        o[L.OPT_P2P_TWOSHOT_MAX] = a.twoshot_max
    return o


def run_sweep(a):
    """Secondary measurements (one JSON line per point, rank 0), SURVEY §8(d) M-1/M-3."""
    import torch
    import torch.distributed as dist
    rank, world, local, dev = _init_dist(a)
    opts = _opts(a)
    out = []
    if a.mode in ("cap-sweep", "nosync"):
        name = a.exposed_model if a.exposed_model != "none" else a.workload
        model, fwd, desc = build_model(name, a.dtype, a.exposed_batch, a.exposed_seq, rank, dev)
        if a.mode == "cap-sweep":
            for cap in [float(c) for c in a.caps.split(",")]:
                r = exposed_for(model, fwd, desc, cap, opts, a.exposed_iters, rank, world, local, dev, a.dtype)
                r.update(mode="cap-sweep", n_gpus=world)
                out.append(r)
        else:
            r = exposed_for(model, fwd, desc, a.cap_mib, opts, a.exposed_iters, rank, world, local, dev, a.dtype,
                            nosync_every=(1, 2, 4, 8), no_overlap=False)
            r.update(mode="nosync", n_gpus=world)
            out.append(r)
    else:
        out = allreduce_sweep(a, rank, world, local, dev, opts)
    if rank == 0:
        for r in out:
            print(json.dumps(r), flush=True)
    if world > 1:
        dist.destroy_process_group()


def allreduce_sweep(a, rank, world, local, dev, opts):
    """M-3 (paper Fig. 2 method): (i) one bucket of S bytes, whole sync
    (pack x1/W + allreduce + unpack / fused kernel) per algorithm, busBW =
    (S/t) 2(W-1)/W; (ii) a fixed total of 60M fp32 parameters split into k equal
    buckets (cap 0: one bucket per gradient), all launched back to back, one wait."""
    import torch
    import torch.distributed as dist
    from paper_2006_15704_b200 import _lib as L
    from paper_2006_15704_b200.ddp import GradReducer
    from synth import device as sdev

    tdt = torch.float32 if a.dtype == "fp32" else torch.bfloat16
    esize = 4 if a.dtype == "fp32" else 2
    stream = torch.cuda.current_stream(dev)
    algos = [L.ALGO_AUTO, L.ALGO_NCCL, L.ALGO_ONESHOT, L.ALGO_TWOSHOT] + (
        [L.ALGO_CE, L.ALGO_CE2, L.ALGO_NVLS, L.ALGO_PUSH] if world > 1 else [])
    nccl_algo = os.environ.get("NCCL_ALGO", "default")
    sizes = [4 << 10, 64 << 10, 256 << 10, 1 << 20, 4 << 20, 16 << 20, 25 << 20, 64 << 20, 256 << 20]
    res = []

    def tmax(x):
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def time_it(fn, reps):
        for _ in range(3):
            fn()
        if world > 1:
            dist.barrier(device_ids=[local])
        torch.cuda.synchronize(dev)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        for _ in range(reps):
            fn()
        e.record(stream)
        torch.cuda.synchronize(dev)
        return tmax(s.elapsed_time(e) / reps)

    for S in sizes:
        n = S // esize
        g = torch.empty(n, dtype=tdt, device=dev)
        sdev.fill(g, 15704, rank, 0, 0, "normal", a.dtype)
        for algo in algos:
            o = dict(opts)
            o[L.OPT_ALGO] = algo
            red = GradReducer([n], a.dtype, S, options=o)

            def one():
                red.grad_ready(0, g, stream)
                red.finalize(stream)
            t = time_it(one, 100 if S <= (64 << 20) else 10)
            bw = S / (t * 1e-3) * 2 * (world - 1) / world / 1e9 if world > 1 else None
            res.append({"mode": "allreduce-sweep", "n_gpus": world, "dtype": a.dtype, "bytes": S,
                        "nccl_algo": nccl_algo, "reps": 100 if S <= (64 << 20) else 10,
                        "algo": red.bucket_algos()[0], "forced": L.ALGO_NAMES[algo] if algo else "auto",
                        "ms": t, "busbw_gbs": bw, "algbw_gbs": S / (t * 1e-3) / 1e9,
                        "includes": "pack x1/W + allreduce + unpack (fused kernel for P2P)"})
            red.close()
        del g
    # (ii) fixed total, k equal gradients, cap 0 (one bucket per gradient), one batched ready call
    total = 60_000_000 if a.dtype == "fp32" else 60_000_000
    for per in (1_000, 10_000, 100_000, 1_000_000, 10_000_000, 60_000_000):
        k = total // per
        flat = torch.empty(k * per, dtype=tdt, device=dev)
        sdev.fill(flat, 15704, rank, 0, 1, "normal", a.dtype)
        for algo in (L.ALGO_AUTO, L.ALGO_NCCL):
            o = dict(opts)
            o[L.OPT_ALGO] = algo
            red = GradReducer([per] * k, a.dtype, 0, options=o)
            batch = L.ReadyBatch(list(range(k - 1, -1, -1)),
                                 [flat[p * per:].data_ptr() for p in range(k - 1, -1, -1)])

            def one():
                red.grads_ready(batch, stream)
                red.finalize(stream)
            t = time_it(one, 3)
            res.append({"mode": "fixed-total-split", "n_gpus": world, "dtype": a.dtype, "total_params": k * per,
                        "params_per_op": per, "ops": k, "algo": red.bucket_algos()[0],
                        "forced": L.ALGO_NAMES[algo] if algo else "auto", "ms_total": t})
            red.close()
        del flat
    return res


def main():
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    elif a.mode == "step":
        run_ours(a)
    else:
        run_sweep(a)


if __name__ == "__main__":
    main()
