"""Summarise ncu output for profiles/ (run here, on the CPU box).

    python tools/ncu_summary.py launches <launches.csv>            # per-kernel share of the launch list
    python tools/ncu_summary.py full <prof.ncu-rep> [label]        # key --set full metrics per launch

`full` also prints a JSON line {"label", "kernel", "traffic_bytes_per_launch", ...}
that can be pasted into profiles/traffic.json (bench.py reads it to fill
roofline.traffic).
"""

import collections
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "launch__occupancy_limit_registers",
    "sm__maximum_warps_per_active_cycle_pct",
    "lts__t_bytes.sum",
    "smsp__inst_executed.sum",
]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1, "usecond": 1, "ms": 1e3,
         "msecond": 1e3, "nsecond": 1e-3}


def launches(path):
    rows = [r for r in csv.DictReader(l for l in open(path) if l.startswith('"'))]
    agg = collections.OrderedDict()
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        k = r["Kernel Name"].split("(")[0].replace("void ", "")
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += float(r["Metric Value"]) * SCALE.get(r["Metric Unit"], 1)
    tot = sum(v[1] for v in agg.values())
    print(f"| kernel | launches | total us | share |\n|---|---|---|---|")
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"| `{k[:90]}` | {n} | {t:.1f} | {100 * t / tot:.1f}% |")


def full(path, label=""):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    col = {h: i for i, h in enumerate(hdr)}
    recs = []
    for r in rows[2:]:
        d = {"kernel": r[col["Kernel Name"]][:90], "grid": r[col["Grid Size"]], "block": r[col["Block Size"]]}
        for k in KEYS:
            if k in col and r[col[k]] not in ("", "n/a"):
                v = float(r[col[k]].replace(",", ""))
                u = units[col[k]]
                if u in SCALE and ("bytes" in k or "time" in k):
                    v *= SCALE[u]
                    u = "byte" if "bytes" in k else "us"
                d[k] = (v, u)
        recs.append(d)
    print(f"### {label or path}\n")
    print("| metric | " + " | ".join(f"launch {i}" for i in range(len(recs))) + " |")
    print("|---|" + "---|" * len(recs))
    print("| kernel | " + " | ".join(f"`{d['kernel']}` grid {d['grid']} block {d['block']}" for d in recs) + " |")
    for k in KEYS:
        if any(k in d for d in recs):
            print(f"| {k} | " + " | ".join(f"{d[k][0]:.4g} {d[k][1]}" if k in d else "" for d in recs) + " |")
    tr = [d["dram__bytes_read.sum"][0] + d["dram__bytes_write.sum"][0] for d in recs
          if "dram__bytes_read.sum" in d and "dram__bytes_write.sum" in d]
    if tr:
        print("\n" + json.dumps({"label": label, "kernel": recs[0]["kernel"],
                                 "traffic_bytes_per_launch": sum(tr) / len(tr),
                                 "ncu_us_per_launch": sum(d["gpu__time_duration.sum"][0] for d in recs) / len(recs)}))


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2])
    else:
        full(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "")
