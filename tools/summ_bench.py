"""One-screen summary of bench.py JSON lines read from stdin."""
import json
import sys

for line in sys.stdin:
    if not line.startswith("{"):
        continue
    d = json.loads(line)
    rf = d.get("roofline") or {}
    print(f"N={d['n_gpus']} {d['config']['workload']} value {d['value']:.4f} ms  algos {d['config']['bucket_algos']}")
    print(f"  roofline {rf.get('kernel')} {rf.get('bound')} {rf.get('achieved', 0):.0f}/{rf.get('peak', 0):.0f} "
          f"frac {rf.get('frac', 0):.3f}  e2e {d.get('e2e') and round(d['e2e']['value'], 3)}")
    bb = d.get("busbw")
    if bb:
        print("  busbw " + "  ".join(f"{k}:{v['algo']}={v['busbw_gbs']:.0f}"
                                     + (f"(nl {v['nonlast']['busbw_gbs']:.0f})" if 'nonlast' in v else "")
                                     for k, v in bb["per_algo"].items()))
    ex = d.get("exposed")
    if ex:
        print(f"  exposed {ex['exposed_ms']:.3f} ms = {ex['exposed_pct_of_bwd']:.2f}% of {ex['t_bwd_ms']:.2f} "
              f"(paired p10/p50/p90 {ex['exposed_paired_pct_of_bwd']['p10']:.2f}/"
              f"{ex['exposed_paired_pct_of_bwd']['p50']:.2f}/{ex['exposed_paired_pct_of_bwd']['p90']:.2f}%) "
              f"algos {ex['bucket_algos']} floor {ex['floor_ms']:.3f}")
    if d.get("cpu_baseline"):
        c = d["cpu_baseline"]
        print(f"  cpu {c['value']:.1f} ms (1 core), all-core {c.get('all_core', {}).get('value')}")
    print(f"  clocks {d.get('clocks')}")
