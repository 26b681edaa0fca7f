"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into per-kernel totals and
shares of the summed kernel time.  Usage: python tools/summarize_launches.py launches.csv out.json "command" """
import csv
import json
import sys
from collections import defaultdict

UNIT = {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0}


def main(path, out, command):
    rows = []
    with open(path, newline="") as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        rows.append((r["Kernel Name"], float(r["Metric Value"].replace(",", "")) * UNIT[r["Metric Unit"]]))
    agg = defaultdict(lambda: [0, 0.0])
    for name, t in rows:
        agg[name][0] += 1
        agg[name][1] += t
    total = sum(t for _, t in rows)
    kernels = [{"name": k, "launches": n, "s": s, "share": s / total if total else 0.0}
               for k, (n, s) in sorted(agg.items(), key=lambda kv: -kv[1][1])]
    json.dump({"command": command, "total_kernel_s": total, "launches": len(rows), "kernels": kernels},
              open(out, "w"), indent=1)
    print(json.dumps({"launches": len(rows), "total_kernel_s": total, "top": kernels[:3]}))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "")
