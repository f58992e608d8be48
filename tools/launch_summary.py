"""ncu --csv launch list -> per-kernel JSON summary (launches, total ms, DRAM GB, share).

    python tools/launch_summary.py launches.csv "command" "note" > profiles/x.json
"""
import collections
import csv
import json
import sys

path, command, note = sys.argv[1], sys.argv[2], sys.argv[3]
rows = list(csv.reader(open(path)))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hi]
per_launch = collections.OrderedDict()
for r in rows[hi + 1:]:
    d = dict(zip(h, r))
    key = (d["ID"], d["Kernel Name"].split("(")[0].replace("void ", ""))
    per_launch.setdefault(key, {})[d["Metric Name"]] = float(d["Metric Value"].replace(",", "") or 0)
kern = collections.OrderedDict()
total = 0.0
for (_, name), v in per_launch.items():
    t = v.get("gpu__time_duration.sum", 0.0) * 1e-6  # ns -> ms
    by = v.get("dram__bytes_read.sum", 0.0) + v.get("dram__bytes_write.sum", 0.0)
    k = kern.setdefault(name, {"launches": 0, "total_ms": 0.0, "dram_GB": 0.0})
    k["launches"] += 1
    k["total_ms"] += t
    k["dram_GB"] += by / 1e9
    total += t
for k in kern.values():
    k["share"] = k["total_ms"] / total if total else 0.0
    k["avg_us"] = 1e3 * k["total_ms"] / k["launches"]
    k["GBps"] = k["dram_GB"] / (k["total_ms"] * 1e-3) if k["total_ms"] else 0.0
out = {"command": command, "note": note, "launches": len(per_launch), "total_ms": total,
       "per_kernel": dict(sorted(kern.items(), key=lambda kv: -kv[1]["total_ms"]))}
print(json.dumps(out, indent=1))
