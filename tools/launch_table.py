"""Summarise an ncu --csv launch list (gpu__time_duration + dram bytes) per launch.

    python tools/launch_table.py gpurun_out/x_launches.csv [--first N]
"""
import collections
import csv
import sys

path = sys.argv[1]
first = int(sys.argv[3]) if len(sys.argv) > 3 and sys.argv[2] == "--first" else None
rows = list(csv.reader(open(path)))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hi]
k = collections.OrderedDict()
for r in rows[hi + 1:]:
    d = dict(zip(h, r))
    key = (d["ID"], d["Kernel Name"].split("(")[0], d["Grid Size"])
    k.setdefault(key, {})[d["Metric Name"]] = d["Metric Value"].replace(",", "")
tot = 0.0
for i, (key, v) in enumerate(k.items()):
    if first is not None and i >= first:
        break
    t = float(v["gpu__time_duration.sum"])
    rb = float(v.get("dram__bytes_read.sum", 0))
    wb = float(v.get("dram__bytes_write.sum", 0))
    tot += t
    print(f"{key[0]:>4} {key[1][:34]:34s} {key[2]:>16s} {t / 1e3:8.1f} us  rd {rb / 1e6:8.1f} MB  wr {wb / 1e6:7.1f} MB  {(rb + wb) / t:6.0f} GB/s")
print(f"total {tot / 1e3:.1f} us")
