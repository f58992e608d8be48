"""Summarise an ncu --set full report (.ncu-rep) into JSON: per launch, the duration, DRAM
bytes and throughput, L2 hit rate, occupancy, registers and the top warp-stall reasons.

    python tools/ncu_full_summary.py report.ncu-rep "command" > profiles/x.json
"""
import csv
import io
import json
import subprocess
import sys

rep, command = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units = rows[0], rows[1]
want = {"gpu__time_duration.sum": "us", "dram__bytes_read.sum": "B", "dram__bytes_write.sum": "B",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "%", "lts__t_sector_hit_rate.pct": "%",
        "sm__warps_active.avg.pct_of_peak_sustained_active": "%", "launch__registers_per_thread": "",
        "launch__grid_size": "", "sm__throughput.avg.pct_of_peak_sustained_elapsed": "%",
        "l1tex__throughput.avg.pct_of_peak_sustained_active": "%"}
scale = {"ns": 1e-3, "us": 1.0, "ms": 1e3, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
out = []
for r in rows[2:]:
    d = dict(zip(h, r))
    u = dict(zip(h, units))
    k = {"kernel": d["Kernel Name"].split("(")[0].replace("void ", "")}
    for m in want:
        if m not in d or d[m] == "":
            continue
        v = float(d[m].replace(",", ""))
        k[m] = v * scale.get(u[m], 1.0) if u[m] in scale else v
    if "gpu__time_duration.sum" in k:
        k["gpu__time_duration.sum"] = float(d["gpu__time_duration.sum"].replace(",", "")) * scale.get(
            u["gpu__time_duration.sum"], 1.0)
        k["time_us"] = k.pop("gpu__time_duration.sum")
    byt = k.get("dram__bytes_read.sum", 0.0) + k.get("dram__bytes_write.sum", 0.0)
    k["dram_bytes"] = byt
    if k.get("time_us"):
        k["dram_GBps"] = byt / (k["time_us"] * 1e-6) / 1e9
    st = {m.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(d[m])
          for m in d if m.startswith("smsp__pcsamp_warps_issue_stalled") and not m.endswith("not_issued")
          and d[m] not in ("", "n/a")}
    tot = sum(st.values()) or 1.0
    k["top_stalls"] = {s: round(v / tot, 3) for s, v in sorted(st.items(), key=lambda kv: -kv[1])[:4]}
    out.append(k)
print(json.dumps({"command": command, "kernels": out}, indent=1))
