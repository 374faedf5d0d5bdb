"""Writes profiles/<tag>_*.txt/json summaries from ncu reports in gpurun_out/.

    python tools/summarize_ncu.py <tag> <report.ncu-rep> <kernel> <workload> [launches.csv]
"""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag, rep, kernel, workload = sys.argv[1:5]
launches = sys.argv[5] if len(sys.argv) > 5 else None
prof = os.path.join(ROOT, "profiles")

raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout.splitlines()
rows = list(csv.reader(raw))
h, u, v = rows[0], rows[1], rows[2]


def metric(name):
    if name not in h:
        return None
    i = h.index(name)
    x = v[i].replace(",", "")
    scale = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0}.get(u[i], 1.0)
    try:
        return float(x) * scale
    except ValueError:
        return x


summary = {
    "tag": tag, "kernel": kernel, "workload": workload,
    "capture": f"ncu --set full --clock-control none --import-source on -k regex:{kernel} -c 1",
    "gpu__time_duration_ms": metric("gpu__time_duration.sum"),
    "dram_bytes_read": metric("dram__bytes_read.sum"),
    "dram_bytes_write": metric("dram__bytes_write.sum"),
    "registers_per_thread": metric("launch__registers_per_thread"),
    "warps_active_pct": metric("sm__warps_active.avg.pct_of_peak_sustained_active"),
    "issue_active_pct": metric("smsp__issue_active.avg.pct_of_peak_sustained_active"),
    "l1tex_hit_rate_pct": metric("l1tex__t_sector_hit_rate.pct"),
    "lts_hit_rate_pct": metric("lts__t_sector_hit_rate.pct"),
    "warp_instructions": metric("smsp__inst_executed.sum"),
    "dram_throughput_pct": metric("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
}
summary["dram_bytes_per_launch"] = (summary["dram_bytes_read"] or 0) + (summary["dram_bytes_write"] or 0)
with open(os.path.join(prof, f"{tag}_{kernel}_ncu.json"), "w") as f:
    json.dump(summary, f, indent=1)
details = subprocess.run(["ncu", "-i", rep, "--page", "details"], capture_output=True,
                         text=True).stdout
hot = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_hot_lines.py"), rep, "30"],
                     capture_output=True, text=True).stdout
with open(os.path.join(prof, f"{tag}_{kernel}_ncu.txt"), "w") as f:
    f.write(f"# ncu --set full, {kernel}, {workload}\n")
    f.write("\n".join(x for x in details.splitlines() if x.strip()) + "\n\n")
    f.write("# hottest source lines (tools/ncu_hot_lines.py)\n" + hot)
if launches:
    with open(launches) as src, open(os.path.join(prof, f"{tag}_launches.csv"), "w") as dst:
        dst.writelines(x for x in src if not x.startswith("=="))
print(json.dumps(summary))
