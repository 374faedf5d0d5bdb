"""Stall-reason breakdown of one ncu report (dev tool):
    python tools/ncu_stalls.py <report.ncu-rep> [n_lines] [steps]
Kernel-wide stall shares, then the hottest CUDA source lines with their top
stall reasons and (with `steps`) executed warp instructions per step."""
import csv
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
steps = float(sys.argv[3]) if len(sys.argv) > 3 else 0.0
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur, hdr, out = None, None, []
for r in csv.reader(txt.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
    elif r[0] == "Line No":
        hdr = r
    elif r[0] != "Function Name" and r[0] and len(r) > 2 and r[2] == "-":
        out.append((cur, r))


def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


idx = {h: i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not" not in h}
i_smp, i_ins = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
tot = sum(f(r[i_smp]) for _, r in out) or 1.0
agg = {k: sum(f(r[i]) for _, r in out) for k, i in idx.items()}
print("stall share (% of warp samples): " + ", ".join(
    f"{k[6:]} {v / tot * 100:.1f}" for k, v in sorted(agg.items(), key=lambda x: -x[1])[:10]))
per_file = {}
for c, r in out:
    per_file.setdefault(c, [0.0, 0.0])
    per_file[c][0] += f(r[i_smp])
    per_file[c][1] += f(r[i_ins])
toti = sum(v[1] for v in per_file.values()) or 1.0
print("by file (% samples / % instructions): " + ", ".join(
    f"{k} {v[0] / tot * 100:.1f}/{v[1] / toti * 100:.1f}"
    for k, v in sorted(per_file.items(), key=lambda x: -x[1][0]) if v[0] / tot > 0.005))
print(f"hottest {n} source lines:")
for c, r in sorted(out, key=lambda x: -f(x[1][i_smp]))[:n]:
    top = sorted(((k[6:], f(r[i])) for k, i in idx.items()), key=lambda x: -x[1])[:3]
    ips = f" {f(r[i_ins]) / steps:6.1f} inst/step" if steps else ""
    print(f"  {f(r[i_smp]) / tot * 100:5.2f}%{ips}  {c}:{r[0]}  "
          + " ".join(f"{k}={v / tot * 100:.2f}" for k, v in top) + "  | " + r[1].strip()[:70])
