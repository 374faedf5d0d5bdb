"""Hottest CUDA source lines of an ncu report (warp-stall samples and executed
warp instructions), from `ncu -i REP --page source --csv --print-source=cuda,sass`."""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows, cur, hdr = [], None, None
for r in csv.reader(out.splitlines()):
    if not r:
        continue
    if r[0] in ("File Path", "File Name"):
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr and r[0].isdigit():
        try:
            s, ins = int(r[4] or 0), int(r[7] or 0)
        except (ValueError, IndexError):
            continue
        rows.append((s, ins, cur, int(r[0]), r[1].strip()[:80]))
ts = sum(x[0] for x in rows) or 1
ti = sum(x[1] for x in rows) or 1
print(f"stall samples {ts}  warp instructions {ti}")
for s, ins, f, ln, src in sorted(rows, reverse=True)[:top]:
    print(f"{100 * s / ts:5.1f}% smp {100 * ins / ti:5.1f}% ins  {f}:{ln}  {src}")
