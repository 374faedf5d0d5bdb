"""Warp-instruction and stall-sample shares of an ncu report by file and by
line range (dev tool): python tools/ncu_by_region.py REP [file:lo-hi ...]"""
import csv
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
ranges = []
for a in sys.argv[2:]:
    f, r = a.split(":")
    lo, hi = r.split("-")
    ranges.append((f, int(lo), int(hi)))
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
cur, hdr = None, None
by_file = defaultdict(lambda: [0, 0])
by_rng = defaultdict(lambda: [0, 0])
ts = ti = 0
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
        ln = int(r[0])
        by_file[cur][0] += s
        by_file[cur][1] += ins
        ts += s
        ti += ins
        for f, lo, hi in ranges:
            if f == cur and lo <= ln <= hi:
                by_rng[f"{f}:{lo}-{hi}"][0] += s
                by_rng[f"{f}:{lo}-{hi}"][1] += ins
print(f"stall samples {ts}  warp instructions {ti}")
for k, (s, i) in sorted(by_file.items(), key=lambda x: -x[1][1]):
    print(f"  {k:28s} {100 * s / ts:5.1f}% smp {100 * i / ti:5.1f}% ins")
for k, (s, i) in by_rng.items():
    print(f"  {k:28s} {100 * s / ts:5.1f}% smp {100 * i / ti:5.1f}% ins")
