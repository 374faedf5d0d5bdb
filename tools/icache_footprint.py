"""Instruction-fetch footprint of a kernel from an ncu report (dev tool):
how many 128-byte I-cache lines hold the instructions that make up a given
share of the executed warp instructions.  The warp engine is fetch-bound
(stall_no_instruction), so this is the number to shrink.
    python tools/icache_footprint.py REP [--kernel regex]"""
import csv
import re
import subprocess
import sys

rep = sys.argv[1]
args = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"]
if len(sys.argv) > 3 and sys.argv[2] == "--kernel":
    args += ["-k", sys.argv[3]]
out = subprocess.run(args, capture_output=True, text=True).stdout
ins = []
for r in csv.reader(out.splitlines()):
    if len(r) >= 3 and r[0].startswith("0x"):
        try:
            ins.append((int(r[0], 16), int(r[2] or 0), r[1].strip()))
        except ValueError:
            pass
if not ins:
    raise SystemExit("no SASS rows")
base = min(a for a, _, _ in ins)
tot = sum(c for _, c, _ in ins)
print(f"{len(ins)} instructions ({len(ins) * 16 / 1024:.0f} KB), {tot} executed")
lines = {}
for a, c, _ in ins:
    lines[(a - base) // 128] = lines.get((a - base) // 128, 0) + c
ranked = sorted(lines.values(), reverse=True)
hot_ins = sorted((c for _, c, _ in ins), reverse=True)
for share in (0.5, 0.8, 0.9, 0.95, 0.99):
    acc, n = 0, 0
    for c in ranked:
        acc += c
        n += 1
        if acc >= share * tot:
            break
    acc2, m = 0, 0
    for c in hot_ins:
        acc2 += c
        m += 1
        if acc2 >= share * tot:
            break
    print(f"  {100 * share:4.0f}% of executed: {n:5d} lines = {n * 128 / 1024:6.1f} KB "
          f"(densely packed: {m} instructions = {m * 16 / 1024:5.1f} KB)")
