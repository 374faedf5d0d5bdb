"""Static SASS size of the hot code per CUDA source line (dev tool): for the
instructions that make up `share` of the executed warp instructions, how
many belong to each source line -- where the fetch footprint comes from.
    python tools/icache_by_line.py REP [share=0.95] [top=40]"""
import csv
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
share = float(sys.argv[2]) if len(sys.argv) > 2 else 0.95
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
ins = []  # (count, file, line, src)
cur_file, cur_line, cur_src = None, None, None
for r in csv.reader(out.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0].isdigit():
        cur_line, cur_src = int(r[0]), r[1].strip()[:70]
        continue
    if len(r) >= 5 and r[2].startswith("0x"):
        try:
            ins.append((int(r[4] or 0), cur_file, cur_line, cur_src))
        except ValueError:
            pass
tot = sum(c for c, *_ in ins)
ins.sort(key=lambda x: -x[0])
acc, hot = 0, []
for x in ins:
    if acc >= share * tot:
        break
    acc += x[0]
    hot.append(x)
by = defaultdict(lambda: [0, 0, ""])
for c, f, ln, src in hot:
    k = (f, ln)
    by[k][0] += 1
    by[k][1] += c
    by[k][2] = src
byf = defaultdict(int)
for (f, ln), (n, c, s) in by.items():
    byf[f] += n
print(f"{len(hot)} hot instructions ({len(hot) * 16 / 1024:.1f} KB) hold {100 * share:.0f}% of execution")
print("  by file:", ", ".join(f"{f} {n}" for f, n in sorted(byf.items(), key=lambda x: -x[1])))
for (f, ln), (n, c, s) in sorted(by.items(), key=lambda x: -x[1][0])[:top]:
    print(f"  {n:4d} instr  {100 * c / tot:5.2f}% exec  {f}:{ln}  {s}")
