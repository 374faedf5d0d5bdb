"""Phase breakdown of the CTA-wide engine on C4 (dev tool).
    tools/build_variant.sh wprof -DFB_WIDE_PROF
    FBGPU_LIB=build/variants/wprof/libfbgpu.so python tools/wide_prof.py [n_inst]"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_14392_b200 import fbgpu, workloads  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
batch = workloads.c4_batch(n_inst=n)
a = fbgpu.Arena(0)
a.load(batch)
L = fbgpu.lib()
buf = (C.c_ulonglong * 24)()
a.run()
a.synchronize()
L.fb_debug_wide_prof(buf, 1)
cbuf = (C.c_ulonglong * 1024)()
L.fb_debug_cta_prof(cbuf, 1)
a.reset()
a.run()
a.synchronize()
ms = a.last_run_ms()
L.fb_debug_wide_prof(buf, 1)
names = ["owner combine+window+cands", "owner sort", "K2 select (later windows)", "cost gather", "K3 scan", "bookkeeping", "moves",
         "tail", "complete", "", "", "K3 prefix"]
tot = sum(buf[i] for i in (0, 1, 2, 3, 4, 5, 6, 7, 8, 11))
steps = buf[10]
print(f"{n} instances, {ms:.3f} ms, {steps} wide steps")
print(f"  windows per step {buf[20] / max(steps, 1):.3f}, fused window load {buf[21] / max(steps, 1) / 1965:.2f} us/step, sort: warp runs {buf[22] / max(steps, 1) / 1965:.2f} merges {buf[23] / max(steps, 1) / 1965:.2f} us/step")
print(f"  first iteration's advance (escalation) wall: {buf[23] / 1965:.1f} us")
print(f"  bin sort: {buf[16]} merge-sort fallbacks, mean rank work {buf[17] / max(steps, 1):.0f}, "
      f"mean window {buf[18] / max(steps, 1):.0f} keys, mean last bin {buf[19] / max(steps, 1):.0f}")
gnames = {12: "advance+barrier", 13: "grid K1+barrier", 14: "grid hist+barrier",
          15: "grid gather+barrier", 9: "owner finish (CTA 0)"}
gt = sum(buf[i] for i in gnames)
print(f"  grid iteration phases (CTA 0 clock), {gt / 1965e3:.3f} ms total:")
for i, nm in gnames.items():
    print(f"    {nm:22s} {100 * buf[i] / max(gt, 1):5.1f}%  {buf[i] / 1965:10.1f} us")
print("  owner-side phases (summed over owners, per step):")
for i, nm in enumerate(names):
    if not nm:
        continue
    print(f"  {nm:12s} {100 * buf[i] / max(tot, 1):5.1f}%  {buf[i] / max(steps, 1) / 1965:8.2f} us/step")

L.fb_debug_cta_prof(cbuf, 1)
import statistics
for k, nm in enumerate(("K1 busy", "hist busy", "gather busy", "owner advance busy")):
    v = [cbuf[c * 4 + k] / 1965.0 for c in range(148)]
    print(f"  per-CTA {nm:18s} mean {statistics.mean(v):9.1f} us  max {max(v):9.1f} us  min {min(v):9.1f} us")
