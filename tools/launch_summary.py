"""Per-kernel shares of a step from an ncu launch list
(ncu --metrics gpu__time_duration.sum --csv --log-file F <cmd>):
    python tools/launch_summary.py F [title]  > profiles/rNN_launches_C2.md"""
import collections
import csv
import io
import sys

txt = open(sys.argv[1]).read()
lines = [l for l in txt.splitlines() if l.startswith('"')]
rows = list(csv.reader(io.StringIO("\n".join(lines))))
h = rows[0]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
d = collections.OrderedDict()
for r in rows[1:]:
    name = r[ki].split("(")[0].replace("snapgpu::", "")
    d.setdefault(name, []).append(float(r[vi].replace(",", "")) / 1e3)
ours = {k: v for k, v in d.items() if k.startswith(("void k_", "k_"))}  # (not torch's)
step = ("k_compute_U", "k_compute_Y", "k_fused_dE", "k_gather")
tot = sum(sum(v) / len(v) for k, v in ours.items() if any(s in k for s in step))
title = sys.argv[2] if len(sys.argv) > 2 else sys.argv[1]
print(f"# launch list: {title}\n")
print("`ncu --metrics gpu__time_duration.sum --clock-control none` (cold, serialised:"
      " compare shares, not absolutes).\n")
print("| kernel | launches | mean µs | share of the step's kernel time |")
print("|---|---|---|---|")
for k, v in d.items():
    m = sum(v) / len(v)
    share = f"{100 * m / tot:.1f} %" if any(s in k for s in step) and k in ours else "-"
    print(f"| `{k}` | {len(v)} | {m:.2f} | {share} |")
