"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per
kernel: launches, total ms, ms per step, share of the hot path.
Usage: python tools/launch_summary.py launches.csv steps out.md [title]"""
import collections
import csv
import sys

path, steps, out = sys.argv[1], int(sys.argv[2]), sys.argv[3]
title = sys.argv[4] if len(sys.argv) > 4 else path
rows = list(csv.reader(open(path)))
hdr = [r for r in rows if len(r) > 5 and r[0] == "ID"][0]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
tot = collections.defaultdict(float)
cnt = collections.Counter()
for r in rows:
    if len(r) != len(hdr) or r[0] == "ID":
        continue
    name = r[ki].split("(")[0].replace("void ", "").split("::")[-1]
    scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0}.get(r[ui], 1e-6)
    tot[name] += float(r[vi].replace(",", "")) * scale
    cnt[name] += 1
setup = {"k_cloud_pack", "k_cloud_pack_batch"}
hot = sum(v for k, v in tot.items() if k not in setup)
lines = [f"# {title}", "", "| kernel | launches | total ms | ms / step | share of hot path |",
         "|---|---|---|---|---|"]
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    share = "(setup)" if k in setup else f"{100 * v / hot:.1f}%"
    lines.append(f"| {k} | {cnt[k]} | {v:.2f} | {v / steps:.2f} | {share} |")
lines.append(f"| **hot path (excl. setup)** | | {hot:.2f} | {hot / steps:.2f} | 100% |")
open(out, "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
