"""Executed-instruction histogram by opcode from an ncu report's source page.
Usage: python tools/sass_hist.py report.ncu-rep kernel_regex [per_unit_count]"""
import csv
import io
import subprocess
import sys
from collections import Counter

rep, kern = sys.argv[1], sys.argv[2]
unit = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "-k", f"regex:{kern}"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ia, isrc, iex = hdr.index("Address"), hdr.index("Source"), hdr.index("Instructions Executed")
ist = hdr.index("Warp Stall Sampling (All Samples)")
c, st = Counter(), Counter()
tot = 0
for r in rows[2:]:
    if len(r) <= iex:
        continue
    s = r[isrc].strip()
    toks = s.split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith("@") else toks[0]
    op = op.split(".")[0]
    try:
        n = int(r[iex] or 0)
    except ValueError:
        continue
    c[op] += n
    st[op] += int(r[ist] or 0)
    tot += n
print(f"total warp instructions {tot}  per unit {tot / unit:.2f}")
for op, n in c.most_common(40):
    print(f"{op:10s} {n:14d} {n / unit:8.3f} {100 * n / tot:6.2f}%  stall samples {st[op]}")
