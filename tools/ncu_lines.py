"""Executed warp instructions per CUDA source line (and the SASS under it) from
an ncu report captured with --import-source on.
Usage: python tools/ncu_lines.py rep kernel_regex [unit] [top]"""
import csv
import io
import subprocess
import sys
from collections import Counter

rep, kern = sys.argv[1], sys.argv[2]
unit = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
top = int(sys.argv[4]) if len(sys.argv) > 4 else 60
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "-k", f"regex:{kern}"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
cur, hdr = None, None
line_n, line_s, line_src, line_ops = Counter(), Counter(), {}, {}
key = None
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        cur, hdr = r[1].split("/")[-1], None
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if not hdr or len(r) != len(hdr):
        continue
    if r[0] not in ("", "-"):  # a CUDA source line row: its own totals
        key = (cur, int(r[0]))
        line_src[key] = r[1].strip()[:100]
        n = int(r[7]) if r[7] not in ("", "-") else 0
        line_n[key] += n
        line_s[key] += int(r[4]) if r[4] not in ("", "-") else 0
        continue
    if key is None or r[7] in ("", "-"):
        continue
    toks = r[3].split()
    if toks:
        op = (toks[1] if toks[0].startswith("@") else toks[0]).split(".")[0]
        line_ops.setdefault(key, Counter())[op] += int(r[7])
tot = sum(line_n.values())
print(f"total {tot / unit:.3f} per unit")
for k, n in line_n.most_common(top):
    ops = " ".join(f"{o}:{c / unit:.2f}" for o, c in line_ops.get(k, Counter()).most_common(6))
    print(f"{n / unit:7.3f} st{line_s[k]:6d} {k[0]}:{k[1]} {line_src.get(k, '')[:70]}\n        {ops}")
