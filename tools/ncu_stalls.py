"""Warp-stall samples per CUDA source line and per SASS instruction, by stall
reason, from the source page of an ncu report captured with --import-source on
(ncu -i rep --page source --csv --print-source cuda,sass, optionally gzipped).
Usage: python tools/ncu_stalls.py src.csv[.gz] [top] [reason ...]
       (reasons: long_sb short_sb wait lg mio math not_selected selected ...;
        default: every reason, lines ranked by all samples)"""
import csv
import gzip
import io
import sys
from collections import defaultdict

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
want = sys.argv[3:]
op = gzip.open if path.endswith(".gz") else open
with op(path, "rt") as f:
    rows = list(csv.reader(io.StringIO(f.read())))

hdr, fname = None, ""
lines, sass = {}, []
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].rsplit("/", 1)[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        idx = {h: i for i, h in enumerate(r)}
        stall_cols = [h for h in r if h.startswith("stall_") and "Not Issued" not in h]
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    rec = {}
    for h in stall_cols:
        v = r[idx[h]]
        rec[h[6:]] = float(v) if v not in ("", "-") else 0.0
    tot = sum(rec.values())
    if r[0]:  # a source line (aggregate of its SASS)
        lines[(fname, int(r[0]))] = (r[1].strip()[:90], rec, tot)
    elif r[2] not in ("", "..."):
        sass.append((fname, r[3].strip()[:70], rec, tot))


def score(rec, tot):
    return sum(rec.get(w, 0.0) for w in want) if want else tot


grand = sum(t for _, _, t in lines.values()) or 1.0
by = defaultdict(float)
for _, rec, _ in lines.values():
    for k, v in rec.items():
        by[k] += v
print("all samples", int(grand), " by reason:",
      ", ".join(f"{k} {v / grand:.3f}" for k, v in sorted(by.items(), key=lambda x: -x[1]) if v / grand > 0.005))
print(f"\ntop source lines by {'+'.join(want) if want else 'all samples'}:")
for (fn, ln), (src, rec, tot) in sorted(lines.items(), key=lambda x: -score(x[1][1], x[1][2]))[:top]:
    parts = ", ".join(f"{k} {v / tot:.2f}" for k, v in sorted(rec.items(), key=lambda x: -x[1])[:4] if tot)
    print(f"{score(rec, tot) / grand:6.3f}  {fn}:{ln}  {src}\n        [{parts}]")
print(f"\ntop SASS instructions by {'+'.join(want) if want else 'all samples'}:")
for fn, ins, rec, tot in sorted(sass, key=lambda x: -score(x[2], x[3]))[:top]:
    parts = ", ".join(f"{k} {v / tot:.2f}" for k, v in sorted(rec.items(), key=lambda x: -x[1])[:3] if tot)
    print(f"{score(rec, tot) / grand:6.3f}  {ins}  [{parts}]")
