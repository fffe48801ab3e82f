"""Per-CUDA-source-line executed instructions / stall samples from
`ncu --page source --csv --print-source cuda,sass`. usage: src_lines.py FILE.csv [N]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
fname, res, hdr = "?", [], None
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r or r[0] == "":
        continue
    try:
        ex = int(float(r[hdr.index("Instructions Executed")] or 0))
        st = int(float(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0))
    except (ValueError, IndexError):
        continue
    if ex or st:
        res.append((ex, st, f"{fname}:{r[0]}", r[1].strip()[:100]))
tot = sum(x[0] for x in res) or 1
tst = sum(x[1] for x in res) or 1
print(f"total inst {tot}  stall samples {tst}")
for ex, st, loc, src in sorted(res, reverse=True)[:n]:
    print(f"{100 * ex / tot:5.1f}% st{100 * st / tst:5.1f}%  {loc:24s} {src}")
