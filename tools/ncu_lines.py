"""Per-CUDA-source-line stall samples / executed instructions of one kernel
from `ncu -i REP --page source --csv --print-source cuda,sass` (mixed mode).
usage: ncu_lines.py FILE.csv [N]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
fname, hdr, res = "?", None, []
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] == "" or r[0] == "Function Name":
        continue
    try:
        st = int(float(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0))
        ex = int(float(r[hdr.index("Instructions Executed")] or 0))
    except (ValueError, IndexError):
        continue
    if st or ex:
        res.append((st, ex, f"{fname}:{r[0]}", r[1].strip()[:90]))
tst = sum(x[0] for x in res) or 1
tex = sum(x[1] for x in res) or 1
print(f"stall samples {tst}  instructions {tex}")
for st, ex, loc, src in sorted(res, reverse=True)[:n]:
    print(f"st{100 * st / tst:5.1f}%  ex{100 * ex / tex:5.1f}%  {loc:26s} {src}")
