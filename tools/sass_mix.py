"""Aggregate an ncu --page source --csv (SASS view) by opcode: executed
instructions and warp-stall samples. usage: python tools/sass_mix.py FILE.csv"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
si, ei, wi = h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
ex, st = collections.Counter(), collections.Counter()
for r in rows[2:]:
    if len(r) <= ei:
        continue
    op = r[si].strip().split()
    if not op:
        continue
    o = op[0]
    if o.startswith("@"):
        o = op[1] if len(op) > 1 else o
    o = o.split(".")[0]
    try:
        ex[o] += int(float(r[ei] or 0))
        st[o] += int(float(r[wi] or 0))
    except ValueError:
        pass
tot, tst = sum(ex.values()), sum(st.values())
print(f"total executed {tot}, stall samples {tst}")
for o, v in ex.most_common(25):
    print(f"{o:10s} {v:10d} {100 * v / tot:5.1f}%   stalls {100 * st[o] / max(tst, 1):5.1f}%")
