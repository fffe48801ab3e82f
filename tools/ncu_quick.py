"""Quick per-kernel digest of an .ncu-rep: key metrics + top stall reasons."""
import csv, io, subprocess, sys
rep = sys.argv[1]
d = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(d)))
h = r[0]
ki, mi, vi, ui = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
want = ("Duration", "DRAM Throughput", "Issue Slots Busy", "Executed Ipc Active", "L1/TEX Hit Rate", "L2 Hit Rate",
        "Registers Per Thread", "Achieved Occupancy", "Mem Busy")
info = {}
for x in r[1:]:
    if x[mi] in want:
        info.setdefault(x[ki], []).append(f"{x[mi]}={x[vi]}{x[ui]}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
h = r[0]
cols = [i for i, k in enumerate(h) if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued")]
for row in r[2:]:
    name = row[h.index("Kernel Name")]
    print("==", name[:70])
    print("   " + "  ".join(info.get(name, [])))
    extra = []
    for m in ("smsp__inst_executed.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
              "dram__bytes_read.sum", "dram__bytes_write.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"):
        if m in h:
            extra.append(f"{m.split('.')[0].replace('sm__pipe_','').replace('smsp__','')}={row[h.index(m)]}")
    print("   " + "  ".join(extra))
    items = []
    for i in cols:
        try:
            items.append((float(row[i].replace(",", "")), h[i].replace("smsp__pcsamp_warps_issue_stalled_", "")))
        except ValueError:
            pass
    t = sum(v for v, k in items) or 1
    print("   stalls: " + "  ".join("%s %.0f%%" % (k, 100 * v / t) for v, k in sorted(items, reverse=True)[:8]))
