"""Summarise an ncu report (+ optional launch-list CSV) into profiles/.

usage: python tools/ncu_summary.py REPORT.ncu-rep OUT_PREFIX [--launches CSV] [--stage-map k=v,...]
Writes OUT_PREFIX.md (human summary) and merges per-kernel DRAM traffic into
profiles/traffic.json keyed by bench stage name (dct_2d.stage0, ...)."""
import argparse, collections, csv, io, json, os, subprocess

M = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
     "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
     "launch__registers_per_thread", "launch__block_size", "launch__grid_size",
     "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
     "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
     "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
     "launch__occupancy_limit_shared_mem", "launch__shared_mem_per_block_dynamic"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"name": r[hdr.index("Kernel Name")]}
        for m in M:
            if m in hdr:
                d[m] = (r[hdr.index(m)], units[hdr.index(m)])
        res.append(d)
    return res


def to_bytes(v, u):
    f = float(v.replace(",", ""))
    return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("out")
    ap.add_argument("--launches")
    ap.add_argument("--stage-map", default="")
    ap.add_argument("--title", default="")
    ap.add_argument("--traffic-prefix", default="", help="key prefix in profiles/traffic.json, e.g. c2:float64:")
    a = ap.parse_args()
    ks = raw(a.report)
    smap = dict(kv.split("=", 1) for kv in a.stage_map.split(";") if kv)
    lines = [f"# ncu summary {a.title}", "", f"report: `{os.path.basename(a.report)}` (ncu --set full --clock-control none)", ""]
    lines.append("| kernel | us | DRAM rd MB | DRAM wr MB | DRAM % | SM % | issue % | FP64 pipe % | regs | block | grid | smem KB | warps act % | smem bank confl |")
    lines.append("|---|---|---|---|---|---|---|---|---|---|---|---|---|---|")
    traffic = {}
    for i, k in enumerate(ks):
        g = lambda m: k.get(m, ("", ""))[0]
        rd = to_bytes(*k["dram__bytes_read.sum"]) if "dram__bytes_read.sum" in k else 0
        wr = to_bytes(*k["dram__bytes_write.sum"]) if "dram__bytes_write.sum" in k else 0
        nm = k["name"][:70]
        lines.append(f"| `{nm}` | {g('gpu__time_duration.sum')} | {rd/1e6:.1f} | {wr/1e6:.1f} | "
                     f"{g('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed')} | "
                     f"{g('sm__throughput.avg.pct_of_peak_sustained_elapsed')} | {g('smsp__issue_active.avg.pct_of_peak_sustained_active')} | "
                     f"{g('sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active')} | "
                     f"{g('launch__registers_per_thread')} | {g('launch__block_size')} | {g('launch__grid_size')} | "
                     f"{float(g('launch__shared_mem_per_block_dynamic') or 0)/1024:.0f} | "
                     f"{g('sm__warps_active.avg.pct_of_peak_sustained_active')} | {g('l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum')} |")
        if i < len(smap):  # stage-map entries name the captured launches in order
            traffic[a.traffic_prefix + list(smap)[i]] = rd + wr
    if a.launches:
        lines += ["", "## launch list (gpu__time_duration.sum, cold-cache, serialised)", ""]
        rows = list(csv.reader(open(a.launches)))
        hdr = None
        tot = collections.Counter()
        order = []
        for r in rows:
            if "Kernel Name" in r:
                hdr = r
                continue
            if hdr and len(r) == len(hdr):
                d = dict(zip(hdr, r))
                if d.get("Metric Name") == "gpu__time_duration.sum":
                    n = d["Kernel Name"].split("(")[0][:60]
                    v = float(d["Metric Value"].replace(",", "")) / (1e3 if d["Metric Unit"] == "ns" else 1)
                    tot[n] += v
                    order.append((n, v))
        s = sum(tot.values())
        lines.append("| kernel | total us | share |")
        lines.append("|---|---|---|")
        for n, v in tot.most_common():
            lines.append(f"| `{n}` | {v:.1f} | {v/s*100:.1f}% |")
    open(a.out + ".md", "w").write("\n".join(lines) + "\n")
    if traffic:
        tp = os.path.join(os.path.dirname(a.out) or ".", "traffic.json")
        cur = json.load(open(tp)) if os.path.exists(tp) else {}
        cur.update(traffic)
        json.dump(cur, open(tp, "w"), indent=1)
    print(open(a.out + ".md").read())


if __name__ == "__main__":
    main()
