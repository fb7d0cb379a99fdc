"""Write profiles/<tag>_*.{md,json} from an ncu --set full report and a launch list.

    python tools/ncu_summary.py TAG REPORT.ncu-rep [LAUNCHES.csv] [WORKLOAD]
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = [
    "gpu__time_duration.sum", "launch__grid_size", "launch__block_size",
    "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
    "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__inst_executed.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "l1tex__t_sector_hit_rate.pct", "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
]


def stall_top(report, n=8):
    """Top warp-stall reasons (pc sampling) of the first kernel in the report."""
    out = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, r = rows[0], rows[2]
    pre = "smsp__pcsamp_warps_issue_stalled_"
    vals = []
    for i, h in enumerate(hdr):
        if h.startswith(pre) and not h.endswith("_not_issued"):
            try:
                vals.append((float(r[i].replace(",", "")), h[len(pre):]))
            except ValueError:
                pass
    tot = sum(v for v, _ in vals) or 1.0
    return [(k, v / tot * 100) for v, k in sorted(vals, reverse=True)[:n]]


def clocks(path):
    """nvidia-smi samples taken while ncu ran: SM clock under load, reasons."""
    rows = list(csv.reader(open(path)))[1:]
    load = [r for r in rows if len(r) > 6 and r[1].strip().split()[0].isdigit()
            and int(r[1].strip().split()[0]) > 500]
    if not load:
        return None
    sm = sorted(int(r[1].strip().split()[0]) for r in load)
    mx = max(int(r[2].strip().split()[0]) for r in load)
    reasons = sorted({r[6].strip() for r in load})
    return {"samples_under_load": len(load), "sm_mhz_median": sm[len(sm) // 2],
            "sm_mhz_min": sm[0], "sm_max_mhz": mx, "reason_masks": reasons}


def raw(report):
    out = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {}
        for m in METRICS:
            if m in hdr:
                i = hdr.index(m)
                d[m] = (r[i], units[i])
        d["Kernel Name"] = r[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        res.append(d)
    return res


def to_bytes(v, u):
    x = float(v.replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
    return x * scale


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, mi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
    tot = {}
    for r in rows[hi + 1:]:
        if len(r) > vi and r[mi] == "gpu__time_duration.sum":
            name = r[ki]
            short = name.split("(")[0].replace("void ", "")
            short = short.split("::")[-1] if "::" in short else short
            tot.setdefault(short, [0.0, 0])
            tot[short][0] += float(r[vi].replace(",", ""))
            tot[short][1] += 1
    return tot


def main():
    tag, report = sys.argv[1], sys.argv[2]
    lpath = sys.argv[3] if len(sys.argv) > 3 and sys.argv[3] else None
    workload = sys.argv[4] if len(sys.argv) > 4 else "C2"
    prof = raw(report)
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    md = [f"# ncu summary `{tag}` ({workload})", "",
          f"Source: `ncu --set full --import-source on --clock-control none` on one warm "
          f"resident solve (tools/profile_one.py {workload}); kernel = persistent dataflow "
          "level kernel (all DP levels in one cooperative launch).", ""]
    for d in prof:
        md.append(f"## {d['Kernel Name'][:140]}")
        md.append("")
        md.append("| metric | value | unit |")
        md.append("|---|---|---|")
        for m in METRICS:
            if m in d:
                md.append(f"| {m} | {d[m][0]} | {d[m][1]} |")
        md.append("")
    if prof:
        d = prof[0]
        traffic = to_bytes(*d["dram__bytes_read.sum"]) + to_bytes(*d["dram__bytes_write.sum"])
        tj = os.path.join(ROOT, "profiles", "traffic.json")
        data = json.load(open(tj)) if os.path.exists(tj) else {}
        data[workload] = traffic
        json.dump(data, open(tj, "w"), indent=1)
        mj = os.path.join(ROOT, "profiles", "ncu_metrics.json")
        mdata = json.load(open(mj)) if os.path.exists(mj) else {}

        def num(m):
            return float(d[m][0].replace(",", "")) if m in d else None

        mdata[workload] = {
            "kernel_ms": num("gpu__time_duration.sum"),
            "issue_active_pct": num("smsp__issue_active.avg.pct_of_peak_sustained_active"),
            "alu_pipe_pct": num("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"),
            "warps_active_pct": num("sm__warps_active.avg.pct_of_peak_sustained_active"),
            "dram_throughput_pct": num("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
            "l2_throughput_pct": num("lts__throughput.avg.pct_of_peak_sustained_elapsed"),
            "l1_hit_pct": num("l1tex__t_sector_hit_rate.pct"),
            "warp_instructions": num("smsp__inst_executed.sum"),
            "registers": num("launch__registers_per_thread"),
            "source": f"profiles/{tag}_ncu.md",
        }
        json.dump(mdata, open(mj, "w"), indent=1)
        md.append(f"DRAM traffic per launch (read + write): **{traffic / 1e6:.2f} MB**.")
        md.append("")
    if prof:
        md += ["## Warp stall reasons (pc sampling, share of samples)", "",
               "| reason | share |", "|---|---|"]
        for k, v in stall_top(report):
            md.append(f"| {k} | {v:.1f}% |")
        md.append("")
    cpath = report.replace(".ncu-rep", "_clocks.csv")
    if os.path.exists(cpath):
        c = clocks(cpath)
        md += ["## Clock record (nvidia-smi every 200 ms while ncu ran; --clock-control none)", "",
               f"`{json.dumps(c)}`", ""]
    if lpath:
        tot = launches(lpath)
        s = sum(v[0] for v in tot.values())
        md += ["## Launch list (ncu gpu__time_duration, cold-cache, serialised)", "",
               "| kernel | launches | total ms | share |", "|---|---|---|---|"]
        for k, v in sorted(tot.items(), key=lambda x: -x[1][0]):
            md.append(f"| {k} | {v[1]} | {v[0] / 1e6:.3f} | {v[0] / s * 100:.1f}% |")
        md.append("")
    open(os.path.join(ROOT, "profiles", f"{tag}_ncu.md"), "w").write("\n".join(md))
    print("\n".join(md))


if __name__ == "__main__":
    main()
