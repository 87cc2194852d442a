#!/usr/bin/env python
"""Summarise an `ncu --set full` report (and optionally an ncu launch list) for profiles/.

    python tools/ncu_summary.py REPORT.ncu-rep --workload c4_multistripe_1GiB \
        [--launches launches.csv] [--out profiles/rNN/ncu_summary.md] [--traffic-json profiles/ncu_traffic.json]

Writes a markdown table of the metrics DESIGN.md cites (DRAM bytes, L2 sectors, shared-memory
wavefronts and bank conflicts, issue activity, stall reasons) and records the per-launch DRAM
traffic (dram__bytes_read.sum + dram__bytes_write.sum) that bench.py reports as
roofline.traffic.
"""
import argparse
import csv
import io
import json
import os
import subprocess

KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_bytes.sum",
    "lts__t_sectors_srcunit_tex_op_read.sum",
    "lts__t_sectors_srcunit_tex_op_write.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
    "smsp__inst_executed.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "launch__shared_mem_per_block_dynamic",
    "smsp__sass_average_data_bytes_per_sector_mem_global_op_ld.pct",
]
STALLS = "smsp__average_warps_issue_stalled_"


def raw(report):
    out = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head, units = rows[0], rows[1]
    kernels = []
    for r in rows[2:]:
        kernels.append({h: (v, u) for h, u, v in zip(head, units, r)})
    return kernels


def to_bytes(v, u):
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    return float(v.replace(",", "")) * mult.get(u, 1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--workload", required=True)
    ap.add_argument("--launches")
    ap.add_argument("--out")
    ap.add_argument("--traffic-json")
    a = ap.parse_args()
    ks = raw(a.report)
    lines = ["# ncu summary: %s (%s)" % (a.workload, os.path.basename(a.report)), ""]
    traffic = None
    for k in ks:
        name = k.get("Kernel Name", ("?", ""))[0]
        lines += ["## `%s`" % name, "", "| metric | unit | value |", "|---|---|---|"]
        for key in KEYS:
            if key in k:
                v, u = k[key]
                lines.append("| %s | %s | %s |" % (key, u, v))
        st = sorted(((float(v.replace(",", "") or 0), h[len(STALLS):]) for h, (v, u) in k.items()
                     if h.startswith(STALLS) and h.endswith("_per_issue_active.ratio")), reverse=True)
        lines += ["", "Top stall reasons (warps per issue):", ""]
        lines += ["- %s: %.3f" % (n.replace("_per_issue_active.ratio", ""), v) for v, n in st[:8]]
        lines.append("")
        if "dram__bytes_read.sum" in k:
            rb = to_bytes(*k["dram__bytes_read.sum"])
            wb = to_bytes(*k["dram__bytes_write.sum"])
            traffic = rb + wb
            lines.append("DRAM traffic per launch: %.0f B (read %.0f + write %.0f)" % (traffic, rb, wb))
            lines.append("")
    if a.launches:
        per = {}
        with open(a.launches) as f:
            rdr = csv.reader(l for l in f if l.startswith('"'))
            head = next(rdr)
            ki, vi = head.index("Kernel Name"), head.index("Metric Value")
            for r in rdr:
                per.setdefault(r[ki].split("(")[0], []).append(float(r[vi].replace(",", "")))
        tot = sum(sum(v) for v in per.values())
        lines += ["## Launch list (`gpu__time_duration.sum`, cold-cache, serialised)", "",
                  "| kernel | launches | mean µs | share |", "|---|---|---|---|"]
        for n, v in sorted(per.items(), key=lambda x: -sum(x[1])):
            lines.append("| `%s` | %d | %.1f | %.1f%% |" % (n[:90], len(v), sum(v) / len(v) / 1e3,
                                                          100 * sum(v) / tot))
        lines.append("")
    text = "\n".join(lines)
    if a.out:
        with open(a.out, "w") as f:
            f.write(text)
    print(text)
    if a.traffic_json and traffic is not None:
        d = {}
        if os.path.exists(a.traffic_json):
            d = json.load(open(a.traffic_json))
        d[a.workload] = {"dram_bytes_per_launch": int(traffic), "report": os.path.basename(a.report)}
        with open(a.traffic_json, "w") as f:
            json.dump(d, f, indent=1)


if __name__ == "__main__":
    main()
