"""The ncu counters BASELINE.json:north_star names, per kernel of an `ncu --set full` report:
achieved DRAM and L2 bandwidth against the B200 peak, global-load/store sectors per request and
load/store efficiency (useful bytes per 32-B sector), shared-memory wavefront utilisation, L2 hit
rate.  CPU only (reads the report):

    python tools/ncu_evidence.py REPORT.ncu-rep [--out profiles/rNN/ncu_evidence_X.md] [--hbm-peak 6459.9]

L2 peak: lts__t_sectors.sum.peak_sustained (sectors/cycle) x 32 B x the measured L2 clock
(lts__cycles_elapsed.avg.per_second), i.e. the hardware's own peak for the run's clock.
"""
import argparse
import csv
import io
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def raw(report):
    out = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    kern = []
    for r in rows[2:]:
        kern.append({h: (v, u) for h, u, v in zip(hdr, units, r)})
    return kern


def num(d, k):
    try:
        v, u = d[k]
        return float(v.replace(",", "")), u
    except (KeyError, ValueError):
        return None, None


def scale(v, u, want):
    f = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "byte/second": 1, "Kbyte/second": 1e3, "Mbyte/second": 1e6, "Gbyte/second": 1e9, "Tbyte/second": 1e12,
         "us": 1e-6, "ms": 1e-3, "ns": 1e-9, "s": 1, "cycle/second": 1, "cycle/nsecond": 1e9, "cycle/usecond": 1e6,
         "hz": 1, "Khz": 1e3, "Mhz": 1e6, "Ghz": 1e9}
    return v * f.get(u, 1) / f.get(want, 1) if v is not None else None


def evidence(d, hbm_peak):
    e = {}
    t, tu = num(d, "gpu__time_duration.sum")
    e["duration_us"] = scale(t, tu, "us")
    rd, ru = num(d, "dram__bytes_read.sum")
    wr, wu = num(d, "dram__bytes_write.sum")
    rd, wr = scale(rd, ru, "byte"), scale(wr, wu, "byte")
    if rd is not None and wr is not None and t:
        e["dram_bytes"] = rd + wr
        e["dram_GBps"] = (rd + wr) / (e["duration_us"] * 1e-6) / 1e9
        e["dram_frac_of_measured_peak"] = e["dram_GBps"] / hbm_peak
    s, _ = num(d, "lts__t_sectors.sum")
    pk, _ = num(d, "lts__t_sectors.sum.peak_sustained")
    clk, cu = num(d, "lts__cycles_elapsed.avg.per_second")
    if s is not None and t:
        e["l2_GBps"] = s * 32 / (e["duration_us"] * 1e-6) / 1e9
        if pk and clk:
            e["l2_peak_GBps"] = pk * 32 * scale(clk, cu, "hz") / 1e9
            e["l2_frac_of_peak"] = e["l2_GBps"] / e["l2_peak_GBps"]
    pct, _ = num(d, "lts__t_sectors.sum.pct_of_peak_sustained_elapsed")
    e["l2_sectors_pct_of_peak_elapsed"] = pct
    if pct and "l2_GBps" in e and "l2_peak_GBps" not in e:
        e["l2_peak_GBps"] = e["l2_GBps"] / (pct / 100.0)   # the peak implied by the report's own %
        e["l2_frac_of_peak"] = pct / 100.0
    for op in ("ld", "st"):
        sec, _ = num(d, "l1tex__t_sectors_pipe_lsu_mem_global_op_%s.sum" % op)
        req, _ = num(d, "l1tex__t_requests_pipe_lsu_mem_global_op_%s.sum" % op)
        if sec is not None and req:
            e["global_%s_sectors_per_request" % op] = sec / req
        bps, _ = num(d, "smsp__sass_average_data_bytes_per_sector_mem_global_op_%s.ratio" % op)
        if bps is not None:
            e["global_%s_efficiency_pct" % op] = 100.0 * bps / 32.0
    for k, name in (("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "shared_wavefronts_pct_of_peak"),
                    ("lts__t_sector_op_read_hit_rate.pct", "l2_read_hit_rate_pct"),
                    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_pct"),
                    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_active_pct")):
        v, _ = num(d, k)
        e[name] = v
    return e


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--out")
    ap.add_argument("--hbm-peak", type=float, default=None)
    a = ap.parse_args()
    peak = a.hbm_peak
    if peak is None:
        try:
            peak = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
        except Exception:
            peak = 6650.0
    lines = ["# ncu evidence (BASELINE.json:north_star counters): `%s`" % os.path.basename(a.report), "",
             "HBM peak for the fraction: %.1f GB/s (MEASURED_PEAKS.json hbm_gbs). L2 peak: the report's own "
             "lts__t_sectors peak x 32 B x L2 clock." % peak, ""]
    for d in raw(a.report):
        name = d.get("Kernel Name", ("?", ""))[0]
        e = evidence(d, peak)
        lines.append("## `%s`" % name[:120])
        lines.append("")
        lines.append("| counter | value |")
        lines.append("|---|---|")
        for k, v in e.items():
            lines.append("| %s | %s |" % (k, "%.4g" % v if isinstance(v, float) else v))
        lines.append("")
    txt = "\n".join(lines) + "\n"
    if a.out:
        open(a.out, "w").write(txt)
    print(txt)


if __name__ == "__main__":
    main()
