#!/usr/bin/env python
"""Benchmark of the Founsure encode hot path on B200 (BASELINE.json metric: encode throughput,
source GB/s, % of HBM roofline).

Workload: BASELINE config 4 -- 1 GiB of seeded uniform bytes split into 256
independent stripes of k=1024 x t=4096 B, precode p=16 checks of degree 3, n=1280 coded symbols
with RSD(c=0.1, delta=0.05).  One step = one pass of the whole hot path (precode + LT over every
stripe of the rank's shard) = one fs_encode_stripes call.  `--scaling strong` (default) shards the
256 stripes over the ranks as BASELINE config 4 states; `--scaling weak` gives every rank its own
1 GiB.  `--config 5` (one 410 MB stripe) partitions the coded rows over the ranks with the source
replicated (reading R16); other configs run on one GPU.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 4] [--impl ours|reference]

N > 1 runs under torchrun (one process per GPU, NCCL): the graph is generated on rank 0 and
broadcast over NCCL (paper_1702_07409_b200/dist.py), work is sharded with no data-path
collective, and the time is the max over ranks of the CUDA-event time of K steps.  Rank 0 prints
one JSON line.
"""
import argparse
import json
import os
import platform
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1702_07409_b200 import configs, dist as fdist, fsb, inputs  # noqa: E402

METRIC = "encode throughput, source GB/s (1/2/4/8 B200), % of HBM roofline"
DATA = "synthetic: seeded counter-form splitmix64 bytes (DESIGN.md R4), graph seed = data seed (R3)"
# Shared-memory gather peak for the secondary (gather-traffic) roofline: parity-paired 64-B row
# gathers, 122 B/clk/SM at 1965 MHz x 148 SMs (tools/microbench/mb3.cu, profiles/r01b/).
SMEM_GATHER_PEAK_GBS = 35595.0
# L2-resident random 512-B row gathers from global memory (the GLOBAL variant's gathers hit L2):
# 66.9 B/clk/SM at 1965 MHz x 148 SMs (tools/microbench/mb7.cu, profiles/r01e/mb7.txt).
L2_GATHER_PEAK_GBS = 19500.0
# The paper's own CPU numbers (context only, another machine): PAPER.md:452-475 (Table 1, encode)
# and PAPER.md:486-489 (Table 2, decode), 2x Intel Xeon E5-2620 (12 threads), 64 MiB test file.
PAPER_CONTEXT = {
    "source": "PAPER.md:452-489 (§4, Tables 1-2); another machine, context only",
    "hardware": "2x Intel Xeon E5-2620 (12 cores / 12 threads used), 2012-era",
    "encode_MBps_best": 2722, "decode_MBps_best": 1691,
    "note": "the paper's library, its own PRNG/graphs and a 64 MiB file: not the same workload",
}
REASONS = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")


def _peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            m = json.load(f)
        return float(m["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def _host_cpu():
    model = platform.processor() or ""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "model": model}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        q = "clocks.sm,clocks.max.sm," + ",".join("clocks_event_reasons." + r for r in REASONS)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), "--query-gpu=" + q, "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.thread.join(timeout=2)
        sm, smax, reasons = [], [], set()
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 2 + len(REASONS):
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for r, v in zip(REASONS, parts[2:]):
                if v.lower().startswith("active"):
                    reasons.add(r)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(smax), "reasons": sorted(reasons),
                "samples": len(sm)}


def _dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


L2_BYTES = 126 * 1024 * 1024
COLL_DEV = "cpu"  # device of the bench's collectives (set in main: the rank's GPU under NCCL)


def plan(cfg, ws, rank, scaling, partition="rows"):
    """This rank's work: ("stripes", first stripe, count), ("rows", row_begin, row_end) or
    ("cols", col_begin, col_end) -- the last two split one large stripe (R16 / NEXT-4)."""
    S_total = cfg["stripes"]
    if S_total == 1 and ws > 1:
        if partition == "cols":
            c0, c1 = fdist.col_shard(cfg["t"], ws, rank)
            return "cols", c0, c1
        r0, r1 = fdist.shard(cfg["n"], ws, rank)
        return "rows", r0, r1
    if scaling == "weak":
        return "stripes", rank * S_total, S_total
    a, b = fdist.shard(S_total, ws, rank)
    return "stripes", a, b - a


def workload_config(cfg, args, ws, kind, S, u0, u1, lt_nnz, max_degree):
    """The `config` object of a bench line; the GPU arm and the reference arm emit the same one."""
    k, p, n, t = cfg["k"], cfg["p"], cfg["n"], cfg["t"]
    rows = n if kind != "rows" else u1 - u0
    cols = u1 - u0 if kind == "cols" else t
    work_bytes = S * (k + p + rows) * cols
    flush = work_bytes < 2 * L2_BYTES
    return {"workload": cfg["name"], "k": k, "p": p, "d_p": cfg["d_p"], "n": n, "t": t,
            "dist": "RSD" if cfg["dist"] == configs.RSD else "Omega",
            "stripes_total": cfg["stripes"] * (ws if args.scaling == "weak" and kind == "stripes" else 1),
            "per_rank": {"stripes": "%d stripes" % S, "rows": "rows [%d,%d)" % (u0, u1),
                         "cols": "bytes [%d,%d)" % (u0, u1)}[kind],
            "parallelism": {"stripes": "stripe-sharded x%d" % ws,
                            "rows": "coded-row partition x%d, source replicated" % ws,
                            "cols": "byte-column partition x%d, nothing replicated" % ws}[kind],
            "variant": args.variant,
            "l2": ("working set %.1f MB per rank < 2x the 126 MB L2: a 252 MiB scratch write "
                   "before each timed step (excluded), steps timed one by one" % (work_bytes / 1e6))
                  if flush else
                  ("working set (%.2f GB per rank) exceeds the 126 MB L2; steps back to back, no flush"
                   % (work_bytes / 1e9)),
            "lt_nnz": int(lt_nnz), "max_degree": int(max_degree)}


def cpu_oracle_sample(cfg, seconds, max_stripes=None):
    """The oracle, as it stands (single-threaded C), on a bounded sample of the workload:
    whole stripes of the config until `seconds` of CPU work (at least one)."""
    import oracle
    go = oracle.generate_graph(cfg)
    S = cfg["stripes"] if max_stripes is None else max_stripes
    done, t_enc = 0, 0.0
    while done < S and (t_enc < seconds or done == 0):
        D = inputs.stripe_data(cfg, stripe_begin=done, num_stripes=1).numpy()
        t0 = time.perf_counter()
        oracle.encode(go, D[0])
        t_enc += time.perf_counter() - t0
        done += 1
    src = done * cfg["k"] * cfg["t"]
    host = _host_cpu()
    return {"value": src / t_enc / 1e9, "unit": "GB/s", "cores": 1, "kind": "oracle",
            "host_cpu": host["model"], "host_nproc": host["nproc"],
            "sample": "%d of %d stripes of %s (%.1f MB source), single-threaded C oracle, %.2f s"
                      % (done, S, cfg["name"], src / 1e6, t_enc)}


def cpu_oracle_sample_mt(cfg, seconds):
    """the same oracle, stripe-parallel over the host's cores (one stripe per
    task, ctypes releases the GIL), mirroring the paper's multi-threaded encoder.
    Context only; `cpu_baseline` stays the single-threaded oracle."""
    import concurrent.futures as cf
    import oracle
    go = oracle.generate_graph(cfg)
    nthreads = os.cpu_count() or 1
    S = cfg["stripes"]
    D = None
    done, t_enc = 0, 0.0
    with cf.ThreadPoolExecutor(nthreads) as ex:
        while done < S and (t_enc < seconds or done == 0):
            batch = min(nthreads, S - done)
            D = inputs.stripe_data(cfg, stripe_begin=done, num_stripes=batch).numpy()
            t0 = time.perf_counter()
            list(ex.map(lambda i: oracle.encode(go, D[i]), range(batch)))
            t_enc += time.perf_counter() - t0
            done += batch
    src = done * cfg["k"] * cfg["t"]
    return {"value": src / t_enc / 1e9, "unit": "GB/s", "cores": nthreads, "kind": "oracle, stripe-parallel",
            "sample": "%d of %d stripes, %d threads, %.2f s" % (done, S, nthreads, t_enc)}


def _reference_config(args, cfg, ws):
    """The GPU arm's config object for the same launch (rank 0's share at this world size)."""
    import numpy as np
    import oracle
    go = oracle.generate_graph(cfg)
    kind, u0, u1 = plan(cfg, ws, 0, args.scaling, args.partition)
    S = u1 if kind == "stripes" else 1
    return workload_config(cfg, args, ws, kind, S, u0, u1, go.nnz, int(np.diff(go.lt_row_ptr).max()))


def run_reference(args, cfg):
    """Reference arm for this tier: the CPU oracle timed as it stands on the host cores, on the
    same config, metric and unit; rank 0 only, the whole run bounded by --ref-seconds."""
    ws, rank, _ = _dist_env()
    if rank != 0:
        return
    steps, warm = args.steps, args.warmup
    per_step = args.ref_seconds / max(1, steps)
    for _ in range(warm):
        cpu_oracle_sample(cfg, 0.0, max_stripes=1)
    vals, secs = [], []
    for _ in range(steps):
        t0 = time.perf_counter()
        vals.append(cpu_oracle_sample(cfg, per_step))
        secs.append(time.perf_counter() - t0)
    v = statistics.median(x["value"] for x in vals)
    cb = dict(vals[0])
    cb["value"] = v
    cb["sample"] = "per step: " + vals[0]["sample"]
    out = {"impl": "reference", "metric": METRIC, "value": v, "unit": "GB/s", "n_gpus": args.gpus,
           "steps": steps, "warmup": warm, "ms_per_step": round(1e3 * statistics.median(secs), 3),
           "higher_is_better": True, "scaling": args.scaling,
           "vs_baseline": None, "dtype": "u8", "data": DATA,
           "config": _reference_config(args, cfg, ws),
           "cpu_baseline": cb, "context": PAPER_CONTEXT,
           "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--scaling", default="strong", choices=["weak", "strong"])
    ap.add_argument("--variant", default="auto", choices=["auto", "smem", "global"])
    ap.add_argument("--partition", default="rows", choices=["rows", "cols"],
                    help="single-stripe configs at N>1: split coded rows (source replicated, BASELINE "
                         "config 5) or byte columns (fs_encode_range, nothing replicated)")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--e2e-chunks", type=int, default=0,
                    help="e2e: chunks per step (0: the library's default for --e2e-api host, 16 for stripes)")
    ap.add_argument("--graph-replay", type=int, default=0,
                    help="also time N steps captured in one CUDA graph (small configs, warm L2)")
    ap.add_argument("--e2e-streams", type=int, default=2, help="e2e: copy/compute streams")
    ap.add_argument("--e2e-api", choices=["host", "stripes"], default="host",
                    help="e2e through fs_encode_host (library staging) or fs_encode_stripes on "
                         "bench-managed staging")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--ref-seconds", type=float, default=60.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--op", default="encode", choices=["encode", "decode", "repair", "update"],
                    help="decode: time fs_decode (Alg 5 DPG plan, NEXT-1); repair: fs_repair of "
                         "--erase-frac erased coded symbols; update: fs_repair of one extra output "
                         "file from the original check data (NEXT-3)")
    ap.add_argument("--erase-frac", type=float, default=0.01,
                    help="repair: fraction of coded symbols erased (seeded random subset)")
    ap.add_argument("--eliminate", action="store_true",
                    help="decode: finish with GF(2) elimination of the residual (FS_DECODE_ELIMINATE)")
    ap.add_argument("--recv-frac", type=float, default=0.95,
                    help="decode: fraction of coded symbols received (seeded random subset)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.op == "decode" and "--config" not in sys.argv:
        args.config = 5
    if args.op in ("repair", "update") and "--config" not in sys.argv:
        args.config = 7
    cfg = configs.get(args.config)
    if args.op != "encode" and _dist_env()[1] != 0:
        return  # the decode / repair / update lines are single-GPU: rank 0 runs them
    if args.op == "decode":
        if args.impl == "reference":
            print(json.dumps({"impl": "reference", "unavailable": "decode reference arm not implemented"}))
            return
        run_decode(args, cfg)
        return
    if args.op in ("repair", "update"):
        if args.impl == "reference":
            print(json.dumps({"impl": "reference", "unavailable": "repair reference arm not implemented"}))
            return
        run_repair(args, cfg)
        return

    if args.impl == "reference":
        run_reference(args, cfg)
        return

    ws, rank, local = _dist_env()
    # one GPU per rank; FSB_BENCH_BACKEND=gloo (host collectives, ranks may share a GPU: local %
    # device count) exists only to exercise the N > 1 code path on a one-GPU box -- its timings
    # are not bench values
    backend = os.environ.get("FSB_BENCH_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    global COLL_DEV
    COLL_DEV = dev if backend == "nccl" else "cpu"
    if ws > 1:
        import torch.distributed as dist
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
        dist.barrier()
        t_bc = time.perf_counter()
        g = fdist.broadcast_graph(cfg, device=COLL_DEV)   # step a2 over NCCL
        torch.cuda.synchronize()
        bcast_ms = fdist.max_over_ranks(1e3 * (time.perf_counter() - t_bc), device=COLL_DEV)
    else:
        g = fsb.Graph.create(cfg)
    if args.variant != "auto":
        g.set_variant(fsb.VARIANT_SMEM if args.variant == "smem" else fsb.VARIANT_GLOBAL)
    kind, u0, u1 = plan(cfg, ws, rank, args.scaling, args.partition)
    k, p, n, t = cfg["k"], cfg["p"], cfg["n"], cfg["t"]
    cols = t
    if kind == "stripes":
        S, rows = u1, n
        data = inputs.stripe_data(cfg, stripe_begin=u0, num_stripes=S, device=dev)
    elif kind == "cols":
        S, rows, cols = 1, n, u1 - u0
        data = inputs.stripe_data(cfg, device=dev)       # only bytes [u0, u1) are read
    else:
        S, rows = 1, u1 - u0
        data = inputs.stripe_data(cfg, device=dev)       # the source is replicated (R16)
    chk = torch.empty((S, p, t), dtype=torch.uint8, device=dev) if p else None
    cod = torch.empty((S, rows, t), dtype=torch.uint8, device=dev)
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.synchronize()

    def step():
        if kind == "stripes":
            g.encode_stripes(data, chk, cod, stream=stream)
        elif kind == "cols":
            g.encode_range(data[0], chk[0] if p else None, cod[0], 0, n, u0, u1, stream=stream)
        else:
            g.encode(data[0], chk[0] if p else None, cod[0], u0, u1, stream=stream)

    for _ in range(args.warmup):
        step()
    launches_per_step = fsb.last_launch_count()
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    # L2 rule: a step whose working set (source + checks + coded) is below 2x the 126 MB L2 would
    # run warm; then each timed step is preceded by an (untimed) write of a 256 MB scratch buffer
    # and timed alone.  Config 4/5 working sets are 0.9-2.4 GB: back-to-back steps, no flush.
    work_bytes = S * (k + p + rows) * (cols if kind == "cols" else t)
    flush = work_bytes < 2 * L2_BYTES
    scratch = torch.empty(2 * L2_BYTES, dtype=torch.uint8, device=dev) if flush else None
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(2 * args.steps if flush else args.steps + 1)]
    torch.cuda.nvtx.range_push("timed")   # ncu --nvtx --nvtx-include "timed/" captures only this
    with torch.cuda.stream(stream):
        if flush:
            for i in range(args.steps):
                scratch.fill_(i & 0xFF)
                evs[2 * i].record(stream)
                step()
                evs[2 * i + 1].record(stream)
        else:
            evs[0].record(stream)
            for i in range(args.steps):
                step()
                evs[i + 1].record(stream)
    stream.synchronize()
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_pop()
    if ws > 1:
        dist.barrier()
    clk = clocks.stop()
    if flush:
        per = [evs[2 * i].elapsed_time(evs[2 * i + 1]) for i in range(args.steps)]
        my_ms = sum(per)
    else:
        my_ms = evs[0].elapsed_time(evs[-1])
        per = [evs[i].elapsed_time(evs[i + 1]) for i in range(args.steps)]
    total_ms = fdist.max_over_ranks(my_ms, device=COLL_DEV) if ws > 1 else my_ms
    ms_per_step = total_ms / args.steps
    if kind == "stripes":
        src_bytes_all = (ws * S if args.scaling == "weak" else cfg["stripes"]) * k * t
    else:
        src_bytes_all = k * t                                # one stripe, rows split over ranks
    value = src_bytes_all / (ms_per_step * 1e-3) / 1e9

    # roofline of the dominant kernel (this rank): algorithmic HBM bytes per launch (one read of
    # the source, one write of checks + coded rows) / mean step time on the stream
    inf = g.info()
    b_hbm = S * (k + p + rows) * cols
    b_gather = S * (inf["lt_nnz"] * rows // n + inf["pre_nnz"]) * cols
    launch_ms = statistics.mean(per)
    peak, peak_src = _peaks()
    achieved = b_hbm / (launch_ms * 1e-3) / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp) and kind == "stripes" and S == cfg["stripes"]:
        try:
            traffic = json.load(open(tp)).get(cfg["name"], {}).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    smem_kernel = launches_per_step == 1
    # the gathers of the SMEM kernel hit shared memory, those of the GLOBAL band kernel L2: each
    # against its own builder-measured peak (microbenchmarks on this pool, not driver-measured)
    if smem_kernel:
        gpeak, gsrc = SMEM_GATHER_PEAK_GBS, ("builder-measured parity-paired 64-B smem row gather "
                                             "(tools/microbench/mb3.cu, profiles/r01b)")
    else:
        gpeak, gsrc = L2_GATHER_PEAK_GBS, ("builder-measured L2-resident random 512-B row gather "
                                           "(tools/microbench/mb7.cu, profiles/r01e/mb7.txt)")
    roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
            "frac": round(achieved / peak, 4), "traffic": traffic,
            "algorithmic_bytes_per_launch": b_hbm, "peak_source": peak_src,
            "kernel": "fsb_smem_encode" if smem_kernel else (
                "fsb_precode_global+fsb_lt_win" if inf.get("lt_windows") and os.environ.get("FSB_BAND_CFG", "5") == "5"
                else "fsb_precode_global+fsb_lt_band"),
            "timing": "CUDA events on the launching stream, mean per step (%d launch%s per step)"
                      % (launches_per_step, "" if smem_kernel else "es"),
            "gather": {"bytes_per_launch": b_gather,
                       "achieved": round(b_gather / (launch_ms * 1e-3) / 1e9, 1),
                       "peak": gpeak, "unit": "GB/s",
                       "frac": round(b_gather / (launch_ms * 1e-3) / 1e9 / gpeak, 4),
                       "peak_source": gsrc}}

    collectives = None
    if ws > 1:
        collectives = {"graph_broadcast_ms": round(bcast_ms, 3),
                       "graph_broadcast": "rank 0 generates, NCCL broadcast of the CSR, every rank "
                                          "rebuilds its schedule; host wall clock, max over ranks"}
        if kind == "stripes" and args.scaling == "strong" and COLL_DEV == "cpu":
            collectives["result_gather"] = {"skipped": "FSB_BENCH_BACKEND=gloo test run (no P2P of device tensors)"}
        elif kind == "stripes" and args.scaling == "strong":
            try:
                collectives["result_gather"] = _time_gather(cod, cfg["stripes"], dev, ws)
            except Exception as e:  # reported, never fatal to the encode line
                collectives["result_gather"] = {"error": repr(e)[:300]}

    e2e = None
    if args.e2e_steps > 0 and kind == "stripes":
        if args.e2e_api == "host":
            e2e = _e2e_host(g, cfg, data, cod, S, args, dev, ws, src_bytes_all)
        else:
            e2e = _e2e(g, cfg, data, cod, S, args, dev, ws, src_bytes_all)

    out = {"metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": ws, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": round(ms_per_step, 5), "higher_is_better": True,
           "scaling": args.scaling if kind == "stripes" else "strong", "vs_baseline": None, "dtype": "u8",
           "data": DATA,
           "config": workload_config(cfg, args, ws, kind, S, u0, u1, inf["lt_nnz"], inf["max_degree"]),
           "roofline": roof, "context": PAPER_CONTEXT, "gpu_launches": launches_per_step * args.steps,
           "step_ms_median": round(statistics.median(per), 5), "step_ms_best": round(min(per), 5),
           "clocks": clk, "e2e": e2e}
    if collectives:
        out["collectives"] = collectives
    if args.graph_replay and ws == 1:
        out["graph_replay"] = _graph_replay(step, stream, args.graph_replay, src_bytes_all)
    if rank == 0 and ws == 1 and not args.no_cpu:
        out["cpu_baseline"] = cpu_oracle_sample(cfg, args.cpu_seconds)
        if cfg["stripes"] > 1:
            out["cpu_baseline_threads"] = cpu_oracle_sample_mt(cfg, args.cpu_seconds / 2)
    if rank == 0:
        print(json.dumps(out))
    if ws > 1:
        dist.destroy_process_group()


def run_decode(args, cfg):
    """NEXT-1: decode throughput of the Alg 5 (DPG) plan, one GPU.  The coded symbols come from one
    (untimed) encode; a seeded random subset of them (--recv-frac) is 'received'; one step = one
    fs_decode call (one launch per DPG level) over every stripe."""
    import numpy as np
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    g = fsb.Graph.create(cfg)
    k, p, n, t, S = cfg["k"], cfg["p"], cfg["n"], cfg["t"], cfg["stripes"]
    K = k + p
    data = inputs.stripe_data(cfg, device=dev)
    chk = torch.empty((S, p, t), dtype=torch.uint8, device=dev) if p else None
    cod = torch.empty((S, n, t), dtype=torch.uint8, device=dev)
    g.encode_stripes(data, chk, cod)
    recv = np.random.default_rng(cfg["seed"]).random(n) < args.recv_frac
    plan = fsb.DecodePlan(g, recv, eliminate=args.eliminate)
    inf = plan.info()
    cod[:, torch.from_numpy(~recv).to(dev)] = 0                 # erased symbols
    inter = torch.zeros((S, K, t), dtype=torch.uint8, device=dev)
    stream = torch.cuda.Stream(device=dev)
    for _ in range(args.warmup):
        plan.decode(cod, inter, stream=stream)
    launches = fsb.last_launch_count()
    stream.synchronize()
    st, _ = plan.state()
    rec = torch.from_numpy(st[:k].astype(bool)).to(dev)
    ok = bool(torch.equal(inter[:, :k][:, rec], data[:, rec]))
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    clocks = ClockSampler(0)
    clocks.start()
    time.sleep(0.3)
    torch.cuda.nvtx.range_push("timed")
    with torch.cuda.stream(stream):
        evs[0].record(stream)
        for i in range(args.steps):
            plan.decode(cod, inter, stream=stream)
            evs[i + 1].record(stream)
    stream.synchronize()
    torch.cuda.nvtx.range_pop()
    clk = clocks.stop()
    ms = evs[0].elapsed_time(evs[-1]) / args.steps
    rec_bytes = S * inf["recovered_data"] * t
    value = rec_bytes / (ms * 1e-3) / 1e9
    # one read of every coded row a plan row uses + one write of every recovered symbol
    b_hbm = S * (int(recv.sum()) + inf["recovered"]) * t
    peak, peak_src = _peaks()
    out = {"op": "decode", "metric": "decode throughput, recovered data GB/s (Alg 5 DPG plan)",
           "value": round(value, 2), "unit": "GB/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": round(ms, 5), "higher_is_better": True, "dtype": "u8", "data": DATA,
           "config": {"workload": cfg["name"], "k": k, "p": p, "n": n, "t": t, "stripes": S,
                      "recv_frac": args.recv_frac, "received": int(recv.sum()),
                      "recovered_data": inf["recovered_data"], "levels": inf["levels"],
                      "eliminated": inf["eliminated"], "elimination": bool(args.eliminate),
                      "xor_sources": inf["xor_sources"]},
           "roofline": {"bound": "hbm", "achieved": round(b_hbm / (ms * 1e-3) / 1e9, 1), "peak": peak,
                        "unit": "GB/s", "frac": round(b_hbm / (ms * 1e-3) / 1e9 / peak, 4),
                        "algorithmic_bytes_per_step": b_hbm, "peak_source": peak_src,
                        "kernel": "fsb_dpg_level x %d launches" % launches},
           "gpu_launches": launches * args.steps, "checked": ok, "clocks": clk}
    if not args.no_cpu:
        out["cpu_baseline"] = _oracle_decode_sample(cfg, recv, cod, args)
    print(json.dumps(out))


def _oracle_decode_sample(cfg, recv, cod, args):
    """The oracle's decoder (Alg 1 BP over LT rows + precode checks, then GF(2) elimination when
    --eliminate), single-threaded C, on whole stripes until ~--cpu-seconds (at least one); metric
    = recovered data bytes per second, as the GPU line's."""
    import numpy as np
    import oracle
    go = oracle.generate_graph(cfg)
    S, k, t = cfg["stripes"], cfg["k"], cfg["t"]
    done, t_dec, rec_bytes = 0, 0.0, 0
    while done < S and (t_dec < args.cpu_seconds or done == 0):
        Y = cod[done].cpu().numpy()
        t0 = time.perf_counter()
        _, state = oracle.decode(go, recv, Y, use_elim=bool(args.eliminate))
        t_dec += time.perf_counter() - t0
        rec_bytes += int(np.count_nonzero(state[:k])) * t
        done += 1
    host = _host_cpu()
    return {"value": rec_bytes / t_dec / 1e9, "unit": "GB/s", "cores": 1, "kind": "oracle",
            "host_cpu": host["model"], "sample": "%d of %d stripes, single-threaded C oracle decoder%s, %.2f s"
            % (done, S, " + elimination" if args.eliminate else "", t_dec)}


def run_repair(args, cfg):
    """NEXT-3 on one GPU.  repair: a seeded random --erase-frac of the coded symbols is erased and
    rebuilt from the local sets (CGA check data); update: the code is extended by one
    output file whose symbols are computed from the ORIGINAL code's check data
    (the data is not read).  One step = one fs_repair call (one launch per level) over every
    stripe.  Metric: rebuilt coded bytes per second."""
    import numpy as np
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    g0 = fsb.Graph.create(cfg)
    t_cga = time.perf_counter()
    checks0 = fsb.Checks.create(g0, fsb.CHECKS_M1 | fsb.CHECKS_M2)
    t_cga = time.perf_counter() - t_cga
    if args.op == "update":
        g = g0.extend(1)
        checks = fsb.Checks.from_data(g, checks0.data())
        erased = np.zeros(g.n, bool)
        erased[g0.n:] = True
    else:
        g, checks = g0, checks0
        rng = np.random.default_rng(cfg["seed"] + 1)
        erased = np.zeros(g.n, bool)
        erased[rng.choice(g.n, max(1, int(round(args.erase_frac * g.n))), replace=False)] = True
    k, p, n, t, S = g.k, g.p, g.n, g.t, cfg["stripes"]
    t_plan = time.perf_counter()
    plan = fsb.RepairPlan(g, checks, erased)
    t_plan = time.perf_counter() - t_plan
    inf = plan.info()
    data = inputs.stripe_data(cfg, device=dev)
    chk = torch.empty((S, p, t), dtype=torch.uint8, device=dev) if p else None
    ref = torch.empty((S, n, t), dtype=torch.uint8, device=dev)
    g.encode_stripes(data, chk, ref)                              # expected symbols (untimed)
    del data, chk
    er_t = torch.from_numpy(erased).to(dev)
    cod = ref.clone()
    cod[:, er_t] = 0
    stream = torch.cuda.Stream(device=dev)
    for _ in range(args.warmup):
        plan.repair(cod, stream=stream)
    launches = fsb.last_launch_count()
    stream.synchronize()
    level_ptr, target, src_ptr, src = plan.rows()
    rebuilt = [int(x) & 0x3FFFFFFF for x in target]
    ok = bool(torch.equal(cod[:, rebuilt], ref[:, rebuilt])) if rebuilt else True
    del ref
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    clocks = ClockSampler(0)
    clocks.start()
    time.sleep(0.3)
    torch.cuda.nvtx.range_push("timed")
    with torch.cuda.stream(stream):
        evs[0].record(stream)
        for i in range(args.steps):
            plan.repair(cod, stream=stream)
            evs[i + 1].record(stream)
    stream.synchronize()
    torch.cuda.nvtx.range_pop()
    clk = clocks.stop()
    ms = evs[0].elapsed_time(evs[-1]) / args.steps
    rows = len(rebuilt)
    distinct_src = len(set(int(v) & 0x3FFFFFFF for v in src))
    value = S * rows * t / (ms * 1e-3) / 1e9
    b_hbm = S * (distinct_src + rows) * t               # each source row read once + each rebuilt row written
    b_gather = S * int(inf["xor_sources"]) * t
    peak, peak_src = _peaks()
    out = {"op": args.op, "metric": "%s throughput, rebuilt coded GB/s (CGA local sets)" % args.op,
           "value": round(value, 2), "unit": "GB/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": round(ms, 5), "higher_is_better": True, "dtype": "u8", "data": DATA,
           "config": {"workload": cfg["name"], "k": k, "p": p, "n": n, "t": t, "stripes": S,
                      "files": g.cfg.get("files", 1), "erased": inf["erased"], "rebuilt": inf["repaired"],
                      "unrepaired": inf["unrepaired"], "levels": inf["levels"], "xor_sources": inf["xor_sources"],
                      "distinct_sources": distinct_src, "cga_s": round(t_cga, 3), "plan_s": round(t_plan, 4),
                      "checks": checks0.info()},
           "roofline": {"bound": "hbm", "achieved": round(b_hbm / (ms * 1e-3) / 1e9, 1), "peak": peak,
                        "unit": "GB/s", "frac": round(b_hbm / (ms * 1e-3) / 1e9 / peak, 4),
                        "algorithmic_bytes_per_step": b_hbm, "peak_source": peak_src,
                        "gather_bytes_per_step": b_gather,
                        "gather_GBps": round(b_gather / (ms * 1e-3) / 1e9, 1),
                        "kernel": "fsb_dpg_level x %d launches" % launches},
           "gpu_launches": launches * args.steps, "checked": ok, "clocks": clk}
    print(json.dumps(out))


def _time_gather(cod, total, dev, ws, reps=3):
    """SURVEY.md §8(e)(ii), reported apart from the encode: every rank's coded stripes to rank 0
    (dist.gather_stripes, NCCL point-to-point).  CUDA events per rep, max over ranks."""
    import torch.distributed as dist
    dist.barrier()
    fdist.gather_stripes(cod, total)                     # warm-up (NCCL P2P setup)
    torch.cuda.synchronize()
    ms = []
    for _ in range(reps):
        dist.barrier()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        out = fdist.gather_stripes(cod, total)
        b.record()
        torch.cuda.synchronize()
        ms.append(fdist.max_over_ranks(a.elapsed_time(b), device=COLL_DEV))
        del out
    moved = (total - fdist.shard(total, ws, 0)[1]) * cod[0].numel()
    best = min(ms)
    return {"ms": round(best, 3), "bytes_to_rank0": moved, "GBps_into_rank0": round(moved / (best * 1e-3) / 1e9, 1),
            "reps": reps, "timing": "CUDA events on the current stream, best of reps, max over ranks"}


def _graph_replay(step, stream, count, src_bytes):
    """for the launch-latency-bound small configs, `count` back-to-back steps captured
    in one CUDA graph and replayed (warm L2, launch overhead amortised); reported beside the
    flushed per-step timing, never as `value`."""
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(stream):
        step()  # warm
        stream.synchronize()
        with torch.cuda.graph(g, stream=stream):
            for _ in range(count):
                step()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        a.record(stream)
        for _ in range(5):
            g.replay()
        b.record(stream)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / (5 * count)
    return {"launches_per_graph": count, "ms_per_step": round(ms, 5),
            "value": round(src_bytes / (ms * 1e-3) / 1e9, 2), "unit": "GB/s", "l2": "warm"}


def _e2e_host(g, cfg, data, cod, S, args, dev, ws, src_bytes_all):
    """The metric through fs_encode_host: every step hands the library the HOST buffers (pinned)
    and it stages them through its own device memory -- H2D of the data, the encode, D2H of
    checks + coded, pipelined over chunks of stripes (or of byte columns for one stripe)."""
    k, p, n, t = cfg["k"], cfg["p"], cfg["n"], cfg["t"]
    h_data = torch.empty((S, k, t), dtype=torch.uint8, pin_memory=True)
    h_data.copy_(data.cpu())
    h_chk = torch.empty((S, p, t), dtype=torch.uint8, pin_memory=True) if p else None
    h_cod = torch.empty((S, n, t), dtype=torch.uint8, pin_memory=True)
    cur = torch.cuda.current_stream(dev)
    g.encode_host(h_data, h_chk, h_cod, chunks=args.e2e_chunks, stream=cur)  # warm: staging allocated
    torch.cuda.synchronize()
    launches = fsb.last_launch_count()
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(cur)
    for _ in range(args.e2e_steps):
        g.encode_host(h_data, h_chk, h_cod, chunks=args.e2e_chunks, stream=cur)
    e1.record(cur)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    ms = (fdist.max_over_ranks(ms, device=COLL_DEV) if ws > 1 else ms) / args.e2e_steps
    ok = bool(torch.equal(h_cod[0].to(dev), cod[0]) and torch.equal(h_cod[S - 1].to(dev), cod[S - 1]))
    return {"value": round(src_bytes_all / (ms * 1e-3) / 1e9, 2), "unit": "GB/s",
            "h2d_bytes_per_step": S * k * t, "d2h_bytes_per_step": S * (p + n) * t,
            "ms_per_step": round(ms, 3), "gpu_launches_per_step": launches,
            "api": "fs_encode_host (library staging, %s chunks of %s, 2 library streams)"
                   % (args.e2e_chunks or "default", "stripes" if S > 1 else "byte columns"), "checked": ok}


def _e2e(g, cfg, data, cod, S, args, dev, ws, src_bytes_all):
    """Same metric through fs_encode_stripes with HOST buffers: per step, H2D of the step's
    data from pinned memory, the encode, and D2H of checks + coded, pipelined over chunks of
    stripes on two streams (copies overlap the kernels of neighbouring chunks)."""
    k, p, n, t = cfg["k"], cfg["p"], cfg["n"], cfg["t"]
    h_data = torch.empty((S, k, t), dtype=torch.uint8, pin_memory=True)
    h_data.copy_(data.cpu())
    h_chk = torch.empty((S, p, t), dtype=torch.uint8, pin_memory=True) if p else None
    h_cod = torch.empty((S, n, t), dtype=torch.uint8, pin_memory=True)
    nchunks = min(S, args.e2e_chunks or 16)
    ns = args.e2e_streams
    bounds = [(i * S // nchunks, (i + 1) * S // nchunks) for i in range(nchunks)]
    streams = [torch.cuda.Stream(device=dev) for _ in range(ns)]
    cs = max(b - a for a, b in bounds)
    d_buf = [torch.empty((cs, k, t), dtype=torch.uint8, device=dev) for _ in range(ns)]
    c_buf = [torch.empty((cs, p, t), dtype=torch.uint8, device=dev) if p else None for _ in range(ns)]
    y_buf = [torch.empty((cs, n, t), dtype=torch.uint8, device=dev) for _ in range(ns)]

    def one_step():
        for i, (a, b) in enumerate(bounds):
            st = streams[i % ns]
            with torch.cuda.stream(st):
                db = d_buf[i % ns][:b - a]
                db.copy_(h_data[a:b], non_blocking=True)
                cb = c_buf[i % ns][:b - a] if p else None
                yb = y_buf[i % ns][:b - a]
                g.encode_stripes(db, cb, yb, stream=st)
                if p:
                    h_chk[a:b].copy_(cb, non_blocking=True)
                h_cod[a:b].copy_(yb, non_blocking=True)

    one_step()
    torch.cuda.synchronize()
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()
    cur = torch.cuda.current_stream(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(cur)
    for st in streams:
        st.wait_stream(cur)
    for _ in range(args.e2e_steps):
        one_step()
    for st in streams:
        cur.wait_stream(st)
    e1.record(cur)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    ms = (fdist.max_over_ranks(ms, device=COLL_DEV) if ws > 1 else ms) / args.e2e_steps
    # spot-check the host result against the device-resident run
    ok = bool(torch.equal(h_cod[0].to(dev), cod[0]) and torch.equal(h_cod[S - 1].to(dev), cod[S - 1]))
    return {"value": round(src_bytes_all / (ms * 1e-3) / 1e9, 2), "unit": "GB/s",
            "h2d_bytes_per_step": S * k * t, "d2h_bytes_per_step": S * (p + n) * t,
            "ms_per_step": round(ms, 3),
            "api": "fs_encode_stripes on pinned-host staging, %d chunks x %d streams" % (nchunks, ns), "checked": ok}


if __name__ == "__main__":
    main()
