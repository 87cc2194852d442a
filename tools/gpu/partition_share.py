"""One rank's share of a single-stripe encode (config 5 by default), timed alone on ONE GPU, for the
two partitions of DESIGN.md §7: coded rows [r n/G, (r+1) n/G) with the whole source read, or byte
columns [c0, c1) (fs_encode_range, nothing replicated).  Per-rank kernel time for G = 1..8 ranks;
no multi-rank execution is emulated (each line is one GPU doing one rank's work).

    python tools/gpu/partition_share.py [config] [steps]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1702_07409_b200 import configs, dist as fdist, fsb, inputs  # noqa: E402

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 5
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 200
cfg = configs.get(cid)
g = fsb.Graph.create(cfg)
k, p, n, t = cfg["k"], cfg["p"], cfg["n"], cfg["t"]
d = inputs.stripe_data(cfg, device="cuda")[0]
chk = torch.empty((p, t), dtype=torch.uint8, device="cuda") if p else None
out = torch.empty((n, t), dtype=torch.uint8, device="cuda")
stream = torch.cuda.Stream()


def timed(fn):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        a.record(stream)
        for _ in range(steps):
            fn()
        b.record(stream)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / steps


res = []
for G in (1, 2, 4, 8):
    r0, r1 = fdist.shard(n, G, 0)
    c0, c1 = fdist.col_shard(t, G, 0)
    ms_rows = timed(lambda: g.encode(d, chk, out[: r1 - r0], r0, r1, stream=stream))
    ms_cols = timed(lambda: g.encode_range(d, chk, out, 0, n, c0, c1, stream=stream))
    res.append({"G": G, "rows_ms": round(ms_rows, 4), "cols_ms": round(ms_cols, 4),
                "rows_GBps_job": round(k * t / ms_rows / 1e6, 1), "cols_GBps_job": round(k * t / ms_cols / 1e6, 1)})
print(json.dumps({"config": cfg["name"], "steps": steps, "per_rank_share": res}))
