"""Per-tile pipeline log of two CTAs of one fsb_smem_encode launch (experiment build, FSB_DEBUG=8):
for each tile, when the TMA thread finished issuing it, when the precode warps saw it land
(`full`), when they released it (`ready`), and the first / last consumer warp's start and end.
Prints the mean intervals: load latency (issue -> full), precode (full -> ready), how long the
first consumer waited past its previous tile (ready late), consumer start / end spreads.
python tools/gpu/tile_log.py [S]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1702_07409_b200 import configs, fsb, inputs  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 256
cfg = configs.get(int(os.environ.get("CFG", "4")))
g = fsb.Graph.create(cfg)
p, n, t = cfg["p"], cfg["n"], cfg["t"]
S = min(S, cfg["stripes"])
d = inputs.stripe_data(cfg, num_stripes=S, device="cuda")
chk = torch.empty((S, p, t), dtype=torch.uint8, device="cuda")
cod = torch.empty((S, n, t), dtype=torch.uint8, device="cuda")
NC = 64 + 16 * 256 + 2 * 128 * 8
for _ in range(5):
    g.encode_stripes(d, chk, cod)
torch.cuda.synchronize()
fsb.debug_counters(NC)
for _ in range(1):  # one launch (the min / max atomics would mix launches)
    g.encode_stripes(d, chk, cod)
torch.cuda.synchronize()
c = np.array(fsb.debug_counters(NC)[64 + 16 * 256:], dtype=np.uint64).reshape(2, 128, 8)
out = {"S": S, "config": cfg["name"]}
for k, name in enumerate(("cta0", "cta_mid")):
    L = c[k]
    ntile = int((L[:, 0] > 0).sum())
    issue, full, ready = L[:ntile, 0].astype(np.float64), L[:ntile, 1].astype(np.float64), L[:ntile, 2].astype(np.float64)
    s_min = (~L[:ntile, 3]).astype(np.float64)
    s_max = L[:ntile, 4].astype(np.float64)
    e_min = (~L[:ntile, 5]).astype(np.float64)
    e_max = L[:ntile, 6].astype(np.float64)
    us = lambda x: round(float(np.mean(x)) / 1e3, 3)  # noqa: E731
    out[name] = {
        "tiles": ntile,
        "tile_period_us": us(np.diff(e_max)),
        "load_us (issue->full)": us(full - issue),
        "precode_us (full->ready)": us(ready - full),
        "release_to_issue_us (last end of tile i-2 -> issue of i)": us(issue[2:] - e_max[:-2]),
        "first_consumer_wait_us (ready - first end of tile i-1)": us(np.maximum(0, ready[1:] - e_min[:-1])),
        "start_spread_us": us(s_max - s_min),
        "end_spread_us": us(e_max - e_min),
        "busy_first_us (end_min - start_min)": us(e_min - s_min),
    }
print(json.dumps(out, indent=1))
