"""Profiling aid: per-warp tile-wait cycles of fsb_smem_encode on config 4 (run with FSB_DEBUG=2)."""
import os, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch
from paper_1702_07409_b200 import configs, fsb, inputs
cfg = configs.get(int(sys.argv[1]) if len(sys.argv) > 1 else 4)
g = fsb.Graph.create(cfg)
S, k, p, n, t = cfg["stripes"], cfg["k"], cfg["p"], cfg["n"], cfg["t"]
d = inputs.stripe_data(cfg, device="cuda")
chk = torch.empty((S, p, t), dtype=torch.uint8, device="cuda")
cod = torch.empty((S, n, t), dtype=torch.uint8, device="cuda")
for _ in range(3):
    g.encode_stripes(d, chk, cod)
torch.cuda.synchronize()
fsb.debug_counters()
for _ in range(10):
    g.encode_stripes(d, chk, cod)
torch.cuda.synchronize()
c = fsb.debug_counters()
W = 24
rows = [{"warp": w, "wait_frac": round(c[2 * w] / max(1, c[2 * w + 1]), 4)} for w in range(W)]
print(json.dumps({"per_warp": rows, "mean_wait_frac": round(sum(r["wait_frac"] for r in rows) / W, 4)}))
