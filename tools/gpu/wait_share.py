"""Share of consumer-warp time spent waiting for tiles in fsb_smem_encode (FSB_DEBUG=2 counters),
each consumer warp's busy cycles relative to the mean, the precode warps' wait on `full` and the
TMA thread's wait on `empty`.  Needs the experiment build:

    FSB_EXPERIMENTS=1 python paper_1702_07409_b200/build.py --force --out /tmp/libexp.so
    FSB_LIB=/tmp/libexp.so FSB_DEBUG=2 python tools/gpu/wait_share.py [config]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1702_07409_b200 import configs, fsb, inputs  # noqa: E402

assert os.environ.get("FSB_DEBUG") == "2", "run with FSB_DEBUG=2"
cid = int(sys.argv[1]) if len(sys.argv) > 1 else 4
cfg = configs.get(cid)
g = fsb.Graph.create(cfg)
S, k, p, n, t = cfg["stripes"], cfg["k"], cfg["p"], cfg["n"], cfg["t"]
d = inputs.stripe_data(cfg, device="cuda")
chk = torch.empty((S, p, t), dtype=torch.uint8, device="cuda")
cod = torch.empty((S, n, t), dtype=torch.uint8, device="cuda")
for _ in range(3):
    g.encode_stripes(d, chk, cod)
torch.cuda.synchronize()
fsb.debug_counters()  # clear
for _ in range(10):
    g.encode_stripes(d, chk, cod)
torch.cuda.synchronize()
c = fsb.debug_counters(64)
waits = [c[2 * w] for w in range(24)]
tots = [c[2 * w + 1] for w in range(24)]
pre = [(c[48 + 2 * w], c[49 + 2 * w]) for w in range(3)]
print({"config": cfg["name"], "wait_share_per_warp": [round(a / b, 4) if b else None for a, b in zip(waits, tots)],
       "wait_share_all": round(sum(waits) / max(1, sum(tots)), 4),
       "busy_cycles_per_warp_rel": [round((b - a) / (sum(tots) - sum(waits)) * 24, 3) for a, b in zip(waits, tots)],
       "precode_wait_share": [round(a / b, 4) if b else None for a, b in pre],
       "tma_empty_wait_share": round(c[60] / max(1, pre[0][1]), 4)})
