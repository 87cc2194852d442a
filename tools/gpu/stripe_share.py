"""Config 4's per-rank share under the stripe partition, timed alone on one GPU: S = 256/N
stripes for N = 1, 2, 4, 8 (what each rank of bench.py --gpus N encodes).  Prints ms per step
and the efficiency against perfect division of the N=1 time.

    python tools/gpu/stripe_share.py [steps]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1702_07409_b200 import configs, fsb, inputs  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 300
cfg = configs.get(4)
g = fsb.Graph.create(cfg)
k, p, n, t = cfg["k"], cfg["p"], cfg["n"], cfg["t"]
d = inputs.stripe_data(cfg, device="cuda")
chk = torch.empty((256, p, t), dtype=torch.uint8, device="cuda")
cod = torch.empty((256, n, t), dtype=torch.uint8, device="cuda")
out = []
base = None
for N in (1, 2, 4, 8):
    S = 256 // N
    for _ in range(20):
        g.encode_stripes(d[:S], chk[:S], cod[:S])
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(steps):
        g.encode_stripes(d[:S], chk[:S], cod[:S])
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / steps
    base = base or ms
    out.append({"N": N, "stripes": S, "ms": round(ms, 5), "efficiency": round(base / (N * ms), 4)})
print(json.dumps({"config": cfg["name"], "per_rank_share": out}))
