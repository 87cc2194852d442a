import sys, os, json
sys.path.insert(0, "/root/repo")
import torch
from paper_1702_07409_b200 import configs, fsb, inputs
cfg = configs.get(4); g = fsb.Graph.create(cfg)
k, p, n, t = cfg["k"], cfg["p"], cfg["n"], cfg["t"]
d = inputs.stripe_data(cfg, device="cuda")
chk = torch.empty((256, p, t), dtype=torch.uint8, device="cuda"); cod = torch.empty((256, n, t), dtype=torch.uint8, device="cuda")
res = []
for S in (3, 5, 10, 14, 19, 24, 32, 64):
    for _ in range(20): g.encode_stripes(d[:S], chk[:S], cod[:S])
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(500): g.encode_stripes(d[:S], chk[:S], cod[:S])
    b.record(); torch.cuda.synchronize()
    tiles = S * 64
    ppc = -(-tiles // 2 // 148) if tiles > 148 else 1
    res.append((S, tiles, ppc, round(a.elapsed_time(b) / 500 * 1000, 2)))
print(res)
