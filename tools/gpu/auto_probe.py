"""SMEM vs GLOBAL variant on small stripe counts (the AUTO rule), warm CUDA-graph replay of 50
encodes and a cold single-launch time.

    python tools/gpu/auto_probe.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1702_07409_b200 import configs, fsb, inputs  # noqa: E402


def timed(g, d, chk, cod, n=50):
    g.encode_stripes(d, chk, cod)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        g.encode_stripes(d, chk, cod)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n * 1000


for cid, S in ((1, 1), (2, 1), (2, 4), (4, 1), (4, 2), (4, 4), (6, 1), (7, 1), (7, 4), (4, 8)):
    cfg = dict(configs.get(cid), stripes=S)
    g = fsb.Graph.create(cfg)
    if not g.info()["smem_eligible"]:
        continue
    d = inputs.stripe_data(cfg, device="cuda")
    chk = torch.empty((S, cfg["p"], cfg["t"]), dtype=torch.uint8, device="cuda") if cfg["p"] else None
    cod = torch.empty((S, cfg["n"], cfg["t"]), dtype=torch.uint8, device="cuda")
    res = []
    for v in (fsb.VARIANT_GLOBAL, fsb.VARIANT_SMEM):
        g.set_variant(v)
        res.append(timed(g, d, chk, cod))
    tiles = S * cfg["t"] // 64
    print("c%d S=%d tiles=%d  global %.1f us  smem %.1f us" % (cid, S, tiles, res[0], res[1]))
