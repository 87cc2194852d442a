"""Cost model of fsb_smem_encode per tile: time ~ a*items + b*gather_steps, fitted on graphs whose
LT rows all have one degree d (finite distribution {d: 1}), config 4's shape otherwise.

    python tools/gpu/item_cost.py
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1702_07409_b200 import configs, fsb, inputs  # noqa: E402

res = []
for d in (2, 3, 4, 6, 8, 12, 16, 24, 32):
    cfg = dict(configs.get(4), dist=configs.FINITE, fin_deg=(d,), fin_prob=(1.0,), seed=7)
    g = fsb.Graph.create(cfg)
    if not g.info()["smem_eligible"]:
        continue
    w, cb, wi, kpad, z = g.schedule()
    items = int(wi[:, 0].sum())
    steps = int(g.info()["sched_steps_avg"]) * 24
    S, k, p, n, t = cfg["stripes"], cfg["k"], cfg["p"], cfg["n"], cfg["t"]
    data = inputs.stripe_data(cfg, device="cuda")
    chk = torch.empty((S, p, t), dtype=torch.uint8, device="cuda")
    cod = torch.empty((S, n, t), dtype=torch.uint8, device="cuda")
    for _ in range(5):
        g.encode_stripes(data, chk, cod)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(100):
        g.encode_stripes(data, chk, cod)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 100
    clk_per_tile = ms * 1e-3 * 1.965e9 / (S * (t // 64) / 148)
    res.append({"d": d, "items": items, "steps_total": int(g.info()["sched_steps_avg"]) * 24,
                "nnz": int(g.info()["lt_nnz"]), "ms": round(ms, 4), "clk_per_tile": round(clk_per_tile)})
    del data, chk, cod, g
X = np.array([[r["items"], r["nnz"] / 8.0] for r in res], float)
y = np.array([r["clk_per_tile"] for r in res], float)
coef, *_ = np.linalg.lstsq(X, y, rcond=None)
print(json.dumps({"runs": res, "fit_clk_per_item": round(coef[0], 1), "fit_clk_per_gather_step": round(coef[1], 2)}))
