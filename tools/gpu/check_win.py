"""Bit-exact check of config 5 through the LT kernel FSB_BAND_CFG selects (run in a fresh
process per setting): the full-row stripe encode, then row ranges (rank partitions G = 2, 3 and
ranges starting / ending mid-window) against the oracle (cached under /tmp like check_cfg.py).
Usage: FSB_BAND_CFG=5 python tools/gpu/check_win.py [CONFIG]"""
import hashlib
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_1702_07409_b200 import configs, fsb, inputs  # noqa: E402

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 5
cfg = configs.get(cid)
go = oracle.generate_graph(cfg)
h = hashlib.sha256()
for arr in (go.pre_row_ptr, go.pre_col, go.lt_row_ptr, go.lt_col):
    h.update(np.ascontiguousarray(arr, dtype="<i4").tobytes())
h.update(repr(sorted((k, v) for k, v in cfg.items() if not isinstance(v, tuple))).encode())
cache = "/tmp/oracle_c%d_%s.npz" % (cid, h.hexdigest()[:16])
if os.path.exists(cache):
    z = np.load(cache)
    C, Y = z["C"], z["Y"]
else:
    C, Y = oracle.encode(go, inputs.stripe_data(cfg).numpy())
    np.savez(cache, C=C, Y=Y)
g = fsb.Graph.create(cfg)
g.set_variant(fsb.VARIANT_GLOBAL)
S, p, n, t = cfg["stripes"], cfg["p"], cfg["n"], cfg["t"]
d = inputs.stripe_data(cfg, device="cuda")
chk = torch.empty((S, p, t), dtype=torch.uint8, device="cuda") if p else None
cod = torch.empty((S, n, t), dtype=torch.uint8, device="cuda")
g.encode_stripes(d, chk, cod)
torch.cuda.synchronize()
bad = []
if not np.array_equal(cod.cpu().numpy(), Y):
    bad.append("full coded")
if p and not np.array_equal(chk.cpu().numpy(), C):
    bad.append("full checks")
ranges = [(r * n // G, (r + 1) * n // G) for G in (2, 3) for r in range(G)]
ranges += [(5, n // 2 + 3), (n // 2 - 1, n), (7, 8), (n - 1, n)]
for a, b in ranges:
    c1 = torch.empty((p, t), dtype=torch.uint8, device="cuda")
    out = torch.full((b - a, t), 0xA5, dtype=torch.uint8, device="cuda")
    g.encode(d[0], c1, out, a, b)
    torch.cuda.synchronize()
    if not np.array_equal(out.cpu().numpy(), Y[0, a:b]):
        bad.append("rows [%d, %d)" % (a, b))
print("c%d band_cfg=%s: %s" % (cid, os.environ.get("FSB_BAND_CFG", "default"), "MISMATCH " + ", ".join(bad) if bad else "ok"))
