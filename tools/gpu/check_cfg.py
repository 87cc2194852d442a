"""Quick bit-exact check of one config through whatever library FSB_LIB selects (A/B builds):
encode on cuda:0, compare checks and coded rows with the oracle (cached under /tmp per config).
Usage: python tools/gpu/check_cfg.py CONFIG [variant: auto|global|smem]"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_1702_07409_b200 import configs, fsb, inputs  # noqa: E402

cid = int(sys.argv[1])
var = sys.argv[2] if len(sys.argv) > 2 else "auto"
cfg = configs.get(cid)
go = oracle.generate_graph(cfg)
# the oracle's output, cached under /tmp by a hash of the oracle's own graph and the config
import hashlib  # noqa: E402
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
if var != "auto":
    g.set_variant(fsb.VARIANT_SMEM if var == "smem" else fsb.VARIANT_GLOBAL)
S, p, n, t = cfg["stripes"], cfg["p"], cfg["n"], cfg["t"]
d = inputs.stripe_data(cfg, device="cuda")
chk = torch.empty((S, p, t), dtype=torch.uint8, device="cuda") if p else None
cod = torch.empty((S, n, t), dtype=torch.uint8, device="cuda")
g.encode_stripes(d, chk, cod)
torch.cuda.synchronize()
ok = np.array_equal(cod.cpu().numpy(), Y) and (not p or np.array_equal(chk.cpu().numpy(), C))
print("c%d %s: %s" % (cid, var, "ok" if ok else "MISMATCH"))
