"""Config 4 time per launch for several stripe counts S (one GPU), to see tile-round quantisation
and the fixed cost per launch.  python tools/gpu/stripe_sweep.py [steps] [S ...]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1702_07409_b200 import configs, fsb, inputs  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 300
Ss = [int(x) for x in sys.argv[2:]] or [5, 10, 20, 32, 37, 64]
cfg = configs.get(4)
g = fsb.Graph.create(cfg)
p, n, t = cfg["p"], cfg["n"], cfg["t"]
d = inputs.stripe_data(cfg, device="cuda")
chk = torch.empty((256, p, t), dtype=torch.uint8, device="cuda")
cod = torch.empty((256, n, t), dtype=torch.uint8, device="cuda")
res = {}
for S in Ss:
    for _ in range(20):
        g.encode_stripes(d[:S], chk[:S], cod[:S])
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(steps):
        g.encode_stripes(d[:S], chk[:S], cod[:S])
    b.record()
    torch.cuda.synchronize()
    res[S] = round(a.elapsed_time(b) / steps * 1e3, 2)
print(json.dumps({"us_per_launch": res, "tail_singles": os.environ.get("FSB_TAIL_SINGLES", "1")}))
