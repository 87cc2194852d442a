import sys, torch
sys.path.insert(0, "/root/repo")
from paper_1702_07409_b200 import configs, fsb, inputs
for t in (512, 1024, 2048, 8192):
    cfg = dict(configs.get(5), t=t)
    g = fsb.Graph.create(cfg)
    d = inputs.stripe_data(cfg, device="cuda")
    chk = torch.empty((1, cfg["p"], t), dtype=torch.uint8, device="cuda")
    cod = torch.empty((1, cfg["n"], t), dtype=torch.uint8, device="cuda")
    for _ in range(5): g.encode_stripes(d, chk, cod)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(50): g.encode_stripes(d, chk, cod)
    b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 50
    gath = (352119 + 2000) * t
    print("t=%d ms=%.4f gather TB/s=%.1f per-band us=%.1f" % (t, ms, gath / ms / 1e9, ms * 1000 / (t / 512)))
