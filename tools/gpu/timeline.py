"""Per-CTA timeline of one fsb_smem_encode launch (experiment build, FSB_DEBUG=4): %globaltimer at
entry, end of prologue (per CTA also: [cta, smid, tiles, last consumer end us], sorted by end), first tile ready, mean / last consumer end, last TMA issue -- where the
fixed cost of a short launch goes.  Needs FSB_LIB = an -DFSB_EXPERIMENTS build and FSB_DEBUG=4.
python tools/gpu/timeline.py S [S ...]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1702_07409_b200 import configs, fsb, inputs  # noqa: E402

cfg = configs.get(4)
g = fsb.Graph.create(cfg)
p, n, t = cfg["p"], cfg["n"], cfg["t"]
d = inputs.stripe_data(cfg, device="cuda")
chk = torch.empty((256, p, t), dtype=torch.uint8, device="cuda")
cod = torch.empty((256, n, t), dtype=torch.uint8, device="cuda")
NC = 64 + 16 * 256
sms = torch.cuda.get_device_properties(0).multi_processor_count
for S in [int(x) for x in sys.argv[1:]] or [32, 256]:
    for _ in range(5):
        g.encode_stripes(d[:S], chk[:S], cod[:S])
    torch.cuda.synchronize()
    fsb.debug_counters(NC)  # clear
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    g.encode_stripes(d[:S], chk[:S], cod[:S])
    b.record()
    torch.cuda.synchronize()
    c = np.array(fsb.debug_counters(NC)[64:], dtype=np.float64).reshape(256, 16)[:sms]
    t0 = c[:, 0].min()
    rel = lambda x: (x - t0) / 1e3  # noqa: E731  (us)
    out = {"S": S, "event_us": round(a.elapsed_time(b) * 1e3, 2)}
    for name, col in (("entry", 0), ("prologue_done", 1), ("first_tile_ready", 2), ("consumer_end_mean", 3),
                      ("consumer_end_max", 4), ("last_tma_issue", 5),
                      ("tmem_alloc_done", 8), ("sched_copy_done", 9), ("tma_gdc_wait_done", 10),
                      ("before_sync", 12), ("after_sync", 13)):
        v = rel(c[:, col])
        out[name] = {"min": round(v.min(), 2), "median": round(float(np.median(v)), 2), "max": round(v.max(), 2)}
    ends = rel(c[:, 4])
    order = np.argsort(ends)
    out["per_cta"] = [[int(i), int(c[i, 6]), int(c[i, 7]), round(float(ends[i]), 1)] for i in order]
    print(json.dumps(out))
