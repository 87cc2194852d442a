"""Stress test: random graphs through the SMEM kernel (paired and unpaired tiles) vs the oracle.

    python tools/gpu/stress_smem.py FIRST_SEED END_SEED
"""
import sys, numpy as np, torch
sys.path.insert(0, "/root/repo")
import oracle
from paper_1702_07409_b200 import configs, fsb, inputs
bad = 0
ran = 0
for seed in range(int(sys.argv[1]), int(sys.argv[2])):
    rng = np.random.default_rng(7000 + seed)
    k = int(rng.integers(1, 1800)); p = int(rng.integers(0, 60)); d_p = int(rng.integers(1, min(k, 6) + 1)) if p else 0
    n = int(rng.integers(1, 2500)); t = int(rng.choice([64, 128, 192, 256, 640, 4096]))
    if rng.random() < 0.5:
        cfg = dict(k=k, p=p, d_p=d_p, n=n, t=t, dist=configs.RSD, rsd_c=float(rng.uniform(0.03, 0.3)),
                   rsd_delta=float(rng.uniform(0.01, 0.5)), seed=int(rng.integers(1, 1 << 40)))
    else:
        cfg = dict(k=k, p=p, d_p=d_p, n=n, t=t, dist=configs.FINITE, seed=int(rng.integers(1, 1 << 40)),
                   fin_deg=configs.OMEGA_DEGREES, fin_prob=configs.OMEGA_PROBS)
    S = int(rng.choice([1, 37, 300])) if k * t <= (1 << 20) else 1
    cfg["stripes"] = S
    try:
        go = oracle.generate_graph(cfg)
    except ValueError:
        continue
    D = inputs.stripe_data(cfg).numpy()
    C, Y = oracle.encode(go, D)
    g = fsb.Graph.create(cfg)
    if not g.info()["smem_eligible"]:
        continue
    g.set_variant(fsb.VARIANT_SMEM)
    d = torch.from_numpy(D).cuda()
    chk = torch.empty((S, p, t), dtype=torch.uint8, device="cuda") if p else None
    cod = torch.empty((S, n, t), dtype=torch.uint8, device="cuda")
    g.encode_stripes(d, chk, cod)
    torch.cuda.synchronize()
    ran += 1
    ok = np.array_equal(cod.cpu().numpy(), Y) and (not p or np.array_equal(chk.cpu().numpy(), C))
    if not ok:
        bad += 1
        print("MISMATCH seed", seed, cfg)
print("done: %d SMEM cases, %d mismatches" % (ran, bad))
