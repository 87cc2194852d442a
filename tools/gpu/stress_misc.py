"""Stress test on random small codes: fs_encode_range over random row x column blocks, the
inactivation-completed decode, repair with the library's check data, and fs_encode_host (random
stripe and chunk counts) -- every result against the oracle (encode bytes, BP + Gauss-Jordan
decode bytes, repair plan replayed by the oracle).

    python tools/gpu/stress_misc.py FIRST_SEED END_SEED
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
from paper_1702_07409_b200 import configs, fsb, inputs  # noqa: E402

bad = {"range": 0, "decode": 0, "repair": 0, "host": 0}
ran = {"range": 0, "decode": 0, "repair": 0, "host": 0}
for seed in range(int(sys.argv[1]), int(sys.argv[2])):
    rng = np.random.default_rng(31000 + seed)
    k = int(rng.integers(1, 300))
    p = int(rng.integers(0, 16))
    n = int(k + p + rng.integers(0, 120))
    t = int(rng.choice([64, 128, 320, 1024]))
    cfg = dict(name="r", k=k, p=p, d_p=int(rng.integers(1, min(k, 5) + 1)) if p else 0, n=n, t=t, stripes=1,
               dist=configs.FINITE, seed=int(rng.integers(1, 1 << 40)),
               fin_deg=configs.OMEGA_DEGREES, fin_prob=configs.OMEGA_PROBS)
    go = oracle.generate_graph(cfg)
    D = inputs.stripe_data(cfg).numpy()
    C, Y = oracle.encode(go, D)
    g = fsb.Graph.create(cfg)
    d = torch.from_numpy(D[0]).cuda()
    # encode_range: a random rows x columns block
    r0, r1 = sorted(int(x) for x in rng.integers(0, n + 1, 2))
    c0, c1 = sorted(16 * int(x) for x in rng.integers(0, t // 16 + 1, 2))
    out = torch.full((max(r1 - r0, 1), t), 0x5A, dtype=torch.uint8, device="cuda")
    chk = torch.empty((p, t), dtype=torch.uint8, device="cuda") if p else None
    if r1 > r0:
        g.encode_range(d, chk, out, r0, r1, c0, c1)
        torch.cuda.synchronize()
        o = out.cpu().numpy()
        ok = np.array_equal(o[:, c0:c1], Y[0][r0:r1, c0:c1]) and (o[:, :c0] == 0x5A).all() and (o[:, c1:] == 0x5A).all()
        ran["range"] += 1
        bad["range"] += 0 if ok else 1
        if not ok:
            print("RANGE mismatch", seed, r0, r1, c0, c1)
    # decode with elimination
    recv = rng.random(n) < float(rng.uniform(0.6, 1.0))
    plan = fsb.DecodePlan(g, recv, eliminate=True)
    Yd = torch.from_numpy(Y).cuda()
    Yd[:, ~torch.from_numpy(recv)] = 0x77
    inter = torch.zeros((1, g.K, t), dtype=torch.uint8, device="cuda")
    plan.decode(Yd, inter)
    torch.cuda.synchronize()
    oI, ostate = oracle.decode(go, recv, Y[0], use_elim=True)
    st, _ = plan.state()
    rec = ostate != 0
    ok = np.array_equal(st != 0, rec) and np.array_equal(inter[0].cpu().numpy()[rec], oI[rec])
    ran["decode"] += 1
    bad["decode"] += 0 if ok else 1
    if not ok:
        print("DECODE mismatch", seed)
    # repair with the library's check data, replayed by the oracle's repair
    ch = fsb.Checks.create(g, 3)
    arr = ch.data()
    er = rng.choice(n, int(rng.integers(1, 4)), replace=False)
    mask = np.zeros(n, bool)
    mask[er] = True
    rp = fsb.RepairPlan(g, ch, mask)
    cod = torch.from_numpy(Y).cuda()
    cod[:, torch.from_numpy(mask).cuda()] = 0xEE
    rp.repair(cod)
    torch.cuda.synchronize()
    y, _, unk = oracle.repair(go, arr, er, np.where(mask[:, None], 0, Y[0]))
    got = cod[0].cpu().numpy()
    want = np.where(np.isin(np.arange(n), list(unk))[:, None], 0xEE, y)
    ok = np.array_equal(got, want)
    ran["repair"] += 1
    bad["repair"] += 0 if ok else 1
    if not ok:
        print("REPAIR mismatch", seed)
    # fs_encode_host: random stripe count and chunking, host buffers (pinned or not)
    S2 = int(rng.integers(1, 6))
    c2 = dict(cfg, stripes=S2)
    D2 = inputs.stripe_data(c2).numpy()
    C2, Y2 = oracle.encode(go, D2)
    pin = bool(rng.integers(0, 2))
    hd = torch.from_numpy(D2).contiguous()
    hd = hd.pin_memory() if pin else hd
    hc = torch.full((S2, p, t), 0xA5, dtype=torch.uint8) if p else None
    hy = torch.full((S2, n, t), 0x5A, dtype=torch.uint8)
    if pin:
        hc = hc.pin_memory() if p else None
        hy = hy.pin_memory()
    g.encode_host(hd, hc, hy, chunks=int(rng.integers(0, 9)))
    torch.cuda.synchronize()
    ok = np.array_equal(hy.numpy(), Y2) and (not p or np.array_equal(hc.numpy(), C2))
    ran["host"] += 1
    bad["host"] += 0 if ok else 1
    if not ok:
        print("HOST mismatch", seed, S2)
print("done:", {key: "%d/%d bad" % (bad[key], ran[key]) for key in ran})
