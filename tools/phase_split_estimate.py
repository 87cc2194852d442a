"""Host estimate of a rejected SMEM design: 128-B columns processed as two half-tiles by
source-row range (low / high rows double-buffered, partial row XORs parked in TMEM between the
halves).  Counts warp-steps, items and shared-port wavefronts per 128-B column for configs 4, 6, 7.
CPU only: python tools/phase_split_estimate.py"""
import sys
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
import numpy as np
from paper_1702_07409_b200 import configs, fsb
for cid in (4, 6, 7):
    c = configs.get(cid)
    g = fsb.Graph.create(c, host_only=True)
    _, _, rp, col = g.csr()
    k, p, n = c["k"], c["p"], c["n"]
    kpad = (k + 63) // 64 * 64
    K = kpad + p
    kh = (K // 2) // 64 * 64
    kh = min(kh, kpad)
    L1 = np.zeros(n, int); L2 = np.zeros(n, int)
    for j in range(n):
        for m in col[rp[j]:rp[j+1]]:
            r = m if m < k else kpad + (m - k)
            if r < kh: L1[j] += 1
            else: L2[j] += 1
    deg = L1 + L2
    for T in (40, 60):
        light = [j for j in range(n) if deg[j] <= T]
        heavy = [j for j in range(n) if deg[j] > T]
        light.sort(key=lambda j: (L1[j] + L2[j], L1[j]))
        steps = 0; items = 0; wavefronts = 0
        for i in range(0, len(light), 4):
            grp = light[i:i+4]
            a, b = max(L1[j] for j in grp), max(L2[j] for j in grp)
            steps += a + b; items += 1
            # wavefronts: real gathers + 1 per padded step (zero row broadcast)
            for ph, Lx in ((a, L1), (b, L2)):
                for e in range(ph):
                    act = sum(1 for j in grp if Lx[j] > e)
                    wavefronts += act + (1 if act < 4 else 0)
        for j in heavy:   # quad split: 4 octets share the row
            a = -(-L1[j] // 4); b = -(-L2[j] // 4)
            steps += a + b; items += 1
            wavefronts += L1[j] + L2[j] + (a * 4 - L1[j] > 0) + (b * 4 - L2[j] > 0)
        nnz = int(deg.sum())
        print("c%d T=%d kh=%d nnz=%d items=%d warp-steps=%d (gathers/4=%.0f) port-wavefronts=%d (x%.3f nnz)" % (
            cid, T, kh, nnz, items, steps, nnz / 4, wavefronts, wavefronts / nnz))
