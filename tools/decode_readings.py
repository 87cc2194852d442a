"""Reading R22: the decoder's BP over the union of LT and precode equations run to
a fixpoint, against the literal reading of PAPER.md:134 ("runs BP algorithm at most twice (once
for the outer graph code and if need be, additional one for the inner Array LDPC precode)"):
Algorithm 1 on the received LT equations to its own fixpoint, then BP on the precode equations
to its fixpoint, and stop.

Graph-only (which symbols are recovered); CPU; calls only oracle/ for the graphs.  Prints one
JSON line per (config, reception) with the recovered counts of both readings.
Usage: python tools/decode_readings.py [trials]
"""
import json
import os
import sys
from collections import deque

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_1702_07409_b200 import configs  # noqa: E402


def peel(eqs, K, known=None):
    """Queue-based peeling closure of a list of equations (member lists) over K unknowns: an
    equation with exactly one unknown member recovers it.  The closure is independent of the
    order equations are visited in.  Returns bool[K] recovered."""
    rec = np.zeros(K, bool) if known is None else known.copy()
    by_sym = [[] for _ in range(K)]
    left = np.zeros(len(eqs), np.int64)
    for e, mem in enumerate(eqs):
        for m in mem:
            by_sym[m].append(e)
        left[e] = sum(1 for m in mem if not rec[m])
    q = deque(e for e in range(len(eqs)) if left[e] == 1)
    while q:
        e = q.popleft()
        if left[e] != 1:
            continue
        x = next(m for m in eqs[e] if not rec[m])
        rec[x] = True
        for f in by_sym[x]:
            left[f] -= 1
            if left[f] == 1:
                q.append(f)
    return rec


def equations(g, recv):
    lt = [list(g.lt_row(j)) for j in range(g.n) if recv[j]]
    pre = [list(g.pre_row(i)) + [g.k + i] for i in range(g.p)]
    return lt, pre


def union_fixpoint(g, recv):
    lt, pre = equations(g, recv)
    return peel(lt + pre, g.K)


def literal_two_pass(g, recv):
    lt, pre = equations(g, recv)
    rec = peel(lt, g.K)
    return peel(pre, g.K, rec) if pre else rec


def main():
    trials = int(sys.argv[1]) if len(sys.argv) > 1 else 5
    rng = np.random.default_rng(2017)
    for cid in (1, 2, 3, 4, 5):
        g = oracle.generate_graph(configs.get(cid))
        for frac in (1.0, 0.95):
            for tr in range(1 if frac == 1.0 else trials):
                recv = np.ones(g.n, bool) if frac == 1.0 else rng.random(g.n) < frac
                u, l = union_fixpoint(g, recv), literal_two_pass(g, recv)
                print(json.dumps({"config": cid, "reception": frac, "trial": tr, "K": g.K, "k": g.k,
                                  "union_fixpoint": int(u.sum()), "literal_two_pass": int(l.sum()),
                                  "union_data": int(u[:g.k].sum()), "literal_data": int(l[:g.k].sum())}))
                sys.stdout.flush()


if __name__ == "__main__":
    main()
