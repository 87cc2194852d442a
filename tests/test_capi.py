"""Host-side tests of the C ABI (no GPU): the library loads, exports every symbol of
include/fsb.h, validates its arguments, and its host graph generator reproduces the
oracle's CSR byte for byte -- two independent implementations."""
import os
import re

import numpy as np
import pytest

import oracle
from paper_1702_07409_b200 import configs, fsb

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "fsb.h")).read()
    return sorted(set(re.findall(r"FSB_API\s+[\w\s\*]+?\b(fs_\w+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    import ctypes
    L = fsb.lib()
    declared = _declared_symbols()
    assert len(declared) >= 10
    assert sorted(fsb.EXPORTS) == declared
    for name in declared:
        assert hasattr(L, name), name
        assert ctypes.cast(getattr(L, name), ctypes.c_void_p).value
    assert "sm_100a" in fsb.version()


@pytest.mark.parametrize("cid", [1, 2, 3, 4, 5])
def test_library_generator_matches_oracle(cid):
    """P2: CSR equality, library (C++) vs oracle (C), all five configs."""
    c = configs.get(cid)
    g = fsb.Graph.create(c, host_only=True)
    o = oracle.generate_graph(c)
    pre_rp, pre_c, lt_rp, lt_c = g.csr()
    assert np.array_equal(lt_rp, o.lt_row_ptr) and np.array_equal(lt_c, o.lt_col)
    if c["p"]:
        assert np.array_equal(pre_rp, o.pre_row_ptr) and np.array_equal(pre_c, o.pre_col)
    inf = g.info()
    assert inf["lt_nnz"] == o.nnz and inf["max_degree"] == int(np.diff(o.lt_row_ptr).max())
    assert inf["device"] == -1


@pytest.mark.parametrize("seed", range(6))
def test_library_generator_matches_oracle_random_params(seed):
    rng = np.random.default_rng(seed)
    k = int(rng.integers(1, 300))
    p = int(rng.integers(0, 20))
    dp = int(rng.integers(1, min(k, 5) + 1))
    n = int(rng.integers(1, 400))
    if seed % 2:
        c = dict(k=k, p=p, d_p=dp, n=n, t=64, dist=configs.FINITE, seed=int(rng.integers(0, 2**63)),
                 fin_deg=configs.OMEGA_DEGREES, fin_prob=configs.OMEGA_PROBS)
    else:
        c = dict(k=max(k, 8), p=p, d_p=dp, n=n, t=64, dist=configs.RSD, seed=int(rng.integers(0, 2**63)),
                 rsd_c=0.1, rsd_delta=0.1)
    try:
        o = oracle.generate_graph(c)
    except ValueError:
        with pytest.raises(fsb.FsError):
            fsb.Graph.create(c, host_only=True)
        return
    g = fsb.Graph.create(c, host_only=True)
    a = g.csr()
    for x, y in zip(a, (o.pre_row_ptr, o.pre_col, o.lt_row_ptr, o.lt_col)):
        if c["p"] or len(y) > 1:
            assert np.array_equal(x, y)


def test_from_csr_roundtrip_and_validation():
    c = configs.get(2)
    g = fsb.Graph.create(c, host_only=True)
    pre_rp, pre_c, lt_rp, lt_c = g.csr()
    g2 = fsb.Graph.from_csr(c, pre_rp, pre_c, lt_rp, lt_c, host_only=True)
    for x, y in zip(g2.csr(), (pre_rp, pre_c, lt_rp, lt_c)):
        assert np.array_equal(x, y)
    bad = lt_c.copy()
    bad[1] = bad[0]                      # duplicate in row 0
    with pytest.raises(fsb.FsError) as e:
        fsb.Graph.from_csr(c, pre_rp, pre_c, lt_rp, bad, host_only=True)
    assert e.value.status == fsb.FS_EINVAL
    bad = lt_c.copy()
    bad[0] = c["k"] + c["p"]             # out of range
    with pytest.raises(fsb.FsError):
        fsb.Graph.from_csr(c, pre_rp, pre_c, lt_rp, bad, host_only=True)
    bad = pre_c.copy()
    bad[0] = c["k"]                      # precode index must be a data index
    with pytest.raises(fsb.FsError):
        fsb.Graph.from_csr(c, pre_rp, bad, lt_rp, lt_c, host_only=True)


@pytest.mark.parametrize("override,status", [
    (dict(k=0), fsb.FS_EINVAL),
    (dict(n=0), fsb.FS_EINVAL),
    (dict(t=100), fsb.FS_EINVAL),
    (dict(t=0), fsb.FS_EINVAL),
    (dict(p=5, d_p=0), fsb.FS_EINVAL),
    (dict(p=5, d_p=2000), fsb.FS_EINVAL),
    (dict(rsd_c=0.0), fsb.FS_EDIST),
    (dict(rsd_delta=1.5), fsb.FS_EDIST),
    (dict(dist=7), fsb.FS_EDIST),
])
def test_param_validation(override, status):
    c = configs.get(2, **override)
    with pytest.raises(fsb.FsError) as e:
        fsb.Graph.create(c, host_only=True)
    assert e.value.status == status


@pytest.mark.parametrize("deg,prob", [
    ((1, 2, 2), (0.3, 0.3, 0.4)),        # not strictly increasing
    ((0, 2), (0.5, 0.5)),                # degree 0
    ((1, 2), (0.5, 0.6)),                # does not sum to 1
    ((1, 2), (-0.1, 1.1)),               # negative weight
    ((), ()),                            # empty support
])
def test_finite_distribution_validation(deg, prob):
    c = configs.get(3, fin_deg=deg, fin_prob=prob)
    with pytest.raises(fsb.FsError) as e:
        fsb.Graph.create(c, host_only=True)
    assert e.value.status == fsb.FS_EDIST


def test_baseline_omega_sum_passes():
    """The BASELINE Omega sums to 0.999998: inside the 1e-5 tolerance (reading R9)."""
    assert abs(sum(configs.OMEGA_PROBS) - 1) < 1e-5
    fsb.Graph.create(configs.get(3), host_only=True)


def test_host_only_graph_refuses_encode():
    import ctypes
    g = fsb.Graph.create(configs.get(1), host_only=True)
    st = fsb.lib().fs_encode(g._h, ctypes.c_void_p(16), None, ctypes.c_void_p(16), 0, 1, None)
    assert st == fsb.FS_EUNSUPPORTED
    assert b"host-only" in fsb.lib().fs_last_error()
    buf = (ctypes.c_uint8 * 64)()
    st = fsb.lib().fs_encode_host(g._h, 1, buf, 0, None, 0, buf, 0, 0, None)
    assert st == fsb.FS_EUNSUPPORTED
    assert fsb.lib().fs_encode_host(None, 1, buf, 0, None, 0, buf, 0, 0, None) == fsb.FS_EINVAL


def test_schedule_balance():
    """The SMEM schedule covers every edge and balances warps: padding (parity + length) below 15%,
    and the heaviest warp's LPT cost (gather steps + 12 per item, the builder's cost model) within
    25% of the mean (items carry 16 rows, ~3.6 per warp on config 4, so the deal is coarse)."""
    for cid in (2, 4):
        g = fsb.Graph.create(configs.get(cid), host_only=True)
        inf = g.info()
        assert inf["smem_eligible"] == 1
        # steps are per group (16 per warp, W warps)
        words, cont_base, info, _, _ = g.schedule()
        W = len(info)
        assert inf["sched_steps_avg"] * W * 16 >= inf["lt_nnz"] - W * 16
        assert inf["sched_steps_avg"] * W * 16 <= 1.15 * inf["lt_nnz"] + W * 16
        heads = words.reshape(-1, 16, 4)[:cont_base]
        cost = []
        for w in range(W):
            nitems, hoff, _ = (int(x) for x in info[w])
            L = [(int(heads[hoff + i, 0, 0]) >> 16) & 0x3FFF for i in range(nitems)]
            assert sum(L) <= inf["sched_steps_max"]
            cost.append(sum(L) + 12 * nitems)
        assert max(cost) <= 1.25 * (sum(cost) / W)


def _simulate_schedule(g, c):
    """Replays the SMEM kernel's consumption of its two chunk streams (fsb_smem_encode) on the
    host: returns {row: sorted tile rows}.  Asserts that every item's control half is identical
    in the 16 groups (the kernel's dispatch and split shuffles rely on it) and the bank rule: in
    every step, groups g and g^2 (the two halves of a pair: half 0 = bit 1 of g clear) read tile
    rows of opposite parity."""
    G = 16
    words, cont_base, info, kpad, z0 = g.schedule()
    words = words.astype(np.int64)
    lo, hi = words & 0x7FF, words >> 21
    slots = np.stack([lo, hi], axis=1).reshape(-1, G, 8)   # [chunk, group, slot position]
    chunks = words.reshape(-1, G, 4)                       # [chunk, group, word]
    heads, conts = chunks[:cont_base], slots[cont_base:]
    head_slots = slots[:cont_base]
    assert np.all((words[cont_base * 4 * G:] >> 11) & 0x3FF == 0)
    rows = {}
    hpos, cpos = 0, 0
    zeros = (z0, z0 + 1)
    for w in range(len(info)):
        nitems, hoff, coff = (int(x) for x in info[w])
        assert (hoff, coff) == (hpos, cpos)
        for _ in range(nitems):
            head = heads[hpos]
            hslots = head_slots[hpos]
            hpos += 1
            pflag = [bool(int(head[h, 1]) & (1 << 11)) for h in range(G)]
            # bits 11..20 of slot words are zero, except the pair-split flag (word 1, bit 11)
            assert all(((int(head[h, j]) >> 11) & 0x3FF) == (1 if j == 1 and pflag[h] else 0)
                       for h in range(G) for j in (1, 2, 3))
            ctrls = set(int(head[h, 0]) >> 16 for h in range(G))
            assert len(ctrls) == 1, "non-uniform item control"
            ctrl = ctrls.pop()
            L, split, psplit = ctrl & 0x3FFF, bool(ctrl & 0x8000), bool(ctrl & 0x4000)
            assert psplit == any(pflag)
            assert L >= 1
            per = [[] for _ in range(G)]
            for e in range(L):
                vals = []
                for h in range(G):
                    if e < 6:
                        v = int(hslots[h, 2 + e])
                    else:
                        f = e - 6
                        v = int(conts[cpos + f // 8, h, f % 8])
                    vals.append(v)
                    if v not in zeros:
                        per[h].append(v)
                for h in range(G):
                    if not h & 2:
                        assert (vals[h] & 1) != (vals[h ^ 2] & 1), "bank rule"
            cpos += 0 if L <= 6 else (L - 6 + 7) // 8
            outs = [int(head[h, 0]) & 0xFFFF for h in range(G)]
            for h0 in range(G):   # pair-split: half 0 (group h0) stores both halves' parts
                if not h0 & 2 and pflag[h0]:
                    h1 = h0 ^ 2
                    assert pflag[h1] and outs[h1] == 0xFFFF and outs[h0] != 0xFFFF
                    per[h0] = per[h0] + per[h1]
                    per[h1] = []
            if split:
                assert len(set(outs)) == 1 and outs[0] != 0xFFFF
                assert outs[0] not in rows
                rows[outs[0]] = sorted(sum(per, []))
            else:
                for h in range(G):
                    if outs[h] == 0xFFFF:
                        assert not per[h]
                        continue
                    assert outs[h] not in rows
                    rows[outs[h]] = sorted(per[h])
    # prefetch padding after each stream
    assert len(heads) - hpos == 2 and np.all(heads[hpos:] == 0)
    assert len(conts) - cpos == 2 and np.all(conts[cpos:] == 0)
    return rows, kpad


@pytest.mark.parametrize("cid", [1, 2, 4, 6, 7])
def test_smem_schedule_covers_every_edge(cid):
    c = configs.get(cid)
    g = fsb.Graph.create(c, host_only=True)
    rows, kpad = _simulate_schedule(g, c)
    _, _, lt_rp, lt_c = g.csr()
    assert sorted(rows) == list(range(c["n"]))
    k = c["k"]
    for j in range(c["n"]):
        want = sorted(m if m < k else kpad + (m - k) for m in lt_c[lt_rp[j]:lt_rp[j + 1]])
        assert rows[j] == want


def _replay_windows(hdr, ent, n):
    """Host replay of the GLOBAL window kernel (fsb_lt_win) over fs_graph_windows: the rows each
    window produces, in order, each as its list of source indices."""
    rows = []
    for w in range(hdr.shape[0]):
        r0, nb = int(hdr[w, 0]), int(hdr[w, 1])
        r1 = int(hdr[w + 1, 0]) if w + 1 < hdr.shape[0] else n
        assert 1 <= nb and 4 * nb <= ent.shape[1]
        assert 1 <= r1 - r0 <= 12
        assert r0 == (len(rows))                   # windows tile the rows in order
        cur = []
        for e in range(4 * nb):
            f = int(ent[w, e])
            if f & (1 << 30):                      # skip slot: only before the first edge
                assert e < 4 and not cur and not (f & (1 << 31))
                continue
            cur.append(f & 0x7FFFFFFF)
            if f & (1 << 31):
                rows.append(cur)
                cur = []
        assert not cur                             # the window ends on a row end
        assert np.all(ent[w, 4 * nb:] == 0)
        assert len(rows) == r1
    return rows


@pytest.mark.parametrize("cid", [3, 5])
def test_lt_windows_cover_every_edge(cid):
    """fs_graph_windows: replaying the window kernel's walk yields every LT row exactly once, in
    order, with exactly its CSR neighbours (bit-exact encode needs nothing more)."""
    c = configs.get(cid)
    g = fsb.Graph.create(c, host_only=True)
    assert g.info()["lt_windows"] > 0
    hdr, ent = g.windows()
    _, _, lt_rp, lt_c = g.csr()
    rows = _replay_windows(hdr, ent, c["n"])
    assert len(rows) == c["n"]
    for j in range(c["n"]):
        assert rows[j] == list(lt_c[lt_rp[j]:lt_rp[j + 1]])


def test_lt_windows_absent_for_heavy_rows():
    """A graph with a row of more than 93 edges has no windows (the band kernels run it)."""
    c = configs.get(4)                             # RSD, max degree 251
    g = fsb.Graph.create(c, host_only=True)
    assert g.info()["max_degree"] > 93 and g.info()["lt_windows"] == 0
    with pytest.raises(fsb.FsError):
        g.windows()


ARRAY_CFGS = [
    dict(k=962, p=74, d_p=0, n=1280, t=4096, dist=configs.RSD, rsd_c=0.1, rsd_delta=0.05, seed=6),
    dict(k=837, p=93, d_p=0, n=1100, t=128, dist=configs.FINITE, seed=7,
         fin_deg=configs.OMEGA_DEGREES, fin_prob=configs.OMEGA_PROBS),
    dict(k=3, p=3, d_p=0, n=9, t=16, dist=configs.FINITE, seed=8, fin_deg=(1, 2), fin_prob=(0.5, 0.5)),
]


@pytest.mark.parametrize("i", range(len(ARRAY_CFGS)))
def test_array_precode_library_matches_oracle(i):
    """NEXT-2: the library's Alg 2 precode + LT rows are byte-identical to the oracle's."""
    c = dict(ARRAY_CFGS[i], precode="array")
    g = fsb.Graph.create(c, host_only=True)
    go = oracle.generate_graph(c)
    pre_rp, pre_c, lt_rp, lt_c = g.csr()
    assert np.array_equal(pre_rp, go.pre_row_ptr) and np.array_equal(pre_c, go.pre_col)
    assert np.array_equal(lt_rp, go.lt_row_ptr) and np.array_equal(lt_c, go.lt_col)
    inf = g.info()
    assert inf["pre_nnz"] == len(pre_c) and inf["d_p"] == int(pre_rp[1])


def test_array_precode_validation():
    for k, p in [(1000, 20), (990, 110), (500, 100)]:   # P does not divide k, or k' > P
        c = dict(ARRAY_CFGS[0], k=k, p=p, precode="array")
        with pytest.raises(fsb.FsError) as e:
            fsb.Graph.create(c, host_only=True)
        assert e.value.status == fsb.FS_EINVAL
    # a CSR whose check reads a LATER check is rejected; the Alg 2 CSR round-trips
    c = dict(ARRAY_CFGS[0], precode="array")
    g = fsb.Graph.create(c, host_only=True)
    pre_rp, pre_c, lt_rp, lt_c = g.csr()
    g2 = fsb.Graph.from_csr(c, pre_rp, pre_c, lt_rp, lt_c, host_only=True)
    assert all(np.array_equal(a, b) for a, b in zip(g.csr(), g2.csr()))
    bad = pre_c.copy()
    bad[0] = c["k"] + 5                                  # check 0 reading check 5
    with pytest.raises(fsb.FsError):
        fsb.Graph.from_csr(c, pre_rp, bad, lt_rp, lt_c, host_only=True)


@pytest.mark.parametrize("cid,files", [(1, 13), (2, 10), (4, 8), (5, 12), (6, 4), (3, 1)])
def test_per_file_streams_library_matches_oracle(cid, files):
    """NEXT-4 / R17: per-file seed streams seed + i, library (threaded) == oracle."""
    c = dict(configs.get(cid), files=files)
    g = fsb.Graph.create(c, host_only=True)
    o = oracle.generate_graph(c)
    a = g.csr()
    for x, y in zip(a, (o.pre_row_ptr, o.pre_col, o.lt_row_ptr, o.lt_col)):
        assert np.array_equal(x, y)
    assert g.info()["max_degree"] == int(np.diff(o.lt_row_ptr).max())


def test_per_file_streams_reject_non_divisor():
    c = dict(configs.get(1), files=7)          # 7 does not divide n = 130
    with pytest.raises(fsb.FsError):
        fsb.Graph.create(c, host_only=True)
    with pytest.raises(ValueError):
        oracle.generate_graph(c)


@pytest.mark.parametrize("pw", ["5", "7"])
def test_smem_schedule_with_more_precode_warps(pw):
    """FSB_PRECODE_WARPS (read once per process, so a fresh pytest process): the schedule is dealt
    over 27 - pw consumer warps and still covers every edge exactly once under the bank rule."""
    import os
    import subprocess
    import sys as _sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, FSB_PRECODE_WARPS=pw)
    r = subprocess.run([_sys.executable, "-m", "pytest", "-q", "-m", "not gpu",
                        os.path.join(root, "tests", "test_capi.py") + "::test_smem_schedule_covers_every_edge"],
                       capture_output=True, text=True, env=env, timeout=600, cwd=root)
    assert r.returncode == 0, (r.stdout + r.stderr)[-3000:]
    code = ("from paper_1702_07409_b200 import configs, fsb; "
            "g = fsb.Graph.create(configs.get(6), host_only=True); print(g.schedule()[2].shape[0])")
    r = subprocess.run([_sys.executable, "-c", code], capture_output=True, text=True, env=env, timeout=300, cwd=root)
    assert r.returncode == 0 and int(r.stdout.strip()) == 27 - int(pw), r.stdout + r.stderr
