"""NEXT-3: repair / update / degraded read (§2.5-2.9, Alg 4 CGA).

CPU (not gpu): the oracle's CGA and repair semantics pinned by a hand-executed Alg 4 example
(tests/golden/cga_k3_n5.txt), the paper's check-data example and Eq 4
(PAPER.md:250-257), and algebraic invariants that hold for any correct execution (B_out = B L,
every Group #3 set XORs to zero and every Group #2 set to its symbol on encoded data, repaired
bytes equal the encoder's); then the library (C++, sparse CGA) against the oracle (dense C),
check data and repair plans element by element.  GPU: fs_repair through the C ABI vs the
oracle's repair, bit-exact.
"""
import os

import numpy as np
import pytest
import torch

import oracle
from paper_1702_07409_b200 import configs, fsb, inputs

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _graph_from_rows(k, rows, t=64):
    cfg = dict(k=k, p=0, n=len(rows), t=t)
    rp = np.cumsum([0] + [len(r) for r in rows]).astype(np.int32)
    return oracle.Graph(cfg, np.zeros(1, np.int32), np.zeros(0, np.int32), rp,
                        np.array(sum([sorted(r) for r in rows], []), np.int32))


def _load_golden():
    rows, data, sweeps = [], None, None
    for line in open(os.path.join(GOLD, "cga_k3_n5.txt")):
        if line.startswith("#") or not line.strip():
            continue
        key, *vals = line.split()
        if key == "lt":
            rows.append([int(v) for v in vals])
        elif key == "data":
            data = [int(v) for v in vals]
        elif key == "sweeps":
            sweeps = int(vals[0])
    return rows, data, sweeps


def _small_cfgs():
    out = [configs.get(1), dict(configs.get(1), files=10), dict(configs.get(1), seed=5),
           dict(configs.get(1), files=2)]
    rng = np.random.default_rng(11)
    for i in range(6):
        k = int(rng.integers(8, 120))
        p = int(rng.integers(0, 12))
        n = int(k + p + rng.integers(1, 60))
        if i % 2:
            out.append(dict(name="rand%d" % i, k=k, p=p, d_p=min(3, k), n=n, t=64, stripes=1, dist=configs.FINITE,
                            seed=int(rng.integers(0, 2 ** 63)), fin_deg=configs.OMEGA_DEGREES,
                            fin_prob=configs.OMEGA_PROBS))
        else:
            out.append(dict(name="rand%d" % i, k=k, p=p, d_p=min(3, k), n=n, t=64, stripes=1, dist=configs.RSD,
                            seed=int(rng.integers(0, 2 ** 63)), rsd_c=0.1, rsd_delta=0.5))
    return out


# ----------------------------------------------------------------------- oracle pins (CPU)
def test_cga_golden_hand_example():
    rows, data, sweeps = _load_golden()
    g = _graph_from_rows(3, rows)
    B, L, sw = oracle.cga(g)
    assert sw == sweeps
    assert [sorted(np.nonzero(B[:, j])[0].tolist()) for j in range(5)] == [[], [1], [], [2], [0]]
    assert [sorted(np.nonzero(L[:, j])[0].tolist()) for j in range(5)] == [[0, 1, 4], [1], [1, 2, 3, 4], [3], [4]]
    arr, _ = oracle.check_data(g)
    assert arr.tolist() == data


def test_check_data_format_paper_example():
    """'0 4 13 56 17 66 1 19 2 11 13 0 2 39 88' = Group #3 {13,56,17,66},
    Group #2 (19; {11,13}), Group #3 {39,88}."""
    arr = [0, 4, 13, 56, 17, 66, 1, 19, 2, 11, 13, 0, 2, 39, 88]
    assert oracle.parse_check_data(arr) == [(3, -1, [13, 56, 17, 66]), (2, 19, [11, 13]), (3, -1, [39, 88])]
    with pytest.raises(ValueError):
        oracle.parse_check_data([2, 1, 0])


def test_set_xor_paper_eq4():
    """the check #1 group (D0, D1, D2) and Eqs (1)-(3) give Eq (4)."""
    assert oracle.set_xor([0, 1, 2], [1, 12, 17, 20, 99], [0, 21, 99]) == {2, 12, 17, 20, 21}


@pytest.mark.parametrize("i", range(10))
def test_cga_invariants(i):
    """Any correct execution of Alg 4's column operations keeps B_out = B L (mod 2), never raises a
    column's weight, and yields local sets that hold on encoded data."""
    c = _small_cfgs()[i]
    g = oracle.generate_graph(c)
    B, L, _ = oracle.cga(g)
    B0 = np.zeros((g.K, g.n), dtype=np.int64)
    for j in range(g.n):
        B0[g.lt_row(j), j] = 1
    assert np.array_equal((B0 @ L.astype(np.int64)) % 2, B)
    assert (B.sum(0) <= B0.sum(0)).all()
    D = inputs.stripe_data(c).numpy()[0]
    C, Y = oracle.encode(g, D)
    I = np.concatenate([D, C]) if g.p else D
    arr, _ = oracle.check_data(g, oracle.CHECKS_M1 | oracle.CHECKS_M2)
    for kind, x, mem in oracle.parse_check_data(arr):
        acc = np.bitwise_xor.reduce(Y[mem], axis=0)
        if kind == 3:
            assert not acc.any()
        else:
            assert np.array_equal(acc, I[x])


def test_cga_converges_on_full_rank_c2():
    """The paper's claim (CGA converges whenever B has full rank) on config 2 (RSD
    c=0.05, B of full rank): n-K zero columns and every symbol with exactly one Group #2 set
    (PAPER.md:315)."""
    g = fsb.Graph.create(configs.get(2), host_only=True)
    inf = fsb.Checks.create(g).info()
    assert inf["zero_columns"] >= g.n - g.K and inf["weight1_columns"] == g.K
    xs = [x for kind, x, _ in oracle.parse_check_data(fsb.Checks.create(g).data()) if kind == 2]
    assert sorted(xs) == list(range(g.K))


def test_cga_on_omega_config3():
    """Config 3 is the Omega(x) code.  Its B is NOT of full rank (8 of the
    10,100 symbols are in no LT row; the column space of B determines 10,091 symbols -- oracle
    GF(2) elimination), so PAPER.md:265's premise fails.  CGA still reaches Alg 4's exit test
    (zero_columns >= n-K, reading R19), every Group #2 symbol is one B determines, and the
    Group #2 sets cover all but 5 of the determined symbols."""
    c = configs.get(3)
    g = fsb.Graph.create(c, host_only=True)
    ch = fsb.Checks.create(g)
    inf = ch.info()
    assert inf["zero_columns"] >= g.n - g.K
    go = oracle.generate_graph(c)
    gg = oracle.Graph(dict(k=go.K, p=0, n=go.n, t=8), np.zeros(1, np.int32), np.zeros(0, np.int32),
                      go.lt_row_ptr, go.lt_col)
    _, st = oracle.decode(gg, np.ones(go.n, bool), np.zeros((go.n, 8), np.uint8))
    det = set(np.nonzero(st)[0].tolist())
    xs = [x for kind, x, _ in oracle.parse_check_data(ch.data()) if kind == 2]
    assert len(xs) == len(set(xs)) == inf["weight1_columns"]
    assert set(xs) <= det
    assert len(det) == 10091 and len(xs) == 10086


@pytest.mark.parametrize("i", range(10))
def test_oracle_repair_reproduces_encoder(i):
    c = _small_cfgs()[i]
    g = oracle.generate_graph(c)
    arr, _ = oracle.check_data(g, 3)
    D = inputs.stripe_data(c).numpy()[0]
    _, Y = oracle.encode(g, D)
    rng = np.random.default_rng(i)
    for ne in (1, 2, 5):
        er = rng.choice(g.n, ne, replace=False)
        Yz = Y.copy()
        Yz[er] = 0
        y, _, unk = oracle.repair(g, arr, er, Yz)
        for x in er:
            if x not in unk:
                assert np.array_equal(y[x], Y[x])


# ----------------------------------------------------------------- library vs oracle (CPU)
@pytest.mark.parametrize("i", range(10))
@pytest.mark.parametrize("flags", [0, 3])
def test_library_check_data_matches_oracle(i, flags):
    c = _small_cfgs()[i]
    g = fsb.Graph.create(c, host_only=True)
    ch = fsb.Checks.create(g, flags)
    arr, sw = oracle.check_data(oracle.generate_graph(c), flags)
    assert np.array_equal(ch.data(), arr)
    assert ch.info()["sweeps"] == sw


def test_library_check_data_golden():
    rows, data, sweeps = _load_golden()
    cfg = dict(k=3, p=0, d_p=0, n=5, t=64, dist=configs.FINITE, seed=1, fin_deg=(1,), fin_prob=(1.0,))
    rp = np.cumsum([0] + [len(r) for r in rows]).astype(np.int32)
    g = fsb.Graph.from_csr(cfg, np.zeros(1, np.int32), np.zeros(0, np.int32), rp,
                           np.array(sum(rows, []), np.int32), host_only=True)
    ch = fsb.Checks.create(g)
    assert ch.data().tolist() == data and ch.info()["sweeps"] == sweeps


def _canon_rows(level_ptr, target, src_ptr, src):
    """{(level, target kind, index, sorted sources with pairs cancelled)}."""
    out = set()
    for L in range(len(level_ptr) - 1):
        for r in range(level_ptr[L], level_ptr[L + 1]):
            tg = int(target[r])
            s = [int(v) & 0x3FFFFFFF for v in src[src_ptr[r]:src_ptr[r + 1]]]
            out.add((L + 1, "c" if tg & (1 << 30) else "i", tg & 0x3FFFFFFF, tuple(sorted(oracle.set_xor(*[[v] for v in s])))))
    return out


def _oracle_rows(g, arr, er, want=()):
    steps, unk, missing = oracle.repair_plan(g, arr, er, want)
    level = {}
    out = set()
    for kind, x, srcs in steps:
        L = 1 + max([level.get(c, 0) for c in srcs] + [0])
        if kind == "c":
            level[x] = L
        out.add((L, kind, x, tuple(sorted(srcs))))
    return out, unk, missing


@pytest.mark.parametrize("i", range(10))
def test_library_repair_plan_matches_oracle(i):
    c = _small_cfgs()[i]
    g = fsb.Graph.create(c, host_only=True)
    og = oracle.generate_graph(c)
    ch = fsb.Checks.create(g, 3)
    arr = ch.data()
    rng = np.random.default_rng(100 + i)
    for ne in (1, 3, max(1, g.n // 10)):
        er = rng.choice(g.n, ne, replace=False)
        mask = np.zeros(g.n, bool)
        mask[er] = True
        want = rng.choice(g.K, min(5, g.K), replace=False)
        rp = fsb.RepairPlan(g, ch, mask, want=want, host_only=True)
        got = _canon_rows(*rp.rows())
        exp, unk, missing = _oracle_rows(og, arr, er, want)
        assert got == exp
        inf = rp.info()
        assert inf["unrepaired"] == len(unk) and inf["want_missing"] == len(missing)
        assert inf["repaired"] == ne - len(unk)


def test_extend_keeps_rows_and_matches_oracle():
    """Update: rows of the original files unchanged, new files from their own
    streams; library == oracle."""
    for c in (dict(configs.get(1), files=10), configs.get(1), dict(configs.get(4), files=8)):
        g = fsb.Graph.create(c, host_only=True)
        g2 = g.extend(2, host_only=True)
        a, b = g.csr(), g2.csr()
        assert np.array_equal(b[2][:g.n + 1], a[2]) and np.array_equal(b[3][:len(a[3])], a[3])
        o = oracle.generate_graph(g2.cfg)
        assert np.array_equal(b[2], o.lt_row_ptr) and np.array_equal(b[3], o.lt_col)
        assert g2.n == g.n + 2 * (g.n // max(1, c.get("files", 1)))


def _omega_small(seed=1, k=100, p=4, n=150, files=5):
    return dict(name="omega_small", k=k, p=p, d_p=3, n=n, t=64, stripes=1, dist=configs.FINITE, seed=seed,
                fin_deg=configs.OMEGA_DEGREES, fin_prob=configs.OMEGA_PROBS, files=files)


def test_update_via_repair_oracle():
    """Update without the data: the new symbols of the extended code, from the
    ORIGINAL code's check data (Group #2 sets), equal the encoder's new rows.  A small Omega(x)
    code where CGA converges: every new symbol is rebuilt."""
    c = _omega_small()
    og = oracle.generate_graph(c)
    arr, _ = oracle.check_data(og, 3)
    c6 = dict(c, n=c["n"] + c["n"] // 5, files=6)
    og6 = oracle.generate_graph(c6)
    D = inputs.stripe_data(c).numpy()[0]
    _, Y6 = oracle.encode(og6, D)
    Y = Y6.copy()
    Y[c["n"]:] = 0
    y, _, unk = oracle.repair(og6, arr, range(c["n"], c6["n"]), Y)
    assert not unk
    assert np.array_equal(y, Y6)


def test_checks_from_data_validation():
    g = fsb.Graph.create(configs.get(1), host_only=True)
    ch = fsb.Checks.from_data(g, [0, 4, 13, 56, 17, 66, 1, 19, 2, 11, 13, 0, 2, 39, 88])
    assert ch.info()["group2"] == 1 and ch.info()["group3"] == 2
    for bad in ([2, 1, 0], [0, 0], [0, 3, 1, 2], [1, 500, 1, 3], [0, 1, 130], [0, 1, -1]):
        with pytest.raises(fsb.FsError):
            fsb.Checks.from_data(g, bad)
    with pytest.raises(fsb.FsError):
        fsb.Checks.create(g, 4)


# --------------------------------------------------------------------------- GPU parity
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.gpu
@pytest.mark.parametrize("cid,S,ne", [(1, 1, 3), (1, 7, 1), (2, 3, 13), (2, 1, 1)])
def test_gpu_repair_parity(cid, S, ne):
    _need_gpu()
    c = configs.get(cid)
    g = fsb.Graph.create(c)
    og = oracle.generate_graph(c)
    ch = fsb.Checks.create(g, 3)
    arr = ch.data()
    D = inputs.stripe_data(c, num_stripes=S).numpy()
    _, Y = oracle.encode(og, D)
    rng = np.random.default_rng(cid * 10 + ne)
    er = rng.choice(g.n, ne, replace=False)
    want = rng.choice(g.k, 4, replace=False)
    mask = np.zeros(g.n, bool)
    mask[er] = True
    rp = fsb.RepairPlan(g, ch, mask, want=want)
    cod = torch.from_numpy(Y).cuda()
    cod[:, er] = 0xEE
    inter = torch.full((S, g.K, g.t), 0x77, dtype=torch.uint8, device="cuda")
    rp.repair(cod, inter)
    torch.cuda.synchronize()
    got, gi = cod.cpu().numpy(), inter.cpu().numpy()
    _, _, missing = oracle.repair_plan(og, arr, er, want)
    for s in range(S):
        y, I, unk = oracle.repair(og, arr, er, np.where(mask[:, None], 0, Y[s]), want)
        assert np.array_equal(got[s], np.where(np.isin(np.arange(g.n), list(unk))[:, None], 0xEE, y))
        for r, x in enumerate(want):
            if int(x) in missing:
                assert (gi[s, x] == 0x77).all()
            else:
                assert np.array_equal(gi[s, x], I[r]) and np.array_equal(I[r], D[s, x])
    assert fsb.last_launch_count() == rp.info()["levels"]


@pytest.mark.gpu
def test_gpu_update_equals_encode():
    """Update on the GPU: the extended code's new rows, computed by fs_repair from the original
    code's check data, equal fs_encode's rows [n, n') (config 2: CGA converges)."""
    _need_gpu()
    c = dict(configs.get(2), files=10)
    g = fsb.Graph.create(c)
    ch = fsb.Checks.create(g, 3)
    g2 = g.extend(1)
    ch2 = fsb.Checks.from_data(g2, ch.data())
    S = 2
    d = inputs.stripe_data(c, num_stripes=S, device="cuda")
    full = torch.empty((S, g2.n, g2.t), dtype=torch.uint8, device="cuda")
    chk = torch.empty((S, g2.p, g2.t), dtype=torch.uint8, device="cuda")
    g2.encode_stripes(d, chk, full)
    mask = np.zeros(g2.n, bool)
    mask[g.n:] = True
    rp = fsb.RepairPlan(g2, ch2, mask)
    cod = full.clone()
    cod[:, g.n:] = 0
    rp.repair(cod)
    torch.cuda.synchronize()
    inf = rp.info()
    done = [j for j in range(g.n, g2.n)]
    assert inf["repaired"] + inf["unrepaired"] == len(done)
    assert inf["repaired"] > 0
    ok = (cod[:, g.n:] == full[:, g.n:]).flatten(2).all(-1).cpu().numpy()    # [S, new rows]
    assert ok.sum(1).tolist() == [inf["repaired"]] * S


@pytest.mark.gpu
def test_gpu_update_long_rows_many_stripes():
    """Update of config 7's code at 64 stripes: one level of 130 new rows of ~234 sources, enough
    units for the long-row level kernel (fsb_dpg_level_q); the rebuilt rows equal fs_encode's."""
    _need_gpu()
    c = dict(configs.get(7), stripes=64)
    g = fsb.Graph.create(c)
    ch = fsb.Checks.create(g, 3)
    g2 = g.extend(1)
    ch2 = fsb.Checks.from_data(g2, ch.data())
    S = c["stripes"]
    d = inputs.stripe_data(c, device="cuda")
    full = torch.empty((S, g2.n, g2.t), dtype=torch.uint8, device="cuda")
    chk = torch.empty((S, g2.p, g2.t), dtype=torch.uint8, device="cuda")
    g2.encode_stripes(d, chk, full)
    mask = np.zeros(g2.n, bool)
    mask[g.n:] = True
    rp = fsb.RepairPlan(g2, ch2, mask)
    inf = rp.info()
    assert inf["xor_sources"] >= 100 * inf["rows"]
    cod = full.clone()
    cod[:, g.n:] = 0
    rp.repair(cod)
    torch.cuda.synchronize()
    ok = (cod[:, g.n:] == full[:, g.n:]).flatten(2).all(-1).cpu().numpy()
    assert ok.sum(1).tolist() == [inf["repaired"]] * S
    assert inf["repaired"] == g2.n - g.n


@pytest.mark.gpu
def test_gpu_long_row_kernel_on_every_level():
    """FSB_DPG_Q=1 routes every plan level through fsb_dpg_level_q (the knob is read once per
    process, so in a child pytest): the decode and repair parity tests must still pass."""
    _need_gpu()
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, FSB_DPG_Q="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
                        "tests/test_decode.py::test_gpu_decode_matches_oracle",
                        "tests/test_decode.py::test_gpu_decode_eliminate_matches_oracle",
                        "tests/test_repair.py::test_gpu_repair_parity",
                        "tests/test_repair.py::test_gpu_update_equals_encode"],
                       cwd=root, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
