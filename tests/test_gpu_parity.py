"""GPU parity: the CUDA path through the C ABI vs the CPU oracle, element by element.

Bar: bit-exact on every output byte (checks and coded symbols) -- the work is
integer XOR.  Full-size configs are compared in full (the C oracle finishes them in
seconds), in the launch configuration bench.py times.
"""
import os

import numpy as np
import pytest
import torch

import oracle
from paper_1702_07409_b200 import configs, fsb, inputs

pytestmark = pytest.mark.gpu

_ORACLE = {}


def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _oracle_case(cfg, S=None):
    key = (tuple(sorted((k, v) for k, v in cfg.items() if not isinstance(v, tuple))), S)
    if key not in _ORACLE:
        g = oracle.generate_graph(cfg)
        D = inputs.stripe_data(cfg, num_stripes=S).numpy()
        C, Y = oracle.encode(g, D)
        _ORACLE.clear()
        _ORACLE[key] = (D, C, Y)
    return _ORACLE[key]


def _run(cfg, variant, S=None, data=None):
    g = fsb.Graph.create(cfg)
    if variant is not None:
        g.set_variant(variant)
    S = cfg["stripes"] if S is None else S
    d = data if data is not None else inputs.stripe_data(cfg, num_stripes=S, device="cuda")
    k, p, n, t = cfg["k"], cfg["p"], cfg["n"], cfg["t"]
    chk = torch.empty((S, p, t), dtype=torch.uint8, device="cuda") if p else None
    cod = torch.empty((S, n, t), dtype=torch.uint8, device="cuda")
    if chk is not None:
        chk.fill_(0xA5)
    cod.fill_(0x5A)
    g.encode_stripes(d, chk, cod)
    torch.cuda.synchronize()
    return g, (chk.cpu().numpy() if chk is not None else None), cod.cpu().numpy()


def _assert_equal(a, b, what):
    if not np.array_equal(a, b):
        bad = np.argwhere(a != b)
        raise AssertionError("%s: %d mismatching bytes, first at %s" % (what, len(bad), bad[:4].tolist()))


@pytest.mark.parametrize("cid", [1, 2, 3, 4, 5])
@pytest.mark.parametrize("variant", [fsb.VARIANT_AUTO, fsb.VARIANT_GLOBAL, fsb.VARIANT_SMEM])
def test_config_parity(cid, variant):
    _need_gpu()
    cfg = configs.get(cid)
    g = fsb.Graph.create(cfg)
    if variant == fsb.VARIANT_SMEM and not g.info()["smem_eligible"]:
        pytest.skip("SMEM variant not eligible for config %d" % cid)
    D, C, Y = _oracle_case(cfg)
    _, c, y = _run(cfg, variant)
    if cfg["p"]:
        _assert_equal(c, C, "checks")
    _assert_equal(y, Y, "coded")


@pytest.mark.parametrize("cid", [3, 5])
def test_row_range_partition_concatenates(cid):
    """P10 / SURVEY §8(e): rows [r*n/G, (r+1)*n/G) per rank concatenate to the full output
    (config 5: BASELINE.json:configs[5]'s coded-symbol range partition, reading R16)."""
    _need_gpu()
    cfg = configs.get(cid)
    g = fsb.Graph.create(cfg)
    D, C, Y = _oracle_case(cfg)
    d = torch.from_numpy(D[0]).cuda()
    n, t = cfg["n"], cfg["t"]
    for G in (2, 3, 8):
        parts = []
        for r in range(G):
            a, b = r * n // G, (r + 1) * n // G
            chk = torch.empty((cfg["p"], t), dtype=torch.uint8, device="cuda")
            out = torch.empty((b - a, t), dtype=torch.uint8, device="cuda")
            g.encode(d, chk, out, a, b)
            parts.append(out)
            _assert_equal(chk.cpu().numpy(), C[0], "checks rank %d" % r)
        torch.cuda.synchronize()
        _assert_equal(torch.cat(parts).cpu().numpy(), Y[0], "row partition G=%d" % G)


@pytest.mark.parametrize("cid,variant", [(5, fsb.VARIANT_AUTO), (3, fsb.VARIANT_GLOBAL),
                                         (4, fsb.VARIANT_SMEM), (4, fsb.VARIANT_GLOBAL)])
def test_col_range_partition_concatenates(cid, variant):
    """NEXT-4: fs_encode_range over byte columns [c0, c1) per rank assembles the full output;
    bytes outside a rank's columns are untouched; 16-B (non-slice) boundaries take GLOBAL."""
    _need_gpu()
    from paper_1702_07409_b200 import dist as fdist
    cfg = dict(configs.get(cid))
    cfg["stripes"] = 1
    g = fsb.Graph.create(cfg)
    g.set_variant(variant)
    D, C, Y = _oracle_case(cfg)
    d = torch.from_numpy(D[0]).cuda()
    k, p, n, t = cfg["k"], cfg["p"], cfg["n"], cfg["t"]
    splits = [[fdist.col_shard(t, G, r) for r in range(G)] for G in (2, 3, 8)]
    splits.append([(0, 16), (16, t - 48), (t - 48, t)])          # 16-B boundaries
    for parts in splits:
        chk = torch.full((p, t), 0xA5, dtype=torch.uint8, device="cuda") if p else None
        out = torch.full((n, t), 0x5A, dtype=torch.uint8, device="cuda")
        for c0, c1 in parts:
            g.encode_range(d, chk, out, 0, n, c0, c1)
            torch.cuda.synchronize()
            o = out.cpu().numpy()
            _assert_equal(o[:, c0:c1], Y[0][:, c0:c1], "coded cols [%d,%d)" % (c0, c1))
            assert (o[:, c1:] == 0x5A).all(), "wrote past col_end"
            if p:
                _assert_equal(chk.cpu().numpy()[:, c0:c1], C[0][:, c0:c1], "checks cols [%d,%d)" % (c0, c1))
        _assert_equal(out.cpu().numpy(), Y[0], "column partition %s" % (parts[:2],))
    # a rows x cols sub-block (row range goes GLOBAL)
    a, b, c0, c1 = n // 3, n // 2, 64 * 5, t - 64
    out = torch.full((b - a, t), 0x5A, dtype=torch.uint8, device="cuda")
    chk = torch.empty((p, t), dtype=torch.uint8, device="cuda") if p else None
    g.encode_range(d, chk, out, a, b, c0, c1)
    torch.cuda.synchronize()
    o = out.cpu().numpy()
    _assert_equal(o[:, c0:c1], Y[0][a:b, c0:c1], "rows x cols block")
    assert (o[:, :c0] == 0x5A).all() and (o[:, c1:] == 0x5A).all()


def test_stripes_equal_single_encodes():
    """P10: fs_encode_stripes over S stripes = S independent fs_encode calls."""
    _need_gpu()
    cfg = configs.get(4)
    g = fsb.Graph.create(cfg)
    S = 5
    d = inputs.stripe_data(cfg, num_stripes=S, device="cuda")
    k, p, n, t = cfg["k"], cfg["p"], cfg["n"], cfg["t"]
    for variant in (fsb.VARIANT_SMEM, fsb.VARIANT_GLOBAL):
        g.set_variant(variant)
        chk = torch.empty((S, p, t), dtype=torch.uint8, device="cuda")
        cod = torch.empty((S, n, t), dtype=torch.uint8, device="cuda")
        g.encode_stripes(d, chk, cod)
        for s in range(S):
            c1 = torch.empty((p, t), dtype=torch.uint8, device="cuda")
            y1 = torch.empty((n, t), dtype=torch.uint8, device="cuda")
            g.encode(d[s], c1, y1)
            torch.cuda.synchronize()
            assert torch.equal(c1, chk[s]) and torch.equal(y1, cod[s])


def test_padded_strides():
    """Strides larger than the minimum: bytes between stripes are left untouched."""
    _need_gpu()
    cfg = configs.get(2)
    k, p, n, t = cfg["k"], cfg["p"], cfg["n"], cfg["t"]
    S = 3
    D = inputs.stripe_data(cfg, num_stripes=S).numpy()
    go = oracle.generate_graph(cfg)
    C, Y = oracle.encode(go, D)
    for variant in (fsb.VARIANT_SMEM, fsb.VARIANT_GLOBAL):
        g = fsb.Graph.create(cfg)
        g.set_variant(variant)
        ds, cs, ys = (k + 3) * t + 16, (p + 1) * t + 32, (n + 2) * t + 48
        dbuf = torch.zeros(S * ds, dtype=torch.uint8, device="cuda")
        for s in range(S):
            dbuf[s * ds:s * ds + k * t] = torch.from_numpy(D[s].reshape(-1)).cuda()
        cbuf = torch.full((S * cs,), 0x33, dtype=torch.uint8, device="cuda")
        ybuf = torch.full((S * ys,), 0x44, dtype=torch.uint8, device="cuda")
        g.encode_stripes_raw(S, dbuf.data_ptr(), ds, cbuf.data_ptr(), cs, ybuf.data_ptr(), ys)
        torch.cuda.synchronize()
        cb, yb = cbuf.cpu().numpy(), ybuf.cpu().numpy()
        for s in range(S):
            _assert_equal(cb[s * cs:s * cs + p * t].reshape(p, t), C[s], "checks")
            _assert_equal(yb[s * ys:s * ys + n * t].reshape(n, t), Y[s], "coded")
            assert np.all(cb[s * cs + p * t:(s + 1) * cs] == 0x33)
            assert np.all(yb[s * ys + n * t:(s + 1) * ys] == 0x44)


EDGE_CASES = [
    # (name, cfg, stripes)
    ("t16_min", dict(k=37, p=3, d_p=2, n=50, t=16, dist=configs.RSD, rsd_c=0.1, rsd_delta=0.05, seed=11), 7),
    ("t48_ragged", dict(k=64, p=5, d_p=3, n=91, t=48, dist=configs.FINITE, seed=12,
                        fin_deg=configs.OMEGA_DEGREES, fin_prob=configs.OMEGA_PROBS), 3),
    ("t1040_ragged", dict(k=300, p=7, d_p=4, n=400, t=1040, dist=configs.RSD, rsd_c=0.1, rsd_delta=0.05,
                          seed=13), 2),
    ("k1_p0", dict(k=1, p=0, d_p=0, n=33, t=256, dist=configs.FINITE, seed=14,
                   fin_deg=configs.OMEGA_DEGREES, fin_prob=configs.OMEGA_PROBS), 4),
    ("deg1_only", dict(k=40, p=0, d_p=0, n=90, t=128, dist=configs.FINITE, seed=15, fin_deg=(1,),
                       fin_prob=(1.0,)), 300),
    ("dense_rows", dict(k=70, p=10, d_p=70, n=64, t=384, dist=configs.FINITE, seed=16,
                        fin_deg=(60, 80), fin_prob=(0.5, 0.5)), 300),
    ("k_not_mult32_many_stripes", dict(k=333, p=40, d_p=3, n=500, t=256, dist=configs.RSD, rsd_c=0.05,
                                       rsd_delta=0.01, seed=17), 400),
    ("p_over_64_checks", dict(k=500, p=150, d_p=5, n=600, t=128, dist=configs.RSD, rsd_c=0.1,
                              rsd_delta=0.05, seed=18), 320),
    # every row of degree 1 on one even source: no even/odd complements at all, so all 20,000 rows
    # go through the cross-class leftover matching (bounded scan) of the SMEM schedule
    ("k1_many_rows", dict(k=1, p=0, d_p=0, n=20000, t=256, dist=configs.FINITE, seed=19,
                          fin_deg=configs.OMEGA_DEGREES, fin_prob=configs.OMEGA_PROBS), 3),
]


@pytest.mark.parametrize("name,cfg,S", EDGE_CASES, ids=[e[0] for e in EDGE_CASES])
def test_edge_cases(name, cfg, S):
    _need_gpu()
    cfg = dict(cfg, stripes=S)
    go = oracle.generate_graph(cfg)
    D = inputs.stripe_data(cfg).numpy()
    C, Y = oracle.encode(go, D)
    variants = [fsb.VARIANT_AUTO, fsb.VARIANT_GLOBAL]
    if fsb.Graph.create(cfg).info()["smem_eligible"]:
        variants.append(fsb.VARIANT_SMEM)
    for v in variants:
        _, c, y = _run(cfg, v, data=torch.from_numpy(D).cuda())
        if cfg["p"]:
            _assert_equal(c, C, "%s checks v%d" % (name, v))
        _assert_equal(y, Y, "%s coded v%d" % (name, v))


def test_empty_calls_are_noops():
    _need_gpu()
    cfg = configs.get(1)
    g = fsb.Graph.create(cfg)
    d = inputs.stripe_data(cfg, device="cuda")
    out = torch.full((4, cfg["t"]), 7, dtype=torch.uint8, device="cuda")
    g.encode(d[0], None, out, 5, 5)                          # empty row range
    g.encode_stripes(d[:0], None, torch.empty((0, cfg["n"], cfg["t"]), dtype=torch.uint8, device="cuda"))
    torch.cuda.synchronize()
    assert torch.all(out == 7)


def test_invalid_arguments_rejected_range():
    _need_gpu()
    cfg = configs.get(1)
    g = fsb.Graph.create(cfg)
    t, n = cfg["t"], cfg["n"]
    d = inputs.stripe_data(cfg, device="cuda")[0]
    chk = torch.empty((cfg["p"], t), dtype=torch.uint8, device="cuda")
    out = torch.empty((n, t), dtype=torch.uint8, device="cuda")
    for c0, c1 in ((8, 64), (0, 24 + 1), (64, 32), (0, t + 16)):
        with pytest.raises(fsb.FsError):
            g.encode_range(d, chk, out, 0, n, c0, c1)
    g.encode_range(d, chk, out, 0, n, 32, 32)                        # empty range: no-op
    assert fsb.last_launch_count() == 0


def test_invalid_arguments_rejected():
    _need_gpu()
    cfg = configs.get(2)
    g = fsb.Graph.create(cfg)
    d = inputs.stripe_data(cfg, device="cuda")
    chk = torch.empty((1, cfg["p"], cfg["t"]), dtype=torch.uint8, device="cuda")
    cod = torch.empty((1, cfg["n"], cfg["t"]), dtype=torch.uint8, device="cuda")
    with pytest.raises(fsb.FsError):
        g.encode(d[0], None, cod[0])                         # p > 0 needs checks
    with pytest.raises(fsb.FsError):
        g.encode(d[0], chk[0], cod[0], 10, 5)                # bad row range
    with pytest.raises(fsb.FsError):
        g.encode_stripes_raw(1, d.data_ptr() + 8, cfg["k"] * cfg["t"], chk.data_ptr(), cfg["p"] * cfg["t"],
                             cod.data_ptr(), cfg["n"] * cfg["t"])   # misaligned
    with pytest.raises(fsb.FsError):
        g.encode_stripes_raw(1, d.data_ptr(), cfg["k"] * cfg["t"] - 16, chk.data_ptr(), cfg["p"] * cfg["t"],
                             cod.data_ptr(), cfg["n"] * cfg["t"])   # stride too small


def test_launch_counts():
    _need_gpu()
    cfg = configs.get(4)
    g = fsb.Graph.create(cfg)
    d = inputs.stripe_data(cfg, num_stripes=16, device="cuda")
    chk = torch.empty((16, cfg["p"], cfg["t"]), dtype=torch.uint8, device="cuda")
    cod = torch.empty((16, cfg["n"], cfg["t"]), dtype=torch.uint8, device="cuda")
    g.set_variant(fsb.VARIANT_SMEM)
    g.encode_stripes(d, chk, cod)
    assert fsb.last_launch_count() == 1
    g.set_variant(fsb.VARIANT_GLOBAL)
    g.encode_stripes(d, chk, cod)
    assert fsb.last_launch_count() == 2
    torch.cuda.synchronize()


def test_decode_gpu_output_roundtrip():
    """P8 on the GPU's bytes: the oracle's decoder recovers the data from a random 95%
    subset of the CUDA path's coded symbols (config 2)."""
    _need_gpu()
    cfg = configs.get(2)
    _, c, y = _run(cfg, fsb.VARIANT_AUTO)
    go = oracle.generate_graph(cfg)
    D = inputs.stripe_data(cfg).numpy()[0]
    recv = np.random.default_rng(3).random(cfg["n"]) < 0.95
    I, state = oracle.decode(go, recv, y[0])
    ok = state[:cfg["k"]] != 0
    assert ok.sum() > 0.9 * cfg["k"]
    assert np.array_equal(I[:cfg["k"]][ok], D[ok])


@pytest.mark.parametrize("seed", range(12))
def test_random_parameters(seed):
    """Random (k, p, d_p, n, t, distribution, stripes): every variant bit-exact vs the oracle
    (covers ragged t, k not a multiple of the TMA box, heavy rows, pair and warp splits)."""
    _need_gpu()
    rng = np.random.default_rng(1000 + seed)
    k = int(rng.integers(1, 1500))
    p = int(rng.integers(0, 60))
    d_p = int(rng.integers(1, min(k, 6) + 1)) if p else 0
    n = int(rng.integers(1, 2200))
    t = int(rng.choice([16, 48, 64, 128, 192, 512, 1088, 4096]))
    if rng.random() < 0.5:
        cfg = dict(k=k, p=p, d_p=d_p, n=n, t=t, dist=configs.RSD, rsd_c=float(rng.uniform(0.03, 0.3)),
                   rsd_delta=float(rng.uniform(0.01, 0.5)), seed=int(rng.integers(1, 1 << 40)))
    else:
        cfg = dict(k=k, p=p, d_p=d_p, n=n, t=t, dist=configs.FINITE, seed=int(rng.integers(1, 1 << 40)),
                   fin_deg=configs.OMEGA_DEGREES, fin_prob=configs.OMEGA_PROBS)
    S = int(rng.choice([1, 3, 150, 400])) if k * t <= (1 << 20) else 1
    cfg["stripes"] = S
    try:
        go = oracle.generate_graph(cfg)
    except ValueError:
        pytest.skip("parameters rejected by the distribution rules (e.g. RSD spike K/R < 1)")
    D = inputs.stripe_data(cfg).numpy()
    C, Y = oracle.encode(go, D)
    variants = [fsb.VARIANT_AUTO, fsb.VARIANT_GLOBAL]
    if fsb.Graph.create(cfg).info()["smem_eligible"]:
        variants.append(fsb.VARIANT_SMEM)
    for v in variants:
        _, c, y = _run(cfg, v, data=torch.from_numpy(D).cuda())
        if p:
            _assert_equal(c, C, "seed %d checks v%d" % (seed, v))
        _assert_equal(y, Y, "seed %d coded v%d" % (seed, v))


@pytest.mark.parametrize("S", [1, 300])
def test_array_precode_parity(S):
    """NEXT-2: the Alg 2 precode (2 levels, checks reading checks) on both variants, bit-exact."""
    _need_gpu()
    cfg = dict(configs.get(6), stripes=S)
    go = oracle.generate_graph(cfg)
    D = inputs.stripe_data(cfg).numpy()
    C, Y = oracle.encode(go, D)
    variants = [fsb.VARIANT_AUTO, fsb.VARIANT_GLOBAL]
    if fsb.Graph.create(cfg).info()["smem_eligible"]:
        variants.append(fsb.VARIANT_SMEM)
    for v in variants:
        _, c, y = _run(cfg, v, data=torch.from_numpy(D).cuda())
        _assert_equal(c, C, "array checks v%d" % v)
        _assert_equal(y, Y, "array coded v%d" % v)


def _check_supports(pre_rp, pre_c, k, p):
    """Data support of each check over GF(2): members < k, or (array precode, Alg 2) an earlier
    check whose support is XORed in."""
    sup = []
    for i in range(p):
        acc = set()
        for m in pre_c[pre_rp[i]:pre_rp[i + 1]]:
            m = int(m)
            acc ^= {m} if m < k else sup[m - k]
        sup.append(acc)
    return sup


def _effective_support(csup, lt_rp, lt_c, k, j):
    """Data symbols of G_eff row j = G_LT . [I_k ; G_pre] over GF(2)."""
    odd = set()
    for m in lt_c[lt_rp[j]:lt_rp[j + 1]]:
        m = int(m)
        odd ^= {m} if m < k else csup[m - k]
    return odd


@pytest.mark.parametrize("cid", [2, 4, 5, 6])
def test_bit_probe_full_scale(cid):
    """P6 at full size, oracle-free: data symbol i = one-hot bit i (k <= 8t), so bit i of Y_j must
    be G_eff[j][i] -- computed from the CSR alone -- on sampled rows (all rows for c2/c4/c6, 3000
    rows incl. the highest-degree ones for c5), in the launch configuration bench.py times."""
    _need_gpu()
    cfg = dict(configs.get(cid), stripes=1)
    g = fsb.Graph.create(cfg)
    k, p, n, t = cfg["k"], cfg["p"], cfg["n"], cfg["t"]
    assert k <= 8 * t
    idx = torch.arange(k, device="cuda")
    d = torch.zeros((1, k, t), dtype=torch.uint8, device="cuda")
    d[0, idx, idx // 8] = (1 << (idx % 8)).to(torch.uint8)
    chk = torch.empty((1, p, t), dtype=torch.uint8, device="cuda") if p else None
    cod = torch.empty((1, n, t), dtype=torch.uint8, device="cuda")
    g.encode_stripes(d, chk, cod)
    torch.cuda.synchronize()
    pre_rp, pre_c, lt_rp, lt_c = g.csr()
    csup = _check_supports(pre_rp, pre_c, k, p)
    if n <= 2000:
        rows = np.arange(n)
    else:
        deg = np.diff(lt_rp)
        rows = np.unique(np.concatenate([np.argsort(-deg)[:200],
                                         np.random.default_rng(cid).choice(n, 2800, replace=False)]))
    got = np.unpackbits(cod[0, torch.from_numpy(rows).cuda()].cpu().numpy(), axis=1, bitorder="little")
    for r, j in enumerate(rows):
        want = np.zeros(8 * t, np.uint8)
        sup = _effective_support(csup, lt_rp, lt_c, k, int(j))
        if sup:
            want[list(sup)] = 1
        assert np.array_equal(got[r], want), "row %d" % j
    if p:
        cb = np.unpackbits(chk[0].cpu().numpy(), axis=1, bitorder="little")
        for i in range(p):
            want = np.zeros(8 * t, np.uint8)
            if csup[i]:
                want[list(csup[i])] = 1
            assert np.array_equal(cb[i], want), "check %d" % i


@pytest.mark.parametrize("t,S", [(128, 300), (192, 200), (4160, 20), (64, 400)])
def test_smem_paired_and_unpaired_tiles(t, S):
    """SMEM kernel with an even slice count (paired tiles: rows leave as full 128-B lines through
    TMEM) and odd slice counts (unpaired 64-B stores), many tiles per CTA so both tile orders
    (odd CTAs run their pairs reversed) and the TMEM column blocks of every warp are exercised."""
    _need_gpu()
    cfg = dict(configs.get(4), t=t, stripes=S)
    g = fsb.Graph.create(cfg)
    assert g.info()["smem_eligible"]
    g.set_variant(fsb.VARIANT_SMEM)
    D = inputs.stripe_data(cfg).numpy()
    go = oracle.generate_graph(cfg)
    C, Y = oracle.encode(go, D)
    _, c, y = _run(cfg, fsb.VARIANT_SMEM, data=torch.from_numpy(D).cuda())
    _assert_equal(c, C, "checks t=%d" % t)
    _assert_equal(y, Y, "coded t=%d" % t)


@pytest.mark.parametrize("cid,S,chunks,pinned", [(4, 6, 0, True), (4, 7, 3, True), (4, 5, 1, False),
                                                 (5, None, 8, True), (5, None, 3, True), (3, None, 0, True),
                                                 (2, None, 4, False), (1, None, 0, True)])
def test_encode_host_matches_oracle(cid, S, chunks, pinned):
    """fs_encode_host: host buffers staged through the library's device buffers, chunked by
    stripes (S > 1) or by byte columns (one stripe), on two library streams -- every output byte
    equals the oracle's; repeated calls with another chunking reuse the staging."""
    _need_gpu()
    cfg = configs.get(cid)
    S = cfg["stripes"] if S is None else S
    D, C, Y = _oracle_case(cfg, S)
    k, p, n, t = cfg["k"], cfg["p"], cfg["n"], cfg["t"]
    g = fsb.Graph.create(cfg)
    h_d = torch.from_numpy(D).contiguous()
    if pinned:
        h_d = h_d.pin_memory()
    h_c = torch.full((S, p, t), 0xA5, dtype=torch.uint8, pin_memory=pinned) if p else None
    h_y = torch.full((S, n, t), 0x5A, dtype=torch.uint8, pin_memory=pinned)
    for ch in (chunks, 2):
        g.encode_host(h_d, h_c, h_y, chunks=ch)
        torch.cuda.synchronize()
        if p:
            _assert_equal(h_c.numpy(), C, "host checks (chunks=%d)" % ch)
        _assert_equal(h_y.numpy(), Y, "host coded (chunks=%d)" % ch)
        h_y.fill_(0x5A)
        if p:
            h_c.fill_(0xA5)
    assert fsb.last_launch_count() >= 1


def test_encode_host_padded_strides_and_validation():
    """fs_encode_host with host strides larger than the symbol block (stripes padded by 4 KiB):
    the padding is neither read into the result nor written; strides below the minimum and NULL
    buffers are rejected with FS_EINVAL."""
    _need_gpu()
    import ctypes
    cfg = configs.get(4)
    S = 3
    D, C, Y = _oracle_case(cfg, S)
    k, p, n, t = cfg["k"], cfg["p"], cfg["n"], cfg["t"]
    g = fsb.Graph.create(cfg)
    pad = 4096
    ds, cs, ys = k * t + pad, p * t + pad, n * t + pad
    h_d = torch.full((S, ds), 0x33, dtype=torch.uint8).pin_memory()
    h_c = torch.full((S, cs), 0xA5, dtype=torch.uint8).pin_memory()
    h_y = torch.full((S, ys), 0x5A, dtype=torch.uint8).pin_memory()
    h_d[:, :k * t] = torch.from_numpy(D.reshape(S, -1))
    L = fsb.lib()
    st = torch.cuda.current_stream()
    ptr = lambda x: ctypes.c_void_p(x.data_ptr())
    s = ctypes.c_void_p(st.cuda_stream)
    assert L.fs_encode_host(g._h, S, ptr(h_d), ds, ptr(h_c), cs, ptr(h_y), ys, 2, s) == fsb.FS_OK
    torch.cuda.synchronize()
    _assert_equal(h_y[:, :n * t].numpy().reshape(S, n, t), Y, "coded (padded strides)")
    _assert_equal(h_c[:, :p * t].numpy().reshape(S, p, t), C, "checks (padded strides)")
    assert (h_y[:, n * t:] == 0x5A).all() and (h_c[:, p * t:] == 0xA5).all()
    assert L.fs_encode_host(g._h, S, ptr(h_d), k * t - 16, ptr(h_c), cs, ptr(h_y), ys, 2, s) == fsb.FS_EINVAL
    assert L.fs_encode_host(g._h, S, ptr(h_d), ds, None, cs, ptr(h_y), ys, 2, s) == fsb.FS_EINVAL
    assert L.fs_encode_host(g._h, S, ptr(h_d), ds, ptr(h_c), cs, None, ys, 2, s) == fsb.FS_EINVAL
    assert L.fs_encode_host(g._h, 0, None, 0, None, 0, None, 0, 0, s) == fsb.FS_OK


def test_encode_host_orders_after_stream_work():
    """fs_encode_host starts after the work already queued on the caller's stream: the input host
    buffer is filled by a device-to-host copy enqueued just before the call (behind a slow kernel),
    and the encode must see the copied bytes, not the stale ones."""
    _need_gpu()
    cfg = configs.get(2)
    D, C, Y = _oracle_case(cfg, 1)
    k, p, n, t = cfg["k"], cfg["p"], cfg["n"], cfg["t"]
    g = fsb.Graph.create(cfg)
    h_d = torch.zeros((1, k, t), dtype=torch.uint8).pin_memory()          # stale input
    h_c = torch.empty((1, p, t), dtype=torch.uint8).pin_memory()
    h_y = torch.empty((1, n, t), dtype=torch.uint8).pin_memory()
    d_src = torch.from_numpy(D).cuda()
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        torch.cuda._sleep(20_000_000)                                      # keep the stream busy
        h_d.copy_(d_src, non_blocking=True)                                # the real input
        g.encode_host(h_d, h_c, h_y, chunks=2, stream=s)
    s.synchronize()
    _assert_equal(h_y.numpy(), Y, "coded after stream-ordered input")
    _assert_equal(h_c.numpy(), C, "checks after stream-ordered input")


@pytest.mark.parametrize("t,S,p,chunks", [(1040, 1, 8, 4), (8208, 1, 8, 8), (512, 5, 0, 2), (4160, 3, 4, 0)])
def test_encode_host_ragged_sizes(t, S, p, chunks):
    """fs_encode_host on sizes off the common grid: t not a multiple of 64 (one stripe: column
    chunks end off a slice boundary, the GLOBAL variant), no precode with several stripes, and an
    odd slice count; every byte against the oracle."""
    _need_gpu()
    cfg = dict(configs.get(2), k=300, p=p, d_p=3 if p else 0, n=390, t=t, stripes=S, seed=77 + t + S)
    D, C, Y = _oracle_case(cfg, S)
    g = fsb.Graph.create(cfg)
    h_d = torch.from_numpy(D).contiguous().pin_memory()
    h_c = torch.full((S, p, t), 0xA5, dtype=torch.uint8).pin_memory() if p else None
    h_y = torch.full((S, cfg["n"], t), 0x5A, dtype=torch.uint8).pin_memory()
    g.encode_host(h_d, h_c, h_y, chunks=chunks)
    torch.cuda.synchronize()
    _assert_equal(h_y.numpy(), Y, "coded")
    if p:
        _assert_equal(h_c.numpy(), C, "checks")


@pytest.mark.parametrize("seed,t,S,dist", [(11, 1008, 160, "omega"), (12, 2064, 96, "rsd"), (13, 528, 300, "omega")])
def test_many_wave_band_kernel_ragged(seed, t, S, dist):
    """fsb_lt_band4 (the GLOBAL band kernel for calls of many waves of warps): a random code with
    a ragged last band (t not a multiple of 512), many stripes, degree-1 rows and a heavy tail;
    every stripe in full against the oracle, plus a row-range partition of one stripe."""
    _need_gpu()
    rng = np.random.default_rng(seed)
    k = int(rng.integers(300, 900))
    p = int(rng.integers(1, 20))
    cfg = dict(name="mw", k=k, p=p, d_p=3, n=int(1.3 * (k + p)), t=t, stripes=S, seed=seed)
    if dist == "omega":
        cfg.update(dist=configs.FINITE, fin_deg=configs.OMEGA_DEGREES, fin_prob=configs.OMEGA_PROBS)
    else:
        cfg.update(dist=configs.RSD, rsd_c=0.1, rsd_delta=0.05)
    g = fsb.Graph.create(cfg)
    g.set_variant(fsb.VARIANT_GLOBAL)
    go = oracle.generate_graph(cfg)
    D = inputs.stripe_data(cfg).numpy()
    C, Y = oracle.encode(go, D)
    d = torch.from_numpy(D).cuda()
    chk = torch.empty((S, p, t), dtype=torch.uint8, device="cuda")
    cod = torch.empty((S, cfg["n"], t), dtype=torch.uint8, device="cuda")
    g.encode_stripes(d, chk, cod)
    torch.cuda.synchronize()
    assert fsb.last_launch_count() == 2
    _assert_equal(chk.cpu().numpy(), C, "checks")
    _assert_equal(cod.cpu().numpy(), Y, "coded")
    a, b = cfg["n"] // 5, cfg["n"] - 3
    out = torch.empty((b - a, t), dtype=torch.uint8, device="cuda")
    g.encode(d[1], chk[1], out, a, b)
    torch.cuda.synchronize()
    _assert_equal(out.cpu().numpy(), Y[1][a:b], "row range")


@pytest.mark.parametrize("S", [5, 20, 77])
def test_smem_pair_rounds_with_tail_singles(S):
    """Paired SMEM tiles whose last partial round of pairs runs as single unpaired tiles (config 4
    geometry, 32 pairs per stripe: S=5 -> 160 pairs = 1 round of 148 + 12 pairs as 24 singles;
    S=20 -> 640 = 4 rounds + 48 pairs as 96 singles; S=77 -> 2464 = 16 rounds + 96 pairs, 2R > 148:
    pairs) -- every stripe against the oracle."""
    _need_gpu()
    cfg = configs.get(4, stripes=S)
    D, C, Y = _oracle_case(cfg)
    _, c, y = _run(cfg, fsb.VARIANT_SMEM)
    _assert_equal(c, C, "checks S=%d" % S)
    _assert_equal(y, Y, "coded S=%d" % S)


@pytest.mark.parametrize("env", [{"FSB_TMEM_HEADS": "0"}, {"FSB_ITEM_OVERHEAD": "3", "FSB_SPLIT1": "40",
                                                            "FSB_SPLIT2": "80"}, {"FSB_PAIR_GLOBAL": "0"}])
def test_smem_schedule_variants_by_env(env):
    """The SMEM kernel's other schedule / layout choices (read once per process, so each runs in a
    fresh process): item heads in shared memory instead of TMEM on a paired launch
    (FSB_TMEM_HEADS=0), another split-threshold / LPT setting (more pair- and warp-splits), and the
    within-class pairing of leftover rows (FSB_PAIR_GLOBAL=0) --
    config 4 (256 stripes) in full against the oracle, SMEM variant."""
    _need_gpu()
    import subprocess
    import sys as _sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([_sys.executable, os.path.join(root, "tools", "gpu", "check_cfg.py"), "4", "smem"],
                       capture_output=True, text=True, env=dict(os.environ, **env), timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    assert r.stdout.strip().endswith("ok"), r.stdout


@pytest.mark.parametrize("band_cfg", ["0", "1", "2", "4"])
def test_band_kernel_instances_by_env(band_cfg):
    """The other GLOBAL band-kernel instances FSB_BAND_CFG selects (read once per process, so each
    runs in a fresh process): 0 = fsb_lt_band<4, 6, lazy> for every call, 1 = the round-1
    fsb_lt_band<2, 8> for many-wave calls, 2 = <8, 4>, 4 = fsb_lt_band4 (round 2 before the edge
    windows) -- config 5 in full against the oracle."""
    _need_gpu()
    import subprocess
    import sys as _sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, FSB_BAND_CFG=band_cfg)
    r = subprocess.run([_sys.executable, os.path.join(root, "tools", "gpu", "check_cfg.py"), "5", "global"],
                       capture_output=True, text=True, env=env, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    assert r.stdout.strip().endswith("ok"), r.stdout


@pytest.mark.parametrize("regs,rows", [("3", "8"), ("3", "16"), ("4", "16"), ("5", "20"), ("5", "32")])
def test_window_kernel_shapes(regs, rows):
    """fsb_lt_win (fixed-size edge windows, FSB_BAND_CFG=5) with 96 / 128 / 160-edge windows and
    8-32 rows per window (FSB_WIN_REGS / FSB_WIN_ROWS, read once per process): config 5's full-row
    encode and its row ranges -- rank partitions G = 2, 3 and ranges that start and end inside a
    window (rows computed but not stored) -- bit-exact against the oracle (tools/gpu/check_win.py)."""
    _need_gpu()
    import subprocess
    import sys as _sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, FSB_BAND_CFG="5", FSB_WIN_REGS=regs, FSB_WIN_ROWS=rows)
    r = subprocess.run([_sys.executable, os.path.join(root, "tools", "gpu", "check_win.py"), "5"],
                       capture_output=True, text=True, env=env, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    assert r.stdout.strip().endswith("ok"), r.stdout


@pytest.mark.parametrize("t,S", [(1040, 3), (528, 2), (2048, 5)])
def test_window_kernel_multi_stripe_ragged(t, S):
    """fsb_lt_win across stripes (unit = stripe x band x window) and with a ragged last band (t not a
    multiple of 512: lanes past the end load a valid address and store nothing): config 3's code
    (Omega, max degree 66, so windows exist) at other symbol sizes, every stripe against the oracle."""
    _need_gpu()
    cfg = dict(configs.get(3), t=t, stripes=S, k=2000, p=40, n=2400)
    g = fsb.Graph.create(cfg)
    assert g.info()["lt_windows"] > 0
    D, C, Y = _oracle_case(cfg, S)
    _, c, y = _run(cfg, fsb.VARIANT_GLOBAL, S=S)
    _assert_equal(c, C, "checks t=%d S=%d" % (t, S))
    _assert_equal(y, Y, "coded t=%d S=%d" % (t, S))
