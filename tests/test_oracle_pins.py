"""Pins of the CPU oracle (oracle/) to things other than itself.

Each test names the pin of SURVEY.md §8(c) it implements and the passage that fixes the
expected value.  No expected value here comes from the CUDA path.
"""
import hashlib
import itertools
import os

import numpy as np
import pytest
import torch

import oracle
from paper_1702_07409_b200 import configs, inputs

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _golden_rows(name):
    rows = []
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.strip()
            if line and not line.startswith("#"):
                rows.append(line.split())
    return rows


# ----------------------------------------------------------------------------- P1: PRNG
def test_splitmix64_known_answers():
    """P1: published splitmix64 vectors (tests/golden/splitmix64_kat.txt)."""
    for row in _golden_rows("splitmix64_kat.txt"):
        seed = int(row[0])
        want = [int(x, 16) for x in row[1:]]
        got = [int(x) for x in oracle.splitmix64(seed, len(want))]
        assert got == want


def test_counter_form_input_generator_matches_sequential_stream():
    """P1 (counter form): inputs.py's counter-form words equal the oracle's sequential
    stream at arbitrary offsets -- two independent implementations (torch vs C)."""
    seq = oracle.splitmix64(4, 5000).astype(np.uint64)
    for start, cnt in [(0, 7), (1, 100), (1234, 3000), (4990, 10)]:
        w = inputs.splitmix64_words(4, start, cnt).numpy().view(np.uint64)
        assert np.array_equal(w, seq[start:start + cnt])


def test_input_bytes_little_endian():
    """R4: byte j = byte (j mod 8), little-endian, of word j//8 (c1
    data[0:8] = c15c0289ec2d0a91, c2 = ce56971cde355897, c3 = ed8f01dbe4140b1d)."""
    for cid, want in [(1, "c15c0289ec2d0a91"), (2, "ce56971cde355897"), (3, "ed8f01dbe4140b1d")]:
        b = inputs.random_bytes(cid, 0, 8).numpy().tobytes().hex()
        assert b == want


# ------------------------------------------------------------------ P3: degree laws
def _pmf(cdf):
    return np.diff(np.concatenate([[0.0], cdf]))


def test_omega_matches_paper_coefficients():
    """the CDF's increments are the printed coefficients / their sum;
    support at degrees 65/66 per BASELINE.json:configs[2] (reading R8)."""
    rows = _golden_rows("omega_paper.txt")
    paper_p = np.array([float(r[1]) for r in rows])
    deg, cdf = oracle.build_cdf(configs.FINITE, 10100, fin_deg=configs.OMEGA_DEGREES,
                                fin_prob=configs.OMEGA_PROBS)
    assert list(deg) == [1, 2, 3, 4, 5, 8, 9, 19, 65, 66]
    assert [int(r[0]) for r in rows][:8] == list(deg[:8])
    np.testing.assert_allclose(_pmf(cdf), paper_p / paper_p.sum(), rtol=0, atol=1e-12)
    assert cdf[-1] == 1.0
    # SPEC.md:68/69-style closed forms: mean 5.8703 (65/66), P(d=2) = 0.49357/0.999998
    mean = float((deg * _pmf(cdf)).sum())
    assert abs(mean - 5.8703) < 5e-4
    assert abs(_pmf(cdf)[1] - 0.49357 / 0.999998) < 1e-9


def test_omega_truncation_merges_into_K():
    """R15 / SPEC.md:59: degrees > K merge into K."""
    deg, cdf = oracle.build_cdf(configs.FINITE, 10, fin_deg=configs.OMEGA_DEGREES,
                                fin_prob=configs.OMEGA_PROBS)
    assert list(deg) == [1, 2, 3, 4, 5, 8, 9, 10]
    s = sum(configs.OMEGA_PROBS)
    assert abs(_pmf(cdf)[-1] - (0.055590 + 0.025023 + 0.003135) / s) < 1e-12


def test_degenerate_distribution_always_one():
    """single term (1, 1.0) -> every coded symbol has degree 1."""
    cfg = dict(k=50, p=0, d_p=0, n=200, t=16, dist=configs.FINITE, seed=9,
               fin_deg=(1,), fin_prob=(1.0,))
    g = oracle.generate_graph(cfg)
    assert np.all(np.diff(g.lt_row_ptr) == 1)


@pytest.mark.parametrize("cid,R,m,beta,dbar", [
    (1, 7.6009, 13, 1.61774, 6.8390),
    (2, 18.4163, 55, 1.21836, 13.0884),
    (4, 32.0643, 32, 1.32344, 11.2262),
])
def test_rsd_structure(cid, R, m, beta, dbar):
    """RSD (Luby): the ideal-soliton part rho sums to exactly 1, so beta =
    1 + sum(tau); the spike sits at m = floor(K/R); beyond m the pmf is rho(i)/beta with
    ratio pmf(i+1)/pmf(i) = (i-1)/(i+1).  Numbers R, m, beta, mean from SURVEY.md §8(c) R10
    (an independent derivation)."""
    c = configs.get(cid)
    K = c["k"] + c["p"]
    deg, cdf = oracle.build_cdf(configs.RSD, K, c["rsd_c"], c["rsd_delta"])
    pmf = _pmf(cdf)
    assert list(deg) == list(range(1, K + 1))
    # beyond the spike: pure soliton shape
    i = np.arange(m + 1, K)            # degrees m+1 .. K-1
    ratio = pmf[i] / pmf[i - 1]        # pmf(d+1)/pmf(d) for d = m+1..K-1  -> (d-1)/(d+1)
    d = i
    np.testing.assert_allclose(ratio, (d - 1) / (d + 1), rtol=1e-6)  # CDF differencing
    # pmf(i) = 1/(i(i-1) beta) for i > m gives beta
    beta_got = 1.0 / (pmf[m] * (m + 1) * m)   # pmf[m] is degree m+1
    assert abs(beta_got - beta) < 5e-5
    # spike: pmf at m exceeds its neighbours
    assert pmf[m - 1] > pmf[m - 2] and pmf[m - 1] > pmf[m]
    mean = float((deg * pmf).sum())
    assert abs(mean - dbar) < 5e-4
    # pmf(1) = (1/K + R/K) / beta
    assert abs(pmf[0] - (1.0 / K + R / K) / beta) < 1e-4


def test_degree_sampling_statistics():
    """P3: 10^6 sampled degrees: chi-square against Omega, mean within 4 SE."""
    n = 1_000_000
    cfg = dict(k=200, p=0, d_p=0, n=n, t=16, dist=configs.FINITE, seed=77,
               fin_deg=configs.OMEGA_DEGREES, fin_prob=configs.OMEGA_PROBS)
    g = oracle.generate_graph(cfg)
    d = np.diff(g.lt_row_ptr)
    sup = np.array(configs.OMEGA_DEGREES)
    p = np.array(configs.OMEGA_PROBS) / sum(configs.OMEGA_PROBS)
    counts = np.array([(d == s).sum() for s in sup])
    assert counts.sum() == n
    chi2 = float((((counts - n * p) ** 2) / (n * p)).sum())
    assert chi2 < 27.9          # 9 dof, p = 0.001
    mean, sd = float((sup * p).sum()), float(np.sqrt((sup ** 2 * p).sum() - (sup * p).sum() ** 2))
    assert abs(d.mean() - mean) < 4 * sd / np.sqrt(n)
    assert abs((d == 2).mean() - 0.49357 / 0.999998) < 4 * 0.0005


# ------------------------------------------------------------- P4: structural validity
@pytest.mark.parametrize("cid", [1, 2, 3, 4, 5])
def test_graph_structure(cid):
    """P4: rows sorted, no duplicates, indices in range, nnz = sum of degrees,
    degree support within the distribution's support; mean degree within 4 SE of d-bar."""
    c = configs.get(cid)
    g = oracle.generate_graph(c)
    K = g.K
    assert g.lt_row_ptr[0] == 0 and np.all(np.diff(g.lt_row_ptr) >= 1)
    assert g.nnz == len(g.lt_col)
    for j in range(g.n):
        r = g.lt_row(j)
        assert np.all(np.diff(r) > 0) and r[0] >= 0 and r[-1] < K
    for i in range(g.p):
        r = g.pre_row(i)
        assert len(r) == c["d_p"] and np.all(np.diff(r) > 0) and r[0] >= 0 and r[-1] < g.k
    deg, cdf = oracle.build_cdf(c["dist"], K, c["rsd_c"], c["rsd_delta"], c["fin_deg"], c["fin_prob"])
    pmf = _pmf(cdf)
    dd = np.diff(g.lt_row_ptr)
    assert set(np.unique(dd)) <= set(deg.tolist())
    mu = float((deg * pmf).sum())
    sd = float(np.sqrt((deg.astype(float) ** 2 * pmf).sum() - mu ** 2))
    assert abs(dd.mean() - mu) < 4 * sd / np.sqrt(g.n)


def test_graph_determinism():
    """same parameters -> identical graphs."""
    c = configs.get(2)
    a, b = oracle.generate_graph(c), oracle.generate_graph(c)
    assert np.array_equal(a.lt_col, b.lt_col) and np.array_equal(a.pre_col, b.pre_col)


def _csr_hash(g):
    h = hashlib.sha256()
    for a in (g.pre_row_ptr, g.pre_col, g.lt_row_ptr, g.lt_col):
        h.update(np.ascontiguousarray(a, dtype="<i4").tobytes())
    return h.hexdigest()[:16]


@pytest.mark.parametrize("cid,nnz,maxdeg,csr,row", [
    (1, 751, 28, "9d336f66423ba021", (0, [19, 35, 61, 90])),
    (2, 15341, 360, "3a65fc1dce1cd74c", (1, [60, 249])),
    (3, 72512, 66, "14aac6fe53a93101", (1, [1817, 3281, 4040, 6597])),
    (4, 13372, 251, "6c0acd9db045f999", (1, [19, 246, 1020])),
    (5, 352119, 66, "52f4395d4e0c42e4", (0, [27672, 32695])),
])
def test_graph_third_vote(cid, nnz, maxdeg, csr, row):
    """P12: values an independent transcription of readings R2-R15 produced at survey
    time -- a third vote on the conventions, not ground truth."""
    g = oracle.generate_graph(configs.get(cid))
    assert g.nnz == nnz
    assert int(np.diff(g.lt_row_ptr).max()) == maxdeg
    assert list(g.lt_row(row[0])) == row[1]
    if g.p:
        assert g.pre_row_ptr[-1] == g.p * configs.get(cid)["d_p"]
    assert _csr_hash(g) == csr


# ---------------------------------------------------------- P5-P7: encoder invariants
def _small_cfg(cid):
    return configs.get(cid)


def _data(c, S=None):
    return inputs.stripe_data(c, num_stripes=S).numpy()


def _dense(g):
    """G_LT (n x K) and G_pre (p x k) as dense 0/1 matrices."""
    A = np.zeros((g.n, g.K), dtype=np.uint8)
    for j in range(g.n):
        A[j, g.lt_row(j)] = 1
    P = np.zeros((g.p, g.k), dtype=np.uint8)
    for i in range(g.p):
        P[i, g.pre_row(i)] = 1
    return A, P


def _geff(g):
    """G_eff = G_LT . [I_k ; G_pre] over GF(2): coded symbols as sums of data symbols."""
    A, P = _dense(g)
    E = np.concatenate([np.eye(g.k, dtype=np.int64), P.astype(np.int64)], axis=0)
    return (A.astype(np.int64) @ E) % 2, P


def test_xor_examples():
    """SPEC.md:283-285 (self-inverse, identity, involution) through the encoder: a graph whose
    rows are {0}, {0,1}, {0,1,1}-free ... built by hand (brute force on a tiny case)."""
    cfg = dict(k=2, p=0, n=3, t=512)
    g = oracle.Graph(cfg, np.zeros(1, np.int32), np.zeros(0, np.int32),
                     np.array([0, 2, 3, 4], np.int32), np.array([0, 1, 0, 1], np.int32))
    rng = np.random.default_rng(1)
    a = rng.integers(0, 256, (2, 512), dtype=np.uint8)
    _, y = oracle.encode(g, a)
    assert np.array_equal(y[0], a[0] ^ a[1])
    assert np.array_equal(y[1], a[0]) and np.array_equal(y[2], a[1])
    same = np.stack([a[0], a[0]])
    _, y = oracle.encode(g, same)
    assert not y[0].any()                                   # x ^ x = 0
    _, y = oracle.encode(g, np.stack([a[0], np.zeros(512, np.uint8)]))
    assert np.array_equal(y[0], a[0])                       # x ^ 0 = x


def test_hand_built_generator_matches_brute_force():
    """random 4-symbol input, hand-built B, byte-by-byte brute-force XOR."""
    cfg = dict(k=4, p=1, n=5, t=64)
    pre_rp = np.array([0, 3], np.int32)
    pre_c = np.array([0, 2, 3], np.int32)
    rows = [[4], [0, 1], [1, 2, 4], [3], [0, 1, 2, 3, 4]]
    lt_rp = np.cumsum([0] + [len(r) for r in rows]).astype(np.int32)
    lt_c = np.array(sum(rows, []), np.int32)
    g = oracle.Graph(cfg, pre_rp, pre_c, lt_rp, lt_c)
    rng = np.random.default_rng(5)
    D = rng.integers(0, 256, (4, 64), dtype=np.uint8)
    C, Y = oracle.encode(g, D)
    chk = [[D[0][b] ^ D[2][b] ^ D[3][b] for b in range(64)]]
    assert C.tolist() == chk
    I = [list(D[m]) for m in range(4)] + chk
    for j, r in enumerate(rows):
        want = [0] * 64
        for m in r:
            want = [want[b] ^ I[m][b] for b in range(64)]
        assert Y[j].tolist() == want


@pytest.mark.parametrize("cid", [1, 2, 4])
def test_encoder_closed_forms(cid):
    """P7: enc(0) = 0; enc(a^b) = enc(a)^enc(b); all-0xFF data gives C_i = 0xFF*(d_p mod 2)
    and Y_j = 0xFF iff row j of G_eff has odd weight."""
    c = _small_cfg(cid)
    g = oracle.generate_graph(c)
    z = np.zeros((g.k, g.t), np.uint8)
    C, Y = oracle.encode(g, z)
    assert not C.any() and not Y.any()
    rng = np.random.default_rng(cid)
    a = rng.integers(0, 256, (g.k, g.t), dtype=np.uint8)
    b = rng.integers(0, 256, (g.k, g.t), dtype=np.uint8)
    Ca, Ya = oracle.encode(g, a)
    Cb, Yb = oracle.encode(g, b)
    Cab, Yab = oracle.encode(g, a ^ b)
    assert np.array_equal(Cab, Ca ^ Cb) and np.array_equal(Yab, Ya ^ Yb)
    ff = np.full((g.k, g.t), 0xFF, np.uint8)
    C, Y = oracle.encode(g, ff)
    if g.p:
        assert np.all(C == (0xFF if c["d_p"] % 2 else 0))
    G, _ = _geff(g)
    odd = G.sum(axis=1) % 2 == 1
    assert np.all(Y[odd] == 0xFF) and not Y[~odd].any()


def test_k1_all_coded_equal_d0():
    """k=1, p=0 -> every coded symbol equals D_0."""
    cfg = dict(k=1, p=0, d_p=0, n=40, t=256, dist=configs.FINITE, seed=3,
               fin_deg=configs.OMEGA_DEGREES, fin_prob=configs.OMEGA_PROBS)
    g = oracle.generate_graph(cfg)
    D = np.random.default_rng(0).integers(0, 256, (1, 256), dtype=np.uint8)
    _, Y = oracle.encode(g, D)
    assert np.all(Y == D[0])


@pytest.mark.parametrize("cid", [1, 2, 4])
def test_bit_probe_recovers_generator(cid):
    """P6: with data symbol i = one-hot bit i, bit i of Y_j is G_eff[j][i] where
    G_eff = G_LT . [I_k ; G_pre] over GF(2) (computed here by dense matrix algebra)."""
    c = _small_cfg(cid)
    g = oracle.generate_graph(c)
    assert g.k <= 8 * g.t
    D = np.zeros((g.k, g.t), np.uint8)
    for i in range(g.k):
        D[i, i // 8] = 1 << (i % 8)
    C, Y = oracle.encode(g, D)
    bits = np.unpackbits(Y, axis=1, bitorder="little")[:, :g.k]
    G, P = _geff(g)
    assert np.array_equal(bits, G.astype(np.uint8))
    if g.p:
        cb = np.unpackbits(C, axis=1, bitorder="little")[:, :g.k]
        assert np.array_equal(cb, P)


def test_lane_permutation_equivariance():
    """P7: permuting byte lanes of every input symbol permutes the outputs the same way."""
    c = _small_cfg(2)
    g = oracle.generate_graph(c)
    D = _data(c)[0]
    perm = np.random.default_rng(9).permutation(g.t)
    C, Y = oracle.encode(g, D)
    Cp, Yp = oracle.encode(g, np.ascontiguousarray(D[:, perm]))
    assert np.array_equal(Cp, C[:, perm]) and np.array_equal(Yp, Y[:, perm])


def test_multistripe_equals_per_stripe():
    """P10 (stripes): encoding S stripes = S independent stripe encodes."""
    c = configs.get(4)
    g = oracle.generate_graph(c)
    D = _data(c, S=3)
    C, Y = oracle.encode(g, D)
    for s in range(3):
        c1, y1 = oracle.encode(g, D[s])
        assert np.array_equal(c1, C[s]) and np.array_equal(y1, Y[s])


# ------------------------------------------------------------- P8/P9: decoder pins
def _determined_by_bruteforce(Gr, P, k):
    """Enumerate all 2^k data vectors; the kernel of the received map decides which data
    symbols (and which checks) are determined (P9)."""
    ker = []
    for bits in itertools.product([0, 1], repeat=k):
        x = np.array(bits, dtype=np.int64)
        if not ((Gr @ x) % 2).any():
            ker.append(x)
    ker = np.array(ker)
    data_det = ~(ker.any(axis=0))
    chk_det = ~(((ker @ P.T.astype(np.int64)) % 2).any(axis=0)) if P.shape[0] else np.zeros(0, bool)
    return data_det, chk_det, len(ker) == 1


@pytest.mark.parametrize("seed", range(12))
def test_decoder_vs_bruteforce_rank(seed):
    """P9: for k <= 12, the decoder recovers data symbol i iff every nonzero message in the
    kernel of the received generator has x_i = 0 (brute force over all 2^k messages)."""
    rng = np.random.default_rng(100 + seed)
    k = int(rng.integers(4, 13))
    p = int(rng.integers(0, 3))
    n = int(rng.integers(k, 2 * k + 3))
    cfg = dict(k=k, p=p, d_p=min(3, k), n=n, t=32, dist=configs.RSD, seed=1000 + seed,
               rsd_c=0.1, rsd_delta=0.5)
    g = oracle.generate_graph(cfg)
    D = rng.integers(0, 256, (k, 32), dtype=np.uint8)
    C, Y = oracle.encode(g, D)
    G, P = _geff(g)
    for trial in range(4):
        recv = rng.random(n) < (0.6 + 0.1 * trial)
        I, state = oracle.decode(g, recv, Y)
        data_det, chk_det, full = _determined_by_bruteforce(G[recv], P, k)
        assert np.array_equal(state[:k] != 0, data_det)
        if p:
            assert np.array_equal(state[k:] != 0, chk_det)
        rec = state[:k] != 0
        assert np.array_equal(I[:k][rec], D[rec])
        if p:
            rc = state[k:] != 0
            assert np.array_equal(I[k:][rc], C[rc])


@pytest.mark.parametrize("cid", [1, 2, 4])
def test_decoder_roundtrip_full(cid):
    """P8: from all n coded symbols the decoder (BP, + elimination)
    recovers every data symbol, and every recovered symbol equals the source."""
    c = configs.get(cid)
    g = oracle.generate_graph(c)
    D = _data(c, S=1)[0]
    C, Y = oracle.encode(g, D)
    I, state = oracle.decode(g, np.ones(g.n, bool), Y)
    assert np.all(state[:g.k] != 0)
    assert np.array_equal(I[:g.k], D)
    if g.p:
        assert np.array_equal(I[g.k:], C)


def _gf2_determined(g, recv):
    """Independent (Python big-int) GF(2) RREF over the same equations: unknown m is
    determined iff e_m is in the row space of the received system."""
    rows = []
    for j in np.nonzero(recv)[0]:
        v = 0
        for m in g.lt_row(j):
            v ^= 1 << int(m)
        rows.append(v)
    for i in range(g.p):
        v = 1 << (g.k + i)
        for m in g.pre_row(i):
            v ^= 1 << int(m)
        rows.append(v)
    piv = {}
    for v in rows:
        for b, r in piv.items():
            if (v >> b) & 1:
                v ^= r
        if v:
            b = v.bit_length() - 1
            for b2 in list(piv):
                if (piv[b2] >> b) & 1:
                    piv[b2] ^= v
            piv[b] = v
    det = np.zeros(g.K, bool)
    for b, r in piv.items():
        if r == (1 << b):
            det[b] = True
    return det


@pytest.mark.parametrize("cid,frac", [(1, 0.95), (2, 0.95), (2, 0.9), (4, 0.95)])
def test_decoder_random_subsets(cid, frac):
    """P8: random subsets of coded symbols: recovered symbols equal the source and the
    unrecovered set equals the rank-deficient set of an independent GF(2) reduction."""
    c = configs.get(cid)
    g = oracle.generate_graph(c)
    D = _data(c, S=1)[0]
    C, Y = oracle.encode(g, D)
    rng = np.random.default_rng(cid * 10 + int(frac * 100))
    for _ in range(2):
        recv = rng.random(g.n) < frac
        I, state = oracle.decode(g, recv, Y)
        I_src = np.concatenate([D, C]) if g.p else D
        ok = state != 0
        assert np.array_equal(I[ok], I_src[ok])
        assert np.array_equal(ok, _gf2_determined(g, recv))


def test_decoder_peeling_only_matches_alg1_closure():
    """Algorithm 1 alone (no elimination): the recovered set is the peeling closure; with
    an identity-like graph (n = k, column j = {j}) everything resolves at once
    (SPEC.md:306)."""
    k = 16
    cfg = dict(k=k, p=0, n=k, t=16)
    g = oracle.Graph(cfg, np.zeros(1, np.int32), np.zeros(0, np.int32),
                     np.arange(k + 1, dtype=np.int32), np.arange(k, dtype=np.int32))
    D = np.random.default_rng(2).integers(0, 256, (k, 16), dtype=np.uint8)
    _, Y = oracle.encode(g, D)
    I, state = oracle.decode(g, np.ones(k, bool), Y, use_elim=False)
    assert np.all(state == 1) and np.array_equal(I, D)
    # all coded erased -> nothing decoded
    I, state = oracle.decode(g, np.zeros(k, bool), Y, use_elim=False)
    assert not state.any()


def _peel_tool():
    import importlib.util
    spec = importlib.util.spec_from_file_location(
        "decode_readings", os.path.join(os.path.dirname(__file__), "..", "tools", "decode_readings.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


@pytest.mark.parametrize("cid,frac", [(1, 1.0), (2, 0.95), (3, 1.0), (4, 1.0), (4, 0.9)])
def test_decoder_bp_set_is_the_union_peeling_closure(cid, frac):
    """Reading R22: the oracle's BP (passes A and B alternated) recovers exactly
    the peeling closure of {received LT equations} U {precode equations} -- checked against an
    independent queue-based peeling (tools/decode_readings.py, graph only; the closure is the
    same whatever the visiting order).  The literal reading (LT BP to its fixpoint, then one
    precode BP) recovers a subset of it (profiles/r02/decode_readings.jsonl: equal on configs
    1-4, 1-2 symbols fewer on config 5)."""
    tool = _peel_tool()
    g = oracle.generate_graph(configs.get(cid))
    recv = np.ones(g.n, bool) if frac == 1.0 else np.random.default_rng(cid).random(g.n) < frac
    t = 16
    Y = np.zeros((g.n, t), np.uint8)
    _, state = oracle.decode(dict_graph_t(g, t), recv, Y, use_elim=False)
    union = tool.union_fixpoint(g, recv)
    assert np.array_equal(state != 0, union)
    lit = tool.literal_two_pass(g, recv)
    assert not np.any(lit & ~union)


def dict_graph_t(g, t):
    """The same graph with symbol size t (the recovered SET does not depend on t)."""
    cfg = dict(k=g.k, p=g.p, n=g.n, t=t)
    return oracle.Graph(cfg, g.pre_row_ptr, g.pre_col, g.lt_row_ptr, g.lt_col)


def test_paper_repair_example_xor_algebra():
    """P11 (off-path, XOR algebra only): Eqs (1)-(3) with the check #1 group
    (D0, D1, D2) give Eq (4): C2 ^ C12 ^ C17 ^ C20 ^ C21 = D0 ^ D1 ^ D2.  Checked on random
    symbols with the encoder: coded symbols built so that Eqs (1)-(3) hold."""
    g0 = {0, 1, 2}                     # D0 = C0 ^ C1 ^ C2
    g1 = {1, 12, 17, 20, 99}           # D1 = C1 ^ C12 ^ C17 ^ C20 ^ C99
    g2 = {0, 21, 99}                   # D2 = C0 ^ C21 ^ C99
    assert (g0 ^ g1 ^ g2) == {2, 12, 17, 20, 21}
    # numeric check: pick random coded symbols, derive D0..D2 with the oracle encoder
    # (rows = the groups above over 100 "source" symbols), then verify Eq (4).
    cfg = dict(k=100, p=0, n=3, t=64)
    rows = [sorted(g0), sorted(g1), sorted(g2)]
    rp = np.cumsum([0] + [len(r) for r in rows]).astype(np.int32)
    g = oracle.Graph(cfg, np.zeros(1, np.int32), np.zeros(0, np.int32), rp,
                     np.array(sum(rows, []), np.int32))
    Cs = np.random.default_rng(4).integers(0, 256, (100, 64), dtype=np.uint8)
    _, Dd = oracle.encode(g, Cs)
    lhs = Cs[2] ^ Cs[12] ^ Cs[17] ^ Cs[20] ^ Cs[21]
    assert np.array_equal(lhs, Dd[0] ^ Dd[1] ^ Dd[2])


# --------------------------------------------------------- NEXT-2: array LDPC precode (Alg 2)
ARRAY_CASES = [(3, 6), (962, 1036), (999, 1036), (837, 930), (34, 51)]


def _lpf(x):
    best, d = 1, 2
    while d * d <= x:
        while x % d == 0:
            best, x = d, x // d
        d += 1
    return x if x > 1 else best


def test_array_precode_golden_k6_b3():
    """tests/golden/array_ldpc_k6_b3.txt: Alg 2 evaluated by hand."""
    rp, col = oracle.array_precode(3, 6)
    want = [[int(r[1])] for r in _golden_rows("array_ldpc_k6_b3.txt")]
    got = [col[rp[i]:rp[i + 1]].tolist() for i in range(3)]
    assert got == want


def _golden_members(name):
    return [[int(x) for x in r[1:]] for r in _golden_rows(name)]


def test_array_precode_golden_k15_K25():
    """tests/golden/array_ldpc_k15_K25.txt: Alg 2 evaluated by hand at a shape
    where every term of the index formula is live: j' = 2, so block row 0 has the slope
    m(j'-j-1) = m, and block row 1 reads the checks of block row 0 (R18)."""
    rp, col = oracle.array_precode(15, 25)
    want = _golden_members("array_ldpc_k15_K25.txt")
    assert len(rp) == 11
    got = [col[rp[i]:rp[i + 1]].tolist() for i in range(10)]
    assert got == want


def _alg2_variant(b, K, slope_shift=-1, offset_shift=-1):
    """Alg 2's index formula with the two '-1' terms of PAPER.md:180 made parameters, for the
    mutation check below only (never used to pin the oracle):
    l = k'P - (j'-j+m-1)P - ((m(j'-j+slope_shift) - i + offset_shift + P) mod P) - 1."""
    P = _lpf(K)
    kp, jp = K // P, K // P - b // P
    return [[kp * P - (jp - j + m - 1) * P - ((m * (jp - j + slope_shift) - i + offset_shift + P) % P) - 1
             for m in range(1, kp - jp + 1)] for j in range(jp) for i in range(P)]


def test_array_precode_golden_rejects_formula_slips():
    """The k15/K25 golden is discriminating: plausible transcription slips of PAPER.md:180 --
    the slope m(j'-j) instead of m(j'-j-1), or '- i' without the '- 1' -- change rows of it (so
    an oracle carrying either slip fails test_array_precode_golden_k15_K25), while the formula
    as printed reproduces it."""
    want = _golden_members("array_ldpc_k15_K25.txt")
    assert _alg2_variant(15, 25) == want
    slope = _alg2_variant(15, 25, slope_shift=0)
    assert sum(a != b for a, b in zip(slope, want)) == 10  # every row moves
    off = _alg2_variant(15, 25, offset_shift=0)
    assert off != want


@pytest.mark.parametrize("k,K", ARRAY_CASES)
def test_array_precode_is_an_array_code(k, K):
    """Array LDPC structure (\\cite{arrayldpc}): the check matrix is built from
    P x P circulant permutation blocks -- for every block row j and member slot m, check i of
    the block row hits one block of P consecutive symbols, and i -> offset is a cyclic shift.
    Encodable in row order (linear-time): members are data or earlier checks."""
    P = _lpf(K)
    kp, jp = K // P, K // P - k // P
    rp, col = oracle.array_precode(k, K)
    d = kp - jp
    assert len(rp) == K - k + 1 and np.all(np.diff(rp) == d)
    rows = [col[rp[r]:rp[r + 1]] for r in range(K - k)]
    for r, mem in enumerate(rows):
        assert len(set(mem.tolist())) == d
        assert np.all(mem >= 0) and np.all(mem < K)
        assert np.all((mem < k) | (mem - k < r)), "references a later check"
    for j in range(jp):
        for m in range(d):
            vals = np.array([rows[i + j * P][m] for i in range(P)])
            blk = vals // P
            assert len(set(blk.tolist())) == 1, "not one block"
            off = vals % P
            shift = (off - np.arange(P)) % P
            assert len(set(shift.tolist())) == 1, "not a circulant permutation"


@pytest.mark.parametrize("k,K", [c for c in ARRAY_CASES if (c[1] // _lpf(c[1])) <= _lpf(c[1])])
def test_array_precode_has_no_four_cycles(k, K):
    """Array codes with k' <= P (Alg 3's realizability condition) have girth >= 6: two check
    groups (members + their own check symbol) share at most one symbol."""
    rp, col = oracle.array_precode(k, K)
    groups = [set(col[rp[r]:rp[r + 1]].tolist()) | {k + r} for r in range(K - k)]
    inc = np.zeros((len(groups), K), dtype=np.int64)
    for r, gset in enumerate(groups):
        inc[r, list(gset)] = 1
    share = inc @ inc.T
    np.fill_diagonal(share, 0)
    assert share.max() <= 1


def test_array_precode_rejects_unrealizable():
    for k, K in [(1000, 1020), (990, 1100), (5, 5), (0, 6)]:
        with pytest.raises(ValueError):
            oracle.array_precode(k, K)


@pytest.mark.parametrize("k,K", ARRAY_CASES[:3])
def test_array_precode_encoding_zero_syndrome(k, K):
    """Every check group XORs to zero after encoding (SPEC.md Check1Sets invariant), and the
    LT stage then reads the checks like data."""
    cfg = dict(k=k, p=K - k, d_p=0, n=int(1.25 * K), t=64, dist=configs.FINITE, seed=5,
               fin_deg=configs.OMEGA_DEGREES, fin_prob=configs.OMEGA_PROBS, precode="array", stripes=2)
    g = oracle.generate_graph(cfg)
    D = inputs.stripe_data(cfg).numpy()
    C, Y = oracle.encode(g, D)
    for s in range(2):
        I = np.concatenate([D[s], C[s]])
        for r in range(K - k):
            acc = I[k + r].copy()
            for m in g.pre_row(r):
                acc ^= I[m]
            assert not acc.any()
        for j in range(0, g.n, 7):
            acc = np.zeros(64, np.uint8)
            for m in g.lt_row(j):
                acc ^= I[m]
            assert np.array_equal(acc, Y[s][j])


# ---------------------------------------------------------- NEXT-4: per-file seed streams (R17)
def _py_rows_from_stream(words, K, deg, cdf, count):
    """Pure-Python transcription of one stream's LT rows (R5, R6, R12): per row one uniform
    u = (x >> 11) 2^-53, degree = first support point with cdf > u (clamped to K), then
    distinct neighbours x mod K by rejection, sorted ascending.  Small cases only."""
    it = iter(int(w) for w in words)
    rows = []
    for _ in range(count):
        u = (next(it) >> 11) * 2.0 ** -53
        i = int(np.searchsorted(cdf, u, side="right"))
        d = min(int(deg[min(i, len(deg) - 1)]), K)
        got = []
        while len(got) < d:
            m = next(it) % K
            if m not in got:
                got.append(m)
        rows.append(sorted(got))
    return rows


@pytest.mark.parametrize("cid,files", [(1, 5), (1, 13), (2, 4)])
def test_per_file_streams(cid, files):
    """PAPER.md:95 ("the seed of the i-th output file"): file i >= 1 is drawn from a fresh stream
    seeded seed + i (pure-Python replay from the splitmix64 known-answer stream), file 0 is the
    single-stream graph's first n/s rows (it continues the base stream after the precode)."""
    c = configs.get(cid)
    cf = dict(c, files=files)
    g1, gs = oracle.generate_graph(c), oracle.generate_graph(cf)
    n, K, per = c["n"], c["k"] + c["p"], c["n"] // files
    assert np.array_equal(gs.pre_col, g1.pre_col)                         # precode unchanged
    for j in range(per):
        assert list(gs.lt_row(j)) == list(g1.lt_row(j))
    deg, cdf = oracle.build_cdf(c["dist"], K, c.get("rsd_c", 0.0), c.get("rsd_delta", 0.0),
                                c.get("fin_deg", ()), c.get("fin_prob", ()))
    m = int(np.count_nonzero(cdf)) or len(cdf)
    deg, cdf = deg[:m], cdf[:m]
    for f in range(1, files):
        words = oracle.splitmix64(c["seed"] + f, per * (int(deg.max()) * 4 + 8))
        want = _py_rows_from_stream(words, K, deg, cdf, per)
        got = [list(gs.lt_row(j)) for j in range(f * per, (f + 1) * per)]
        assert got == want, "file %d" % f
    assert oracle.generate_graph(dict(c, files=1)).nnz == g1.nnz
