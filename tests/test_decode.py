"""Decoder: the Alg 5 (DPG) plan on the host and fs_decode on the GPU.

The oracle's decoder with elimination switched off is Alg 1 (BP) run to convergence over the LT
rows and the precode checks; its recovered set -- the peeling closure -- is
unique, so the plan must recover exactly that set ("upon convergence ...") and the
GPU must reproduce the oracle's recovered bytes bit for bit.
"""
import numpy as np
import pytest
import torch

import oracle
from paper_1702_07409_b200 import configs, fsb, inputs


def _recv(n, frac, seed):
    if frac >= 1.0:
        return np.ones(n, dtype=bool)
    return np.random.default_rng(seed).random(n) < frac


def _small(cid):
    c = configs.get(cid)
    if cid == 3:
        c = dict(c, k=1200, p=24, n=1450)
    return c


CASES = [(1, 1.0), (1, 0.97), (2, 1.0), (2, 0.95), (3, 1.0), (3, 0.98), (4, 1.0), (4, 0.9)]


def _plan_rows(plan_obj):
    """Decode rows from the C plan (via the state/level views and the graph): (level, target)."""
    st, lev = plan_obj.state()
    return st, lev


@pytest.mark.parametrize("cid,frac", CASES)
def test_plan_recovers_the_peeling_closure(cid, frac):
    c = _small(cid)
    g = fsb.Graph.create(c, host_only=True)
    recv = _recv(c["n"], frac, 7 + cid)
    plan = fsb.DecodePlan(g, recv, host_only=True)
    st, lev = plan.state()
    go = oracle.generate_graph(c)
    D = inputs.stripe_data(c, num_stripes=1).numpy()[0]
    _, Y = oracle.encode(go, D)
    _, ostate = oracle.decode(go, recv, Y, use_elim=False)
    assert np.array_equal(st, (ostate == 1).astype(np.uint8))
    inf = plan.info()
    assert inf["recovered"] == int(st.sum()) == inf["rows"]
    assert inf["received"] == int(recv.sum())
    assert np.all((lev >= 0) == (st == 1))
    assert inf["levels"] == (int(lev.max()) + 1 if st.any() else 0)


def _py_dpg_levels(c, recv):
    """Independent transcription of Alg 5's level structure in Python: the
    level at which each intermediate symbol becomes decodable (one unknown left)."""
    go = oracle.generate_graph(c)
    k, p, n = c["k"], c["p"], c["n"]
    K = k + p
    eqs = [set(go.lt_row(j).tolist()) for j in range(n) if recv[j]]
    eqs += [set(go.pre_row(i).tolist()) | {k + i} for i in range(p)]
    level = np.full(K, -1)
    known = set()
    L = 0
    while True:
        ready = {next(iter(e - known)) for e in eqs if len(e - known) == 1}
        if not ready:
            break
        for f in ready:
            level[f] = L
        known |= ready
        L += 1
    return level


@pytest.mark.parametrize("cid,frac", [(1, 1.0), (2, 0.95), (4, 0.9)])
def test_plan_levels_match_alg5(cid, frac):
    c = _small(cid)
    recv = _recv(c["n"], frac, 3)
    g = fsb.Graph.create(c, host_only=True)
    _, lev = fsb.DecodePlan(g, recv, host_only=True).state()
    assert np.array_equal(lev, _py_dpg_levels(c, recv))


def test_plan_rejects_bad_arguments():
    c = configs.get(1)
    g = fsb.Graph.create(c, host_only=True)
    with pytest.raises(ValueError):
        fsb.DecodePlan(g, np.ones(c["n"] - 1, dtype=bool), host_only=True)
    plan = fsb.DecodePlan(g, np.zeros(c["n"], dtype=bool), host_only=True)
    assert plan.info()["recovered"] == 0 and plan.info()["levels"] == 0


@pytest.mark.gpu
@pytest.mark.parametrize("cid,frac,S", [(1, 0.97, 3), (2, 0.95, 2), (3, 0.98, 1), (4, 1.0, 5), (4, 0.9, 3)])
def test_gpu_decode_matches_oracle(cid, frac, S):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    c = dict(_small(cid), stripes=S)
    recv = _recv(c["n"], frac, 11 + cid)
    go = oracle.generate_graph(c)
    D = inputs.stripe_data(c).numpy()
    C, Y = oracle.encode(go, D)
    g = fsb.Graph.create(c)
    plan = fsb.DecodePlan(g, recv)
    K, t = c["k"] + c["p"], c["t"]
    Yd = torch.from_numpy(Y).cuda()
    Yd[:, ~torch.from_numpy(recv)] = 0x77          # erased rows must never be read
    inter = torch.full((S, K, t), 0xA5, dtype=torch.uint8, device="cuda")
    plan.decode(Yd, inter)
    torch.cuda.synchronize()
    I = inter.cpu().numpy()
    st, _ = plan.state()
    for s in range(S):
        oI, ostate = oracle.decode(go, recv, Y[s], use_elim=False)
        rec = ostate == 1
        assert np.array_equal(st.astype(bool), rec)
        assert np.array_equal(I[s][rec], oI[rec])
        assert np.all(I[s][~rec] == 0xA5)                     # unrecovered rows untouched
        data_rec = rec[:c["k"]]
        assert np.array_equal(I[s][:c["k"]][data_rec], D[s][data_rec])   # recovered data = source
        if c["p"]:
            chk_rec = rec[c["k"]:]
            assert np.array_equal(I[s][c["k"]:][chk_rec], C[s][chk_rec])


@pytest.mark.parametrize("cid,frac", [(1, 1.0), (1, 0.97), (2, 0.95), (3, 0.98), (4, 1.0), (4, 0.9)])
def test_plan_elimination_matches_oracle(cid, frac):
    """FS_DECODE_ELIMINATE: the plan recovers exactly the symbols the received equations determine
    (the oracle's BP + Gauss-Jordan state: 1 = peeled, 2 = eliminated), every peeled one in the
    same way as without elimination."""
    c = _small(cid)
    recv = _recv(c["n"], frac, 11 + cid)
    go = oracle.generate_graph(c)
    g = fsb.Graph.create(c, host_only=True)
    D = inputs.stripe_data(c).numpy()[0]
    _, Y = oracle.encode(go, D)
    _, ostate = oracle.decode(go, recv, Y, use_elim=True)
    plan = fsb.DecodePlan(g, recv, host_only=True, eliminate=True)
    st, lev = plan.state()
    assert np.array_equal(st, ostate)
    inf = plan.info()
    assert inf["eliminated"] == int((ostate == 2).sum()) and not inf["elim_skipped"]
    base = fsb.DecodePlan(g, recv, host_only=True).state()
    assert np.array_equal(base[0], (st == 1).astype(base[0].dtype)) and np.array_equal(base[1][st == 1], lev[st == 1])


def test_plan_with_array_precode_matches_oracle():
    """Decoding through Alg 2 checks (checks whose members include earlier checks)."""
    c = dict(configs.get(6), n=1150)
    recv = _recv(c["n"], 0.97, 5)
    g = fsb.Graph.create(c, host_only=True)
    st, _ = fsb.DecodePlan(g, recv, host_only=True).state()
    go = oracle.generate_graph(c)
    D = inputs.stripe_data(c, num_stripes=1).numpy()[0]
    _, Y = oracle.encode(go, D)
    _, ostate = oracle.decode(go, recv, Y, use_elim=False)
    assert np.array_equal(st, (ostate == 1).astype(np.uint8))


@pytest.mark.gpu
@pytest.mark.parametrize("cid,frac,S", [(1, 0.97, 3), (1, 1.0, 1), (2, 0.9, 2), (4, 1.0, 2), (4, 0.9, 2),
                                         (4, 0.82, 1), (3, 0.98, 1), (3, 0.9, 1)])
def test_gpu_decode_eliminate_matches_oracle(cid, frac, S):
    """GPU bytes of the peeling levels + the inactivation-decoding rows = the oracle's BP +
    Gauss-Jordan decode, = the source data for every determined data symbol."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    c = dict(_small(cid), stripes=S)
    recv = _recv(c["n"], frac, 11 + cid)
    go = oracle.generate_graph(c)
    D = inputs.stripe_data(c).numpy()
    C, Y = oracle.encode(go, D)
    g = fsb.Graph.create(c)
    plan = fsb.DecodePlan(g, recv, eliminate=True)
    K, t = c["k"] + c["p"], c["t"]
    Yd = torch.from_numpy(Y).cuda()
    Yd[:, ~torch.from_numpy(recv)] = 0x77
    inter = torch.full((S, K, t), 0xA5, dtype=torch.uint8, device="cuda")
    plan.decode(Yd, inter)
    torch.cuda.synchronize()
    I = inter.cpu().numpy()
    st, _ = plan.state()
    for s in range(S):
        oI, ostate = oracle.decode(go, recv, Y[s], use_elim=True)
        rec = ostate != 0
        assert np.array_equal(st != 0, rec)
        assert np.array_equal(I[s][rec], oI[rec])           # (unrecovered rows may hold partials)
        assert np.array_equal(I[s][:c["k"]][rec[:c["k"]]], D[s][rec[:c["k"]]])


@pytest.mark.parametrize("seed", range(16))
def test_plan_elimination_random_graphs(seed):
    """Random small codes and reception patterns (incl. p = 0, all / none received): the
    inactivation-completed plan = the oracle's BP + Gauss-Jordan state."""
    rng = np.random.default_rng(500 + seed)
    k = int(rng.integers(1, 80))
    p = int(rng.integers(0, 8))
    n = int(rng.integers(1, 160))
    c = dict(name="r", k=k, p=p, d_p=int(rng.integers(1, min(k, 4) + 1)) if p else 0, n=n, t=16, stripes=1,
             dist=configs.FINITE, seed=int(rng.integers(1, 1 << 40)),
             fin_deg=configs.OMEGA_DEGREES, fin_prob=configs.OMEGA_PROBS)
    go = oracle.generate_graph(c)
    g = fsb.Graph.create(c, host_only=True)
    D = inputs.stripe_data(c).numpy()[0]
    _, Y = oracle.encode(go, D)
    for frac in (0.0, 0.5, 0.8, 1.0):
        recv = rng.random(n) < frac
        _, ostate = oracle.decode(go, recv, Y, use_elim=True)
        st, lev = fsb.DecodePlan(g, recv, host_only=True, eliminate=True).state()
        assert np.array_equal(st, ostate), (seed, frac)
        assert np.all((lev >= 0) == (st != 0))


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(6))
def test_gpu_decode_eliminate_random_graphs(seed):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    rng = np.random.default_rng(900 + seed)
    k = int(rng.integers(8, 300))
    p = int(rng.integers(0, 12))
    n = int(k + p + rng.integers(0, 80))
    c = dict(name="r", k=k, p=p, d_p=int(rng.integers(1, min(k, 4) + 1)) if p else 0, n=n,
             t=int(rng.choice([16, 512, 1040])), stripes=2, dist=configs.RSD, rsd_c=0.1, rsd_delta=0.5,
             seed=int(rng.integers(1, 1 << 40)))
    try:
        go = oracle.generate_graph(c)
    except ValueError:
        pytest.skip("RSD parameters rejected")
    D = inputs.stripe_data(c).numpy()
    _, Y = oracle.encode(go, D)
    recv = rng.random(n) < float(rng.uniform(0.8, 1.0))
    g = fsb.Graph.create(c)
    plan = fsb.DecodePlan(g, recv, eliminate=True)
    Yd = torch.from_numpy(Y).cuda()
    Yd[:, ~torch.from_numpy(recv)] = 0x77
    inter = torch.full((2, g.K, c["t"]), 0xA5, dtype=torch.uint8, device="cuda")
    plan.decode(Yd, inter)
    torch.cuda.synchronize()
    I = inter.cpu().numpy()
    for s in range(2):
        oI, ostate = oracle.decode(go, recv, Y[s], use_elim=True)
        rec = ostate != 0
        assert np.array_equal(I[s][rec], oI[rec])

