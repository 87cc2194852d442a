"""Multi-GPU host logic on CPU: world_size-2 gloo process groups.

Covers step a2 (rank 0 generates the graph, the CSR is broadcast, the other ranks rebuild it with
fs_graph_from_csr), the max-over-ranks timing reduction, and bench.py's work partition (stripes
for multi-stripe configs, coded rows for a single stripe).  No GPU is touched: graphs are
host-only.
"""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from paper_1702_07409_b200 import configs, dist as fdist, fsb  # noqa: E402


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, ws, port, cid, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=ws)
        cfg = configs.get(cid)
        g = fdist.broadcast_graph(cfg, device="cpu", host_only=True)
        local = fsb.Graph.create(cfg, host_only=True)      # independent regeneration
        same = all(np.array_equal(a, b) for a, b in zip(g.csr(), local.csr()))
        t = fdist.max_over_ranks(1.5 + rank, device="cpu")
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, same, t, g.info()["lt_nnz"]))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, "error", repr(e), None))


@pytest.mark.parametrize("cid", [2, 4])
def test_graph_broadcast_gloo_world2(cid):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, cid, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    res.sort()
    for rank, same, t, nnz in res:
        assert same is True, (rank, same, t)
        assert t == 2.5                                     # max over ranks
    assert res[0][3] == res[1][3]


def test_shard_covers_exactly_once():
    for total in (0, 1, 7, 256, 60000):
        for ws in (1, 2, 3, 4, 8):
            seen = []
            for r in range(ws):
                a, b = fdist.shard(total, ws, r)
                assert 0 <= a <= b <= total
                assert b - a in (total // ws, total // ws + 1)
                seen.extend(range(a, b))
            assert seen == list(range(total))
    with pytest.raises(ValueError):
        fdist.shard(10, 2, 2)


def test_bench_plan():
    import bench
    c4, c5 = configs.get(4), configs.get(5)
    for ws in (1, 2, 4, 8):
        stripes = [bench.plan(c4, ws, r, "strong") for r in range(ws)]
        assert all(k == "stripes" for k, _, _ in stripes)
        assert sum(cnt for _, _, cnt in stripes) == c4["stripes"]
        assert [s0 for _, s0, _ in stripes] == sorted(s0 for _, s0, _ in stripes)
        weak = [bench.plan(c4, ws, r, "weak") for r in range(ws)]
        assert all(cnt == c4["stripes"] and s0 == r * c4["stripes"] for r, (_, s0, cnt) in enumerate(weak))
        rows = [bench.plan(c5, ws, r, "strong") for r in range(ws)]
        if ws == 1:
            assert rows == [("stripes", 0, 1)]
        else:
            assert all(k == "rows" for k, _, _ in rows)
            assert rows[0][1] == 0 and rows[-1][2] == c5["n"]
            assert all(rows[i][2] == rows[i + 1][1] for i in range(ws - 1))


def test_col_shard_covers_exactly_once():
    for t in (16, 64, 80, 4096, 320 * 1024, 1000016):
        for ws in (1, 2, 3, 4, 8):
            parts = [fdist.col_shard(t, ws, r) for r in range(ws)]
            assert parts[0][0] == 0 and parts[-1][1] == t
            for (a, b), (c, d) in zip(parts, parts[1:]):
                assert b == c
            for a, b in parts:
                assert a <= b and a % 64 == 0 and (b % 64 == 0 or b == t)


def test_bench_plan_cols():
    import bench
    c5 = configs.get(5)
    for ws in (2, 4, 8):
        parts = [bench.plan(c5, ws, r, "strong", "cols") for r in range(ws)]
        assert all(k == "cols" for k, _, _ in parts)
        assert parts[0][1] == 0 and parts[-1][2] == c5["t"]


def _gather_worker(rank, ws, port, total, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=ws)
        b, e = fdist.shard(total, ws, rank)
        # stripe s of the job = bytes (s * 7 + column) & 0xFF: rank 0 can check every slice
        local = ((torch.arange(b, e).view(-1, 1, 1) * 7 + torch.arange(96).view(1, 1, -1)) & 0xFF)
        local = local.expand(e - b, 3, 96).to(torch.uint8).contiguous()
        out = fdist.gather_stripes(local, total)
        ok = None
        if rank == 0:
            want = ((torch.arange(total).view(-1, 1, 1) * 7 + torch.arange(96).view(1, 1, -1)) & 0xFF)
            ok = bool(torch.equal(out, want.expand(total, 3, 96).to(torch.uint8)))
        else:
            ok = out is None
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, ok))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e)))


@pytest.mark.parametrize("ws,total", [(2, 5), (3, 7), (3, 2)])
def test_gather_stripes_to_rank0(ws, total):
    """§8(e)(ii): every rank's contiguous stripe shard lands in its slice of rank 0's output
    (ragged shards, and a rank with no stripes)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gather_worker, args=(r, ws, port, total, q)) for r in range(ws)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert all(ok is True for _, ok in res), res
