"""Multi-rank encode on the hardware this build has: two processes share cuda:0
and talk over gloo, so the sharded encode path -- graph broadcast from rank 0, rebuild with
fs_graph_from_csr, each rank's share of the units through the C ABI, result gather to rank 0 --
runs end to end and rank 0 compares the gathered output bit for bit with the oracle.

The ranks' kernels never wait on one another (no data-path collective: the units are
independent), so sharing one GPU changes only timing, not what is computed.
The NCCL branch itself needs one GPU per rank; `test_nccl_world1_collectives` runs the same
dist.py helpers on an NCCL group of one rank (device tensors, `device_id` init).
"""
import os
import socket
import sys

import numpy as np
import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, ws, port, cid, mode, q):
    """One rank: mode 'stripes' (config 4), 'rows' or 'cols' (config 5)."""
    try:
        import torch.distributed as dist

        from paper_1702_07409_b200 import configs, dist as fdist, inputs
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=ws)
        cfg = configs.get(cid)
        g = fdist.broadcast_graph(cfg, device="cpu")          # step a2: rank 0 generates
        k, p, n, t, S = cfg["k"], cfg["p"], cfg["n"], cfg["t"], cfg["stripes"]
        if mode == "stripes":
            a, b = fdist.shard(S, ws, rank)
            d = inputs.stripe_data(cfg, a, b - a, device="cuda")   # rank-local counter-form data
            chk = torch.empty((b - a, p, t), dtype=torch.uint8, device="cuda")
            cod = torch.empty((b - a, n, t), dtype=torch.uint8, device="cuda")
            g.encode_stripes(d, chk, cod)
            torch.cuda.synchronize()
            Y = fdist.gather_stripes(cod.cpu(), S)             # gloo point-to-point to rank 0
            C = fdist.gather_stripes(chk.cpu(), S)
        else:
            d = inputs.stripe_data(cfg, device="cuda")[0]      # the full source on every rank (R16)
            chk = torch.empty((p, t), dtype=torch.uint8, device="cuda")
            if mode == "rows":
                a, b = fdist.shard(n, ws, rank)
                cod = torch.empty((b - a, t), dtype=torch.uint8, device="cuda")
                g.encode(d, chk, cod, a, b)
                torch.cuda.synchronize()
                Y = fdist.gather_stripes(cod.cpu(), n)         # rows are the units here
            else:
                c0, c1 = fdist.col_shard(t, ws, rank)
                cod = torch.full((n, t), 0x5A, dtype=torch.uint8, device="cuda")
                g.encode_range(d, chk, cod, 0, n, c0, c1)
                torch.cuda.synchronize()
                # this rank's column block of coded rows and checks (rows first, then checks)
                blk = torch.cat([cod[:, c0:c1], chk[:, c0:c1]]).contiguous().cpu()
                untouched = bool((cod[:, :c0] == 0x5A).all() and (cod[:, c1:] == 0x5A).all())
                parts = [None] * ws
                dist.all_gather_object(parts, (c0, c1, untouched))
                if rank == 0:
                    full = torch.empty((n + p, t), dtype=torch.uint8)
                    full[:, c0:c1] = blk
                    for r in range(1, ws):
                        r0, r1, _ = parts[r]
                        tmp = torch.empty((n + p, r1 - r0), dtype=torch.uint8)
                        dist.recv(tmp, r)
                        full[:, r0:r1] = tmp
                    assert all(u for _, _, u in parts), "bytes outside a rank's columns were written"
                    Y, chk_all = full[:n], full[n:]
                else:
                    dist.send(blk, 0)
                    Y = None
            if mode == "rows":
                chk_all = chk.cpu()                            # every rank computes all p checks
            C = chk_all[None] if rank == 0 else None
            if Y is not None:
                Y = Y[None]
        dist.barrier()
        dist.destroy_process_group()
        if rank == 0:
            np.save(os.path.join(q, "Y.npy"), Y.numpy())
            np.save(os.path.join(q, "C.npy"), C.numpy())
    except Exception as e:  # pragma: no cover - reported to the parent
        with open(os.path.join(q, "err%d.txt" % rank), "w") as f:
            import traceback
            f.write(repr(e) + "\n" + traceback.format_exc())
        raise


def _run(cid, mode, tmp_path, ws=2):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, ws, port, cid, mode, str(tmp_path))) for r in range(ws)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
    errs = [open(os.path.join(tmp_path, f)).read() for f in os.listdir(tmp_path) if f.startswith("err")]
    assert not errs, errs
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    return np.load(os.path.join(tmp_path, "Y.npy")), np.load(os.path.join(tmp_path, "C.npy"))


def _oracle(cid):
    import oracle
    from paper_1702_07409_b200 import configs, inputs
    cfg = configs.get(cid)
    go = oracle.generate_graph(cfg)
    D = inputs.stripe_data(cfg).numpy()
    return oracle.encode(go, D)


@pytest.mark.parametrize("cid,mode", [(4, "stripes"), (5, "rows"), (5, "cols")])
def test_sharded_encode_two_ranks(cid, mode, tmp_path):
    """PAPER.md:80 / SURVEY.md §8(e): the world-2 partition of config 4's 256 stripes, and of
    config 5's coded rows (R16) and byte columns (NEXT-4), gathered on rank 0 = the oracle's
    output for the whole workload, bit for bit."""
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    Y, C = _run(cid, mode, tmp_path)
    Co, Yo = _oracle(cid)
    if Yo.ndim == 2:
        Yo, Co = Yo[None], Co[None]
    assert Y.shape == Yo.shape
    bad = np.nonzero((Y != Yo).any(axis=-1))
    assert bad[0].size == 0, "coded rows differ: %s" % (list(zip(*bad))[:5],)
    assert np.array_equal(C, Co)


def test_nccl_world1_collectives():
    """The NCCL branch of dist.py / bench.py on the one GPU a lease gives: init with device_id,
    broadcast_graph on device tensors, max_over_ranks, gather_stripes -- then an encode with the
    broadcast graph equals the oracle."""
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    port = _free_port()
    q = ctx.Queue()
    p = ctx.Process(target=_nccl_worker, args=(port, q))
    p.start()
    res = q.get(timeout=300)
    p.join(timeout=60)
    assert res == "ok", res


def _nccl_worker(port, q):
    try:
        import torch.distributed as dist

        import oracle
        from paper_1702_07409_b200 import configs, dist as fdist, inputs
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dev = torch.device("cuda", 0)
        torch.cuda.set_device(dev)
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
        cfg = configs.get(4, stripes=8)
        g = fdist.broadcast_graph(cfg, device=dev)
        m = fdist.max_over_ranks(2.5, device=dev)
        d = inputs.stripe_data(cfg, device="cuda")
        chk = torch.empty((8, cfg["p"], cfg["t"]), dtype=torch.uint8, device="cuda")
        cod = torch.empty((8, cfg["n"], cfg["t"]), dtype=torch.uint8, device="cuda")
        g.encode_stripes(d, chk, cod)
        out = fdist.gather_stripes(cod, 8)
        torch.cuda.synchronize()
        dist.destroy_process_group()
        go = oracle.generate_graph(cfg)
        C, Y = oracle.encode(go, d.cpu().numpy())
        ok = m == 2.5 and np.array_equal(out.cpu().numpy(), Y) and np.array_equal(chk.cpu().numpy(), C)
        q.put("ok" if ok else "mismatch (max %r)" % m)
    except Exception as e:  # pragma: no cover
        q.put(repr(e))
