"""bench.py contract (CPU): the reference arm (the oracle, this tier's reference) and the GPU arm
describe the same launch with an identical `config` object, so the driver's same-config check
holds (round-1 VERDICT: the arms emitted different key sets)."""
import argparse
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_1702_07409_b200 import configs, fsb  # noqa: E402


@pytest.mark.parametrize("cid,ws,partition", [(4, 1, "rows"), (4, 2, "rows"), (4, 8, "rows"),
                                              (5, 1, "rows"), (5, 4, "rows"), (5, 4, "cols")])
def test_reference_and_gpu_arm_configs_identical(cid, ws, partition):
    args = argparse.Namespace(scaling="strong", partition=partition, variant="auto")
    cfg = configs.get(cid)
    ref = bench._reference_config(args, cfg, ws)
    g = fsb.Graph.create(cfg, host_only=True)
    inf = g.info()
    kind, u0, u1 = bench.plan(cfg, ws, 0, args.scaling, args.partition)
    S = u1 if kind == "stripes" else 1
    ours = bench.workload_config(cfg, args, ws, kind, S, u0, u1, inf["lt_nnz"], inf["max_degree"])
    assert ref == ours
