"""The row-partitioned layer with the real kernels (and the hub split) on one
GPU: 2 ranks of a gloo group share cuda:0, so the multi-GPU host path —
partition, padded all-gather, owned/remote split, per-rank hub block — runs
through libgnnc; outputs are compared with the single-process oracle."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, comp, order, overlap, q):
    import sys
    from pathlib import Path

    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2306_15155_b200 as gc
        from paper_2306_15155_b200 import graphs, hub
        from paper_2306_15155_b200.distributed import RowPartition, all_gather_rows, dist_gcn_layer

        hub.HUB_SPLIT = "64"
        dev = torch.device("cuda", 0)
        a = graphs.powerlaw_graph(2500, 40, seed=11, device=dev)
        g = gc.NormalizedGraph.from_adjacency(a).with_precomputed()
        rng = np.random.default_rng(8)
        h = torch.from_numpy(rng.uniform(-0.5, 0.5, (2500, 40)).astype(np.float32)).to(dev)
        w = torch.from_numpy(rng.uniform(-0.5, 0.5, (40, 24)).astype(np.float32)).to(dev)
        gc.set_gemm_precision("fp32")
        part = RowPartition.of(g.n_tilde if comp == "precompute" else g.a_tilde, rank, world)
        out = dist_gcn_layer(part, h[part.lo:part.hi], w, composition=comp, order=order,
                             d=g.d_inv_sqrt.to(dev), overlap=overlap, hub_unit=True)
        used = any(k[0] == "hubsplit" for k in part.padded()._plans) or \
            any(k[0] == "hubsplit" for k in part.split_local_remote()[1]._plans)
        full = all_gather_rows(out.cpu(), part)
        if rank == 0:
            q.put((full.numpy(), used))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("overlap", [False, True])
@pytest.mark.parametrize("comp,order", [("dynamic", "update_first"), ("precompute", "aggregate_first")])
def test_partitioned_layer_with_hub_split_on_gpu(oracle, comp, order, overlap):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, comp, order, overlap, q))
             for r in range(2)]
    for p in procs:
        p.start()
    full, used = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert used
    import paper_2306_15155_b200 as gc
    from paper_2306_15155_b200 import graphs

    a = graphs.powerlaw_graph(2500, 40, seed=11, device="cuda")
    rp, ci, v = a.numpy()
    og = oracle.GcnGraph.from_adjacency(oracle.Csr(2500, 2500, rp, ci, v))
    rng = np.random.default_rng(8)
    h = rng.uniform(-0.5, 0.5, (2500, 40)).astype(np.float32)
    w = rng.uniform(-0.5, 0.5, (40, 24)).astype(np.float32)
    ref = oracle.gcn_layer(og, h.astype(np.float64), w.astype(np.float64), comp, order)
    assert oracle.rel_err(full, ref) <= 1e-4
    _ = gc


def _gat_worker(rank, world, port, comp, att, heads, q, half=False):
    import sys
    from pathlib import Path

    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2306_15155_b200 as gc
        from paper_2306_15155_b200 import graphs
        from paper_2306_15155_b200.distributed import RowPartition, all_gather_rows, dist_gat_layer

        dev = torch.device("cuda", 0)
        at = gc.add_self_loops(graphs.powerlaw_graph(3000, 30, seed=12, device=dev))
        rng = np.random.default_rng(21)
        k1, k2 = 48, 32
        h = torch.from_numpy(rng.uniform(-0.5, 0.5, (3000, k1)).astype(np.float32)).to(dev)
        w = rng.uniform(-0.5, 0.5, (k1, k2 * heads)).astype(np.float32)
        a_s = rng.uniform(-0.5, 0.5, k2 * heads).astype(np.float32)
        a_d = rng.uniform(-0.5, 0.5, k2 * heads).astype(np.float32)
        from paper_2306_15155_b200 import distributed, gcn

        used = []
        if half:  # TF32 class with fp16 gathers at test size
            gcn.HALF_MIN_BYTES = 0
            real = distributed.all_gather_half_multi
            distributed.all_gather_half_multi = lambda *a, **k: used.append(1) or real(*a, **k)
        gc.set_gemm_precision("tf32" if half else "fp32")
        spec = gc.GatLayerSpec(k1, k2, w, a_s, a_d, composition=comp, attention=att, heads=heads)
        part = RowPartition.of(at, rank, world)
        out = dist_gat_layer(part, h[part.lo:part.hi], spec)
        full = all_gather_rows(out.cpu(), part)
        if rank == 0:
            q.put((full.numpy(), bool(used)) if half else full.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("comp,att", [("reuse", "reassoc"), ("reuse", "sddmm"),
                                      ("recompute", "reassoc"), ("recompute", "sddmm")])
@pytest.mark.parametrize("heads", [1, 4])
def test_partitioned_gat_layer_on_gpu(oracle, comp, att, heads):
    """dist_gat_layer with the real kernels (2 gloo ranks sharing cuda:0):
    the concatenated rank outputs equal the single-process oracle (fp32 mode,
    1e-4)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gat_worker, args=(r, 2, port, comp, att, heads, q))
             for r in range(2)]
    for p in procs:
        p.start()
    full = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from paper_2306_15155_b200 import graphs

    rp, ci, v = graphs.powerlaw_graph(3000, 30, seed=12, device="cuda").numpy()
    at = oracle.add_self_loops(oracle.Csr(3000, 3000, rp, ci, v))
    rng = np.random.default_rng(21)
    k1, k2 = 48, 32
    h = rng.uniform(-0.5, 0.5, (3000, k1)).astype(np.float32).astype(np.float64)
    w = rng.uniform(-0.5, 0.5, (k1, k2 * heads)).astype(np.float32).astype(np.float64)
    a_s = rng.uniform(-0.5, 0.5, k2 * heads).astype(np.float32).astype(np.float64)
    a_d = rng.uniform(-0.5, 0.5, k2 * heads).astype(np.float32).astype(np.float64)
    ref = oracle.gat_layer_multihead(at, h, w, a_s, a_d, heads, 0.2, comp, "relu")
    assert oracle.rel_err(full, ref) <= 1e-4


@pytest.mark.parametrize("comp", ["reuse", "recompute"])
@pytest.mark.parametrize("heads", [1, 4])
def test_partitioned_gat_layer_fp16_gather_on_gpu(oracle, comp, heads):
    """TF32 class: the reassoc GAT partition all-gathers fp16 rows (one set of
    row scales per head) and t in one collective; against the oracle at the
    class's tolerance."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gat_worker, args=(r, 2, port, comp, "reassoc", heads, q, True))
             for r in range(2)]
    for p in procs:
        p.start()
    full, used = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert used, "the fp16 all-gather did not run"
    from paper_2306_15155_b200 import graphs

    rp, ci, v = graphs.powerlaw_graph(3000, 30, seed=12, device="cuda").numpy()
    at = oracle.add_self_loops(oracle.Csr(3000, 3000, rp, ci, v))
    rng = np.random.default_rng(21)
    k1, k2 = 48, 32
    h = rng.uniform(-0.5, 0.5, (3000, k1)).astype(np.float32).astype(np.float64)
    w = rng.uniform(-0.5, 0.5, (k1, k2 * heads)).astype(np.float32).astype(np.float64)
    a_s = rng.uniform(-0.5, 0.5, k2 * heads).astype(np.float32).astype(np.float64)
    a_d = rng.uniform(-0.5, 0.5, k2 * heads).astype(np.float32).astype(np.float64)
    ref = oracle.gat_layer_multihead(at, h, w, a_s, a_d, heads, 0.2, comp, "relu")
    assert oracle.rel_err(full, ref) <= 5e-3


def _half_worker(rank, world, port, comp, order, overlap, q):
    import sys
    from pathlib import Path

    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2306_15155_b200 as gc
        from paper_2306_15155_b200 import gcn, graphs, hub
        from paper_2306_15155_b200.distributed import RowPartition, all_gather_rows, dist_gcn_layer

        gcn.HALF_MIN_BYTES = 0  # fp16 gathers at test size
        hub.HUB_SPLIT = "stair:40"
        dev = torch.device("cuda", 0)
        a = graphs.synthetic_graph("rmat", 6000, 300000, seed=5, device=dev)
        g = gc.NormalizedGraph.from_adjacency(a).with_precomputed()
        rng = np.random.default_rng(9)
        h = torch.from_numpy(rng.uniform(-0.5, 0.5, (6000, 40)).astype(np.float32)).to(dev)
        w = torch.from_numpy(rng.uniform(-0.5, 0.5, (40, 32)).astype(np.float32)).to(dev)
        gc.set_gemm_precision("tf32")
        part = RowPartition.of(g.n_tilde if comp == "precompute" else g.a_tilde, rank, world)
        out = dist_gcn_layer(part, h[part.lo:part.hi], w, composition=comp, order=order,
                             d=g.d_inv_sqrt.to(dev), overlap=overlap, hub_unit=True)
        full = all_gather_rows(out.cpu(), part)
        if rank == 0:
            q.put(full.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("overlap", [False, True])
@pytest.mark.parametrize("comp,order", [("dynamic", "update_first"), ("dynamic", "aggregate_first"),
                                        ("precompute", "update_first")])
def test_partitioned_layer_fp16_gather_on_gpu(oracle, comp, order, overlap):
    """TF32 class, fp16 rows + scales all-gathered in one collective (half the
    bytes), the staircase split on each rank reading the same fp16 rows:
    against the oracle at the class's tolerance."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_half_worker, args=(r, 2, port, comp, order, overlap, q))
             for r in range(2)]
    for p in procs:
        p.start()
    full = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from paper_2306_15155_b200 import graphs

    rp, ci, v = graphs.synthetic_graph("rmat", 6000, 300000, seed=5, device="cuda").numpy()
    og = oracle.GcnGraph.from_adjacency(oracle.Csr(6000, 6000, rp, ci, v))
    rng = np.random.default_rng(9)
    h = rng.uniform(-0.5, 0.5, (6000, 40)).astype(np.float32).astype(np.float64)
    w = rng.uniform(-0.5, 0.5, (40, 32)).astype(np.float32).astype(np.float64)
    ref = oracle.gcn_layer(og, h, w, comp, order)
    assert oracle.rel_err(full, ref) <= 3e-3
