"""Multi-GPU host logic on CPU: world_size-2 (and 3) gloo process groups run
the row-partitioned GCN layer (partition -> padded all-gather -> local SpMM
-> local GEMM) with the oracle standing in for the CUDA kernels; the
concatenated per-rank outputs must equal the single-process oracle layer and
the partition bounds must be bit-exact."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


class OracleOps:
    """CPU stand-ins with the CudaOps signatures (float64 oracle arithmetic)."""

    @staticmethod
    def gemm(a, w, row_scale=None, relu=False):
        from oracle import gnn_oracle as orc

        out = orc.gemm(a.double().numpy(), w.double().numpy())
        if row_scale is not None:
            out = orc.scale_rows(row_scale.double().numpy(), out)
        if relu:
            out = np.maximum(out, 0)
        return torch.from_numpy(out)

    @staticmethod
    def spmm(a, b, d_row=None, d_col=None, relu=False, weighted=True, out=None, accumulate=False,
             hub_d=None):  # hub split = same product (GPU-only kernel choice)
        from oracle import gnn_oracle as orc

        rp, ci, v = a.numpy()
        oa = orc.Csr(a.n_rows, a.n_cols, rp, ci, v)
        bb = b.double().numpy()
        if d_col is not None:
            bb = orc.scale_rows(d_col.double().numpy(), bb)
        res = orc.spmm(oa, bb) if weighted else orc.spmm_unweighted(oa, bb)
        if d_row is not None:
            res = orc.scale_rows(d_row.double().numpy(), res)
        if accumulate:
            res = res + out.double().numpy()
        if relu:
            res = np.maximum(res, 0)
        return torch.from_numpy(res)


def _worker(rank, world, port, comp, order, q, overlap=False):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        from pathlib import Path

        root = Path(__file__).resolve().parents[1]
        sys.path.insert(0, str(root))
        import paper_2306_15155_b200 as gc
        from paper_2306_15155_b200 import graphs
        from paper_2306_15155_b200.distributed import RowPartition, all_gather_rows, dist_gcn_layer

        a = graphs.synthetic_graph("rmat", 700, 9000, seed=4, device="cpu")
        at = gc.add_self_loops(a)
        d = gc.inv_sqrt_degrees(at).double()
        rng = np.random.default_rng(5)
        h = torch.from_numpy(rng.uniform(-0.5, 0.5, (700, 12)))
        w = torch.from_numpy(rng.uniform(-0.5, 0.5, (12, 9)))
        if comp == "precompute":
            rp, ci, _ = at.numpy()
            rows = np.repeat(np.arange(700), np.diff(rp))
            dn = d.numpy()
            base = gc.CsrMatrix(700, 700, rp, ci, dn[rows] * dn[ci], device="cpu")
        else:
            base = at
        part = RowPartition.of(base, rank, world)
        # hub_unit: the hub-split plumbing (d_row/d_col of each pass); the
        # oracle ops compute the same product either way
        out = dist_gcn_layer(part, h[part.lo:part.hi], w, composition=comp, order=order,
                             d=d, ops=OracleOps, overlap=overlap, hub_unit=world == 2)
        full = all_gather_rows(out, part)
        if rank == 0:
            q.put((part.bounds.tolist(), full.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,overlap", [(2, False), (3, False), (2, True), (3, True)])
@pytest.mark.parametrize("comp,order", [("dynamic", "aggregate_first"), ("dynamic", "update_first"),
                                        ("precompute", "aggregate_first"),
                                        ("precompute", "update_first")])
def test_partitioned_layer_matches_single_process(oracle, world, overlap, comp, order):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, comp, order, q, overlap))
             for r in range(world)]
    for p in procs:
        p.start()
    bounds, full = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    import paper_2306_15155_b200 as gc
    from paper_2306_15155_b200 import graphs

    a = graphs.synthetic_graph("rmat", 700, 9000, seed=4, device="cpu")
    rp, ci, v = a.numpy()
    g = oracle.GcnGraph.from_adjacency(oracle.Csr(700, 700, rp, ci, v))
    rng = np.random.default_rng(5)
    h = rng.uniform(-0.5, 0.5, (700, 12))
    w = rng.uniform(-0.5, 0.5, (12, 9))
    ref = oracle.gcn_layer(g, h, w, comp, order)
    assert oracle.rel_err(full, ref) < 1e-6
    # nnz-balanced partition, bit-exact with the oracle restatement
    at_rp = oracle.add_self_loops(oracle.Csr(700, 700, rp, ci, v)).row_ptr
    assert bounds == oracle.partition_rows(at_rp, world).tolist()
    _ = gc
