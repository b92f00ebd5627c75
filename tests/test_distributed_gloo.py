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


def _into(res: np.ndarray, out):
    t = torch.from_numpy(np.ascontiguousarray(res))
    if out is None:
        return t
    out.copy_(t)
    return out


def _ocsr(a):
    from oracle import gnn_oracle as orc

    rp, ci, v = a.numpy()
    return orc.Csr(a.n_rows, a.n_cols, rp, ci, v)


class OracleOps:
    """CPU stand-ins with the CudaOps signatures (float64 oracle arithmetic)."""

    @staticmethod
    def gemm(a, w, row_scale=None, relu=False, out=None):
        from oracle import gnn_oracle as orc

        res = orc.gemm(a.double().numpy(), w.double().numpy()) if a.shape[0] else \
            np.zeros((0, w.shape[1]))
        if row_scale is not None:
            res = orc.scale_rows(row_scale.double().numpy(), res)
        if relu:
            res = np.maximum(res, 0)
        return _into(res, out)

    @staticmethod
    def node_scores(x, a_src, a_dst, heads, width, head_stride):
        xs = x.double().numpy()
        s = np.stack([xs[:, h * head_stride:h * head_stride + width]
                      @ a_src.double().numpy()[h * width:(h + 1) * width] for h in range(heads)])
        t = np.stack([xs[:, h * head_stride:h * head_stride + width]
                      @ a_dst.double().numpy()[h * width:(h + 1) * width] for h in range(heads)])
        return torch.from_numpy(s.reshape(heads, -1)), torch.from_numpy(t.reshape(heads, -1))

    @staticmethod
    def gat_aggregate(a, s, t, slope, b, relu=False, out=None):
        """edge softmax (gat.py:72-95) then spmm(alpha, B) on the oracle."""
        from oracle import gnn_oracle as orc

        oa = _ocsr(a)
        alpha = orc.edge_softmax(oa, s.double().numpy(), t.double().numpy(), slope)
        res = orc.spmm(oa.with_values(alpha), b.double().numpy())
        return _into(np.maximum(res, 0) if relu else res, out)

    @staticmethod
    def gat_sddmm_aggregate(a, a_src, a_dst, slope, b, b_self, relu=False, out=None):
        s = b_self.double().numpy() @ a_src.double().numpy()
        t = b.double().numpy() @ a_dst.double().numpy()
        return OracleOps.gat_aggregate(a, torch.from_numpy(s), torch.from_numpy(t), slope, b,
                                       relu=relu, out=out)

    @staticmethod
    def attn_sddmm(a, hw, hw_self, a_src, a_dst, slope, heads, k2):
        from oracle import gnn_oracle as orc

        oa = _ocsr(a)
        hwn, hsn = hw.double().numpy(), hw_self.double().numpy()
        al = [orc.edge_softmax(oa, hsn[:, h * k2:(h + 1) * k2] @ a_src.double().numpy()[h * k2:(h + 1) * k2],
                               hwn[:, h * k2:(h + 1) * k2] @ a_dst.double().numpy()[h * k2:(h + 1) * k2],
                               slope) for h in range(heads)]
        return torch.from_numpy(np.stack(al))

    @staticmethod
    def spmm(a, b, d_row=None, d_col=None, relu=False, weighted=True, out=None, accumulate=False,
             hub_d=None):  # hub split = same product (GPU-only kernel choice)
        from oracle import gnn_oracle as orc

        rp, ci, v = a.numpy()
        oa = orc.Csr(a.n_rows, a.n_cols, rp, ci, v)
        bb = b.double().numpy()
        if d_col is not None:
            bb = orc.scale_rows(d_col.double().numpy(), bb)
        res = (orc.spmm(oa, bb) if weighted else orc.spmm_unweighted(oa, bb)) if a.n_rows else \
            np.zeros((0, bb.shape[1]))
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


# ---- GAT partition (reuse gathers HW_p and t_p, recompute H_p and t_p) ----

N_GAT, E_GAT, K1, K2 = 600, 7000, 12, 8


def _gat_worker(rank, world, port, comp, att, heads, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        from pathlib import Path

        sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
        import paper_2306_15155_b200 as gc
        from paper_2306_15155_b200 import graphs
        from paper_2306_15155_b200.distributed import RowPartition, all_gather_rows, dist_gat_layer

        at = gc.add_self_loops(graphs.synthetic_graph("rmat", N_GAT, E_GAT, seed=6, device="cpu"))
        rng = np.random.default_rng(9)
        h = torch.from_numpy(rng.uniform(-0.5, 0.5, (N_GAT, K1)))
        w = rng.uniform(-0.5, 0.5, (K1, K2 * heads))
        a_s, a_d = rng.uniform(-0.5, 0.5, K2 * heads), rng.uniform(-0.5, 0.5, K2 * heads)
        spec = gc.GatLayerSpec(K1, K2, w, a_s, a_d, composition=comp, attention=att, heads=heads)
        part = RowPartition.of(at, rank, world)
        out = dist_gat_layer(part, h[part.lo:part.hi], spec, ops=OracleOps)
        full = all_gather_rows(out.double(), part)
        if rank == 0:
            q.put(full.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("comp,att", [("reuse", "reassoc"), ("reuse", "sddmm"),
                                      ("recompute", "reassoc"), ("recompute", "sddmm")])
@pytest.mark.parametrize("heads", [1, 2])
def test_partitioned_gat_layer_matches_single_process(oracle, world, comp, att, heads):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gat_worker, args=(r, world, port, comp, att, heads, q))
             for r in range(world)]
    for p in procs:
        p.start()
    full = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from paper_2306_15155_b200 import graphs

    rp, ci, v = graphs.synthetic_graph("rmat", N_GAT, E_GAT, seed=6, device="cpu").numpy()
    at = oracle.add_self_loops(oracle.Csr(N_GAT, N_GAT, rp, ci, v))
    rng = np.random.default_rng(9)
    h = rng.uniform(-0.5, 0.5, (N_GAT, K1))
    w = rng.uniform(-0.5, 0.5, (K1, K2 * heads))
    # the spec holds float32 copies of W and the attention vectors
    w = w.astype(np.float32).astype(np.float64)
    a_s = rng.uniform(-0.5, 0.5, K2 * heads).astype(np.float32).astype(np.float64)
    a_d = rng.uniform(-0.5, 0.5, K2 * heads).astype(np.float32).astype(np.float64)
    ref = oracle.gat_layer_multihead(at, h, w, a_s, a_d, heads, 0.2, comp, "relu")
    assert full.shape == ref.shape
    assert oracle.rel_err(full, ref) < 1e-6


def _empty_worker(rank, world, port, q):
    """world > n: some ranks own no rows: they still join every
    collective and return 0-row outputs."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        from pathlib import Path

        sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
        import paper_2306_15155_b200 as gc
        from paper_2306_15155_b200.distributed import (RowPartition, all_gather_rows, dist_gat_layer,
                                                       dist_gcn_layer)

        # a 2-node graph (one edge) on 3 ranks
        at = gc.add_self_loops(gc.CsrMatrix.from_coo(2, 2, [0, 1], [1, 0], [1.0, 1.0], device="cpu"))
        d = gc.inv_sqrt_degrees(at).double()
        rng = np.random.default_rng(1)
        h = torch.from_numpy(rng.uniform(-0.5, 0.5, (2, 4)))
        w = torch.from_numpy(rng.uniform(-0.5, 0.5, (4, 4)))
        part = RowPartition.of(at, rank, world)
        res = {}
        for overlap in (False, True):
            for order in ("aggregate_first", "update_first"):
                y = dist_gcn_layer(part, h[part.lo:part.hi], w, composition="dynamic", order=order,
                                   d=d, ops=OracleOps, overlap=overlap)
                res[(overlap, order)] = all_gather_rows(y.double(), part).numpy()
        spec = gc.GatLayerSpec(4, 4, w.numpy(), np.ones(4) * 0.1, np.ones(4) * 0.2)
        y = dist_gat_layer(part, h[part.lo:part.hi], spec, ops=OracleOps)
        res["gat"] = all_gather_rows(y.double(), part).numpy()
        if rank == 0:
            q.put((part.bounds.tolist(), res))
    finally:
        dist.destroy_process_group()


def test_partition_with_empty_ranks(oracle):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_empty_worker, args=(r, 3, port, q)) for r in range(3)]
    for p in procs:
        p.start()
    bounds, res = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert 0 in np.diff(bounds)  # some rank owns no rows
    og = oracle.GcnGraph.from_adjacency(oracle.Csr(2, 2, [0, 1, 2], [1, 0], [1.0, 1.0]))
    rng = np.random.default_rng(1)
    h = rng.uniform(-0.5, 0.5, (2, 4))
    w = rng.uniform(-0.5, 0.5, (4, 4))
    for (overlap, order), full in ((k, v) for k, v in res.items() if k != "gat"):
        ref = oracle.gcn_layer(og, h, w, "dynamic", order)
        assert oracle.rel_err(full, ref) < 1e-6, (overlap, order)
    w32 = w.astype(np.float32).astype(np.float64)
    ref = oracle.gat_layer(og.a_tilde, h, w32, np.full(4, np.float32(0.1)), np.full(4, np.float32(0.2)))
    assert oracle.rel_err(res["gat"], ref) < 1e-6
