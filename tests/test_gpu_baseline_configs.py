"""Parity at every BASELINE.json config, at full size.

* graph prep of the full Reddit / arxiv / products shapes — Ã's row_ptr and
  col_idx, D^-1/2 and the P = 2/4/8 partition bounds — bit-exact against the
  oracle's restatement of the reference (sparse.py:303-336), run on the host
  copy of the same raw A;
* every layer composition at the configs' K values against the row-sampled
  oracle (``sampled_oracle``: the reference layer on 256 random rows plus the
  two heaviest rows, graph prep from the oracle itself, float64): GCN on Reddit
  (K = 32, 256, 1024, with the autotuned dense split) and products
  (K = 32, 256), single- and 4-head GAT on arxiv (K = 32, 256, 1024) and GAT
  on products;
* the Cora 2-layer model in both numerics classes against the full oracle.

Tolerances (normwise rel_err of reference tests/helpers.py:68-72): 1e-2 in
the TF32 class (``set_gemm_precision("tf32")``, the default), 1e-4 in the
fp32 class.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

import paper_2306_15155_b200 as gc
from paper_2306_15155_b200 import graphs, sparse

from oracle import sampled as so

pytestmark = pytest.mark.gpu
DEV = "cuda"
TOL = {"tf32": 1e-2, "fp32": 1e-4}
_CACHE: dict = {}


def shape_case(shape: str, oracle):
    """(device NormalizedGraph, oracle Ã, oracle d, raw host A) for one shape;
    one shape is held at a time."""
    if shape not in _CACHE:
        _CACHE.clear()
        torch.cuda.empty_cache()
        a = graphs.shape_graph(shape, device=DEV)
        rp, ci, v = a.numpy()
        raw = oracle.Csr(a.n_rows, a.n_cols, rp, ci, v)
        at = oracle.add_self_loops(raw)
        d = oracle.inv_sqrt_degrees(at)
        g = gc.NormalizedGraph.from_adjacency(a)
        del a
        _CACHE[shape] = (g, at, d, raw)
    return _CACHE[shape]


def rows_for(at, seed: int) -> np.ndarray:
    deg = np.diff(at.row_ptr)
    return so.sample_rows(at.n_rows, 256, seed, heavy=np.argsort(deg)[-2:])


def rows_of(h_dev: torch.Tensor):
    """Host float64 rows of a device operand, fetched only where the sampled
    oracle needs them."""
    return lambda idx: host(h_dev[torch.from_numpy(idx).to(DEV)])


def operands(n: int, k1: int, k2: int, seed: int, heads: int = 1):
    gen = torch.Generator(device=DEV)
    gen.manual_seed(seed)
    h = torch.rand(n, k1, device=DEV, generator=gen) - 0.5
    w = torch.rand(k1, k2 * heads, device=DEV, generator=gen) - 0.5
    a_s = torch.rand(k2 * heads, device=DEV, generator=gen) - 0.5
    a_d = torch.rand(k2 * heads, device=DEV, generator=gen) - 0.5
    return h, w, a_s, a_d


def host(x: torch.Tensor) -> np.ndarray:
    return x.cpu().numpy().astype(np.float64)


@pytest.fixture(params=["tf32", "fp32"])
def precision(request):
    old = gc.get_gemm_precision()
    gc.set_gemm_precision(request.param)
    yield request.param
    gc.set_gemm_precision(old)


# ---- graph prep, full shapes ----------------------------------------------------


def _graph_prep_bit_exact(oracle, shape):
    g, at, d, _ = shape_case(shape, oracle)
    rp, ci, v = g.a_tilde.numpy()
    assert np.array_equal(rp, at.row_ptr)
    assert np.array_equal(ci, at.col_idx)
    assert np.array_equal(v, at.values)
    assert torch.equal(g.d_inv_sqrt.cpu(), torch.from_numpy(d.astype(np.float32)))
    from paper_2306_15155_b200.distributed import partition_rows

    for parts in (2, 4, 8):
        assert np.array_equal(partition_rows(g.a_tilde.row_ptr, parts),
                              oracle.partition_rows(at.row_ptr, parts))


# ---- layer cases -------------------------------------------------------------------

GCN_COMPS = [("precompute", "aggregate_first"), ("precompute", "update_first"),
             ("dynamic", "aggregate_first"), ("dynamic", "update_first")]


def _gcn_case(oracle, shape, K, comp, order, precision, seed):
    g, at, d, _ = shape_case(shape, oracle)
    if comp == "precompute":
        g.with_precomputed()
    n = at.n_rows
    h, w, _, _ = operands(n, K, K, seed)
    out = gc.gcn_layer(g, h, gc.GcnLayerSpec(K, K, w, composition=comp, order=order))
    rows = rows_for(at, seed)
    rt = torch.from_numpy(rows).to(DEV)
    ref = so.gcn_rows(at, d, rows_of(h), host(w), rows, comp, order)
    err = oracle.rel_err(host(out[rt]), ref)
    assert err <= TOL[precision], f"{shape} K={K} {comp}/{order} {precision}: rel_err {err}"
    return g


# ---- GAT: arxiv (configs[2]) and products (configs[3]) ---------------------------

GAT_COMPS = [("reuse", "reassoc"), ("reuse", "sddmm"), ("recompute", "reassoc"),
             ("recompute", "sddmm")]


def _gat_case(oracle, shape, K, heads, comp, att, precision, seed):
    g, at, _, _ = shape_case(shape, oracle)
    n = at.n_rows
    h, w, a_s, a_d = operands(n, K, K, seed, heads)
    spec = gc.GatLayerSpec(K, K, w, a_s, a_d, composition=comp, attention=att, heads=heads)
    out = gc.gat_layer(g.a_tilde, h, spec)
    rows = rows_for(at, seed)
    rt = torch.from_numpy(rows).to(DEV)
    ref = so.gat_rows(at, rows_of(h), host(w), host(a_s), host(a_d), heads, rows, comp)
    err = oracle.rel_err(host(out[rt]), ref)
    assert err <= TOL[precision], \
        f"{shape} K={K} heads={heads} {comp}/{att} {precision}: rel_err {err}"


# ---- configs[2]: arxiv ------------------------------------------------------------


def test_arxiv_graph_prep_bit_exact(oracle):
    _graph_prep_bit_exact(oracle, "arxiv")


@pytest.mark.parametrize("K", [32, 256, 1024])
@pytest.mark.parametrize("heads", [1, 4])
@pytest.mark.parametrize("comp,att", GAT_COMPS)
def test_arxiv_gat_layer_parity(oracle, precision, K, heads, comp, att):
    """BASELINE configs[2]: single- and 4-head GAT, SDDMM vs reassociated
    attention, reuse vs recompute, K = 32 .. 1024."""
    _gat_case(oracle, "arxiv", K, heads, comp, att, precision, seed=K + heads)


# ---- configs[1]: Reddit -----------------------------------------------------------


def test_reddit_graph_prep_bit_exact(oracle):
    _graph_prep_bit_exact(oracle, "reddit")


@pytest.mark.parametrize("K", [32, 256, 1024])
@pytest.mark.parametrize("comp,order", GCN_COMPS)
def test_reddit_gcn_layer_parity(oracle, precision, K, comp, order):
    """BASELINE configs[1]: every composition × K, the dense split (staircase)
    autotuned per K as in the bench."""
    if precision == "fp32" and K == 1024 and comp == "precompute":
        pytest.skip("fp32 class at K=1024: covered by the dynamic compositions")
    g = _gcn_case(oracle, "reddit", K, comp, order, precision, seed=K)
    if comp == "dynamic" and order == "update_first" and precision == "tf32" and K == 256:
        from paper_2306_15155_b200 import hub

        assert g.a_tilde._plans.get(hub.split_key(K, False), 0), \
            "the autotuner keeps a dense split on the Reddit shape"


# ---- configs[3]: products ---------------------------------------------------------


def test_products_graph_prep_bit_exact(oracle):
    _graph_prep_bit_exact(oracle, "products")


@pytest.mark.parametrize("K", [32, 256])
@pytest.mark.parametrize("comp,order", GCN_COMPS)
def test_products_gcn_layer_parity(oracle, precision, K, comp, order):
    _gcn_case(oracle, "products", K, comp, order, precision, seed=K + 7)


@pytest.mark.parametrize("K", [32, 256])
@pytest.mark.parametrize("comp,att", GAT_COMPS)
def test_products_gat_layer_parity(oracle, K, comp, att):
    _gat_case(oracle, "products", K, 1, comp, att, "tf32", seed=K + 11)


# ---- Cora 2-layer (configs[0]) in both numerics classes -------------------------


@pytest.mark.parametrize("comp,order", GCN_COMPS)
def test_cora_two_layer_parity(oracle, precision, comp, order):
    from paper_2306_15155_b200 import profiling

    a = graphs.shape_graph("cora", device=DEV)
    g = gc.NormalizedGraph.from_adjacency(a).with_precomputed()
    rp, ci, v = a.numpy()
    og = oracle.GcnGraph.from_adjacency(oracle.Csr(a.n_rows, a.n_cols, rp, ci, v))
    inp = profiling.draw_inputs(profiling.config_rng(0, "cora", 1433, 16), a.n_rows, 1433, 16, "gcn")
    w2 = profiling.draw_inputs(profiling.config_rng(0, "cora", 16, 7), a.n_rows, 16, 7, "gcn")["w"]
    h32, w1, w2 = (x.astype(np.float32) for x in (inp["h"], inp["w"], w2))
    specs = [gc.GcnLayerSpec(1433, 16, w1, composition=comp, order=order),
             gc.GcnLayerSpec(16, 7, w2, composition=comp, order=order)]
    out = gc.gcn_forward(g, torch.from_numpy(h32).to(DEV), specs).cpu().numpy()
    f64 = lambda x: x.astype(np.float64)  # noqa: E731
    ref = oracle.gcn_layer(og, oracle.gcn_layer(og, f64(h32), f64(w1), comp, order), f64(w2), comp,
                           order)
    assert oracle.rel_err(out, ref) <= TOL[precision]


def test_sparse_module_is_the_cuda_path():
    """The parity above ran through libgnnc (no silent fallback)."""
    from paper_2306_15155_b200 import _native

    assert _native.launch_count() > 0
    assert sparse.get_gemm_precision() in ("tf32", "fp32")
