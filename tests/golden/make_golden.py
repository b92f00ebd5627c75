"""Generate the golden vectors that pin the oracle and the host logic.

Run HERE (the build container), never on the GPU box: it imports the
reference package ``gnncompose`` straight from ``/root/reference/pkg/src``
(read-only; bytecode/numba caches redirected to /tmp) and records its outputs
on small seeded inputs.  The outputs are committed as
``tests/golden/golden.npz`` and ``tests/golden/selector_golden.json``.

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden.py

Every dense input is rounded to float32 first (then fed to the reference as
float64) so that a float32 device path differs from these vectors only by
its arithmetic, never by its inputs.
"""

from __future__ import annotations

import json
import os
import sys
from pathlib import Path

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.dont_write_bytecode = True
REF_SRC = "/root/reference/pkg/src"
sys.path.insert(0, REF_SRC)

import numpy as np  # noqa: E402

import gnncompose as ref  # noqa: E402  (the reference, read-only)
from gnncompose import gat as ref_gat  # noqa: E402
from gnncompose import gcn as ref_gcn  # noqa: E402
from gnncompose import graphs as ref_graphs  # noqa: E402
from gnncompose import profiling as ref_prof  # noqa: E402
from gnncompose import selector as ref_sel  # noqa: E402

OUT = Path(__file__).resolve().parent


def f32(x):
    return np.asarray(x, dtype=np.float64).astype(np.float32).astype(np.float64)


def weighted_symmetric(n, density, seed):
    rng = np.random.default_rng(seed)
    upper = np.triu(rng.random((n, n)) < density, k=1)
    r, c = np.nonzero(upper)
    v = f32(rng.uniform(0.5, 2.0, size=r.size))
    return ref.CsrMatrix.from_coo(n, n, np.concatenate((r, c)), np.concatenate((c, r)),
                                  np.concatenate((v, v)))


def with_some_diagonal(n, seed):
    rng = np.random.default_rng(seed)
    a = ref_graphs.random_graph(n, 0.1, seed=seed)
    d = np.flatnonzero(rng.random(n) < 0.4)
    rows = np.concatenate((a.row_of_nnz(), d))
    cols = np.concatenate((a.col_idx, d))
    vals = np.concatenate((a.values, np.full(d.size, 1.0)))
    return ref.CsrMatrix.from_coo(n, n, rows, cols, vals)


def graphs():
    return {
        "path3": ref_graphs.path_graph(3),
        "star5": ref_graphs.star_graph(5),
        "grid4x5": ref_graphs.grid_graph(4, 5),
        "powerlaw200": ref_graphs.powerlaw_graph(200, 4, seed=7),
        "random120": ref_graphs.random_graph(120, 0.05, seed=3),
        "weighted40": weighted_symmetric(40, 0.15, seed=11),
        "diag30": with_some_diagonal(30, seed=5),
    }


SIZES = [(6, 3), (3, 6), (5, 5)]


def put_csr(store, key, a):
    store[f"{key}/shape"] = np.array([a.n_rows, a.n_cols], dtype=np.int64)
    store[f"{key}/row_ptr"] = a.row_ptr
    store[f"{key}/col_idx"] = a.col_idx
    store[f"{key}/values"] = a.values


def main():
    store: dict[str, np.ndarray] = {}
    meta = {"graphs": [], "sizes": SIZES, "reference": "gnncompose " + ref.__version__}

    # ---- kernel-level cases (sparse.py) ---------------------------------
    rng = np.random.default_rng(20240817)
    dense = (rng.random((12, 9)) < 0.35) * f32(rng.uniform(0.5, 2.0, size=(12, 9)))
    dense[4, :] = 0.0  # an empty row
    a = ref.CsrMatrix.from_dense(dense)
    b = f32(rng.standard_normal((9, 5)))
    bs = f32(rng.standard_normal((12, 3)))
    cs = f32(rng.standard_normal((9, 3)))
    put_csr(store, "kern/a", a)
    store["kern/b"] = b
    store["kern/spmm"] = ref.spmm(a, b)
    store["kern/spmm_unweighted"] = ref.spmm_unweighted(a, b)
    store["kern/sddmm_b"] = bs
    store["kern/sddmm_c"] = cs
    store["kern/sddmm"] = ref.sddmm(a, bs, cs).values
    # from_coo with duplicates and unsorted input
    rr = np.array([3, 0, 1, 3, 0, 2, 3, 0], dtype=np.int64)
    cc = np.array([1, 2, 0, 1, 2, 2, 0, 0], dtype=np.int64)
    vv = f32(np.array([1.5, 2.0, 3.0, 0.25, 4.0, 1.0, 2.0, 7.0]))
    coo = ref.CsrMatrix.from_coo(4, 3, rr, cc, vv)
    store["coo/rows"], store["coo/cols"], store["coo/vals"] = rr, cc, vv
    put_csr(store, "coo/out", coo)

    # ---- per-graph cases -------------------------------------------------
    for gid, A in graphs().items():
        meta["graphs"].append(gid)
        put_csr(store, f"{gid}/A", A)
        feats = ref.extract_features(A)
        store[f"{gid}/features"] = feats.vector()
        g = ref.NormalizedGraph.from_adjacency(A, precompute=True)
        put_csr(store, f"{gid}/At", g.a_tilde)
        store[f"{gid}/d"] = g.d_inv_sqrt
        store[f"{gid}/Nt"] = g.n_tilde.values
        n = A.n_rows
        for k1, k2 in SIZES:
            key = f"{gid}/{k1}x{k2}"
            r = ref_prof._config_rng(0, gid, k1, k2)
            inp = ref_prof._draw_inputs(r, n, k1, k2, "gat", "relu")
            h, w = f32(inp["h"]), f32(inp["w"])
            a_s, a_d = f32(inp["attn_src"]), f32(inp["attn_dst"])
            store[f"{key}/h"], store[f"{key}/w"] = h, w
            store[f"{key}/attn_src"], store[f"{key}/attn_dst"] = a_s, a_d
            # GCN: heuristic layer for both compositions ...
            for comp in ("precompute", "dynamic"):
                spec = ref.GcnLayerSpec(k1, k2, w, composition=comp)
                store[f"{key}/gcn/{comp}/heuristic"] = ref.gcn_layer(g, h, spec)
            # ... and both forced orders through the reference's own
            # _aggregate_update (gcn.py:119-122), as gcn_layer_* would.
            for order in (ref.AggregationOrder.AGGREGATE_FIRST, ref.AggregationOrder.UPDATE_FIRST):
                pre = ref_gcn._relu(ref_gcn._aggregate_update(ref.spmm, g.n_tilde, h, w, order))
                agg = ref.spmm_unweighted if g.a_tilde.has_unit_values else ref.spmm
                sc = ref.scale_rows(g.d_inv_sqrt, h)
                dyn = ref_gcn._relu(ref.scale_rows(
                    g.d_inv_sqrt, ref_gcn._aggregate_update(agg, g.a_tilde, sc, w, order)))
                store[f"{key}/gcn/precompute/{order.value}"] = pre
                store[f"{key}/gcn/dynamic/{order.value}"] = dyn
            # GAT
            for slope in (0.2, 0.1):
                spec = ref.GatLayerSpec(k1, k2, w, a_s, a_d, leaky_slope=slope)
                hw = ref.gemm(h, w)
                store[f"{key}/gat/s{slope}/alpha"] = ref.atten_calc(g.a_tilde, hw, spec).alpha.values
                for comp in ("reuse", "recompute"):
                    for act in ("relu", "none"):
                        spec = ref.GatLayerSpec(k1, k2, w, a_s, a_d, leaky_slope=slope,
                                                composition=comp, activation=act)
                        store[f"{key}/gat/s{slope}/{comp}/{act}"] = ref.gat_layer(g.a_tilde, h, spec)

    # ---- input recipe (profiling.py:127-130, 251-259) -----------------------
    r = ref_prof._config_rng(0, "cora", 5, 3)
    inp = ref_prof._draw_inputs(r, 7, 5, 3, "gat", "relu")
    for k in ("h", "w", "attn_src", "attn_dst"):
        store[f"recipe/{k}"] = inp[k]

    np.savez_compressed(OUT / "golden.npz", **store)

    # ---- selector (selector.py) --------------------------------------------
    sel = {}
    recs = []
    rng = np.random.default_rng(7)
    gfeat = {}
    for gi in range(14):
        n = int(rng.integers(100, 5000))
        nnz = int(n * rng.uniform(2, 40))
        gfeat[f"g{gi}"] = ref.GraphFeatures(
            n_rows=n, n_nnzs=nnz, nnz_den=nnz / (n * n), nnz_mean=nnz / n,
            d_min=int(rng.integers(1, 3)), d_max=int(rng.integers(10, 500)),
            d_dentr=float(rng.uniform(0.1, 0.9)), e_dentr=float(rng.uniform(0.5, 1.0)))
    for model, comps in ref_sel.COMPOSITIONS.items():
        for gid, f in gfeat.items():
            for k1, k2 in [(32, 32), (32, 256), (256, 32)]:
                for ci, comp in enumerate(comps):
                    # synthetic timing rule with a feature-dependent crossover
                    base = f.n_nnzs * (k1 if ci == 0 else k2) * 1e-9
                    t = base * (1.0 + 0.3 * ci * (f.nnz_mean > 20)) + 1e-6 * (ci + 1)
                    recs.append(ref_prof.ProfileRecord(
                        graph_id=gid, model=model, k1=k1, k2=k2, composition=comp,
                        features=f, hw_tag="golden", median_time_s=float(t), iterations=3))
        # one incomplete group (must be dropped with a warning)
        recs.append(ref_prof.ProfileRecord(
            graph_id="lonely", model=model, k1=64, k2=64, composition=comps[0],
            features=gfeat["g0"], hw_tag="golden", median_time_s=1.0, iterations=3))
    sel["records"] = [r.to_dict() for r in recs]
    hyper = ref.SelectorHyperparams(n_estimators=12, learning_rate=0.1, max_depth=3, reg_lambda=1.0)
    import warnings

    for model in ("gcn", "gat"):
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            m = ref.train(recs, model, hyper)
        sel[f"{model}/model"] = m.to_dict()
        picks = []
        for gid, f in list(gfeat.items())[:6]:
            for k1, k2 in [(32, 32), (64, 512), (512, 64)]:
                inp = ref.SelectorInput(features=f, k1=k1, k2=k2)
                comp, scores = ref.select_with_scores(m, inp)
                picks.append({"graph": gid, "k1": k1, "k2": k2, "choice": comp,
                              "scores": {k: float(v) for k, v in scores.items()}})
        sel[f"{model}/picks"] = picks
        sel[f"{model}/importance"] = [[n, float(v)] for n, v in ref.feature_importance(m)]
    # a constant (no-tree) model must reproduce the defaults
    (OUT / "selector_golden.json").write_text(json.dumps(sel))
    (OUT / "golden_meta.json").write_text(json.dumps(meta, indent=1))
    print("wrote", OUT / "golden.npz", len(store), "arrays")


if __name__ == "__main__":
    main()
