"""Host-side logic on CPU: CSR construction/validation semantics, graph prep
bit-exactness, features, the input recipe, the selector (trained trees must
equal the reference's on the same records), synthetic generators."""

from __future__ import annotations

import json
import warnings

import numpy as np
import pytest
import torch

import paper_2306_15155_b200 as gc
from paper_2306_15155_b200 import graphs, profiling, selector

from conftest import GOLDEN

CPU = "cpu"
GRAPHS = ["path3", "star5", "grid4x5", "powerlaw200", "random120", "weighted40", "diag30"]


def gcsr(golden, key):
    n_rows, n_cols = (int(x) for x in golden[f"{key}/shape"])
    return gc.CsrMatrix(n_rows, n_cols, golden[f"{key}/row_ptr"], golden[f"{key}/col_idx"],
                        golden[f"{key}/values"], device=CPU)


# ---- CsrMatrix semantics (reference tests/test_sparse.py:32-68) ----------------


def test_from_coo_sums_duplicates():
    a = gc.CsrMatrix.from_coo(2, 2, [0, 0, 1], [1, 1, 0], [2.0, 3.0, 1.0], device=CPU)
    assert a.nnz == 2 and a.to_dense()[0, 1] == 5.0


def test_from_coo_matches_reference_golden(golden):
    a = gc.CsrMatrix.from_coo(4, 3, golden["coo/rows"], golden["coo/cols"], golden["coo/vals"],
                              device=CPU)
    rp, ci, v = a.numpy()
    assert np.array_equal(rp, golden["coo/out/row_ptr"])
    assert np.array_equal(ci, golden["coo/out/col_idx"])
    assert np.array_equal(v, golden["coo/out/values"].astype(np.float32))


def test_from_coo_rejects_out_of_range_before_merging():
    """an out-of-range column must raise, not alias a valid entry
    of the next row and be summed into it (reference lexsort + _check)."""
    with pytest.raises(gc.ShapeError, match="column index out of range"):
        gc.CsrMatrix.from_coo(3, 3, [1, 0], [0, 3], [1, 1], device=CPU)
    with pytest.raises(gc.ShapeError, match="column index out of range"):
        gc.CsrMatrix.from_coo(3, 3, [0], [-1], [1.0], device=CPU)
    with pytest.raises(gc.ShapeError):
        gc.CsrMatrix.from_coo(2, 2, [2], [0], [1.0], device=CPU)
    with pytest.raises(ValueError):
        gc.CsrMatrix.from_coo(2, 2, [-1], [0], [1.0], device=CPU)


def test_validation_rejects_bad_row_ptr():
    with pytest.raises(gc.ShapeError):
        gc.CsrMatrix(2, 2, np.array([0, 1]), np.array([0]), np.array([1.0]), device=CPU)
    with pytest.raises(gc.ShapeError):
        gc.CsrMatrix(2, 2, np.array([0, 2, 1]), np.array([0, 1]), np.ones(2), device=CPU)


def test_validation_rejects_bad_columns():
    with pytest.raises(gc.ShapeError):
        gc.CsrMatrix(2, 2, np.array([0, 1, 2]), np.array([0, 5]), np.ones(2), device=CPU)
    with pytest.raises(gc.ShapeError):
        gc.CsrMatrix(1, 3, np.array([0, 2]), np.array([2, 0]), np.ones(2), device=CPU)
    gc.CsrMatrix(2, 3, np.array([0, 1, 2]), np.array([2, 0]), np.ones(2), device=CPU)


def test_unit_value_flag():
    assert gc.CsrMatrix(3, 3, np.arange(4), np.arange(3), np.ones(3), device=CPU).has_unit_values
    a = gc.CsrMatrix(1, 2, np.array([0, 2]), np.array([0, 1]), np.array([1.0, 2.0]), device=CPU)
    assert not a.has_unit_values


def test_dense_matrix_rejects_non_finite():
    with pytest.raises(ValueError):
        gc.dense_matrix(np.array([[1.0, np.nan]]))


@pytest.mark.parametrize("gid", GRAPHS)
def test_graph_prep_bit_exact(golden, gid):
    a = gcsr(golden, f"{gid}/A")
    at = gc.add_self_loops(a)
    rp, ci, v = at.numpy()
    assert np.array_equal(rp, golden[f"{gid}/At/row_ptr"])
    assert np.array_equal(ci, golden[f"{gid}/At/col_idx"])
    assert np.array_equal(v, golden[f"{gid}/At/values"].astype(np.float32))
    assert gc.add_self_loops(at).same_pattern(at)  # idempotent
    d = gc.inv_sqrt_degrees(at).numpy()
    assert np.array_equal(d, golden[f"{gid}/d"].astype(np.float32))
    f = gc.extract_features(a).vector()
    assert np.array_equal(f, golden[f"{gid}/features"])


def test_add_self_loops_edge_cases():
    e = gc.CsrMatrix(2, 2, np.zeros(3, np.int64), np.array([], np.int64), np.array([]), device=CPU)
    assert torch.equal(gc.add_self_loops(e).to_dense(), torch.eye(2))
    with pytest.raises(gc.ShapeError):
        gc.add_self_loops(gc.CsrMatrix(2, 3, np.zeros(3, np.int64), np.array([], np.int64),
                                       np.array([]), device=CPU))


@pytest.mark.parametrize("seed", range(20))
def test_add_self_loops_random_counting(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 30))
    dense = (rng.random((n, n)) < rng.uniform(0, 0.8)) * rng.uniform(0.5, 2, (n, n))
    a = gc.CsrMatrix.from_dense(dense, device=CPU)
    missing = int((np.diag(dense) == 0).sum())
    out = gc.add_self_loops(a)
    assert out.nnz == a.nnz + missing
    ref = dense.copy()
    ref[np.diag_indices(n)] = np.where(np.diag(dense) != 0, np.diag(dense), 1.0)
    assert np.allclose(out.to_dense().numpy(), ref)
    out._check()


def test_inv_sqrt_degrees_errors_and_values():
    a = gc.CsrMatrix(2, 2, np.array([0, 1, 1]), np.array([0]), np.ones(1), device=CPU)
    with pytest.raises(gc.DegenerateNodeError):
        gc.inv_sqrt_degrees(a)
    a = gc.CsrMatrix(1, 4, np.array([0, 4]), np.arange(4), np.ones(4), device=CPU)
    assert gc.inv_sqrt_degrees(a)[0].item() == 0.5


# ---- layer specs (reference gcn.py:58-73, gat.py:30-57) ------------------------------


def test_spec_validation():
    with pytest.raises(gc.ShapeError):
        gc.GcnLayerSpec(3, 2, np.ones((2, 3)))
    with pytest.raises(ValueError):
        gc.GcnLayerSpec(0, 2, np.ones((0, 2)))
    with pytest.raises(ValueError):
        gc.GatLayerSpec(2, 2, np.ones((2, 2)), np.ones(2), np.ones(2), leaky_slope=1.5)
    with pytest.raises(ValueError):
        gc.GatLayerSpec(2, 2, np.ones((2, 2)), np.ones(2), np.ones(2), activation="tanh")
    with pytest.raises(gc.ShapeError):
        gc.GatLayerSpec(2, 2, np.ones((2, 2)), np.ones(3), np.ones(2))
    s = gc.GatLayerSpec(2, 3, np.ones((2, 6)), np.ones(6), np.ones(6), heads=2)
    assert s.heads == 2


def test_ordering_heuristic_known_answers():
    assert gc.ordering_heuristic(1024, 32) is gc.AggregationOrder.UPDATE_FIRST
    assert gc.ordering_heuristic(32, 256) is gc.AggregationOrder.AGGREGATE_FIRST
    assert gc.ordering_heuristic(64, 64) is gc.AggregationOrder.AGGREGATE_FIRST
    with pytest.raises(ValueError):
        gc.ordering_heuristic(0, 3)


def test_input_recipe_matches_reference(golden):
    inp = profiling.draw_inputs(profiling.config_rng(0, "cora", 5, 3), 7, 5, 3, "gat")
    for k in ("h", "w", "attn_src", "attn_dst"):
        assert np.array_equal(inp[k], golden[f"recipe/{k}"])


# ---- selector: same trees as the reference on the same records ----------------


@pytest.fixture(scope="module")
def sel_golden():
    return json.loads((GOLDEN / "selector_golden.json").read_text())


@pytest.mark.parametrize("model", ["gcn", "gat"])
def test_selector_trains_reference_identical_trees(sel_golden, model):
    recs = [profiling.ProfileRecord.from_dict(d) for d in sel_golden["records"]]
    hyper = gc.SelectorHyperparams(n_estimators=12, learning_rate=0.1, max_depth=3, reg_lambda=1.0)
    with warnings.catch_warnings(record=True) as w:
        warnings.simplefilter("always")
        m = gc.train(recs, model, hyper)
    assert any("single composition" in str(x.message) for x in w)
    exp = sel_golden[f"{model}/model"]
    got = m.to_dict()
    assert got["feature_names"] == exp["feature_names"]
    assert len(got["trees"]) == len(exp["trees"])
    for tg, te in zip(got["trees"], exp["trees"]):
        assert tg["feature"] == te["feature"]
        assert tg["left"] == te["left"] and tg["right"] == te["right"]
        np.testing.assert_array_equal(tg["threshold"], te["threshold"])
        np.testing.assert_allclose(tg["value"], te["value"], rtol=1e-12, atol=1e-15)
    np.testing.assert_allclose(got["feature_gain"], exp["feature_gain"], rtol=1e-12)
    # the reference's model file loads and scores identically here
    ref_model = gc.SelectorModel.from_dict(exp)
    for pick in sel_golden[f"{model}/picks"]:
        feats = recs[[r.graph_id for r in recs].index(pick["graph"])].features
        inp = gc.SelectorInput(features=feats, k1=pick["k1"], k2=pick["k2"])
        choice, scores = gc.select_with_scores(ref_model, inp)
        assert choice == pick["choice"]
        for k, v in pick["scores"].items():
            assert scores[k] == pytest.approx(v, rel=1e-12, abs=1e-15)
    imp = gc.feature_importance(ref_model)
    assert [n for n, _ in imp] == [n for n, _ in sel_golden[f"{model}/importance"]]


def test_selector_errors_and_defaults(sel_golden):
    recs = [profiling.ProfileRecord.from_dict(d) for d in sel_golden["records"]][:10]
    with pytest.raises(gc.InsufficientDataError):
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            gc.train(recs, "gcn")
    with pytest.raises(ValueError):
        gc.train(recs, "mlp")
    empty = gc.SelectorModel("gcn", selector.feature_layout(0))
    inp = gc.SelectorInput(features=recs[0].features, k1=8, k2=8)
    assert gc.select(empty, inp) == "dynamic"
    with pytest.raises(gc.SchemaError):
        gc.SelectorModel.from_dict({"format_version": 99})
    with pytest.raises(gc.SchemaError):
        empty.score(np.zeros(3))


def test_selector_multiway_roundtrip(tmp_path, sel_golden):
    base = [profiling.ProfileRecord.from_dict(d) for d in sel_golden["records"] if d["model"] == "gcn"]
    comps = selector.B200_COMPOSITIONS["gcn"]
    recs = []
    for r in base:
        if r.composition != "precompute":
            continue
        for i, c in enumerate(comps):
            t = r.median_time_s * (1 + 0.1 * ((i + r.k1 // 32) % 4))
            recs.append(profiling.ProfileRecord.from_dict({**r.to_dict(), "composition": c,
                                                           "median_time_s": t}))
    m = gc.train(recs, "gcn", gc.SelectorHyperparams(n_estimators=20, learning_rate=0.3, max_depth=3),
                 compositions=comps)
    p = tmp_path / "m.json"
    m.save(p)
    m2 = gc.SelectorModel.load(p)
    assert m2.candidates == comps
    inp = gc.SelectorInput(features=recs[0].features, k1=recs[0].k1, k2=recs[0].k2)
    assert gc.select(m2, inp) in comps


# ---- synthetic generators ------------------------------------------------------


@pytest.mark.parametrize("kind,n,nnz", [("uniform", 500, 3000), ("rmat", 1000, 20000),
                                        ("rmat", 3000, 40000)])
def test_synthetic_graph_exact_and_symmetric(kind, n, nnz):
    a = graphs.synthetic_graph(kind, n, nnz, seed=1, device=CPU)
    assert a.nnz == nnz and a.n_rows == n
    a._check()
    d = a.to_dense()
    assert torch.equal(d, d.T) and not bool(torch.diagonal(d).any())
    b = graphs.synthetic_graph(kind, n, nnz, seed=1, device=CPU)
    assert a.same_pattern(b)
    c = graphs.synthetic_graph(kind, n, nnz, seed=2, device=CPU)
    assert not a.same_pattern(c)


def test_synthetic_graph_is_a_prefix_in_counter_order():
    # a smaller target is the earliest-generated subset of a larger one
    small = graphs.synthetic_graph("rmat", 2000, 10000, seed=3, device=CPU)
    big = graphs.synthetic_graph("rmat", 2000, 14000, seed=3, device=CPU)
    ds, db = small.to_dense(), big.to_dense()
    assert bool((db[ds > 0] > 0).all())


def test_rmat_is_power_law():
    a = graphs.synthetic_graph("rmat", 4096, 80000, seed=0, device=CPU)
    f = gc.extract_features(a)
    assert f.d_max > 20 * f.nnz_mean
    u = graphs.synthetic_graph("uniform", 4096, 80000, seed=0, device=CPU)
    assert gc.extract_features(u).d_max < 3 * f.nnz_mean


def test_hash_matches_python_reference():
    x = torch.tensor([0, 1, 12345, -7], dtype=torch.int64)
    got = graphs.splitmix64(x).tolist()
    exp = [graphs._s64(graphs._splitmix64_int(v & graphs._M64)) for v in (0, 1, 12345, -7)]
    assert got == exp


def test_sweep_plan_and_train_roundtrip(tmp_path, sel_golden, monkeypatch):
    from paper_2306_15155_b200 import sweep

    plan = sweep.graph_plan()
    assert len(plan) > 30 and {k for _, k, _, _ in plan} == {"uniform", "rmat"}
    assert all(nnz <= sweep.MAX_NNZ and nnz % 2 == 0 for _, _, _, nnz in plan)
    assert [p[0] for p in sweep.named_plan()] == ["arxiv", "reddit", "products"]
    # synthetic 4-composition records -> train/evaluate/save through the CLI
    base = [profiling.ProfileRecord.from_dict(d) for d in sel_golden["records"] if d["model"] == "gcn"]
    comps = selector.B200_COMPOSITIONS["gcn"]
    recs = []
    for r in base:
        if r.composition != "precompute":
            continue
        for i, c in enumerate(comps):
            fast = (i == 3) if r.features.nnz_mean > 20 else (i == 0)
            recs.append(profiling.ProfileRecord.from_dict(
                {**r.to_dict(), "composition": c, "median_time_s": r.median_time_s * (1 if fast else 1.5)}))
    path = tmp_path / "r.ndjson"
    profiling.write_records(path, recs)
    monkeypatch.setattr(selector, "MODEL_DIR", tmp_path / "models")
    rep = tmp_path / "rep.json"
    sweep.main(["train", "--records", str(path), "--trees", "20", "--lr", "0.3", "--depth", "3",
                "--report", str(rep)])
    report = json.loads(rep.read_text())
    assert report["gcn"]["train"]["selected_over_oracle_geomean"] < 1.05
    assert (tmp_path / "models" / "gcn_b200.json").exists()


def test_hub_plan_partitions_the_pattern():
    """Host-side structure of the hub split (hub.py): the hub block and the
    tail partition the edges of Ã; the hub columns are the T most referenced."""
    from paper_2306_15155_b200 import hub

    a = graphs.synthetic_graph("rmat", 1500, 40000, seed=2, device="cpu")
    T = 128
    plan = hub.HubPlan(a, T)
    counts = torch.bincount(a.col_idx.long(), minlength=a.n_cols)
    assert plan.hub_cols.numel() == T and bool((plan.hub_cols[1:] > plan.hub_cols[:-1]).all())
    assert int(counts[plan.hub_cols.long()].min()) >= int(
        counts[torch.ones(a.n_cols, dtype=torch.bool).index_fill_(0, plan.hub_cols.long(), False)].max())
    assert plan.hub_edges + plan.tail.nnz == a.nnz
    assert int(plan.a_hub.float().sum()) == plan.hub_edges
    dense = a.to_dense()
    hub_dense = torch.zeros_like(dense)
    hub_dense[:, plan.hub_cols.long()] = plan.a_hub.float()
    assert torch.equal(hub_dense + plan.tail.to_dense(), dense)
    rows = plan.tail_block(None, 100, 700)
    assert torch.equal(rows.to_dense(), plan.tail.to_dense()[100:700])
    with pytest.raises(gc.ShapeError):
        hub.HubPlan(a, 100)


@pytest.mark.parametrize("abits", [True, False])
def test_stair_plan_partitions_the_pattern(abits, monkeypatch):
    """The degree-rank staircase (hub.StairPlan): blocks + tail partition the
    edges, rows shrink along the staircase, block cells are the adjacency of
    the rank-ordered rows/columns — stored as 16-bit blocks or as bitmaps
    (GC_HUB_A_BITS word layout: word (k, r) at k * rpad + r, zero padding)."""
    from paper_2306_15155_b200 import hub

    monkeypatch.setattr(hub, "HUB_ABITS", abits)
    a = graphs.synthetic_graph("rmat", 6000, 300000, seed=5, device="cpu")
    plan = hub.StairPlan(a, 0.05, n_clusters=1, first_band=256)
    assert len(plan.steps) >= 2
    rows_seq = [r for r, _, _ in plan.steps]
    assert rows_seq == sorted(rows_seq, reverse=True)
    for (_, c0, w), (_, c1, _) in zip(plan.steps, plan.steps[1:]):
        assert c1 == c0 + w and w % 64 == 0
    dense = a.to_dense()
    cover = torch.zeros_like(dense)
    edges = 0
    for s, (R, c0, W) in enumerate(plan.steps):
        blk = plan.dense_block(s)
        r_ids = plan.row_map[:R].long()
        c_ids = plan.hub_cols[c0:c0 + W].long()
        assert torch.equal(blk, dense[r_ids][:, c_ids])
        cover[r_ids.unsqueeze(1), c_ids.unsqueeze(0)] = blk
        edges += int(blk.sum())
        if abits:  # padding rows R..rpad stay zero
            rpad = -(-R // 256) * 256
            words = plan.blocks[s].view(W // 64, rpad)
            assert plan.blocks[s].dtype == torch.int64 and not bool(words[:, R:].any())
    assert torch.equal(cover + plan.tail.to_dense(), dense)
    assert plan.hub_edges + plan.tail.nnz == a.nnz
    assert plan.hub_edges == edges


# ---- .gcsr binary CSR files -----------------------------


@pytest.mark.parametrize("name", ["weighted40", "powerlaw200", "diag30"])
def test_gcsr_round_trip(golden, tmp_path, name):
    a = gcsr(golden, f"{name}/A")
    p = tmp_path / f"{name}.gcsr"
    a.save(p)
    b = gc.CsrMatrix.load(p, device=CPU)
    assert (b.n_rows, b.n_cols, b.nnz) == (a.n_rows, a.n_cols, a.nnz)
    assert torch.equal(b.row_ptr, a.row_ptr) and torch.equal(b.col_idx, a.col_idx)
    assert torch.equal(b.values, a.values)
    assert b.has_unit_values == a.has_unit_values


def test_gcsr_unit_values_not_stored(tmp_path):
    a = graphs.powerlaw_graph(300, 3, seed=1, device=CPU)
    assert a.has_unit_values
    p = tmp_path / "u.gcsr"
    a.save(p)
    size = p.stat().st_size
    rp_bytes = (a.n_rows + 1) * 4 + (-(a.n_rows + 1) * 4) % 64
    ci_bytes = a.nnz * 4 + (-a.nnz * 4) % 64
    assert size == 64 + rp_bytes + ci_bytes
    b = gc.CsrMatrix.load(p, device=CPU)
    assert b.has_unit_values and torch.equal(b.values, torch.ones(a.nnz))
    assert b.same_pattern(a)


def test_gcsr_empty_and_rectangular(tmp_path):
    for a in (gc.CsrMatrix(0, 0, [0], [], [], device=CPU),
              gc.CsrMatrix(3, 5, [0, 0, 2, 2], [1, 4], [0.5, -2.0], device=CPU)):
        p = tmp_path / "m.gcsr"
        a.save(p)
        b = gc.CsrMatrix.load(p, device=CPU)
        assert torch.equal(b.to_dense(), a.to_dense()) and b.n_cols == a.n_cols


@pytest.mark.parametrize("name", ["weighted40", "powerlaw200"])
def test_gcsr_row_range_load_equals_take_rows(golden, tmp_path, name):
    """CsrMatrix.load(rows=(lo, hi)) reads only that row block: equal to
    take_rows of the whole matrix (rebased row_ptr, global column ids)."""
    a = gcsr(golden, f"{name}/A")
    p = tmp_path / f"{name}.gcsr"
    a.save(p)
    assert np.array_equal(gc.CsrMatrix.read_row_ptr(p), a.row_ptr.numpy().astype(np.int64))
    n = a.n_rows
    for lo, hi in ((0, n), (0, 0), (3, 17), (n // 2, n), (n, n)):
        blk = gc.CsrMatrix.load(p, device=CPU, rows=(lo, hi))
        ref = a.take_rows(lo, hi)
        assert blk.n_rows == hi - lo and blk.n_cols == a.n_cols
        for x, y in zip(blk.numpy(), ref.numpy()):
            assert np.array_equal(x, y)
    with pytest.raises(gc.ShapeError):
        gc.CsrMatrix.load(p, device=CPU, rows=(5, 2))


def test_partition_from_file_matches_in_memory(golden, tmp_path, oracle):
    """The capacity path: each rank reads only its rows of Ã from the file;
    bounds, block and D^-1/2 equal the in-memory partition of the same Ã."""
    from paper_2306_15155_b200.distributed import RowPartition

    at = gc.add_self_loops(gcsr(golden, "powerlaw200/A"))
    p = tmp_path / "at.gcsr"
    at.save(p)
    d_ref = gc.inv_sqrt_degrees(at)
    for world in (1, 2, 3, 5):
        for rank in range(world):
            part, d = RowPartition.from_file(p, rank, world, device=CPU)
            ref = RowPartition.of(at, rank, world)
            assert np.array_equal(part.bounds, ref.bounds)
            assert np.array_equal(part.bounds, oracle.partition_rows(
                at.row_ptr.numpy().astype(np.int64), world))
            for x, y in zip(part.local.numpy(), ref.local.numpy()):
                assert np.array_equal(x, y)
            assert torch.equal(d, d_ref.to(torch.float32))


def test_gcsr_rejects_bad_files(tmp_path):
    a = gc.CsrMatrix(2, 2, [0, 1, 2], [1, 0], [3.0, 4.0], device=CPU)
    p = tmp_path / "m.gcsr"
    a.save(p)
    raw = p.read_bytes()
    (tmp_path / "trunc.gcsr").write_bytes(raw[:-70])
    with pytest.raises(gc.ShapeError):
        gc.CsrMatrix.load(tmp_path / "trunc.gcsr", device=CPU)
    (tmp_path / "empty.gcsr").write_bytes(b"")
    with pytest.raises(gc.ShapeError):
        gc.CsrMatrix.load(tmp_path / "empty.gcsr", device=CPU)
    (tmp_path / "foreign.gcsr").write_bytes(b"%%MatrixMarket" + raw[14:])
    with pytest.raises(gc.ShapeError):
        gc.CsrMatrix.load(tmp_path / "foreign.gcsr", device=CPU)
    bad = bytearray(raw)
    bad[64 + 4] = 7  # row_ptr[1] = 7 > nnz: invariant check on load
    (tmp_path / "bad.gcsr").write_bytes(bytes(bad))
    with pytest.raises(gc.ShapeError):
        gc.CsrMatrix.load(tmp_path / "bad.gcsr", device=CPU)
    assert gc.CsrMatrix.load(tmp_path / "bad.gcsr", device=CPU, validate=False).nnz == 2
