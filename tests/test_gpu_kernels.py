"""Parity of every C-ABI kernel with the CPU oracle (float64 restatement of the
reference), on seeded inputs.  Tolerances (normwise rel_err, the reference's
tests/helpers.py:68-72 metric): 1e-5 for fp32 sparse kernels, 1e-4 for the
exact-fp32 GEMM, 1e-2 for the TF32 tensor-core GEMM.  Integer/pattern outputs
are compared bit-exactly."""

from __future__ import annotations

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

import paper_2306_15155_b200 as gc  # noqa: E402
from paper_2306_15155_b200 import graphs, sparse  # noqa: E402

DEV = "cuda"
SP_TOL = 1e-5
# the hybrid aggregation in the default TF32 mode rounds the dense part's
# operand to one fp16 term (11 significant bits, TF32's input rounding): the
# layer's stated 1e-2 class; measured ~1e-4 on these graphs
HUB_F16_TOL = 1e-3


def hub_tol() -> float:
    from paper_2306_15155_b200 import _native as nat
    from paper_2306_15155_b200 import hub
    return HUB_F16_TOL if hub.term_format() == nat.GC_HUB_F16 else SP_TOL


def to_oracle(oracle, a: gc.CsrMatrix):
    rp, ci, v = a.numpy()
    return oracle.Csr(a.n_rows, a.n_cols, rp, ci, v)


def f32(x):
    return np.asarray(x, dtype=np.float32)


def rand_csr(rng, n_rows, n_cols, density, unit=False, empty_rows=()):
    dense = (rng.random((n_rows, n_cols)) < density).astype(np.float64)
    if not unit:
        dense *= f32(rng.uniform(0.5, 2.0, size=dense.shape))
    for r in empty_rows:
        dense[r] = 0
    return gc.CsrMatrix.from_dense(dense, device=DEV)


@pytest.fixture(scope="module")
def plgraph():
    a = graphs.powerlaw_graph(1500, 6, seed=3, device=DEV)
    return gc.add_self_loops(a)


KS = [1, 3, 4, 7, 16, 32, 33, 64, 100, 128, 256, 300, 512]


@pytest.mark.parametrize("K", KS)
@pytest.mark.parametrize("algo", ["row", "split"])
def test_spmm_weighted_unweighted(oracle, plgraph, K, algo, monkeypatch):
    if algo == "split":
        monkeypatch.setattr(sparse, "SPLIT_CHUNK", 16)  # force many split rows
    rng = np.random.default_rng(K)
    a = plgraph.with_values(torch.from_numpy(f32(rng.uniform(0.5, 2, plgraph.nnz))).to(DEV))
    oa = to_oracle(oracle, a)
    b = f32(rng.standard_normal((a.n_cols, K)))
    bt = torch.from_numpy(b).to(DEV)
    out = gc.spmm(a, bt, algo=algo).cpu().numpy()
    assert oracle.rel_err(out, oracle.spmm(oa, b)) < SP_TOL
    outu = gc.spmm_unweighted(a, bt, algo=algo).cpu().numpy()
    assert oracle.rel_err(outu, oracle.spmm_unweighted(oa, b)) < SP_TOL
    # fused dynamic normalisation: d_i * sum_j w_ij d_j b_j, then ReLU
    d = torch.from_numpy(f32(rng.uniform(0.1, 1.0, a.n_rows))).to(DEV)
    outd = gc.spmm(a, bt, d_row=d, d_col=d, relu=True, algo=algo).cpu().numpy()
    dn = d.cpu().numpy().astype(np.float64)
    ref = np.maximum(oracle.scale_rows(dn, oracle.spmm(oa, oracle.scale_rows(dn, b))), 0)
    assert oracle.rel_err(outd, ref) < SP_TOL


@pytest.mark.parametrize("K", [4, 12, 32, 64, 256, 1024])
def test_pack_rows_f16_semantics(K):
    """gc_pack_rows_f16: with y = fp32(d * x), xh = fp16_rn(y * 2^-e) with
    max|y_j| * 2^-e in [2^14, 2^15) and sigma = 2^e (a power of two, d folded
    into the values); rows of zeros -> sigma = 1."""
    rng = np.random.default_rng(K)
    x = f32(rng.uniform(-1, 1, (300, K)) * 2.0 ** rng.integers(-30, 30, (300, 1)))
    x[7] = 0
    d = f32(rng.uniform(0.1, 1, 300))
    hr = sparse.pack_rows_f16(torch.from_numpy(x).to(DEV), torch.from_numpy(d).to(DEV))
    y = f32(x * d[:, None])
    mx = np.abs(y).max(1)
    e = np.where(mx > 0, np.frexp(mx)[1] - 1 - 14, 0)
    ref_h = (y * np.ldexp(1.0, -e)[:, None]).astype(np.float16)
    assert np.array_equal(hr.xh[:, :K].cpu().numpy(), ref_h)
    assert np.array_equal(hr.sigma.cpu().numpy(), f32(np.ldexp(1.0, e)))
    # dequantised rows carry 11 significant bits
    deq = hr.xh[:, :K].float().cpu().numpy() * hr.sigma.cpu().numpy()[:, None]
    rel = np.abs(deq - x * d[:, None]).max(1) / np.maximum(np.abs(x * d[:, None]).max(1), 1e-30)
    assert rel.max() <= 2.0 ** -11


@pytest.mark.parametrize("K", [8, 64, 256, 1024])
@pytest.mark.parametrize("n_proj", [2, 8])
def test_pack_rows_f16_projections(K, n_proj):
    """The node scores fused into the pack (gc_pack_rows_f16_proj): the same
    fp16 rows as the plain pack, projections equal to X @ P^T (float64
    reference, 1e-6), and bit-identical to node_proj_kernel when the lane
    layout matches (K a multiple of 128)."""
    from paper_2306_15155_b200.gat import GatLayerSpec, _projections
    rng = np.random.default_rng(K + n_proj)
    x = torch.from_numpy(f32(rng.standard_normal((500, K)))).to(DEV)
    P = torch.from_numpy(f32(rng.uniform(-0.5, 0.5, (n_proj, K)))).to(DEV)
    hr, pr = sparse.pack_rows_f16(x, proj=P)
    plain = sparse.pack_rows_f16(x)
    assert torch.equal(hr.xh.view(torch.int16), plain.xh.view(torch.int16))
    assert torch.equal(hr.sigma, plain.sigma)
    ref = (P.double() @ x.double().T).cpu().numpy()
    assert np.abs(pr.cpu().numpy() - ref).max() <= 1e-6 * max(1.0, np.abs(ref).max())
    if K % 128 == 0 and n_proj == 2:
        spec = GatLayerSpec(K, K, np.zeros((K, K)), P[0].cpu().numpy(), P[1].cpu().numpy())
        s, t = _projections(x, spec, P[0].contiguous(), P[1].contiguous(), K, K)
        assert torch.equal(s[0], pr[0]) and torch.equal(t[0], pr[1])


@pytest.mark.parametrize("K", [8, 32, 128, 200, 256, 512])
@pytest.mark.parametrize("algo", ["row", "split"])
@pytest.mark.parametrize("weighted", [False, True])
@pytest.mark.parametrize("scales", ["d", "pow2", "mixed"])
def test_spmm_fp16_operand_bit_exact_to_dequantised(plgraph, K, algo, weighted, scales,
                                                    monkeypatch):
    """GC_SPMM_B_F16: the fp16-row gather computes exactly what the fp32 kernel
    computes on the dequantised rows with d_col = sigma (same order), and
    plain ReLU / accumulate epilogues.  scales "pow2": sigma_j pure powers of
    two, so unit-valued batches take the fp16-weight FMA (fma.rn.f32.f16);
    "mixed": some rows scaled out of fp16 range (sigma < 2^-24), so batches
    switch between the two FMA forms within a row."""
    if algo == "split":
        monkeypatch.setattr(sparse, "SPLIT_CHUNK", 16)
    rng = np.random.default_rng(K + 5)
    if weighted and scales != "d":
        vals = np.where(rng.random(plgraph.nnz) < 0.9, 1.0, rng.uniform(0.5, 2, plgraph.nnz))
    else:
        vals = rng.uniform(0.5, 2, plgraph.nnz)
    a = plgraph.with_values(torch.from_numpy(f32(vals)).to(DEV))
    xn = rng.standard_normal((a.n_cols, K))
    if scales == "mixed":
        xn[rng.random(a.n_cols) < 0.3] *= 1e-12
    x = torch.from_numpy(f32(xn)).to(DEV)
    d = torch.from_numpy(f32(rng.uniform(0.1, 1, a.n_rows))).to(DEV)
    hr = sparse.pack_rows_f16(x, d if scales == "d" else None)
    deq = hr.xh[:, :K].float().contiguous()
    f = gc.spmm if weighted else gc.spmm_unweighted
    got = f(a, hr, d_row=d, relu=True, algo=algo)
    ref = f(a, deq, d_row=d, d_col=hr.sigma, relu=True, algo=algo)
    assert torch.equal(got, ref)
    acc = torch.ones_like(got)
    f(a, hr, d_row=d, out=acc, accumulate=True, algo=algo)
    ref2 = torch.ones_like(got)
    f(a, deq, d_row=d, d_col=hr.sigma, out=ref2, accumulate=True, algo=algo)
    assert torch.equal(acc, ref2)


def test_spmm_unweighted_bit_identical_to_unit_weights(plgraph):
    rng = np.random.default_rng(1)
    b = torch.from_numpy(f32(rng.standard_normal((plgraph.n_cols, 64)))).to(DEV)
    ones = plgraph.with_values(torch.ones(plgraph.nnz, device=DEV))
    assert torch.equal(gc.spmm_unweighted(plgraph, b), gc.spmm(ones, b))


def test_spmm_unweighted_never_reads_values(plgraph):
    rng = np.random.default_rng(2)
    b = torch.from_numpy(f32(rng.standard_normal((plgraph.n_cols, 32)))).to(DEV)
    expected = gc.spmm(plgraph.with_values(torch.ones(plgraph.nnz, device=DEV)), b)
    poisoned = plgraph.with_values(torch.full((plgraph.nnz,), float("nan"), device=DEV))
    assert torch.equal(gc.spmm_unweighted(poisoned, b), expected)


def test_spmm_known_answers():
    a = gc.CsrMatrix(2, 2, np.array([0, 1, 1]), np.array([1]), np.array([2.0]), device=DEV)
    out = gc.spmm(a, np.array([[1.0, 1.0], [3.0, 4.0]]))
    assert isinstance(out, np.ndarray) and np.array_equal(out, [[6.0, 8.0], [0.0, 0.0]])
    a = gc.CsrMatrix(1, 3, np.array([0, 2]), np.array([1, 2]), np.ones(2), device=DEV)
    assert np.array_equal(gc.spmm_unweighted(a, np.array([[9.0, 9], [1, 2], [3, 4]])), [[4.0, 6.0]])
    ident = gc.CsrMatrix(3, 3, np.arange(4), np.arange(3), np.ones(3), device=DEV)
    b = np.random.default_rng(0).random((3, 2)).astype(np.float32)
    assert np.array_equal(gc.spmm(ident, b), b)


def test_spmm_empty_and_zero_rows(oracle):
    rng = np.random.default_rng(3)
    a = rand_csr(rng, 40, 30, 0.2, empty_rows=(0, 7, 39))
    b = f32(rng.standard_normal((30, 12)))
    out = gc.spmm(a, b)
    assert np.array_equal(out[[0, 7, 39]], np.zeros((3, 12), np.float32))
    assert oracle.rel_err(out, oracle.spmm(to_oracle(oracle, a), b)) < SP_TOL
    z = gc.CsrMatrix(3, 3, np.zeros(4, np.int64), np.array([], np.int64), np.array([]), device=DEV)
    assert np.array_equal(gc.spmm(z, np.ones((3, 2))), np.zeros((3, 2)))
    e = gc.CsrMatrix(0, 5, np.zeros(1, np.int64), np.array([], np.int64), np.array([]), device=DEV)
    assert gc.spmm(e, np.ones((5, 4))).shape == (0, 4)


def test_spmm_shape_errors():
    a = gc.CsrMatrix(3, 3, np.arange(4), np.arange(3), np.ones(3), device=DEV)
    with pytest.raises(gc.ShapeError):
        gc.spmm(a, np.ones((4, 2)))
    with pytest.raises(RuntimeError):  # no CPU fallback
        gc.spmm(a.to("cpu"), torch.ones(3, 2))


def test_spmm_strided_output_and_accumulate(oracle, plgraph):
    rng = np.random.default_rng(4)
    b = torch.from_numpy(f32(rng.standard_normal((plgraph.n_cols, 64)))).to(DEV)
    big = torch.zeros(plgraph.n_rows, 128, device=DEV)
    gc.spmm(plgraph, b, out=big[:, 64:])
    ref = gc.spmm(plgraph, b)
    assert torch.equal(big[:, 64:], ref) and not big[:, :64].any()
    gc.spmm(plgraph, b, out=big[:, 64:], accumulate=True)
    assert torch.allclose(big[:, 64:], 2 * ref, rtol=1e-6, atol=1e-6)


# ---------------------------------------------------------------------------
# SDDMM
# ---------------------------------------------------------------------------


@pytest.mark.parametrize("k", [1, 3, 16, 65])
def test_sddmm(oracle, k):
    rng = np.random.default_rng(k)
    a = rand_csr(rng, 50, 37, 0.3)
    b, c = f32(rng.standard_normal((50, k))), f32(rng.standard_normal((37, k)))
    out = gc.sddmm(a, b, c)
    assert out.same_pattern(a)
    ref = oracle.sddmm(to_oracle(oracle, a), b, c).values
    assert oracle.rel_err(out.values.cpu().numpy(), ref) < SP_TOL


def test_sddmm_identity_and_empty():
    rng = np.random.default_rng(5)
    a = rand_csr(rng, 6, 6, 0.5)
    ones = np.ones((6, 1))
    assert torch.equal(gc.sddmm(a, ones, ones).values, a.values)
    z = gc.CsrMatrix(3, 3, np.zeros(4, np.int64), np.array([], np.int64), np.array([]), device=DEV)
    assert gc.sddmm(z, np.ones((3, 2)), np.ones((3, 2))).nnz == 0
    with pytest.raises(gc.ShapeError):
        gc.sddmm(a, np.ones((5, 2)), np.ones((6, 2)))


def test_normalized_adjacency_matches_golden(golden):
    for gid in ("path3", "grid4x5", "powerlaw200", "weighted40", "diag30"):
        rp, ci, v = (golden[f"{gid}/A/{k}"] for k in ("row_ptr", "col_idx", "values"))
        n = int(golden[f"{gid}/A/shape"][0])
        a = gc.CsrMatrix(n, n, rp, ci, v, device=DEV)
        g = gc.NormalizedGraph.from_adjacency(a, precompute=True)
        assert np.array_equal(g.a_tilde.row_ptr.cpu().numpy(), golden[f"{gid}/At/row_ptr"])
        assert np.array_equal(g.a_tilde.col_idx.cpu().numpy(), golden[f"{gid}/At/col_idx"])
        np.testing.assert_allclose(g.n_tilde.values.cpu().numpy(), golden[f"{gid}/Nt"], rtol=2e-7)


# ---------------------------------------------------------------------------
# GEMM
# ---------------------------------------------------------------------------

GEMM_SHAPES = [(1, 1, 1), (5, 3, 7), (130, 33, 16), (300, 32, 32), (1000, 64, 200),
               (513, 256, 256), (700, 100, 300), (257, 1433, 16), (2000, 256, 1024),
               (129, 7, 33), (4097, 512, 128)]


@pytest.mark.parametrize("M,K,N", GEMM_SHAPES)
@pytest.mark.parametrize("prec,tol", [("fp32", 2e-5), ("simt", 1e-5), ("tf32", 1e-2)])
def test_gemm(oracle, M, K, N, prec, tol):
    rng = np.random.default_rng(M + K + N)
    a, w = f32(rng.uniform(-0.5, 0.5, (M, K))), f32(rng.uniform(-0.5, 0.5, (K, N)))
    out = gc.gemm(torch.from_numpy(a).to(DEV), torch.from_numpy(w).to(DEV), precision=prec)
    assert oracle.rel_err(out.cpu().numpy(), oracle.gemm(a, w)) <= tol
    rs = torch.from_numpy(f32(rng.uniform(0.1, 1, M))).to(DEV)
    out = gc.gemm(torch.from_numpy(a).to(DEV), torch.from_numpy(w).to(DEV), precision=prec,
                  row_scale=rs, relu=True)
    ref = np.maximum(oracle.scale_rows(rs.cpu().numpy(), oracle.gemm(a, w)), 0)
    assert oracle.rel_err(out.cpu().numpy(), ref) <= tol


def test_gemm_tf32_uses_tensor_cores_accuracy_profile(oracle):
    # TF32 drops 13 mantissa bits: visibly less exact than fp32, within 1e-2.
    rng = np.random.default_rng(9)
    a, w = f32(rng.uniform(-0.5, 0.5, (1024, 512))), f32(rng.uniform(-0.5, 0.5, (512, 256)))
    ref = oracle.gemm(a, w)
    e32 = oracle.rel_err(gc.gemm(a, w, precision="fp32"), ref)
    etf = oracle.rel_err(gc.gemm(a, w, precision="tf32"), ref)
    assert e32 < 1e-5 < etf < 1e-2


def test_gemm_3xtf32_wide_dynamic_range(oracle):
    """3xTF32 (the fp32 class): operands spanning 2^-20 .. 2^20 keep fp32-class
    normwise error — the hi/lo split carries 22+ significant bits per operand."""
    rng = np.random.default_rng(17)
    a = f32(rng.uniform(-1, 1, (777, 96)) * 2.0 ** rng.integers(-20, 20, (777, 96)))
    w = f32(rng.uniform(-1, 1, (96, 80)) * 2.0 ** rng.integers(-4, 4, (96, 80)))
    ref = oracle.gemm(a, w)
    out = gc.gemm(torch.from_numpy(a).to(DEV), torch.from_numpy(w).to(DEV), precision="fp32")
    err = float(np.abs(out.cpu().numpy() - ref).max() / np.abs(ref).max())
    assert err < 4e-6, err
    tf = gc.gemm(torch.from_numpy(a).to(DEV), torch.from_numpy(w).to(DEV), precision="tf32")
    assert float(np.abs(tf.cpu().numpy() - ref).max() / np.abs(ref).max()) > 10 * err


@pytest.mark.parametrize("M,K,N", [(1, 8, 8), (300, 64, 40), (1000, 256, 256), (4097, 128, 16),
                                   (2000, 1433, 16), (777, 96, 200)])
@pytest.mark.parametrize("scaled", [False, True])
def test_gemm_f16rows_epilogue_equals_pack(M, K, N, scaled):
    """gc_gemm_f16rows_f32 (the TF32 GEMM emitting the fp16 gather operand
    from TMEM) is bit-identical to gc_pack_rows_f16 of the TF32 GEMM's fp32
    output (same row max, same power-of-two scale, same two roundings)."""
    rng = np.random.default_rng(M + K + N)
    a = torch.from_numpy(f32(rng.uniform(-0.5, 0.5, (M, K)) * 2.0 ** rng.integers(-6, 6, (M, 1)))).to(DEV)
    w = torch.from_numpy(f32(rng.uniform(-0.5, 0.5, (K, N)))).to(DEV)
    if K % 4:  # TMA needs a 16-byte row pitch (gemm pads; the fused path does not)
        ap = torch.zeros(M, (K + 3) // 4 * 4, device=DEV)
        ap[:, :K] = a
        a = ap[:, :K]
    rs = torch.from_numpy(f32(rng.uniform(0.1, 1.0, M))).to(DEV) if scaled else None
    hr = sparse.gemm_f16rows(a, w, row_scale=rs)
    assert hr is not None and hr.K == N
    ref = sparse.pack_rows_f16(gc.gemm(a, w, row_scale=rs, precision="tf32"))
    assert torch.equal(hr.xh.view(torch.int16), ref.xh.view(torch.int16))
    assert torch.equal(hr.sigma, ref.sigma)


def test_gemm_known_and_errors():
    out = gc.gemm(np.array([[1.0, 2.0], [3.0, 4.0]]), np.array([[5.0], [6.0]]), precision="fp32")
    assert np.array_equal(out, [[17.0], [39.0]])
    with pytest.raises(gc.ShapeError):
        gc.gemm(np.ones((2, 3)), np.ones((2, 3)))


def test_scale_rows(oracle):
    rng = np.random.default_rng(6)
    d, b = f32(rng.uniform(0.5, 2, 10)), f32(rng.standard_normal((10, 6)))
    assert np.array_equal(gc.scale_rows(d, b), d[:, None] * b)
    assert np.array_equal(gc.scale_rows(np.array([2.0, 3.0]), np.ones((2, 2))), [[2, 2], [3, 3]])
    with pytest.raises(gc.ShapeError):
        gc.scale_rows(np.ones(3), np.ones((4, 2)))


# ---------------------------------------------------------------------------
# attention
# ---------------------------------------------------------------------------


@pytest.mark.parametrize("k2", [1, 5, 16, 64, 130])
@pytest.mark.parametrize("form", ["reassoc", "sddmm"])
def test_attention_matches_oracle(oracle, plgraph, k2, form):
    rng = np.random.default_rng(k2)
    hw = f32(rng.standard_normal((plgraph.n_rows, k2)))
    a_s, a_d = f32(rng.uniform(-0.5, 0.5, k2)), f32(rng.uniform(-0.5, 0.5, k2))
    spec = gc.GatLayerSpec(3, k2, np.zeros((3, k2)), a_s, a_d, leaky_slope=0.2, attention=form)
    att = gc.atten_calc(plgraph, torch.from_numpy(hw).to(DEV), spec)
    ref = oracle.atten_calc(to_oracle(oracle, plgraph), hw, a_s, a_d, 0.2).values
    assert oracle.rel_err(att.alpha.values.cpu().numpy(), ref) < 1e-5
    sums = att.row_sums().cpu().numpy()
    np.testing.assert_allclose(sums, 1.0, atol=1e-5)


@pytest.fixture(scope="module")
def hubgraph():
    """Power-law graph plus two hub rows far above the softmax lane-group
    threshold (and an empty-row-free Ã), so the CTA-per-heavy-row path runs."""
    n = 3000
    rng = np.random.default_rng(5)
    src = [0] * (n - 1) + [7] * 1500 + list(rng.integers(0, n, 6000))
    dst = list(range(1, n)) + list(rng.choice(np.arange(8, n), 1500, replace=False)) + \
        list(rng.integers(0, n, 6000))
    rows, cols = np.array(src + dst), np.array(dst + src)
    keep = rows != cols
    a = gc.CsrMatrix.from_coo(n, n, rows[keep], cols[keep], np.ones(int(keep.sum())), device=DEV)
    a = gc.CsrMatrix(n, n, a.row_ptr, a.col_idx, torch.ones_like(a.values), device=DEV)
    return gc.add_self_loops(a)


@pytest.mark.parametrize("heads", [1, 3])
@pytest.mark.parametrize("form", ["reassoc", "sddmm"])
@pytest.mark.parametrize("k2", [8, 64])
def test_attention_heavy_rows(oracle, hubgraph, heads, form, k2):
    assert hubgraph.softmax_heavy_rows().numel() >= 2
    rng = np.random.default_rng(heads * 100 + k2)
    hw = f32(rng.standard_normal((hubgraph.n_rows, heads * k2)))
    a_s, a_d = f32(rng.uniform(-0.5, 0.5, heads * k2)), f32(rng.uniform(-0.5, 0.5, heads * k2))
    spec = gc.GatLayerSpec(3, k2, np.zeros((3, heads * k2)), a_s, a_d, heads=heads, attention=form)
    att = gc.atten_calc(hubgraph, torch.from_numpy(hw).to(DEV), spec)
    oa = to_oracle(oracle, hubgraph)
    for h in range(heads):
        ref = oracle.atten_calc(oa, hw[:, h * k2:(h + 1) * k2], a_s[h * k2:(h + 1) * k2],
                                a_d[h * k2:(h + 1) * k2], 0.2).values
        assert oracle.rel_err(att.head(h).values.cpu().numpy(), ref) < 1e-5
    np.testing.assert_allclose(att.row_sums().cpu().numpy(), 1.0, atol=1e-5)
    # the heavy-row CTAs and the lane groups agree with the unsplit launch
    again = gc.atten_calc(hubgraph, torch.from_numpy(hw).to(DEV), spec)
    assert torch.equal(att.alpha.values, again.alpha.values)


def test_normalized_adjacency_heavy_rows(oracle, hubgraph):
    g = gc.NormalizedGraph.from_adjacency(hubgraph, precompute=True)
    og = oracle.GcnGraph.from_adjacency(to_oracle(oracle, hubgraph))
    np.testing.assert_allclose(g.n_tilde.values.cpu().numpy(), og.n_tilde.values, rtol=2e-7)


def test_attention_singleton_and_ties():
    a = gc.CsrMatrix(1, 1, np.array([0, 1]), np.array([0]), np.ones(1), device=DEV)
    spec = gc.GatLayerSpec(1, 1, np.ones((1, 1)), np.ones(1), np.ones(1))
    assert gc.atten_calc(a, np.ones((1, 1)), spec).alpha.values.item() == 1.0
    a2 = gc.CsrMatrix(2, 2, np.array([0, 2, 2]), np.array([0, 1]), np.ones(2), device=DEV)
    spec = gc.GatLayerSpec(1, 1, np.ones((1, 1)), np.zeros(1), np.zeros(1))
    att = gc.atten_calc(a2, np.ones((2, 1)), spec)
    assert np.allclose(att.alpha.values.cpu().numpy(), [0.5, 0.5])


# ---------------------------------------------------------------------------
# layers against the reference's own golden outputs
# ---------------------------------------------------------------------------

GRAPHS = ["path3", "star5", "grid4x5", "powerlaw200", "random120", "weighted40", "diag30"]
SIZES = [(6, 3), (3, 6), (5, 5)]


def golden_graph(golden, gid):
    n = int(golden[f"{gid}/A/shape"][0])
    return gc.CsrMatrix(n, n, golden[f"{gid}/A/row_ptr"], golden[f"{gid}/A/col_idx"],
                        golden[f"{gid}/A/values"], device=DEV)


@pytest.mark.parametrize("prec,tol", [("fp32", 1e-4), ("tf32", 1e-2)])
@pytest.mark.parametrize("gid", GRAPHS)
def test_gcn_layers_vs_reference_golden(golden, gid, prec, tol):
    gc.set_gemm_precision(prec)
    try:
        g = gc.NormalizedGraph.from_adjacency(golden_graph(golden, gid), precompute=True)
        for k1, k2 in SIZES:
            key = f"{gid}/{k1}x{k2}"
            h, w = golden[f"{key}/h"], golden[f"{key}/w"]
            for comp in ("precompute", "dynamic"):
                out = gc.gcn_layer(g, h, gc.GcnLayerSpec(k1, k2, w, composition=comp))
                exp = golden[f"{key}/gcn/{comp}/heuristic"]
                assert out.shape == exp.shape and _rel(out, exp) <= tol, (key, comp)
                for order in ("aggregate_first", "update_first"):
                    spec = gc.GcnLayerSpec(k1, k2, w, composition=comp, order=order)
                    out = gc.gcn_layer(g, torch.from_numpy(f32(h)).to(DEV), spec).cpu().numpy()
                    assert _rel(out, golden[f"{key}/gcn/{comp}/{order}"]) <= tol, (key, comp, order)
    finally:
        gc.set_gemm_precision("tf32")


@pytest.mark.parametrize("prec,tol", [("fp32", 1e-4), ("tf32", 1e-2)])
@pytest.mark.parametrize("gid", GRAPHS)
def test_gat_layers_vs_reference_golden(golden, gid, prec, tol):
    gc.set_gemm_precision(prec)
    try:
        at = gc.add_self_loops(golden_graph(golden, gid))
        for k1, k2 in SIZES:
            key = f"{gid}/{k1}x{k2}"
            h, w = golden[f"{key}/h"], golden[f"{key}/w"]
            a_s, a_d = golden[f"{key}/attn_src"], golden[f"{key}/attn_dst"]
            for slope in (0.2, 0.1):
                for comp in ("reuse", "recompute"):
                    for act in ("relu", "none"):
                        for form in ("reassoc", "sddmm"):
                            spec = gc.GatLayerSpec(k1, k2, w, a_s, a_d, leaky_slope=slope,
                                                   composition=comp, activation=act, attention=form)
                            out = gc.gat_layer(at, h, spec)
                            exp = golden[f"{key}/gat/s{slope}/{comp}/{act}"]
                            assert _rel(out, exp) <= tol, (key, slope, comp, act, form)
    finally:
        gc.set_gemm_precision("tf32")


def _rel(a, e):
    a = np.asarray(a, dtype=np.float64)
    e = np.asarray(e, dtype=np.float64)
    return float(np.abs(a - e).max()) / max(1.0, float(np.abs(e).max()))


@pytest.mark.parametrize("heads", [2, 4])
@pytest.mark.parametrize("comp", ["reuse", "recompute"])
@pytest.mark.parametrize("form", ["reassoc", "sddmm"])
def test_multihead_gat(oracle, plgraph, heads, comp, form):
    rng = np.random.default_rng(heads)
    k1, k2 = 24, 16
    h = f32(rng.uniform(-0.5, 0.5, (plgraph.n_rows, k1)))
    w = f32(rng.uniform(-0.5, 0.5, (k1, heads * k2)))
    a_s, a_d = f32(rng.uniform(-0.5, 0.5, heads * k2)), f32(rng.uniform(-0.5, 0.5, heads * k2))
    spec = gc.GatLayerSpec(k1, k2, w, a_s, a_d, composition=comp, heads=heads, attention=form)
    gc.set_gemm_precision("fp32")
    try:
        out = gc.gat_layer(plgraph, h, spec)
    finally:
        gc.set_gemm_precision("tf32")
    ref = oracle.gat_layer_multihead(to_oracle(oracle, plgraph), h, w, a_s, a_d, heads,
                                     composition=comp)
    assert oracle.rel_err(out, ref) <= 1e-4


def test_layers_are_deterministic(plgraph):
    rng = np.random.default_rng(11)
    h = torch.from_numpy(f32(rng.uniform(-0.5, 0.5, (plgraph.n_rows, 64)))).to(DEV)
    w = f32(rng.uniform(-0.5, 0.5, (64, 64)))
    g = gc.NormalizedGraph(plgraph, gc.inv_sqrt_degrees(plgraph)).with_precomputed()
    for comp in ("precompute", "dynamic"):
        spec = gc.GcnLayerSpec(64, 64, w, composition=comp)
        assert torch.equal(gc.gcn_layer(g, h, spec), gc.gcn_layer(g, h, spec))
    spec = gc.GatLayerSpec(64, 64, w, np.ones(64) * 0.1, np.ones(64) * -0.1)
    assert torch.equal(gc.gat_layer(plgraph, h, spec), gc.gat_layer(plgraph, h, spec))


def test_spmm_fn_hook_is_used(golden):
    g = gc.NormalizedGraph.from_adjacency(golden_graph(golden, "grid4x5"), precompute=True)
    calls = []

    @gc.device_hook
    def my_spmm(a, b):
        calls.append(a.nnz)
        return gc.spmm(a, b)

    key = "grid4x5/5x5"
    h, w = golden[f"{key}/h"], golden[f"{key}/w"]
    for comp in ("precompute", "dynamic"):
        out = gc.gcn_layer(g, h, gc.GcnLayerSpec(5, 5, w, composition=comp), spmm_fn=my_spmm)
        assert _rel(out, golden[f"{key}/gcn/{comp}/heuristic"]) <= 1e-2
    assert len(calls) == 2


def test_host_spmm_fn_hook_gets_reference_operands(golden, oracle):
    """An unmarked hook gets the reference's host contract (a CsrMatrix-like
    view with int64/float64 numpy arrays, a float64 ndarray) — e.g. the
    reference's own numpy/numba spmm, here its oracle restatement."""
    g = gc.NormalizedGraph.from_adjacency(golden_graph(golden, "grid4x5"), precompute=True)
    seen = []

    def host_spmm(a, b):
        assert isinstance(b, np.ndarray) and b.dtype == np.float64
        assert a.row_ptr.dtype == np.int64 and a.values.dtype == np.float64
        seen.append(a.nnz)
        return oracle.spmm(oracle.Csr(a.n_rows, a.n_cols, a.row_ptr, a.col_idx, a.values), b)

    key = "grid4x5/5x5"
    h, w = golden[f"{key}/h"], golden[f"{key}/w"]
    for comp in ("precompute", "dynamic"):
        out = gc.gcn_layer(g, h, gc.GcnLayerSpec(5, 5, w, composition=comp), spmm_fn=host_spmm)
        assert _rel(out, golden[f"{key}/gcn/{comp}/heuristic"]) <= 1e-2
    rng = np.random.default_rng(3)
    a_s, a_d = rng.uniform(-0.5, 0.5, 5), rng.uniform(-0.5, 0.5, 5)
    for comp in ("reuse", "recompute"):
        spec = gc.GatLayerSpec(5, 5, w, a_s, a_d, composition=comp)
        ref = gc.gat_layer(g.a_tilde, torch.as_tensor(h, dtype=torch.float32, device=DEV), spec)
        out = gc.gat_layer(g.a_tilde, torch.as_tensor(h, dtype=torch.float32, device=DEV), spec,
                           spmm_fn=host_spmm)
        assert _rel(out.cpu().numpy(), ref.cpu().numpy()) <= 1e-5
    assert len(seen) == 4


@pytest.mark.parametrize("K", [1, 7, 32, 64, 256])
@pytest.mark.parametrize("algo", ["row", "split"])
def test_fused_gat_aggregate_matches_oracle(oracle, plgraph, K, algo, monkeypatch):
    """gc_gat_aggregate_f32 == edge softmax (gat.py:72-95) then spmm(alpha, B)."""
    if algo == "split":
        monkeypatch.setattr(sparse, "SPLIT_CHUNK", 16)
    rng = np.random.default_rng(K + 100)
    n = plgraph.n_rows
    s = f32(rng.standard_normal(n) * 3)
    t = f32(rng.standard_normal(n) * 3)
    b = f32(rng.standard_normal((n, K)))
    dev = lambda x: torch.from_numpy(x).to(DEV)  # noqa: E731
    for relu, slope in ((False, 0.2), (True, 0.05)):
        out = sparse.gat_aggregate(plgraph, dev(s), dev(t), slope, dev(b), relu=relu,
                                   algo=algo).cpu().numpy()
        oa = to_oracle(oracle, plgraph)
        alpha = oracle.edge_softmax(oa, s, t, slope)
        ref = oracle.spmm(oa.with_values(alpha), b)
        if relu:
            ref = np.maximum(ref, 0)
        assert oracle.rel_err(out, ref) < 2e-5, (K, algo, relu)


@pytest.mark.parametrize("K", [8, 32, 256, 512])
@pytest.mark.parametrize("algo", ["row", "split"])
def test_fused_gat_fp16_rows_match_oracle_on_dequantised(oracle, plgraph, K, algo, monkeypatch):
    """GC_SPMM_B_F16 in both GAT modes: the reassociated-score aggregation
    and the SDDMM-score aggregation over fp16 rows equal the oracle run on the
    dequantised rows sigma_j * xh_j (the score's source rows stay fp32)."""
    if algo == "split":
        monkeypatch.setattr(sparse, "SPLIT_CHUNK", 16)
    rng = np.random.default_rng(K + 300)
    n = plgraph.n_rows
    dev = lambda x: torch.from_numpy(x).to(DEV)  # noqa: E731
    hw = f32(rng.uniform(-1, 1, (n, K)) * 2.0 ** rng.integers(-3, 3, (n, 1)))
    hr = sparse.pack_rows_f16(dev(hw))
    deq = hr.xh[:, :K].double().cpu().numpy() * hr.sigma.double().cpu().numpy()[:, None]
    oa = to_oracle(oracle, plgraph)
    s, t = f32(rng.standard_normal(n) * 3), f32(rng.standard_normal(n) * 3)
    out = sparse.gat_aggregate(plgraph, dev(s), dev(t), 0.2, hr, relu=True, algo=algo)
    ref = np.maximum(oracle.spmm(oa.with_values(oracle.edge_softmax(oa, s, t, 0.2)), deq), 0)
    assert oracle.rel_err(out.cpu().numpy(), ref) < 2e-5
    a_s, a_d = f32(rng.uniform(-0.5, 0.5, K)), f32(rng.uniform(-0.5, 0.5, K))
    out = sparse.gat_sddmm_aggregate(plgraph, dev(a_s), dev(a_d), 0.2, hr, b_self=dev(hw),
                                     algo=algo)
    assert out is not None
    ss = hw.astype(np.float64) @ a_s.astype(np.float64)
    tt = deq @ a_d.astype(np.float64)
    ref = oracle.spmm(oa.with_values(oracle.edge_softmax(oa, ss, tt, 0.2)), deq)
    assert oracle.rel_err(out.cpu().numpy(), ref) < 2e-5
    with pytest.raises(gc.ShapeError):
        sparse.gat_sddmm_aggregate(plgraph, dev(a_s), dev(a_d), 0.2, hr)


def test_fused_gat_aggregate_empty_rows(oracle):
    rng = np.random.default_rng(7)
    a = rand_csr(rng, 60, 60, 0.1, unit=True, empty_rows=(0, 13, 59))
    s, t = f32(rng.standard_normal(60)), f32(rng.standard_normal(60))
    b = f32(rng.standard_normal((60, 8)))
    out = sparse.gat_aggregate(a, torch.from_numpy(s).to(DEV), torch.from_numpy(t).to(DEV), 0.2,
                               torch.from_numpy(b).to(DEV)).cpu().numpy()
    assert np.all(out[[0, 13, 59]] == 0) and np.isfinite(out).all()
    oa = to_oracle(oracle, a)
    ref = oracle.spmm(oa.with_values(oracle.edge_softmax(oa, s, t, 0.2)), b)
    assert oracle.rel_err(out, ref) < 2e-5


@pytest.mark.parametrize("comp", ["precompute", "dynamic"])
@pytest.mark.parametrize("order", ["aggregate_first", "update_first"])
def test_host_pipelined_layer_matches_device_path(plgraph, comp, order):
    """Pinned host H in -> pinned host out (row-blocked, D2H overlapped) must
    equal the device-resident path."""
    rng = np.random.default_rng(21)
    g = gc.NormalizedGraph(plgraph, gc.inv_sqrt_degrees(plgraph)).with_precomputed()
    h = torch.from_numpy(f32(rng.uniform(-0.5, 0.5, (plgraph.n_rows, 48)))).pin_memory()
    spec = gc.GcnLayerSpec(48, 40, f32(rng.uniform(-0.5, 0.5, (48, 40))), composition=comp,
                           order=order)
    out = gc.gcn_layer(g, h, spec)
    assert not out.is_cuda and out.is_pinned()
    ref = gc.gcn_layer(g, h.to(DEV), spec).cpu()
    assert torch.allclose(out, ref, rtol=1e-5, atol=1e-6)


def test_cuda_graph_captured_forward_matches_eager(plgraph):
    from paper_2306_15155_b200.capture import GraphedForward

    rng = np.random.default_rng(31)
    g = gc.NormalizedGraph(plgraph, gc.inv_sqrt_degrees(plgraph)).with_precomputed()
    specs = [gc.GcnLayerSpec(40, 16, f32(rng.uniform(-0.5, 0.5, (40, 16))), composition="dynamic"),
             gc.GcnLayerSpec(16, 7, f32(rng.uniform(-0.5, 0.5, (16, 7))), composition="precompute")]
    h = torch.from_numpy(f32(rng.uniform(-0.5, 0.5, (plgraph.n_rows, 40)))).to(DEV)
    eager = gc.gcn_forward(g, h, specs)
    fwd = GraphedForward(lambda x: gc.gcn_forward(g, x, specs), h)
    assert torch.equal(fwd(h), eager)
    h2 = h * 0.5
    assert torch.equal(fwd(h2), gc.gcn_forward(g, h2, specs))


@pytest.mark.parametrize("K", [16, 32, 64, 128, 256])
@pytest.mark.parametrize("shrink", ["0", "1", "2"])
@pytest.mark.parametrize("hints", ["0", "1"])
def test_spmm_and_gat_kernel_variants(oracle, plgraph, K, shrink, hints, monkeypatch):
    """Every lane-group shape x hub-tag variant the autotuner can pick is exact."""
    if K <= 16 and shrink == "2":
        pytest.skip("no such variant")
    monkeypatch.setattr(sparse, "PLAN_MIN_NNZ", 0)
    monkeypatch.setattr(sparse, "SPMM_SHRINK", shrink)
    monkeypatch.setattr(sparse, "HUB_HINTS", hints)
    monkeypatch.setattr(sparse, "HUB_L1_BUDGET", 64 * K)  # tag ~16 hub columns
    rng = np.random.default_rng(K)
    a = plgraph.with_values(torch.from_numpy(f32(rng.uniform(0.5, 2, plgraph.nnz))).to(DEV))
    oa = to_oracle(oracle, a)
    b = f32(rng.standard_normal((a.n_cols, K)))
    d = f32(rng.uniform(0.1, 1.0, a.n_rows))
    bt, dt = torch.from_numpy(b).to(DEV), torch.from_numpy(d).to(DEV)
    out = gc.spmm(a, bt, d_row=dt, d_col=dt).cpu().numpy()
    ref = oracle.scale_rows(d, oracle.spmm(oa, oracle.scale_rows(d, b)))
    assert oracle.rel_err(out, ref) < SP_TOL
    s, t = f32(rng.standard_normal(a.n_rows)), f32(rng.standard_normal(a.n_rows))
    outg = sparse.gat_aggregate(a, torch.from_numpy(s).to(DEV), torch.from_numpy(t).to(DEV), 0.2,
                                bt).cpu().numpy()
    refg = oracle.spmm(oa.with_values(oracle.edge_softmax(oa, s, t, 0.2)), b)
    assert oracle.rel_err(outg, refg) < 2e-5


@pytest.mark.parametrize("K", [64, 128, 256, 512])
@pytest.mark.parametrize("shrink", ["0", "1", "2"])
@pytest.mark.parametrize("algo", ["row", "split"])
def test_fp16_row_kernel_variants(oracle, plgraph, K, shrink, algo, monkeypatch):
    """Every fp16-row lane-group shape computes the SpMM bit-identically to
    the fp32 kernel on the dequantised rows, and the GAT reassoc aggregation
    to 2e-5."""
    monkeypatch.setattr(sparse, "PLAN_MIN_NNZ", 0)
    monkeypatch.setattr(sparse, "SPMM_SHRINK", shrink)
    if algo == "split":
        monkeypatch.setattr(sparse, "SPLIT_CHUNK", 16)
    rng = np.random.default_rng(K + int(shrink))
    n = plgraph.n_rows
    x = torch.from_numpy(f32(rng.standard_normal((n, K)))).to(DEV)
    d = torch.from_numpy(f32(rng.uniform(0.1, 1, n))).to(DEV)
    hr = sparse.pack_rows_f16(x, d)
    deq = hr.xh[:, :K].float().contiguous()
    got = gc.spmm_unweighted(plgraph, hr, d_row=d, algo=algo)
    monkeypatch.setattr(sparse, "SPMM_SHRINK", "0")
    ref = gc.spmm_unweighted(plgraph, deq, d_row=d, d_col=hr.sigma, algo=algo)
    assert torch.equal(got, ref)
    monkeypatch.setattr(sparse, "SPMM_SHRINK", shrink)
    s, t = f32(rng.standard_normal(n) * 3), f32(rng.standard_normal(n) * 3)
    out = sparse.gat_aggregate(plgraph, torch.from_numpy(s).to(DEV), torch.from_numpy(t).to(DEV),
                               0.2, hr, algo=algo)
    oa = to_oracle(oracle, plgraph)
    deq64 = hr.xh[:, :K].double().cpu().numpy() * hr.sigma.double().cpu().numpy()[:, None]
    ref = oracle.spmm(oa.with_values(oracle.edge_softmax(oa, s, t, 0.2)), deq64)
    assert oracle.rel_err(out.cpu().numpy(), ref) < 2e-5


def test_variant_autotune_caches_a_choice(monkeypatch):
    monkeypatch.setattr(sparse, "HUB_AUTOTUNE_MIN_NNZ", 0)
    monkeypatch.setattr(sparse, "PLAN_MIN_NNZ", 0)
    a = gc.add_self_loops(graphs.synthetic_graph("rmat", 4096, 60000, seed=2, device=DEV))
    b = torch.rand(a.n_cols, 64, device=DEV)
    r1 = gc.spmm(a, b)
    assert ("variant", "spmm", 64) in a._plans
    assert torch.equal(gc.spmm(a, b), r1)  # cached variant, deterministic


@pytest.mark.parametrize("K", [4, 16, 64, 256, 384, 1024])
@pytest.mark.parametrize("algo", ["row", "split"])
@pytest.mark.parametrize("shrink", ["0", "2"])
def test_fused_sddmm_attention_aggregate(oracle, plgraph, K, algo, shrink, monkeypatch):
    if K > 256 and shrink != "0":
        pytest.skip("wide rows use one lane-group shape")
    """gc_gat_sddmm_aggregate_f32 == SDDMM-form attention (gat.py:98-114) then
    spmm(alpha, HW) (gat.py:127)."""
    if algo == "split":
        monkeypatch.setattr(sparse, "SPLIT_CHUNK", 16)
    monkeypatch.setattr(sparse, "SPMM_SHRINK", shrink)
    rng = np.random.default_rng(K + 7)
    n = plgraph.n_rows
    hw = f32(rng.uniform(-1, 1, (n, K)))
    a_s, a_d = f32(rng.uniform(-0.5, 0.5, K)), f32(rng.uniform(-0.5, 0.5, K))
    dev = lambda x: torch.from_numpy(x).to(DEV)  # noqa: E731
    for relu in (False, True):
        out = sparse.gat_sddmm_aggregate(plgraph, dev(a_s), dev(a_d), 0.2, dev(hw), relu=relu,
                                         algo=algo)
        assert out is not None
        oa = to_oracle(oracle, plgraph)
        alpha = oracle.atten_calc(oa, hw, a_s, a_d, 0.2)
        ref = oracle.spmm(alpha, hw)
        if relu:
            ref = np.maximum(ref, 0)
        assert oracle.rel_err(out.cpu().numpy(), ref) < 2e-5, (K, algo, relu)


def test_fused_sddmm_attention_falls_back_outside_range(plgraph):
    hw = torch.rand(plgraph.n_rows, 6, device=DEV)
    assert sparse.gat_sddmm_aggregate(plgraph, torch.rand(8, device=DEV)[:6],
                                      torch.rand(8, device=DEV)[:6], 0.2, hw) is None
    hw = torch.rand(plgraph.n_rows, 1028, device=DEV)
    assert sparse.gat_sddmm_aggregate(plgraph, torch.rand(1028, device=DEV),
                                      torch.rand(1028, device=DEV), 0.2, hw) is None


def test_reference_side_binding(oracle, plgraph):
    """INTEGRATION.md's reference-side ctypes stub, fed a reference-style CSR."""
    from paper_2306_15155_b200.refbind import b200_spmm

    oa = to_oracle(oracle, plgraph.with_values(torch.rand(plgraph.nnz, device=DEV)))
    b = np.random.default_rng(5).standard_normal((oa.n_cols, 24))
    out = b200_spmm(oa, b)
    assert out.dtype == np.float64
    assert oracle.rel_err(out, oracle.spmm(oa, b.astype(np.float32))) < SP_TOL


# ---------------------------------------------------------------------------
# hybrid aggregation: dense hub block on tcgen05 (BF16 x3) + sparse tail
# ---------------------------------------------------------------------------


@pytest.fixture(scope="module")
def hub_pl():
    """Power-law graph dense enough for a 64/128-column hub block."""
    a = graphs.powerlaw_graph(2500, 40, seed=11, device=DEV)
    return gc.add_self_loops(a)


@pytest.mark.parametrize("K", [1, 7, 16, 32, 100, 256, 300, 512])
@pytest.mark.parametrize("T", [64, 128])
@pytest.mark.parametrize("fmt", ["bf16x3", "f16x2", "f16", "f16mn"])
def test_hub_gemm_term_split(oracle, K, T, fmt):
    """Dense 0/1 block times the packed terms of D·X: bf16x3 is the exact fp32
    split (1e-6 normwise with rows spanning six decades), f16x2 carries 22
    significant bits relative to max|D·X| (absolute error <= 2^-23 max), f16
    11 (TF32's input rounding: 1e-3 normwise here)."""
    from paper_2306_15155_b200 import _native as nat
    f = {"f16x2": nat.GC_HUB_F16X2, "f16": nat.GC_HUB_F16, "f16mn": nat.GC_HUB_F16_MN,
         "bf16x3": nat.GC_HUB_BF16X3}[fmt]
    if fmt == "f16mn" and not nat.load().gc_hub_f16_mn_supported(K):
        pytest.skip("MN-major one-term operand needs CTA pairs and K > 64")
    dt = torch.bfloat16 if fmt == "bf16x3" else torch.float16
    terms = {"f16x2": 2, "f16": 1, "f16mn": 1, "bf16x3": 3}[fmt]
    rng = np.random.default_rng(K * 7 + T)
    n, ncols = 777, 3000
    a_hub = (rng.random((n, T)) < 0.3).astype(np.float32)
    x = f32(rng.standard_normal((ncols, K)) * 10.0 ** rng.integers(-3, 3, (ncols, 1)))
    hub_cols = np.sort(rng.choice(ncols, T, replace=False)).astype(np.int32)
    d = f32(rng.uniform(0.05, 1.0, ncols))
    dr = f32(rng.uniform(0.05, 1.0, n))
    lib = nat.load()
    kp = lib.gc_hub_terms_rows(K)
    bt = torch.empty(terms * kp * T, dtype=dt, device=DEV)
    sc = torch.empty(2, dtype=torch.float32, device=DEV)
    xt, ht, dtt = (torch.from_numpy(v).to(DEV) for v in (x, hub_cols, d))
    drt = torch.from_numpy(dr).to(DEV)
    at = torch.from_numpy(a_hub).to(DEV).to(dt)
    out = torch.full((n, K), float("nan"), device=DEV)
    st = torch.cuda.current_stream().cuda_stream
    nat.check(lib.gc_hub_pack(xt.data_ptr(), K, K, ht.data_ptr(), T, dtt.data_ptr(), f,
                              bt.data_ptr(), sc.data_ptr(), st), "pack")
    nat.check(lib.gc_hub_gemm(at.data_ptr(), T, n, T, bt.data_ptr(), K, f, sc.data_ptr(),
                              out.data_ptr(), K, drt.data_ptr(), 0, st), "gemm")
    ref = dr.astype(np.float64)[:, None] * (a_hub.astype(np.float64) @ (
        x.astype(np.float64)[hub_cols] * d.astype(np.float64)[hub_cols][:, None]))
    assert oracle.rel_err(out.cpu().numpy(), ref) < (1e-3 if fmt in ("f16", "f16mn") else 1e-6)


@pytest.mark.parametrize("K", [8, 32, 96, 256, 512])
@pytest.mark.parametrize("fmt", ["f16", "f16mn"])
@pytest.mark.parametrize("with_d", [False, True])
def test_hub_pack_from_fp16_rows_bit_exact(K, fmt, with_d):
    """gc_hub_pack_f16rows (the dense part reading the fp16 gather operand)
    packs exactly what gc_hub_pack packs from the dequantised fp32 rows
    sigma_j * xh_j (exact in fp32: sigma is a power of two here)."""
    from paper_2306_15155_b200 import _native as nat
    f = {"f16": nat.GC_HUB_F16, "f16mn": nat.GC_HUB_F16_MN}[fmt]
    lib = nat.load()
    if fmt == "f16mn" and not lib.gc_hub_f16_mn_supported(K):
        pytest.skip("MN-major one-term operand needs CTA pairs and K > 64")
    rng = np.random.default_rng(K + 31)
    ncols, T = 3000, 128
    x = torch.from_numpy(f32(rng.standard_normal((ncols, K)) * 4.0 ** rng.integers(-4, 4, (ncols, 1)))).to(DEV)
    hr = sparse.pack_rows_f16(x)
    deq = (hr.xh[:, :K].float() * hr.sigma[:, None]).contiguous()
    hub_cols = torch.from_numpy(np.sort(rng.choice(ncols, T, replace=False)).astype(np.int32)).to(DEV)
    d = torch.from_numpy(f32(rng.uniform(0.05, 1.0, ncols))).to(DEV) if with_d else None
    kp = lib.gc_hub_terms_rows(K)
    st = torch.cuda.current_stream().cuda_stream
    outs = []
    for half in (True, False):
        bt = torch.empty(kp * T, dtype=torch.float16, device=DEV)
        sc = torch.empty(2, dtype=torch.float32, device=DEV)
        dp = None if d is None else d.data_ptr()
        if half:
            rc = lib.gc_hub_pack_f16rows(hr.xh.data_ptr(), hr.xh.stride(0), hr.sigma.data_ptr(), K,
                                         hub_cols.data_ptr(), T, dp, f, bt.data_ptr(),
                                         sc.data_ptr(), st)
        else:
            rc = lib.gc_hub_pack(deq.data_ptr(), K, K, hub_cols.data_ptr(), T, dp, f,
                                 bt.data_ptr(), sc.data_ptr(), st)
        nat.check(rc, "pack")
        outs.append((bt.cpu(), sc[1:].cpu()))
    assert torch.equal(outs[0][0].view(torch.int16), outs[1][0].view(torch.int16))
    assert torch.equal(outs[0][1], outs[1][1])


@pytest.mark.parametrize("K", [3, 32, 256])
@pytest.mark.parametrize("T", [64, 128])
@pytest.mark.parametrize("precompute", [False, True])
def test_hybrid_aggregate_matches_oracle(oracle, hub_pl, K, T, precompute):
    from paper_2306_15155_b200 import hub
    g = gc.NormalizedGraph.from_adjacency(hub_pl).with_precomputed()
    og = oracle.GcnGraph.from_adjacency(to_oracle(oracle, hub_pl))
    rng = np.random.default_rng(K + T)
    x = f32(rng.uniform(-0.5, 0.5, (hub_pl.n_rows, K)))
    d = g.d_inv_sqrt.to(DEV)
    vals = g.n_tilde.values if precompute else None
    out = hub.hybrid_aggregate(g.a_tilde, torch.from_numpy(x).to(DEV), d, T, values=vals,
                               relu=True)
    ref = np.maximum(oracle.spmm(og.n_tilde, x), 0)
    assert oracle.rel_err(out.cpu().numpy(), ref) < hub_tol()
    plan = hub.hub_plan(g.a_tilde, T)
    assert plan.hub_edges + plan.tail.nnz == g.a_tilde.nnz
    assert plan.hub_edges == int(plan.a_hub.float().sum())


@pytest.mark.parametrize("comp", ["precompute", "dynamic"])
@pytest.mark.parametrize("order", ["aggregate_first", "update_first"])
@pytest.mark.parametrize("split", ["0", "128"])
def test_gcn_layer_fp16_gathers_tf32_class(oracle, hub_pl, comp, order, split, monkeypatch):
    """TF32 class with the fp16 gather operand forced on a small graph (the
    size threshold lifted): plain SpMM and the hybrid split's tail, every
    composition, against the oracle at the class's 1e-2 (and well inside)."""
    from paper_2306_15155_b200 import gcn, hub
    monkeypatch.setattr(gcn, "HALF_MIN_BYTES", 0)
    monkeypatch.setattr(hub, "HUB_SPLIT", split)
    g = gc.NormalizedGraph.from_adjacency(hub_pl).with_precomputed()
    og = oracle.GcnGraph.from_adjacency(to_oracle(oracle, hub_pl))
    rng = np.random.default_rng(4)
    k1, k2 = 48, 32
    h = f32(rng.uniform(-0.5, 0.5, (hub_pl.n_rows, k1)))
    w = f32(rng.uniform(-0.5, 0.5, (k1, k2)))
    spec = gc.GcnLayerSpec(k1, k2, w, composition=comp, order=order)
    assert gc.get_gemm_precision() == "tf32"
    packs = []  # the fp16 rows come from the pack kernel or the GEMM epilogue
    real_pack, real_gemm = gcn.pack_rows_f16, gcn.gemm_f16rows
    monkeypatch.setattr(gcn, "pack_rows_f16", lambda *a, **k: packs.append(1) or real_pack(*a, **k))
    monkeypatch.setattr(gcn, "gemm_f16rows", lambda *a, **k: packs.append(2) or real_gemm(*a, **k))
    out = gc.gcn_layer(g, torch.from_numpy(h).to(DEV), spec).cpu().numpy()
    assert packs, "the fp16 gather operand was used"
    ref = oracle.gcn_layer(og, h.astype(np.float64), w.astype(np.float64), comp, order)
    assert oracle.rel_err(out, ref) <= 3e-3


@pytest.mark.parametrize("comp", ["precompute", "dynamic"])
@pytest.mark.parametrize("order", ["aggregate_first", "update_first"])
def test_gcn_layer_with_hub_split(oracle, hub_pl, comp, order, monkeypatch):
    from paper_2306_15155_b200 import hub
    monkeypatch.setattr(hub, "HUB_SPLIT", "128")
    g = gc.NormalizedGraph.from_adjacency(hub_pl).with_precomputed()
    og = oracle.GcnGraph.from_adjacency(to_oracle(oracle, hub_pl))
    rng = np.random.default_rng(3)
    k1, k2 = 48, 32
    h = f32(rng.uniform(-0.5, 0.5, (hub_pl.n_rows, k1)))
    w = f32(rng.uniform(-0.5, 0.5, (k1, k2)))
    spec = gc.GcnLayerSpec(k1, k2, w, composition=comp, order=order)
    gc.set_gemm_precision("fp32")
    try:
        launches = sparse.kernel_timing("spmm")
        with launches:
            out = gc.gcn_layer(g, torch.from_numpy(h).to(DEV), spec).cpu().numpy()
        torch.cuda.synchronize()
    finally:
        gc.set_gemm_precision("tf32")
    assert ("hubsplit", 128) in g.a_tilde._plans
    ref = oracle.gcn_layer(og, h.astype(np.float64), w.astype(np.float64), comp, order)
    assert oracle.rel_err(out, ref) <= 1e-4


@pytest.mark.parametrize("comp", ["precompute", "dynamic"])
@pytest.mark.parametrize("order", ["aggregate_first", "update_first"])
def test_host_pipelined_layer_with_hub_split(oracle, hub_pl, comp, order, monkeypatch):
    """Pinned host H through the row-block pipeline with the hub split on
    every block (the e2e path of bench.py)."""
    from paper_2306_15155_b200 import gcn as gcn_mod
    from paper_2306_15155_b200 import hub
    monkeypatch.setattr(hub, "HUB_SPLIT", "64")
    monkeypatch.setattr(gcn_mod, "HOST_PIPELINE_BLOCKS", 3)
    g = gc.NormalizedGraph.from_adjacency(hub_pl).with_precomputed()
    og = oracle.GcnGraph.from_adjacency(to_oracle(oracle, hub_pl))
    rng = np.random.default_rng(4)
    k1, k2 = 40, 24
    h = f32(rng.uniform(-0.5, 0.5, (hub_pl.n_rows, k1)))
    w = f32(rng.uniform(-0.5, 0.5, (k1, k2)))
    spec = gc.GcnLayerSpec(k1, k2, w, composition=comp, order=order)
    gc.set_gemm_precision("fp32")
    try:
        out = gc.gcn_layer(g, torch.from_numpy(h).pin_memory(), spec)
    finally:
        gc.set_gemm_precision("tf32")
    assert not out.is_cuda
    blocks = list(g.__dict__.get("_unit_block_cache", {}).values()) + \
        [b for (_, _, b) in sum(g.__dict__.get("_row_block_cache", {}).values(), [])]
    assert any(("hubsplit", 64) in b._plans for b in blocks)  # each row block splits
    ref = oracle.gcn_layer(og, h.astype(np.float64), w.astype(np.float64), comp, order)
    assert oracle.rel_err(out.numpy(), ref) <= 1e-4


@pytest.fixture(scope="module")
def stair_pl():
    a = graphs.synthetic_graph("rmat", 6000, 300000, seed=5, device=DEV)
    return gc.add_self_loops(a)


@pytest.mark.parametrize("K", [24, 32, 64, 96, 128, 256, 512])
@pytest.mark.parametrize("precompute", [False, True])
@pytest.mark.parametrize("abits", [True, False])
def test_stair_split_matches_oracle(oracle, stair_pl, K, precompute, abits, monkeypatch):
    """Multi-step staircase (rank-ordered rows scattered by row_map, rows
    outside every step zero-filled before the tail) vs the oracle, with the
    0/1 blocks as bitmaps (expanded in shared memory) or 16-bit tiles."""
    from paper_2306_15155_b200 import _native as nat
    from paper_2306_15155_b200 import hub
    monkeypatch.setattr(hub, "HUB_ABITS", abits)
    if not nat.load().gc_hub_stair_supported(K):
        pytest.skip("no CTA-pair tile for this K")
    g = gc.NormalizedGraph.from_adjacency(stair_pl).with_precomputed()
    a = g.a_tilde
    spec = ("stair", 50, 10)
    a._plans[("hubsplit", spec)] = hub.StairPlan(a, 0.05, n_clusters=1, first_band=256)
    plan = hub.hub_plan(a, spec)
    assert len(plan.steps) >= 2 and plan.rows0 < a.n_rows
    _, _, _, ws, fx = plan.schedule(K, torch.device(DEV))
    if K <= 256:  # the top tile outlasts the mean pair load: split-K items + fixups
        assert fx is not None and ws is not None
    og = oracle.GcnGraph.from_adjacency(to_oracle(oracle, stair_pl))
    rng = np.random.default_rng(K)
    x = f32(rng.uniform(-0.5, 0.5, (a.n_rows, K)))
    d = g.d_inv_sqrt.to(DEV)
    vals = g.n_tilde.values if precompute else None
    out = hub.hybrid_aggregate(a, torch.from_numpy(x).to(DEV), d, spec, values=vals, relu=True)
    ref = np.maximum(oracle.spmm(og.n_tilde, x), 0)
    assert oracle.rel_err(out.cpu().numpy(), ref) < hub_tol()
    # accumulate form (used by the multi-GPU remote pass)
    base = torch.from_numpy(f32(rng.uniform(-1, 1, (a.n_rows, K)))).to(DEV)
    acc = base.clone()
    hub.hybrid_aggregate(a, torch.from_numpy(x).to(DEV), d, spec, values=vals, out=acc,
                         accumulate=True)
    ref2 = base.cpu().numpy().astype(np.float64) + oracle.spmm(og.n_tilde, x)
    assert oracle.rel_err(acc.cpu().numpy(), ref2) < hub_tol()


def test_host_pipelined_layer_with_stair_split(oracle, stair_pl, monkeypatch):
    from paper_2306_15155_b200 import gcn as gcn_mod
    from paper_2306_15155_b200 import hub
    g = gc.NormalizedGraph.from_adjacency(stair_pl).with_precomputed()
    a = g.a_tilde
    spec = ("stair", 50, 10)
    a._plans[("hubsplit", spec)] = hub.StairPlan(a, 0.05, n_clusters=1, first_band=256)
    monkeypatch.setattr(hub, "HUB_SPLIT", "stair:50:10")
    monkeypatch.setattr(hub, "STAIR_FIRST_BAND", 256)
    monkeypatch.setattr(gcn_mod, "HOST_PIPELINE_BLOCKS", 3)
    og = oracle.GcnGraph.from_adjacency(to_oracle(oracle, stair_pl))
    rng = np.random.default_rng(9)
    h = f32(rng.uniform(-0.5, 0.5, (a.n_rows, 64)))
    w = f32(rng.uniform(-0.5, 0.5, (64, 32)))
    for comp, order in (("precompute", "update_first"), ("dynamic", "aggregate_first")):
        spec_l = gc.GcnLayerSpec(64, 32, w, composition=comp, order=order)
        gc.set_gemm_precision("fp32")
        try:
            out = gc.gcn_layer(g, torch.from_numpy(h).pin_memory(), spec_l)
            dev_out = gc.gcn_layer(g, torch.from_numpy(h).to(DEV), spec_l).cpu()
        finally:
            gc.set_gemm_precision("tf32")
        ref = oracle.gcn_layer(og, h.astype(np.float64), w.astype(np.float64), comp, order)
        assert oracle.rel_err(out.numpy(), ref) <= 1e-4
        assert oracle.rel_err(dev_out.numpy(), ref) <= 1e-4
    blocks = list(g.__dict__.get("_unit_block_cache", {}).values()) + \
        [b for (_, _, b) in sum(g.__dict__.get("_row_block_cache", {}).values(), [])]
    assert any(("hubsplit", ("stair", 50, 10)) in b._plans for b in blocks)


def test_host_pipelined_stair_split_tf32_mode(oracle, stair_pl, monkeypatch):
    """The bench's e2e configuration: TF32 mode (one-term MN-major dense
    operand on every row block), pinned host H, row-block pipeline; layer
    parity in the TF32 class (1e-2, measured ~1e-3)."""
    from paper_2306_15155_b200 import gcn as gcn_mod
    from paper_2306_15155_b200 import hub
    g = gc.NormalizedGraph.from_adjacency(stair_pl).with_precomputed()
    monkeypatch.setattr(hub, "HUB_SPLIT", "stair:50:10")
    monkeypatch.setattr(hub, "STAIR_FIRST_BAND", 256)
    monkeypatch.setattr(gcn_mod, "HOST_PIPELINE_BLOCKS", 3)
    og = oracle.GcnGraph.from_adjacency(to_oracle(oracle, stair_pl))
    rng = np.random.default_rng(12)
    h = f32(rng.uniform(-0.5, 0.5, (stair_pl.n_rows, 256)))
    w = f32(rng.uniform(-0.5, 0.5, (256, 256)))
    assert gc.get_gemm_precision() == "tf32"
    for comp, order in (("dynamic", "update_first"), ("precompute", "aggregate_first")):
        spec_l = gc.GcnLayerSpec(256, 256, w, composition=comp, order=order)
        out = gc.gcn_layer(g, torch.from_numpy(h).pin_memory(), spec_l)
        dev_out = gc.gcn_layer(g, torch.from_numpy(h).to(DEV), spec_l).cpu()
        ref = oracle.gcn_layer(og, h.astype(np.float64), w.astype(np.float64), comp, order)
        assert oracle.rel_err(out.numpy(), ref) <= 1e-2
        assert oracle.rel_err(dev_out.numpy(), ref) <= 1e-2
    blocks = list(g.__dict__.get("_unit_block_cache", {}).values()) + \
        [b for (_, _, b) in sum(g.__dict__.get("_row_block_cache", {}).values(), [])]
    assert any(("hubsplit", ("stair", 50, 10)) in b._plans for b in blocks)
    from paper_2306_15155_b200 import _native as nat
    assert nat.load().gc_hub_f16_mn_supported(256)


def test_stair_split_on_rectangular_block(oracle, stair_pl):
    """A row block of Ã (local rows x all columns, as a rank's remote pass or an
    e2e row block sees it) through the staircase with separate d_row / d_col."""
    from paper_2306_15155_b200 import hub
    g = gc.NormalizedGraph.from_adjacency(stair_pl).with_precomputed()
    d = g.d_inv_sqrt.to(DEV)
    lo, hi = 0, 3000  # the high-degree half of the RMAT rows
    blk = g.a_tilde.take_rows(lo, hi)
    blk._unit = True
    spec = ("stair", 40, 10)
    blk._plans[("hubsplit", spec)] = hub.StairPlan(blk, 0.04, n_clusters=4, first_band=256)
    plan = hub.hub_plan(blk, spec)
    assert len(plan.steps) >= 2
    rng = np.random.default_rng(2)
    x = torch.from_numpy(f32(rng.uniform(-0.5, 0.5, (blk.n_cols, 128)))).to(DEV)
    out = hub.hybrid_aggregate(blk, x, d, spec, d_row=d[lo:hi], relu=True)
    ref = gc.spmm_unweighted(blk, x, d_row=d[lo:hi], d_col=d, relu=True)
    assert oracle.rel_err(out.cpu().numpy(), ref.cpu().numpy().astype(np.float64)) < hub_tol()


def test_gcsr_load_to_device_and_partition(tmp_path, oracle):
    """.gcsr file -> device CSR (same arrays), then the on-device partition
    equals the C-ABI/oracle bounds."""
    from paper_2306_15155_b200.distributed import partition_rows_device

    a = graphs.synthetic_graph("rmat", 20000, 400000, seed=3, device=DEV)
    p = tmp_path / "g.gcsr"
    a.save(p)
    b = gc.CsrMatrix.load(p, device=DEV)
    assert b.device.type == "cuda" and b.same_pattern(a) and b.has_unit_values
    rp = a.row_ptr.cpu().numpy().astype(np.int64)
    for parts in (2, 3, 8):
        assert np.array_equal(partition_rows_device(b.row_ptr, parts), oracle.partition_rows(rp, parts))


@pytest.fixture(scope="module")
def reddit_full():
    """BASELINE configs[1] at full size: Reddit-shaped RMAT (n = 232,965,
    nnz(A) = 114.6 M) with self loops, on the device."""
    return gc.NormalizedGraph.from_adjacency(graphs.shape_graph("reddit", device=DEV))


def test_full_size_reddit_layer_parity(oracle, reddit_full):
    """The bench's configuration at full size: the selected dynamic layer with
    the autotuned dense split vs the fp64 oracle on 512 sampled rows (TF32
    class, 1e-2), and the size-independent property that the hybrid
    aggregation equals the plain SpMM (1e-3 of max in the one-term mode)."""
    from paper_2306_15155_b200 import hub
    g = reddit_full
    a = g.a_tilde
    n, K = a.n_rows, 256
    rng = np.random.default_rng(1)
    h = f32(rng.uniform(-0.5, 0.5, (n, K)))
    w = f32(rng.uniform(-0.5, 0.5, (K, K)))
    spec = gc.GcnLayerSpec(K, K, w, composition="dynamic", order="update_first")
    out = gc.gcn_layer(g, torch.from_numpy(h).to(DEV), spec)
    split = a._plans.get(hub.split_key(K, False), 0)
    assert split, "the autotuner keeps a dense split on the Reddit shape"
    # oracle on sampled rows: relu(D Ã D (H W)) restricted to those rows
    rows = np.sort(rng.choice(n, size=512, replace=False))
    rp, ci, _ = a.numpy()
    d = g.d_inv_sqrt.cpu().numpy().astype(np.float64)
    hw = h.astype(np.float64) @ w.astype(np.float64)
    ref = np.zeros((rows.size, K))
    for k, r in enumerate(rows):
        cols = ci[rp[r]:rp[r + 1]]
        ref[k] = d[r] * (d[cols][:, None] * hw[cols]).sum(0)
    ref = np.maximum(ref, 0)
    got = out[torch.from_numpy(rows).to(DEV)].cpu().numpy()
    assert oracle.rel_err(got, ref) <= 1e-2
    # hybrid == plain on the whole output (same HW operand)
    x = torch.from_numpy(f32(hw)).to(DEV)
    dd = g.d_inv_sqrt.to(DEV)
    plain = sparse.spmm_unweighted(a, x, d_row=dd, d_col=dd)
    hyb = hub.hybrid_aggregate(a, x, dd, split)
    err = float((hyb - plain).abs().max() / plain.abs().max())
    assert err <= 1e-3, err


@pytest.mark.parametrize("shape", ["products", "reddit", "arxiv"])
def test_full_size_normalisation_sddmm_exact(shape):
    """Ñ = D Ã D at the full BASELINE shapes through the edge-parallel window
    kernel: every value equals fp32(d_i * d_j) bit for bit (rows of every
    length, including runs of short rows that cross many row ends per step)."""
    a = gc.add_self_loops(graphs.shape_graph(shape, device=DEV))
    d = sparse.inv_sqrt_degrees(a).to(DEV)
    nt = sparse.sddmm_norm(a, d)
    vals = nt.values if hasattr(nt, "values") else nt
    ref = d[a.row_of_nnz()] * d[a.col_idx.long()]
    assert torch.equal(vals, ref)


# ---- aggregate-first layer with W fused into the SpMM epilogue --


@pytest.mark.parametrize("K1", [4, 8, 16, 32, 64, 128, 200, 256])
@pytest.mark.parametrize("K2", [1, 7, 16, 32])
@pytest.mark.parametrize("weighted", [False, True])
def test_spmm_gemm_matches_oracle(oracle, K1, K2, weighted):
    """gc_spmm_gemm_f32 = relu(D_row A D_col B) W (reference gcn.py:119-122
    `gemm(spmm(a, h), w)`) to fp32 accuracy, including empty rows."""
    rng = np.random.default_rng(K1 * 100 + K2)
    a = rand_csr(rng, 300, 280, 0.04, unit=not weighted, empty_rows=(0, 17, 299))
    oa = to_oracle(oracle, a)
    b = f32(rng.standard_normal((280, K1)))
    w = f32(rng.standard_normal((K1, K2)))
    dr, dc = f32(rng.uniform(0.1, 1, 300)), f32(rng.uniform(0.1, 1, 280))
    t = lambda x: torch.from_numpy(x).to(DEV)  # noqa: E731
    out = sparse.spmm_gemm(a, t(b), t(w), weighted=weighted, d_row=t(dr), d_col=t(dc),
                           relu=True).cpu().numpy()
    agg = oracle.spmm(oa, oracle.scale_rows(dc, b)) if weighted else \
        oracle.spmm_unweighted(oa, oracle.scale_rows(dc, b))
    ref = np.maximum(oracle.gemm(oracle.scale_rows(dr, agg), w), 0)
    assert oracle.rel_err(out, ref) < 1e-5
    assert np.all(out[[0, 17, 299]] == 0)
    plain = sparse.spmm_gemm(a, t(b), t(w), weighted=weighted).cpu().numpy()
    ref_plain = oracle.gemm(oracle.spmm(oa, b) if weighted else oracle.spmm_unweighted(oa, b), w)
    assert oracle.rel_err(plain, ref_plain) < 1e-5


def test_spmm_gemm_rejects_unsupported_shapes():
    rng = np.random.default_rng(1)
    a = rand_csr(rng, 20, 20, 0.2)
    b = torch.rand(20, 6, device=DEV)
    from paper_2306_15155_b200._native import NativeError

    with pytest.raises(NativeError):
        sparse.spmm_gemm(a, b, torch.rand(6, 4, device=DEV))  # K1 % 4 != 0
    b = torch.rand(20, 8, device=DEV)
    with pytest.raises(NativeError):
        sparse.spmm_gemm(a, b, torch.rand(8, 33, device=DEV))  # K2 > 32
    with pytest.raises(gc.ShapeError):
        sparse.spmm_gemm(a, b, torch.rand(7, 4, device=DEV))


@pytest.mark.parametrize("comp", ["precompute", "dynamic"])
@pytest.mark.parametrize("k1,k2", [(16, 7), (64, 32), (128, 16), (256, 8)])
def test_gcn_aggregate_first_fused_update(oracle, comp, k1, k2, monkeypatch):
    """The aggregate-first layer takes the fused kernel on a bounded-degree
    graph (no nnz-split plan) and matches the oracle layer and the two-kernel
    form; the fp32 class to 1e-4."""
    gc.set_gemm_precision("fp32")
    try:
        A = graphs.synthetic_graph("uniform", 3000, 24000, seed=k1 + k2, device=DEV)
        g = gc.NormalizedGraph.from_adjacency(A).with_precomputed()
        assert sparse.spmm_gemm_eligible(g.a_tilde, torch.empty(1, k1, device=DEV), k2)
        rng = np.random.default_rng(k1 + k2)
        h = f32(rng.uniform(-0.5, 0.5, (g.a_tilde.n_rows, k1)))
        w = f32(rng.uniform(-0.5, 0.5, (k1, k2)))
        spec = gc.GcnLayerSpec(k1, k2, w, composition=comp, order="aggregate_first")
        calls = []
        from paper_2306_15155_b200 import gcn as gcn_mod

        real = sparse.spmm_gemm
        monkeypatch.setattr(gcn_mod, "spmm_gemm", lambda *a, **k: calls.append(1) or real(*a, **k))
        fused = gc.gcn_layer(g, torch.from_numpy(h).to(DEV), spec).cpu().numpy()
        assert calls, "the fused kernel did not run"
        host = g.a_tilde.numpy()
        at = oracle.Csr(g.a_tilde.n_rows, g.a_tilde.n_cols, *host)
        og = oracle.GcnGraph(at, oracle.inv_sqrt_degrees(at))
        ref = oracle.gcn_layer(og, h, w, comp, "aggregate_first")
        assert oracle.rel_err(fused, ref) < 1e-4
        monkeypatch.setattr(sparse, "SPMM_GEMM", False)
        two = gc.gcn_layer(g, torch.from_numpy(h).to(DEV), spec).cpu().numpy()
        assert oracle.rel_err(fused, two) < 1e-5
    finally:
        gc.set_gemm_precision("tf32")


@pytest.mark.parametrize("kind", ["uniform", "rmat"])
@pytest.mark.parametrize("seed", [0, 1, 2])
@pytest.mark.parametrize("K", [64, 256, 512])
def test_fp16_spmm_random_graphs_bit_exact_and_oracle(oracle, kind, seed, K):
    """Random uniform / power-law graphs (seeded): the fp16-row SpMM (fp16-
    weight FMA for unit edges, split plans for the heavy rows) equals the fp32
    kernel on the dequantised rows bit for bit, and the oracle on the
    dequantised rows to fp32 accuracy."""
    a = gc.add_self_loops(graphs.synthetic_graph(kind, 5000 + 700 * seed, 120000 + 20000 * seed,
                                                 seed=seed, device=DEV))
    rng = np.random.default_rng(seed * 10 + K)
    x = torch.from_numpy(f32(rng.standard_normal((a.n_cols, K))
                             * 2.0 ** rng.integers(-8, 8, (a.n_cols, 1)))).to(DEV)
    d = gc.inv_sqrt_degrees(a).to(DEV)
    hr = sparse.pack_rows_f16(x, d)
    got = gc.spmm_unweighted(a, hr, d_row=d, relu=False)
    deq = hr.xh[:, :K].float().contiguous()
    assert torch.equal(got, gc.spmm_unweighted(a, deq, d_row=d, d_col=hr.sigma))
    deq64 = hr.xh[:, :K].double().cpu().numpy() * hr.sigma.double().cpu().numpy()[:, None]
    ref = oracle.scale_rows(d.double().cpu().numpy(),
                            oracle.spmm_unweighted(to_oracle(oracle, a), deq64))
    assert oracle.rel_err(got.cpu().numpy(), ref) < 1e-5


# ---- fp16 rows with one scale per 256-column chunk (gemm_f16rows, N > 256) ----


def _chunked_rows(x: torch.Tensor) -> "sparse.HalfRows":
    """HalfRows with one scale per 256-column chunk, built by packing each
    chunk on its own (what the GEMM epilogue emits per N tile)."""
    parts = [sparse.pack_rows_f16(x[:, c:c + 256].contiguous()) for c in range(0, x.shape[1], 256)]
    xh = torch.cat([p.xh for p in parts], 1).contiguous()
    return sparse.HalfRows(xh, torch.stack([p.sigma for p in parts], 1).contiguous(), x.shape[1])


@pytest.mark.parametrize("M,K,N", [(1000, 64, 512), (3001, 200, 1024), (777, 256, 768)])
@pytest.mark.parametrize("scaled", [False, True])
def test_gemm_f16rows_chunked_scales_equal_chunk_packs(M, K, N, scaled):
    """N a multiple of 256: the epilogue emits one scale per row and 256-column
    N tile, bit-identical to packing each chunk of the TF32 GEMM's output."""
    rng = np.random.default_rng(M + N)
    a = torch.from_numpy(f32(rng.uniform(-0.5, 0.5, (M, K)) * 2.0 ** rng.integers(-6, 6, (M, 1)))).to(DEV)
    w = torch.from_numpy(f32(rng.uniform(-0.5, 0.5, (K, N)) * 2.0 ** rng.integers(-4, 4, (1, N)))).to(DEV)
    rs = torch.from_numpy(f32(rng.uniform(0.1, 1.0, M))).to(DEV) if scaled else None
    hr = sparse.gemm_f16rows(a, w, row_scale=rs)
    assert hr is not None and hr.chunks == N // 256
    ref = _chunked_rows(gc.gemm(a, w, row_scale=rs, precision="tf32"))
    assert torch.equal(hr.xh.view(torch.int16), ref.xh.view(torch.int16))
    assert torch.equal(hr.sigma, ref.sigma)


@pytest.mark.parametrize("K", [512, 1024])
@pytest.mark.parametrize("algo", ["row", "split"])
@pytest.mark.parametrize("shrink", ["0", "1", "2"])
def test_spmm_and_gat_chunked_scales(oracle, plgraph, K, algo, shrink, monkeypatch):
    """SpMM over chunked-scale fp16 rows: each 256-column pass equals the fp32
    kernel on that chunk's dequantised rows with d_col = the chunk's scales
    (bit for bit); GAT reassoc against the oracle on the dequantised rows."""
    monkeypatch.setattr(sparse, "PLAN_MIN_NNZ", 0)
    monkeypatch.setattr(sparse, "SPMM_SHRINK", shrink)
    if algo == "split":
        monkeypatch.setattr(sparse, "SPLIT_CHUNK", 16)
    rng = np.random.default_rng(K + int(shrink))
    n = plgraph.n_rows
    x = torch.from_numpy(f32(rng.standard_normal((n, K)) * 2.0 ** rng.integers(-5, 5, (1, K)))).to(DEV)
    d = torch.from_numpy(f32(rng.uniform(0.1, 1, n))).to(DEV)
    hr = _chunked_rows(x)
    got = gc.spmm_unweighted(plgraph, hr, d_row=d, algo=algo)
    monkeypatch.setattr(sparse, "SPMM_SHRINK", "0")
    for c in range(K // 256):
        cs = slice(c * 256, (c + 1) * 256)
        deq = hr.xh[:, cs].float().contiguous()
        ref = gc.spmm_unweighted(plgraph, deq, d_row=d, d_col=hr.sigma[:, c].contiguous(), algo=algo)
        assert torch.equal(got[:, cs], ref), f"chunk {c}"
    monkeypatch.setattr(sparse, "SPMM_SHRINK", shrink)
    s, t = f32(rng.standard_normal(n) * 3), f32(rng.standard_normal(n) * 3)
    out = sparse.gat_aggregate(plgraph, torch.from_numpy(s).to(DEV), torch.from_numpy(t).to(DEV),
                               0.2, hr, algo=algo)
    sig = np.repeat(hr.sigma.double().cpu().numpy(), 256, axis=1)
    deq64 = hr.xh.double().cpu().numpy() * sig
    oa = to_oracle(oracle, plgraph)
    ref = oracle.spmm(oa.with_values(oracle.edge_softmax(oa, s, t, 0.2)), deq64)
    assert oracle.rel_err(out.cpu().numpy(), ref) < 2e-5


@pytest.mark.parametrize("K", [512, 1024])
@pytest.mark.parametrize("fmt", ["f16", "f16mn"])
def test_hub_pack_chunked_scales_bit_exact(K, fmt):
    from paper_2306_15155_b200 import _native as nat
    f = {"f16": nat.GC_HUB_F16, "f16mn": nat.GC_HUB_F16_MN}[fmt]
    lib = nat.load()
    if fmt == "f16mn" and not lib.gc_hub_f16_mn_supported(K):
        pytest.skip("MN-major one-term operand needs CTA pairs")
    rng = np.random.default_rng(K + 7)
    ncols, T = 3000, 128
    x = torch.from_numpy(f32(rng.standard_normal((ncols, K)) * 2.0 ** rng.integers(-4, 4, (1, K)))).to(DEV)
    hr = _chunked_rows(x)
    deq = (hr.xh.float() * torch.repeat_interleave(hr.sigma, 256, dim=1)).contiguous()
    hub_cols = torch.from_numpy(np.sort(rng.choice(ncols, T, replace=False)).astype(np.int32)).to(DEV)
    kp = lib.gc_hub_terms_rows(K)
    st = torch.cuda.current_stream().cuda_stream
    outs = []
    for half in (True, False):
        bt = torch.empty(kp * T, dtype=torch.float16, device=DEV)
        sc = torch.empty(2, dtype=torch.float32, device=DEV)
        if half:
            rc = lib.gc_hub_pack_f16rows(hr.xh.data_ptr(), hr.xh.stride(0), hr.sigma.data_ptr(), K,
                                         hub_cols.data_ptr(), T, None,
                                         f | nat.GC_HUB_SIG_CHUNKS(K // 256), bt.data_ptr(),
                                         sc.data_ptr(), st)
        else:
            rc = lib.gc_hub_pack(deq.data_ptr(), K, K, hub_cols.data_ptr(), T, None, f,
                                 bt.data_ptr(), sc.data_ptr(), st)
        nat.check(rc, "pack")
        outs.append((bt.view(torch.int16).clone(), sc.clone()))
    assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])


@pytest.mark.parametrize("comp", ["precompute", "dynamic"])
def test_gcn_update_first_chunked_fp16_rows(oracle, hub_pl, comp, monkeypatch):
    """Update-first at k2 = 512 in the TF32 class: the GEMM epilogue emits
    fp16 rows with two scales per row, consumed by the plain SpMM and by the
    hybrid split's dense part and tail; against the oracle."""
    from paper_2306_15155_b200 import gcn, hub
    monkeypatch.setattr(gcn, "HALF_MIN_BYTES", 0)
    g = gc.NormalizedGraph.from_adjacency(hub_pl).with_precomputed()
    og = oracle.GcnGraph.from_adjacency(to_oracle(oracle, hub_pl))
    rng = np.random.default_rng(5)
    k1, k2 = 64, 512
    h = f32(rng.uniform(-0.5, 0.5, (hub_pl.n_rows, k1)))
    w = f32(rng.uniform(-0.5, 0.5, (k1, k2)))
    spec = gc.GcnLayerSpec(k1, k2, w, composition=comp, order="update_first")
    seen = []
    real = gcn.gemm_f16rows
    monkeypatch.setattr(gcn, "gemm_f16rows",
                        lambda *a, **k: (lambda r: seen.append(r.chunks) or r)(real(*a, **k)))
    ref = oracle.gcn_layer(og, h.astype(np.float64), w.astype(np.float64), comp, "update_first")
    for split in ("0", "128"):
        monkeypatch.setattr(hub, "HUB_SPLIT", split)
        out = gc.gcn_layer(g, torch.from_numpy(h).to(DEV), spec).cpu().numpy()
        assert oracle.rel_err(out, ref) <= 3e-3, split
    assert seen and all(c == 2 for c in seen)
