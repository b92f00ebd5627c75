"""The C-ABI library builds for sm_100a, loads without a GPU, and exports every
symbol include/gnnc.h declares.  Host-only entry points (planner, partition)
are exercised here; compute entry points are GPU tests."""

from __future__ import annotations

import ctypes
import subprocess

import numpy as np
import pytest
import torch

from paper_2306_15155_b200 import _build, _native


@pytest.fixture(scope="module")
def lib():
    _build.build()
    return _native.load()


def test_header_declares_the_boundary():
    syms = _native.header_symbols()
    for s in ("gc_spmm_f32", "gc_sddmm_f32", "gc_sddmm_norm_f32", "gc_gemm_f32",
              "gc_edge_softmax_f32", "gc_attn_sddmm_f32", "gc_node_proj_f32",
              "gc_partition_rows", "gc_spmm_plan_count", "gc_spmm_plan_fill", "gc_hub_pack",
              "gc_hub_gemm", "gc_hub_stair_gemm"):
        assert s in syms


def test_every_header_symbol_is_exported(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", str(_native.lib_path())],
                         capture_output=True, text=True, check=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if line.strip()}
    missing = [s for s in _native.header_symbols() if s not in exported]
    assert not missing, missing
    for s in _native.header_symbols():
        assert s in _native._SIGNATURES, f"{s} has no ctypes signature"


def test_library_is_sm100a_only(lib):
    out = subprocess.run(["cuobjdump", "--list-elf", str(_native.lib_path())],
                         capture_output=True, text=True, check=True).stdout
    assert "sm_100a" in out


def test_tcgen05_and_tma_in_sass(lib):
    out = subprocess.run(["cuobjdump", "-sass", str(_native.lib_path())], capture_output=True,
                         text=True, check=True).stdout
    assert "UTCHMMA" in out or "UTCMMA" in out or "UTC" in out  # tcgen05.mma
    assert "UTMALDG" in out  # TMA tensor loads
    assert "LDTM" in out  # tcgen05.ld


def test_abi_version_and_counters(lib):
    assert lib.gc_abi_version() == _native.ABI_VERSION == 2
    assert isinstance(_native.launch_count(), int)


def test_error_codes_without_launch(lib):
    # validation happens before any CUDA call, so this works without a GPU
    rc = lib.gc_spmm_f32(None, None, None, None, None, None, 1, -1, 1, 1, None, 1, 0, 1, None, 0,
                         None, 0, None, 0, None)
    assert rc == _native.GC_ERR_SHAPE
    assert b"negative" in lib.gc_last_error()
    rc = lib.gc_gemm_f32(None, 4, None, 4, 4, 4, 4, None, 4, None, 0, None, 0, None)
    assert rc == _native.GC_ERR_VALUE
    # dense-split entry points: unknown term format, bad shapes, bad staircase
    rc = lib.gc_hub_pack(None, 8, 8, None, 64, None, 7, None, None, None)
    assert rc == _native.GC_ERR_VALUE and b"format" in lib.gc_last_error()
    rc = lib.gc_hub_pack(None, 8, 8, None, 64, None, _native.GC_HUB_F16X2, None, None, None)
    assert rc == _native.GC_ERR_VALUE  # null operands (f16x2 also needs the scale workspace)
    rc = lib.gc_hub_pack(None, 8, 8, None, 64, None, _native.GC_HUB_F16, None, None, None)
    assert rc == _native.GC_ERR_VALUE  # one-term f16: known format, null operands
    assert b"null" in lib.gc_last_error()
    rc = lib.gc_hub_stair_gemm(None, None, None, None, 1, None, None, None, 0, None, None, 0, None,
                               64, 32, _native.GC_HUB_F16, None, None, 32, None, 0, None)
    assert rc == _native.GC_ERR_VALUE  # f16 needs the scale workspace
    rc = lib.gc_hub_gemm(None, 63, 10, 64, None, 8, _native.GC_HUB_BF16X3, None, None, 8, None,
                         0, None)
    assert rc == _native.GC_ERR_SHAPE  # lda < T
    rc = lib.gc_hub_stair_gemm(None, None, None, None, 0, None, None, None, 0, None, None, 0, None,
                               64, 32, 0, None, None, 32, None, 0, None)
    assert rc == _native.GC_ERR_VALUE  # no steps
    assert lib.gc_hub_terms_rows(256) % 128 == 0 and lib.gc_hub_terms_rows(0) == 0


def _plan(lib, rp, chunk, flags=0):
    rp = np.ascontiguousarray(rp, dtype=np.int32)
    ni, ns, nsr = (np.zeros(1, np.int64) for _ in range(3))
    assert lib.gc_spmm_plan_count(rp.ctypes.data, rp.size - 1, chunk,
                                  ni.ctypes.data_as(_native._i64p), ns.ctypes.data_as(_native._i64p),
                                  nsr.ctypes.data_as(_native._i64p)) == 0
    items = np.zeros((ni[0], 4), np.int32)
    split = np.zeros((max(nsr[0], 1), 4), np.int32)
    assert lib.gc_spmm_plan_fill(rp.ctypes.data, rp.size - 1, chunk, flags, items.ctypes.data,
                                 split.ctypes.data) == 0
    return items, split[: nsr[0]], int(ns[0])


@pytest.mark.parametrize("flags", [0, 1])
def test_spmm_plan_covers_every_edge_once(lib, flags):
    rng = np.random.default_rng(0)
    deg = rng.integers(0, 50, size=200)
    deg[[3, 77]] = [500, 1000]
    rp = np.concatenate(([0], np.cumsum(deg)))
    items, split, n_slots = _plan(lib, rp, 64, flags)
    lens = items[:, 2] - items[:, 1]
    if flags:  # longest length class first, stable within a class
        cls = np.where(lens == 0, 0, np.floor(np.log2(np.maximum(lens, 1))).astype(int) + 1)
        assert np.all(np.diff(cls) <= 0)
        for c in np.unique(cls):
            r = items[cls == c, 0]
            assert np.all(np.diff(r) >= 0)
    else:
        assert np.all(np.diff(items[:, 0]) >= 0)
    covered = np.zeros(rp[-1], np.int32)
    for r, b, e, s in items:
        assert rp[r] <= b <= e <= rp[r + 1] and e - b <= 64
        covered[b:e] += 1
    assert (covered == 1).all()
    # every row appears; split rows are exactly those over the chunk
    assert set(items[:, 0]) == set(range(200))
    assert set(split[:, 0]) == set(np.flatnonzero(deg > 64))
    assert n_slots == (items[:, 3] >= 0).sum() == split[:, 2].sum()


@pytest.mark.parametrize("parts", [1, 2, 3, 4, 8])
def test_partition_bit_exact_with_oracle(lib, oracle, parts):
    rng = np.random.default_rng(parts)
    deg = rng.zipf(1.7, size=3000).clip(max=5000)
    rp = np.concatenate(([0], np.cumsum(deg))).astype(np.int64)
    out = np.zeros(parts + 1, np.int64)
    assert lib.gc_partition_rows(rp.ctypes.data, rp.size - 1, parts, out.ctypes.data) == 0
    assert np.array_equal(out, oracle.partition_rows(rp, parts))


def test_default_chunk(lib):
    assert lib.gc_spmm_default_chunk(100, 1000, 256, 148) == 128
    assert lib.gc_spmm_default_chunk(233_000, 115_000_000, 256, 148) == 4096
    c = lib.gc_spmm_default_chunk(169_343, 2_500_000, 32, 148)
    assert 128 <= c <= 512 and c & (c - 1) == 0


def test_partition_edge_cases(lib, oracle):
    for rp in (np.array([0], np.int64), np.array([0, 0, 0], np.int64), np.array([0, 10], np.int64)):
        out = np.zeros(5, np.int64)
        assert lib.gc_partition_rows(rp.ctypes.data, rp.size - 1, 4, out.ctypes.data) == 0
        assert np.array_equal(out, oracle.partition_rows(rp, 4))
    assert lib.gc_partition_rows(ctypes.c_void_p(0), 0, 2, ctypes.c_void_p(0)) == _native.GC_ERR_VALUE


@pytest.mark.parametrize("parts", [1, 2, 3, 4, 8])
def test_partition_device_form_matches_abi(oracle, parts):
    """partition_rows_device (searchsorted where row_ptr lives) gives the
    same bounds as the C ABI / oracle; run here on a CPU tensor."""
    from paper_2306_15155_b200.distributed import partition_rows_device

    rng = np.random.default_rng(10 + parts)
    for deg in (rng.zipf(1.7, size=3000).clip(max=5000), np.zeros(7, np.int64), np.array([10])):
        rp = np.concatenate(([0], np.cumsum(deg))).astype(np.int64)
        want = oracle.partition_rows(rp, parts)
        got = partition_rows_device(torch.from_numpy(rp.astype(np.int32)), parts)
        assert np.array_equal(got, want)
