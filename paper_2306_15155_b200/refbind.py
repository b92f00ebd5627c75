"""The reference-side binding: a ``spmm_fn`` for the reference package.

``gnncompose``'s layer functions accept ``spmm_fn(a, b) -> ndarray``
(gcn.py:125-161, gat.py:121-153).  This module is the stub a maintainer of the
reference would add to route that aggregation through ``libgnnc.so``: it only
uses ctypes, numpy and torch (for device memory and the stream) and accepts
any object with the reference ``CsrMatrix`` attributes (``n_rows``,
``n_cols``, ``row_ptr``, ``col_idx``, ``values``, int64 / float64 host
arrays), returning a float64 ndarray like the reference's ``spmm``.

    from paper_2306_15155_b200.refbind import b200_spmm
    gnncompose.gcn_layer(g, h, spec, spmm_fn=b200_spmm)
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from ._build import LIB

_lib = None


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(str(LIB))
        p, i = ctypes.c_void_p, ctypes.c_int64
        lib.gc_spmm_f32.argtypes = [p, p, p, p, p, p, i, i, i, i, p, i, ctypes.c_uint32, ctypes.c_int,
                                    p, i, p, i, p, ctypes.c_size_t, p]
        lib.gc_last_error.restype = ctypes.c_char_p
        _lib = lib
    return _lib


def b200_spmm(a, b) -> np.ndarray:
    """C = A @ B for a reference CsrMatrix ``a`` and a host dense ``b``."""
    lib = _load()
    dev = torch.device("cuda", torch.cuda.current_device())
    b = np.ascontiguousarray(b, dtype=np.float32)
    if b.ndim != 2 or b.shape[0] != a.n_cols:
        raise ValueError(f"spmm: a is {a.n_rows}x{a.n_cols}, b has shape {b.shape}")
    rp = torch.from_numpy(np.asarray(a.row_ptr, dtype=np.int32)).to(dev)
    ci = torch.from_numpy(np.asarray(a.col_idx, dtype=np.int32)).to(dev)
    va = torch.from_numpy(np.asarray(a.values, dtype=np.float32)).to(dev)
    bt = torch.from_numpy(b).to(dev)
    k = b.shape[1]
    out = torch.empty(a.n_rows, k, dtype=torch.float32, device=dev)
    rc = lib.gc_spmm_f32(rp.data_ptr(), ci.data_ptr(), va.data_ptr(), None, None, bt.data_ptr(),
                         max(k, 1), a.n_rows, a.n_cols, k, out.data_ptr(), max(k, 1), 0, 1, None, 0,
                         None, 0, None, 0, torch.cuda.current_stream(dev).cuda_stream)
    if rc:
        raise RuntimeError(lib.gc_last_error().decode())
    return out.cpu().numpy().astype(np.float64)
