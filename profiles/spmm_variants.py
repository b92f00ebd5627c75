"""Micro-benchmark behind the SpMM design decisions (run on the B200 box).

Times the dominant aggregation kernel on the BASELINE graph shapes with and
without the hub-column L1 policy tags, the fused GAT aggregation against the
two-step edge-softmax + SpMM, and the raw host<->device copy bandwidth that
bounds ``e2e``.  CUDA events on the launching stream, median of 10 after 3
warm-ups.  Prints one JSON document.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import paper_2306_15155_b200 as gc  # noqa: E402
from paper_2306_15155_b200 import graphs, sparse  # noqa: E402
from paper_2306_15155_b200.gat import _projections  # noqa: E402


def timed(fn, reps=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in ev:
        a.record()
        fn()
        b.record()
    torch.cuda.synchronize()
    t = sorted(a.elapsed_time(b) for a, b in ev)
    return t[len(t) // 2]


def main():
    dev = torch.device("cuda", 0)
    out = {"spmm": [], "gat": [], "pcie": {}}
    for shape, ks in (("reddit", (32, 256, 1024)), ("products", (32, 256)), ("arxiv", (32, 256))):
        A = graphs.shape_graph(shape, device=dev)
        at = gc.add_self_loops(A)
        del A
        d = gc.inv_sqrt_degrees(at).to(dev)
        n, m = at.n_rows, at.nnz
        for K in ks:
            h = torch.rand(n, K, device=dev) - 0.5
            row = {"shape": shape, "K": K, "m": m}
            for hints in (False, True):
                sparse.HUB_HINTS = "1" if hints else "0"
                ms = timed(lambda: gc.spmm_unweighted(at, h, d_row=d, d_col=d))
                row["hints" if hints else "plain"] = ms
            sparse.HUB_HINTS = "auto"
            row["gain"] = row["plain"] / row["hints"]
            out["spmm"].append(row)
            print(json.dumps(row), file=sys.stderr, flush=True)
            if shape in ("arxiv", "products") and K == 256:
                spec = gc.GatLayerSpec(K, K, torch.eye(K, device=dev), torch.rand(K, device=dev) - 0.5,
                                       torch.rand(K, device=dev) - 0.5)
                s, t = _projections(h, spec, spec.attn_src, spec.attn_dst, K, K)
                fused = timed(lambda: sparse.gat_aggregate(at, s[0], t[0], 0.2, h))

                def two_step():
                    att = gc.atten_calc(at, h, spec)
                    gc.spmm(att.alpha, h)
                two = timed(two_step)
                out["gat"].append({"shape": shape, "K": K, "fused_ms": fused, "two_step_ms": two})
            del h
        del at
        torch.cuda.empty_cache()
    nbytes = 238_556_160
    host = torch.empty(nbytes // 4, dtype=torch.float32, pin_memory=True)
    devb = torch.empty(nbytes // 4, dtype=torch.float32, device=dev)
    h2d = timed(lambda: devb.copy_(host, non_blocking=True))
    d2h = timed(lambda: host.copy_(devb, non_blocking=True))
    out["pcie"] = {"bytes": nbytes, "h2d_ms": h2d, "d2h_ms": d2h,
                   "h2d_gbs": nbytes / h2d / 1e6, "d2h_gbs": nbytes / d2h / 1e6}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
