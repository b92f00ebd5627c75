"""Timeline of the host-pipelined GCN layer (pinned H in, pinned out): CUDA
events on the compute and copy streams for every row block, to see how much
of the D2H hides behind the next block's SpMM.  Reddit-shaped, K = 256."""

from __future__ import annotations

import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import paper_2306_15155_b200 as gc  # noqa: E402
from paper_2306_15155_b200 import gcn, graphs  # noqa: E402
from paper_2306_15155_b200.sparse import spmm  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    K = 256
    A = graphs.shape_graph("reddit", device=dev)
    g = gc.NormalizedGraph.from_adjacency(A).with_precomputed()
    del A
    n = g.a_tilde.n_rows
    h_pin = (torch.rand(n, K) - 0.5).pin_memory()
    spec = gc.GcnLayerSpec(K, K, torch.rand(K, K, device=dev) - 0.5, composition="precompute",
                           order="aggregate_first")
    res = {}
    for blocks in (0, 1, 4):
        gcn.HOST_PIPELINE_BLOCKS = blocks
        for _ in range(3):
            gc.gcn_layer(g, h_pin, spec)
        torch.cuda.synchronize()
        # manual replica of _host_pipelined with events
        comp = torch.cuda.current_stream()
        copy = gcn._COPY_STREAMS[dev]
        ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
        t0 = ev()
        t0.record(comp)
        h_dev = h_pin.to(dev, non_blocking=True)
        t_h2d = ev()
        t_h2d.record(comp)
        out = torch.empty(n, K, pin_memory=True)
        marks = []
        for lo, hi, blk in gcn._row_blocks(g, g.n_tilde, blocks):
            a0 = ev()
            a0.record(comp)
            y = gc.gemm(spmm(blk, h_dev), spec.weights, relu=True)  # precompute, aggregate-first
            a1 = ev()
            a1.record(comp)
            copy.wait_event(a1)
            c0 = ev()
            c0.record(copy)
            with torch.cuda.stream(copy):
                out[lo:hi].copy_(y, non_blocking=True)
            c1 = ev()
            c1.record(copy)
            y.record_stream(copy)
            marks.append((a0, a1, c0, c1))
        torch.cuda.synchronize()
        res[blocks] = {"h2d_ms": t0.elapsed_time(t_h2d),
                       "blocks": [{"compute": (t0.elapsed_time(a0), t0.elapsed_time(a1)),
                                   "copy": (t0.elapsed_time(c0), t0.elapsed_time(c1))}
                                  for a0, a1, c0, c1 in marks]}
        print(json.dumps({blocks: res[blocks]}), file=sys.stderr, flush=True)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
