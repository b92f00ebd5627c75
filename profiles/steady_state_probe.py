"""Is the headline step slower right after setup than in the sweep?  Times 60
consecutive GCN layer steps (Reddit-shaped, K = 256) one by one with CUDA
events and prints the sequence, plus nvidia-smi clocks before/after."""

from __future__ import annotations

import json
import subprocess
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import paper_2306_15155_b200 as gc  # noqa: E402
from paper_2306_15155_b200 import graphs, profiling  # noqa: E402


def clocks():
    try:
        return subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks.mem,power.draw,temperature.gpu",
                               "--format=csv,noheader"], capture_output=True, text=True).stdout.strip()
    except OSError:
        return None


def main():
    dev = torch.device("cuda", 0)
    K = 256
    A = graphs.shape_graph("reddit", device=dev)
    g = gc.NormalizedGraph.from_adjacency(A).with_precomputed()
    n = g.a_tilde.n_rows
    inp = profiling.draw_inputs(profiling.config_rng(0, "reddit", K, K), n, K, K, "gcn")
    h = torch.from_numpy(inp["h"].astype(np.float32)).to(dev)
    out = {"clocks_start": clocks()}
    for comp in ("precompute:update_first", "precompute:aggregate_first"):
        base, order = comp.split(":")
        spec = gc.GcnLayerSpec(K, K, inp["w"].astype(np.float32), composition=base, order=order)
        ts = []
        for _ in range(60):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            gc.gcn_layer(g, h, spec)
            b.record()
            torch.cuda.synchronize()
            ts.append(round(a.elapsed_time(b), 3))
        out[comp] = ts
        out[f"clocks_after_{comp}"] = clocks()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
