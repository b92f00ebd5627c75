"""CUDA-graph capture of layer stacks (launch-latency-bound small graphs).

A Cora-sized 2-layer GCN is a handful of microsecond kernels; host-side
Python + ctypes launch overhead dominates eager execution.  ``GraphedForward``
captures the whole forward once (our kernels are launched on the current
stream, so they record into the graph like any CUDA work) and replays it with
one ``cudaGraphLaunch``.  Inputs are copied into static buffers; the output
buffer is reused across replays.
"""

from __future__ import annotations

from typing import Callable

import torch


class GraphedForward:
    def __init__(self, fn: Callable[..., torch.Tensor], *example_inputs: torch.Tensor,
                 warmup: int = 2):
        if not all(isinstance(x, torch.Tensor) and x.is_cuda for x in example_inputs):
            raise ValueError("graph capture needs CUDA tensor inputs")
        self.inputs = [x.clone() for x in example_inputs]
        cur = torch.cuda.current_stream()
        side = torch.cuda.Stream()
        side.wait_stream(cur)
        with torch.cuda.stream(side):  # warm-up: plans, caches, lazy library load
            for _ in range(warmup):
                fn(*self.inputs)
        cur.wait_stream(side)
        torch.cuda.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self.output = fn(*self.inputs)

    def __call__(self, *inputs: torch.Tensor) -> torch.Tensor:
        for dst, src in zip(self.inputs, inputs):
            if src is not dst:
                dst.copy_(src, non_blocking=True)
        self.graph.replay()
        return self.output
