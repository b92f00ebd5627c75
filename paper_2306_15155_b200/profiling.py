"""Offline timing harness (SENSEi stage 1) on the GPU: run every layer
composition across graphs and sizes, emit selector training records.

Mirror of ``gnncompose/profiling.py``: same ``ProfileRecord`` NDJSON schema,
same seeded input recipe (``default_rng([seed, crc32(graph_id), k1, k2])``,
h/w/attn_src/attn_dst ~ U(-0.5, 0.5) in that order), same warmup/median/CV
semantics.  Timing uses CUDA events on the launching stream instead of
``perf_counter``; the timed region is exactly one layer forward with its
inputs already on the device.  Out-of-memory configurations are skipped with
a warning, as in the reference.
"""

from __future__ import annotations

import json
import time
import warnings
import zlib
from dataclasses import dataclass
from pathlib import Path

import numpy as np
import torch

from .features import GraphFeatures, extract_features
from .gat import AttentionForm, GatComposition, GatLayerSpec, gat_layer
from .gcn import AggregationOrder, GcnComposition, GcnLayerSpec, NormalizedGraph, gcn_layer
from .selector import B200_COMPOSITIONS
from .sparse import CsrMatrix, add_self_loops, inv_sqrt_degrees

MODEL_TAGS = ("gcn", "gat")


def default_hw_tag() -> str:
    if torch.cuda.is_available():
        p = torch.cuda.get_device_properties(torch.cuda.current_device())
        return f"{p.name.replace(' ', '_')}-{p.multi_processor_count}sm"
    import os
    import platform

    return f"{platform.machine()}-{os.cpu_count()}cpu"


@dataclass
class ProfileRecord:
    """One timed (graph, sizes, composition) observation (profiling.py:39-108)."""

    graph_id: str
    model: str
    k1: int
    k2: int
    composition: str
    features: GraphFeatures
    hw_tag: str
    median_time_s: float
    iterations: int
    setup_time_s: float = 0.0
    cv: float = 0.0
    unreliable: bool = False
    opt_config: object | None = None
    hw_desc: tuple[float, ...] = ()

    def __post_init__(self):
        if self.median_time_s <= 0:
            raise ValueError("median_time_s must be positive")
        if self.iterations < 3:
            raise ValueError("iterations must be >= 3")

    def to_dict(self) -> dict:
        return {
            "graph_id": self.graph_id, "model": self.model, "k1": self.k1, "k2": self.k2,
            "composition": self.composition, "features": self.features.to_dict(),
            "opt_config": self.opt_config if isinstance(self.opt_config, (dict, type(None))) else None,
            "hw_tag": self.hw_tag, "hw_desc": list(self.hw_desc),
            "median_time_s": self.median_time_s, "setup_time_s": self.setup_time_s, "cv": self.cv,
            "iterations": self.iterations, "unreliable": self.unreliable,
        }

    @classmethod
    def from_dict(cls, d: dict) -> "ProfileRecord":
        opt = d.get("opt_config")
        return cls(graph_id=d["graph_id"], model=d["model"], k1=int(d["k1"]), k2=int(d["k2"]),
                   composition=d["composition"], features=GraphFeatures(**d["features"]),
                   hw_tag=d["hw_tag"], median_time_s=float(d["median_time_s"]),
                   iterations=int(d["iterations"]), setup_time_s=float(d.get("setup_time_s", 0.0)),
                   cv=float(d.get("cv", 0.0)), unreliable=bool(d.get("unreliable", False)),
                   opt_config=tuple(opt.values()) if isinstance(opt, dict) else opt,
                   hw_desc=tuple(d.get("hw_desc", ())))


def write_records(path, records: list[ProfileRecord]) -> None:
    with Path(path).open("w") as fh:
        for rec in records:
            fh.write(json.dumps(rec.to_dict()) + "\n")


def read_records(path) -> list[ProfileRecord]:
    out = []
    with Path(path).open() as fh:
        for line in fh:
            line = line.strip()
            if line:
                out.append(ProfileRecord.from_dict(json.loads(line)))
    return out


def config_rng(seed: int, graph_id: str, k1: int, k2: int) -> np.random.Generator:
    """Stable across processes (no salted hash); shared by all compositions of a
    group so they see identical inputs (profiling.py:127-130)."""
    return np.random.default_rng([seed, zlib.crc32(graph_id.encode()), k1, k2])


_config_rng = config_rng


def draw_inputs(rng, n: int, k1: int, k2: int, model: str, activation: str = "relu",
                heads: int = 1) -> dict:
    """h, w, [attn_src, attn_dst] ~ U(-0.5, 0.5) in the reference's order
    (profiling.py:251-259); multi-head draws w as k1 x heads*k2 and the
    attention vectors head after head."""
    h = rng.uniform(-0.5, 0.5, size=(n, k1))
    w = rng.uniform(-0.5, 0.5, size=(k1, k2 * heads))
    inputs = {"h": h, "w": w, "k1": k1, "k2": k2}
    if model == "gat":
        inputs["attn_src"] = rng.uniform(-0.5, 0.5, size=k2 * heads)
        inputs["attn_dst"] = rng.uniform(-0.5, 0.5, size=k2 * heads)
        inputs["activation"] = activation
    return inputs


_draw_inputs = draw_inputs


def time_iterations(run, warmup: int, reps: int) -> tuple[float, float]:
    """Warm up, then time ``reps`` runs with CUDA events; returns (median s, CV)."""
    for _ in range(warmup):
        run()
    stream = torch.cuda.current_stream()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(reps)]
    torch.cuda.synchronize()
    for a, b in ev:
        a.record(stream)
        run()
        b.record(stream)
    torch.cuda.synchronize()
    times = np.array([a.elapsed_time(b) * 1e-3 for a, b in ev])
    med = float(np.median(times))
    mean = float(times.mean())
    return med, (float(times.std() / mean) if mean > 0 else 0.0)


def split_composition(model: str, comp: str) -> tuple[str, str | None]:
    if ":" in comp:
        a, b = comp.split(":", 1)
        return a, b
    return comp, None


def make_runner(model: str, comp: str, graph, inputs: dict, heads: int = 1):
    """A zero-argument callable running one layer forward of ``comp`` on
    device-resident inputs."""
    base, variant = split_composition(model, comp)
    dev = graph.a_tilde.device if model == "gcn" else graph.device
    h = torch.as_tensor(inputs["h"], dtype=torch.float32, device=dev)
    if model == "gcn":
        spec = GcnLayerSpec(inputs["k1"], inputs["k2"],
                            torch.as_tensor(inputs["w"], dtype=torch.float32, device=dev),
                            composition=GcnComposition(base),
                            order=AggregationOrder(variant) if variant else None)
        if spec.composition is GcnComposition.PRECOMPUTE:
            graph.with_precomputed()
        return lambda: gcn_layer(graph, h, spec)
    spec = GatLayerSpec(inputs["k1"], inputs["k2"],
                        torch.as_tensor(inputs["w"], dtype=torch.float32, device=dev),
                        inputs["attn_src"], inputs["attn_dst"], composition=GatComposition(base),
                        activation=inputs.get("activation", "relu"), heads=heads,
                        attention=AttentionForm(variant) if variant else AttentionForm.REASSOC)
    return lambda: gat_layer(graph, h, spec)


def profile(graphs: list[tuple[str, CsrMatrix]], sizes: list[tuple[int, int]], model: str,
            reps: int = 10, *, warmup: int = 3, seed: int = 0, amortize_precompute: bool = True,
            hw_tag: str | None = None, hw_desc: tuple[float, ...] = (),
            compositions: tuple[str, ...] | None = None, activation: str = "relu",
            heads: int = 1) -> list[ProfileRecord]:
    """Time every (graph, size, composition); one record per combination
    (profiling.py:147-217).  Default compositions: the B200 set."""
    if model not in MODEL_TAGS:
        raise ValueError(f"unknown model {model!r}")
    if reps < 3:
        raise ValueError("reps must be >= 3")
    hw_tag = hw_tag if hw_tag is not None else default_hw_tag()
    comps = compositions or B200_COMPOSITIONS[model]
    records: list[ProfileRecord] = []
    for graph_id, a in graphs:
        feats = extract_features(a)
        a_tilde = add_self_loops(a)
        setup_s = 0.0
        if model == "gcn":
            graph = NormalizedGraph(a_tilde=a_tilde, d_inv_sqrt=inv_sqrt_degrees(a_tilde))
            if any(c.startswith("precompute") for c in comps):
                s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s0.record()
                graph.with_precomputed()
                s1.record()
                torch.cuda.synchronize()
                setup_s = s0.elapsed_time(s1) * 1e-3
        else:
            graph = a_tilde
        for k1, k2 in sizes:
            rng = config_rng(seed, graph_id, k1, k2)
            inputs = draw_inputs(rng, a.n_rows, k1, k2, model, activation, heads)
            for comp in comps:
                try:
                    run = make_runner(model, comp, graph, inputs, heads)
                    # first call: plan builds and the kernel-variant / dense-split
                    # autotuners run once per (pattern, K); their cost beyond a
                    # steady-state call is setup, reported in setup_time_s
                    torch.cuda.synchronize()
                    t0 = time.perf_counter()
                    run()
                    torch.cuda.synchronize()
                    first_s = time.perf_counter() - t0
                    med, cv = time_iterations(run, warmup, reps)
                except torch.cuda.OutOfMemoryError:
                    warnings.warn(f"{graph_id} {k1}x{k2} {comp}: skipped (out of memory)")
                    torch.cuda.empty_cache()
                    continue
                su = (setup_s if comp.startswith("precompute") else 0.0) + max(first_s - med, 0.0)
                if not amortize_precompute and su:
                    med += su / reps
                # multi-head GAT: the record's k2 is the layer's output width
                # heads*k2 (what a selector sees for a multi-head layer), and
                # the group id carries the head count
                records.append(ProfileRecord(graph_id=graph_id if heads == 1 else
                                             f"{graph_id}/h{heads}", model=model, k1=k1,
                                             k2=k2 * heads,
                                             composition=comp, features=feats, hw_tag=hw_tag,
                                             median_time_s=med, iterations=reps, setup_time_s=su,
                                             cv=cv, unreliable=cv > 0.3, hw_desc=tuple(hw_desc)))
    return records
