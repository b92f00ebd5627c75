#!/usr/bin/env python
"""Benchmark: one GCN layer on the Reddit-shaped power-law graph (BASELINE.json
configs[1]) through the B200 composition engine.

A "step" is one forward pass of the selected GCN layer composition over the
whole graph (n = 232,965, nnz(A) = 114,615,892, m = nnz(Ã) = nnz(A) + n) at
k1 = k2 = K (default 256), inputs resident in HBM.  ``value`` is whole-job
edges/s = m / step time, in the TF32 numerics class (parity 1e-2);
``fp32_class`` times the same step in the fp32 class (3xTF32 GEMM, two-term
dense operand; parity 1e-4).  ``e2e`` is the same layer through the public
API with HOST (pinned) H in and the host result out, copies inside the timed
region.  ``sweep`` times every composition at K in {32..1024}; ``roofline``
is the dominant kernel against measured HBM bandwidth; every timed row
carries its row-sampled parity against the CPU oracle (``rel_err`` <=
``tol``).  ``cpu_baseline`` is the CPU oracle (the reference's algorithm,
float64, numba-equivalent C/OpenMP + OpenBLAS, calibrated against the
reference itself: profiles/data/cpu_calibration.json) on the FULL graph.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 (torchrun, one rank per GPU, NCCL): rank 0 writes Ã as a .gcsr file and
every rank reads only its nnz-balanced row block (the capacity path); each
step is the partitioned layer with its one all-gather per layer; the time is
the max over ranks (strong scaling of the same graph).  ``partitioned``
adds BASELINE configs[3]: GCN + GAT on the products shape, row-partitioned.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

BASELINE = json.loads((ROOT / "BASELINE.json").read_text())
METRIC = BASELINE["metric"]
UNIT = "edges/s"
KSWEEP = (32, 64, 128, 256, 512, 1024)


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=("ours", "reference"), default="ours")
    p.add_argument("--shape", default="reddit")
    p.add_argument("--k", type=int, default=256)
    p.add_argument("--composition", default="auto",
                   help="auto (selector) or '<precompute|dynamic>:<aggregate_first|update_first>'")
    p.add_argument("--no-sweep", action="store_true")
    p.add_argument("--sweep-ks", default=",".join(map(str, KSWEEP)))
    p.add_argument("--sweep-reps", type=int, default=5)
    p.add_argument("--cpu-ks", default="32,256,1024",
                   help="K values of the full-graph CPU-oracle baseline")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--no-fp32-class", action="store_true")
    p.add_argument("--no-extra", action="store_true",
                   help="skip the Cora / GAT-on-arxiv / products configs (BASELINE configs[0], [2], [3])")
    p.add_argument("--parity-rows", type=int, default=128,
                   help="random rows (plus the heaviest row) per row-sampled oracle check")
    p.add_argument("--backend", default="nccl", help="process-group backend for N > 1")
    p.add_argument("--no-overlap", action="store_true",
                   help="N > 1: all-gather, then SpMM (default: owned-column edges overlap the gather)")
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--out", default=None, help="also write the JSON line to this file")
    return p.parse_args()


# ---------------------------------------------------------------------------
# helpers
# ---------------------------------------------------------------------------


def peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": float(d["hbm_gbs"]), "bf16_tflops": float(d["bf16_tflops"]),
                "source": "measured (MEASURED_PEAKS.json)"}
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "source": "fallback (B200_PROFILING.md)"}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 50 ms around and
    during the timed region (the profiling recipe's clocks line).  The first
    sample is taken before the region starts and one more after it ends, so a
    region shorter than the sampling period is still bracketed."""

    Q = ("index,clocks.sm,clocks.max.sm,utilization.gpu,power.draw,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[tuple[float, str]] = []
        self.t0 = self.t1 = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            deadline = time.time() + 3.0
            while not self.lines and time.time() < deadline:
                time.sleep(0.01)
        except (FileNotFoundError, OSError):
            self.proc = None
        self.t0 = time.time()
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def __exit__(self, *exc):
        self.t1 = time.time()
        if self.proc is not None:
            n = len(self.lines)
            deadline = time.time() + 1.0
            while len(self.lines) <= n and time.time() < deadline:
                time.sleep(0.01)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        rows = []
        inside = 0
        for ts, ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                rows.append((float(f[1]), float(f[2]), float(f[3]), f[5:9], ts))
            except ValueError:
                continue
            if self.t0 is not None and self.t1 is not None and self.t0 <= ts <= self.t1:
                inside += 1
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        # samples inside the region plus the ones bracketing it
        lo = max([r for r in rows if r[4] < (self.t0 or 0)], key=lambda r: r[4], default=None)
        hi = min([r for r in rows if r[4] > (self.t1 or 0)], key=lambda r: r[4], default=None)
        win = [r for r in rows if self.t0 <= r[4] <= self.t1] + [r for r in (lo, hi) if r is not None]
        win = win or rows
        load = [r for r in win if r[2] >= 50] or win
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = sorted({names[i] for r in load for i, v in enumerate(r[3]) if v == "Active"})
        return {"sm_mhz": float(np.median([r[0] for r in load])), "sm_max_mhz": rows[0][1],
                "reasons": reasons, "samples": len(win), "samples_inside_region": inside,
                "samples_under_load": len(load), "interval_ms": 50}


def spmm_alg_bytes(n_rows: int, m: int, K: int, weighted: bool, dcol: bool, drow: bool,
                   half: bool = False) -> int:
    """Edge-gather model of SURVEY.md §8(d): row_ptr + col_idx + (values) +
    (d_j gathers) + one K-row of B per edge + the output (+ d_i).  ``half``:
    the TF32 class's fp16 rows — 2K bytes per gathered row plus its 4-byte
    scale (which carries d_j)."""
    b = 4 * (n_rows + 1) + 4 * m + (2 if half else 4) * m * K + 4 * n_rows * K
    b += 4 * m if weighted else 0
    b += 4 * m if (dcol or half) else 0
    b += 4 * n_rows if drow else 0
    return b


def uses_half(gc, n_cols: int, K: int) -> bool:
    """Whether the TF32 class gathers fp16 rows for an n_cols x K operand
    (gcn.half_gather's rule)."""
    from paper_2306_15155_b200 import gcn

    return (gcn.HALF_GATHER and gc.get_gemm_precision() == "tf32" and K % 8 == 0
            and n_cols * K * 4 > gcn.HALF_MIN_BYTES)


def layer_flops(n: int, m: int, k1: int, k2: int, order: str) -> int:
    k_agg = k1 if order == "aggregate_first" else k2
    return 2 * m * k_agg + 2 * n * k1 * k2


def choose_composition(arg: str, feats, k1: int, k2: int) -> tuple[str, str]:
    if arg != "auto":
        return arg, "forced"
    from paper_2306_15155_b200 import selector

    model = selector.load_b200_model("gcn")
    if model is not None:
        inp = selector.SelectorInput(features=feats, k1=k1, k2=k2)
        return selector.select(model, inp), "selector (B200-trained)"
    from paper_2306_15155_b200.gcn import ordering_heuristic

    return f"dynamic:{ordering_heuristic(k1, k2).value}", "reference default (dynamic + heuristic)"


# ---------------------------------------------------------------------------
# CPU oracle (cpu_baseline leg and the --impl reference arm) and parity checks
# ---------------------------------------------------------------------------


def cpu_oracle_layer(orc, at, d, h, w):
    """The reference default for k1 == k2 on the FULL graph: dynamic
    composition, heuristic order (aggregate first) — gcn.py:137-155:
    relu(D ((Ã (D H)) W)) with the oracle's float64 kernels."""
    order = orc.ordering_heuristic(w.shape[0], w.shape[1])
    scaled = orc.scale_rows(d, h)
    agg = orc.spmm_unweighted if at.has_unit_values else orc.spmm
    if order == orc.UPDATE_FIRST:
        out = agg(at, orc.gemm(scaled, w))
    else:
        out = orc.gemm(agg(at, scaled), w)
    return np.maximum(orc.scale_rows(d, out), 0.0)


def time_cpu(fn, warmup: int, reps: int) -> float:
    for _ in range(warmup):
        fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return float(np.median(ts))


def host_graph(A_dev):
    """Reference-dtype host copy (int64 / float64) of a device CSR."""
    from oracle import gnn_oracle as orc

    rp, ci, v = A_dev.numpy()
    return orc.Csr(A_dev.n_rows, A_dev.n_cols, rp, ci, v)


def cpu_model() -> str:
    try:
        for ln in Path("/proc/cpuinfo").read_text().splitlines():
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def calibration() -> dict | None:
    """The port-vs-reference factor measured in the build container
    (profiles/probes/calibrate_cpu.py): same graphs, inputs and threads, the
    reference's numba kernels vs the oracle's C port."""
    p = ROOT / "profiles" / "data" / "cpu_calibration.json"
    if not p.exists():
        return None
    d = json.loads(p.read_text())
    return {"source": "profiles/data/cpu_calibration.json", "threads": d.get("threads"),
            "rows": [{k: r[k] for k in ("shape", "K", "reference_s", "port_s",
                                        "port_over_reference", "max_abs_diff")}
                     for r in d.get("rows", [])]}


class Parity:
    """Row-sampled oracle checks at full size (oracle/sampled.py, SURVEY.md
    §8(c) step 5): the reference layer on ``count`` random rows plus the
    heaviest row of the host copy of Ã (bit-exact with the oracle's graph
    prep: tests/test_gpu_baseline_configs.py), operand rows fetched only where
    the oracle needs them."""

    def __init__(self, a_tilde_dev, count: int, seed: int = 0):
        from oracle import gnn_oracle as orc
        from oracle import sampled

        self.orc, self.so = orc, sampled
        self.at = host_graph(a_tilde_dev)
        self.d = orc.inv_sqrt_degrees(self.at)
        deg = np.diff(self.at.row_ptr)
        self.rows = sampled.sample_rows(self.at.n_rows, count, seed, heavy=np.argsort(deg)[-1:])

    def _fetch(self, x):
        import torch

        return lambda idx: x[torch.from_numpy(idx).to(x.device)].double().cpu().numpy()

    def _got(self, out):
        import torch

        return out[torch.from_numpy(self.rows).to(out.device)].double().cpu().numpy()

    def gcn(self, out, h, w, comp: str, tol: float) -> dict:
        base, order = comp.split(":")
        ref = self.so.gcn_rows(self.at, self.d, self._fetch(h), w.double().cpu().numpy(), self.rows,
                               base, order)
        err = self.orc.rel_err(self._got(out), ref)
        return {"rel_err": err, "tol": tol, "ok": bool(err <= tol), "rows_checked": int(self.rows.size)}

    def gat(self, out, h, w, a_s, a_d, heads: int, comp: str, tol: float) -> dict:
        base = comp.split(":")[0]
        ref = self.so.gat_rows(self.at, self._fetch(h), w.double().cpu().numpy(),
                               a_s.double().cpu().numpy(), a_d.double().cpu().numpy(), heads,
                               self.rows, base)
        err = self.orc.rel_err(self._got(out), ref)
        return {"rel_err": err, "tol": tol, "ok": bool(err <= tol), "rows_checked": int(self.rows.size)}


def tol_of(gc) -> float:
    return 1e-2 if gc.get_gemm_precision() == "tf32" else 1e-4


def _dram_side(traffic, kernel_ms, pk, alg_bytes) -> dict:
    """The DRAM-side rate of a gather kernel: its ncu-measured DRAM bytes per
    launch over the live launch time.  The algorithmic model counts every
    K-wide row gather; most of those hit the 126 MB L2, so ``frac`` (model
    bytes / HBM peak) can exceed 1 while the DRAM side stays below peak."""
    if not traffic or not kernel_ms:
        return {}
    gbs = traffic / (kernel_ms * 1e-3) / 1e9
    return {"dram_gbs": round(gbs, 1), "dram_frac": round(gbs / pk["hbm_gbs"], 3),
            "dram_over_model": round(traffic / alg_bytes, 3)}


def e2e(gc, g, spec, h_host32, args, m, n, K) -> dict:
    """Same layer through the public API with a pinned HOST H in and the
    pinned host result out; the H2D and D2H are inside the timed region
    (the API overlaps the D2H of finished row blocks with the next block)."""
    import torch

    h_pin = torch.from_numpy(h_host32).pin_memory()
    for _ in range(max(args.warmup, 2)):
        res = gc.gcn_layer(g, h_pin, spec)
    torch.cuda.synchronize()
    ts = []
    t_all = time.perf_counter()
    for _ in range(args.steps):
        t0 = time.perf_counter()
        res = gc.gcn_layer(g, h_pin, spec)  # returns only after the D2H completed
        ts.append(time.perf_counter() - t0)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t_all) / args.steps
    # raw link speed for context
    dev_buf = torch.empty_like(h_pin, device="cuda")
    c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    c0.record()
    dev_buf.copy_(h_pin, non_blocking=True)
    c1.record()
    torch.cuda.synchronize()
    h2d_ms = c0.elapsed_time(c1)
    return {"value": round(m / dt, 1), "unit": UNIT, "ms_per_step": round(dt * 1e3, 3),
            "ms_per_step_median": round(float(np.median(ts)) * 1e3, 3),
            "h2d_bytes_per_step": int(h_pin.numel() * 4), "d2h_bytes_per_step": int(res.numel() * 4),
            "raw_h2d_ms": round(h2d_ms, 3),
            "api": "paper_2306_15155_b200.gcn_layer(NormalizedGraph, pinned host H, spec)"}


# ---------------------------------------------------------------------------
# main
# ---------------------------------------------------------------------------


def _events():
    import torch

    return torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def load_partition(args, rank: int, world: int, dev, shape: str):
    """The capacity path: rank 0 generates the graph, adds self loops and
    writes Ã as .gcsr; every rank then reads only its nnz-balanced row block
    (RowPartition.from_file) and the O(n) row_ptr for D^-1/2.  Returns
    (partition, full D^-1/2, raw-graph features, m, prep seconds)."""
    import torch
    import torch.distributed as dist

    import paper_2306_15155_b200 as gc
    from paper_2306_15155_b200 import graphs
    from paper_2306_15155_b200.distributed import RowPartition

    obj = [None, None]
    if rank == 0:
        A = graphs.shape_graph(shape, seed=args.seed, device=dev)
        feats = gc.extract_features(A)
        at = gc.add_self_loops(A)
        del A
        path = f"/tmp/gnnc_{shape}_s{args.seed}_p{os.getpid()}.gcsr"
        at.save(path)
        obj = [path, feats]
        del at
        torch.cuda.empty_cache()
    dist.broadcast_object_list(obj, src=0)
    path, feats = obj
    t0 = time.perf_counter()
    part, d = RowPartition.from_file(path, rank, world, device=dev)
    torch.cuda.synchronize()
    prep_s = time.perf_counter() - t0
    m = int(gc.CsrMatrix.read_row_ptr(path)[-1])
    dist.barrier()
    if rank == 0:
        os.unlink(path)
    return part, d, feats, m, prep_s


def normalized_block(part, d):
    """Ñ's values on this rank's block: d_i d_j over the rows it owns (setup)."""
    loc = part.local
    rows = loc.row_of_nnz() + part.lo
    nt = loc.with_values(d[rows] * d[loc.col_idx.long()])
    nt._unit = False
    return nt


def main():
    args = parse()
    import torch
    import torch.distributed as dist

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)

    local = local % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if args.backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:  # e.g. gloo: lets the N > 1 path be exercised with several ranks on one GPU
            dist.init_process_group(args.backend)

    import paper_2306_15155_b200 as gc
    from paper_2306_15155_b200 import _native, graphs, hub, profiling, sparse
    from paper_2306_15155_b200.distributed import RowPartition, dist_gcn_layer

    _native.load()
    shape = graphs.SHAPES[args.shape]
    K = args.k
    setup: dict = {}
    part = None
    if world > 1:
        part, d_full, feats, m, prep_s = load_partition(args, rank, world, dev, args.shape)
        n = int(part.bounds[-1])
        setup.update({"partition_load_s": round(prep_s, 3), "rows_local": part.rows,
                      "edges_local": part.local.nnz})
    else:
        t0 = time.perf_counter()
        A = graphs.shape_graph(args.shape, seed=args.seed, device=dev)
        torch.cuda.synchronize()
        setup["graph_gen_s"] = round(time.perf_counter() - t0, 2)
        t0 = time.perf_counter()
        feats = gc.extract_features(A)
        setup["features_s"] = round(time.perf_counter() - t0, 4)
        t0 = time.perf_counter()
        g = gc.NormalizedGraph.from_adjacency(A)
        torch.cuda.synchronize()
        setup["prep_s"] = round(time.perf_counter() - t0, 3)
        g.with_precomputed()  # first call allocates Ñ's values
        e0, e1 = _events()
        e0.record()
        gc.precompute_normalized(g)
        e1.record()
        torch.cuda.synchronize()
        setup["normalize_sddmm_ms"] = round(e0.elapsed_time(e1), 3)
        del A
        n, m = g.a_tilde.n_rows, g.a_tilde.nnz
    t0 = time.perf_counter()
    comp, selected_by = choose_composition(args.composition, feats, K, K)
    setup["select_s"] = round(time.perf_counter() - t0, 4)
    base, order = comp.split(":")
    dyn = base == "dynamic"

    rng = profiling.config_rng(args.seed, args.shape, K, K)
    inp = profiling.draw_inputs(rng, n, K, K, "gcn")
    h_host32 = inp["h"].astype(np.float32)
    w_dev = torch.from_numpy(inp["w"].astype(np.float32)).to(dev)
    spec = gc.GcnLayerSpec(K, K, w_dev, composition=base, order=order)

    if part is not None:
        if not dyn:
            part.local = normalized_block(part, d_full)
        h_dev = torch.from_numpy(h_host32[part.lo:part.hi]).to(dev)

        def step():
            return dist_gcn_layer(part, h_dev, w_dev, composition=base, order=order,
                                  d=d_full, overlap=not args.no_overlap, hub_unit=True)
    else:
        h_dev = torch.from_numpy(h_host32).to(dev)

        def step():
            return gc.gcn_layer(g, h_dev, spec)

    def barrier():
        if world > 1:
            dist.barrier()

    # ---- first call (plans + autotuners), warmup, timed region --------------
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    step()
    torch.cuda.synchronize()
    first_call_s = time.perf_counter() - t0
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    launches0 = _native.launch_count()
    t_start, t_end = _events()
    with ClockSampler(local) as clocks, \
            sparse.kernel_timing("spmm", "gemm", "hub_gemm", "spmm_tail") as kt:
        # cudaProfilerStart/Stop bracket the timed region so that
        # `ncu --profile-from-start off` captures exactly its launches
        torch.cuda.profiler.start()
        t_start.record()
        for _ in range(args.steps):
            out = step()
        t_end.record()
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
        barrier()
        torch.cuda.synchronize()
    launches = _native.launch_count() - launches0
    ms = t_start.elapsed_time(t_end) / args.steps
    if world > 1:
        tt = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())

    def kms(name):
        v = kt.durations_ms(name)
        return float(np.mean(v)) if v else None

    spmm_ms, gemm_ms = kms("spmm"), kms("gemm")
    hub_ms, tail_ms = kms("hub_gemm"), kms("spmm_tail")
    value = m / (ms * 1e-3)

    # ---- roofline of the dominant kernel -------------------------------------
    pk = peaks()
    a_used = part.padded() if part is not None else (g.a_tilde if dyn else g.n_tilde)
    weighted = not dyn
    skey = hub.split_key(K, not dyn)
    pat = a_used if part is not None else g.a_tilde
    split = pat._plans.get(skey, 0)
    roof, hub_roof = None, None
    if split and tail_ms:
        # hybrid aggregation: the tail SpMM is the dominant kernel (HBM/L2
        # roofline over its own edges, + the read-modify-write of C); the
        # dense part is a tensor-core GEMM
        plan = hub.hub_plan(pat, split)
        mt = plan.tail.nnz
        nr = pat.n_rows
        half = uses_half(gc, pat.n_cols, K)
        tail_bytes = spmm_alg_bytes(nr, mt, K, weighted, dyn, dyn, half) + 4 * nr * K
        ach = tail_bytes / (tail_ms * 1e-3) / 1e9
        traffic = traffic_lookup(f"{args.shape}/K{K}/{comp}/tail/{hub.spec_label(split)}", world)
        roof = {"kernel": "spmm_kernel (tail of the dense split)", "bound": "hbm",
                "achieved": round(ach, 1), "peak": pk["hbm_gbs"], "unit": "GB/s",
                "frac": round(ach / pk["hbm_gbs"], 3), "traffic": traffic,
                "alg_bytes_per_launch": tail_bytes, "kernel_ms": round(tail_ms, 4),
                "share_of_step": round(tail_ms / ms, 3), "peak_source": pk["source"],
                "model": "edge-gather over the tail edges: 4(n+1)+4m_t[+4m_t values][+4m_t d_j]"
                         "+4m_tK (2m_tK + 4m_t scales with fp16 rows)+4nK(+4nK C read)[+4n]; "
                         "frac > 1 = gathered rows served by L2",
                "fp16_rows": half,
                "tail_edges": mt}
        roof.update(_dram_side(traffic, tail_ms, pk, tail_bytes))
        roof["l2_side"] = l2_lookup(f"{args.shape}/K{K}/{comp}/tail/{hub.spec_label(split)}",
                                    world, tail_ms)
        cell_flops = 2 * plan.cells * K * hub.term_count()
        useful = 2 * plan.hub_edges * K
        tf = cell_flops / (hub_ms * 1e-3) / 1e12
        blk = plan.cells * (0.125 if getattr(plan, "abits", False) else 2)
        hub_roof = {"kernel": "gemm_hub_pair_tcgen05 (dense part)", "bound": "tensor",
                    "achieved": round(tf, 1), "peak": pk["bf16_tflops"], "unit": "TFLOP/s",
                    "frac": round(tf / pk["bf16_tflops"], 3), "kernel_ms": round(hub_ms, 4),
                    "share_of_step": round(hub_ms / ms, 3), "split": hub.spec_label(split),
                    "dense_cells": plan.cells, "dense_edges": plan.hub_edges,
                    "cell_flops_per_launch": cell_flops, "useful_flops_per_launch": useful,
                    "useful_tflops": round(useful / (hub_ms * 1e-3) / 1e12, 1),
                    "cell_density": round(plan.hub_edges / plan.cells, 4),
                    "steps": getattr(plan, "steps", None),
                    "terms": hub.FORMAT_NAMES[hub.term_format()],
                    "block_bytes": int(blk),
                    "block_hbm_frac": round(blk / (hub_ms * 1e-3) / 1e9 / pk["hbm_gbs"], 3),
                    "model": "cell flops 2·cells·K per 16-bit term (f16: 1 term, TF32-equivalent "
                             "11-bit rounding of D·X; f16x2: 2 terms); useful flops 2·edges·K"}
    elif spmm_ms:
        spmm_bytes = spmm_alg_bytes(a_used.n_rows, a_used.nnz, K, weighted, dyn, dyn,
                                    uses_half(gc, a_used.n_cols, K))
        ach = spmm_bytes / (spmm_ms * 1e-3) / 1e9
        traffic = traffic_lookup(f"{args.shape}/K{K}/{comp}", world)
        roof = {"kernel": "spmm_kernel", "bound": "hbm", "achieved": round(ach, 1),
                "peak": pk["hbm_gbs"], "unit": "GB/s", "frac": round(ach / pk["hbm_gbs"], 3),
                "traffic": traffic, "alg_bytes_per_launch": spmm_bytes,
                "kernel_ms": round(spmm_ms, 4), "share_of_step": round(spmm_ms / ms, 3),
                "peak_source": pk["source"],
                "model": "edge-gather: 4(n+1)+4m[+4m values][+4m d_j]+4mK+4nK[+4n]"}
        roof.update(_dram_side(traffic, spmm_ms, pk, spmm_bytes))
    stats = pat._plans.get(skey + ("stats",), {})
    layer_s = ms * 1e-3
    setup.update({"first_call_s": round(first_call_s, 3),
                  "dense_split_plan_build_s": stats.get("plan_build_s"),
                  "dense_split_autotune_s": stats.get("autotune_s"),
                  "dense_split_peak_extra_bytes": stats.get("peak_extra_bytes"),
                  "dense_split_resident_bytes": stats.get("resident_plan_bytes"),
                  })
    sel_s = (setup.get("features_s") or 0.0) + setup["select_s"] + (stats.get("autotune_s") or 0.0)
    setup["selection_overhead_iterations"] = round(sel_s / layer_s, 1)
    setup["selection_overhead_note"] = ("(features + selector inference + dense-split autotune) / "
                                        "layer time, as the reference's cli.py:257-258")
    result = {
        "metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "tf32" if gc.get_gemm_precision() == "tf32" else "f32",
        "data": f"synthetic {shape.kind.upper()} graph, {args.shape}-shaped (n={n}, "
                f"nnz(A)={shape.nnz}); H,W ~ U(-0.5,0.5) by the reference recipe",
        "config": {"workload": f"gcn_layer/{args.shape}/k1=k2={K}", "shape": args.shape, "n": n,
                   "nnz_A": shape.nnz, "m_tilde": m, "K": K, "composition": comp,
                   "selected_by": selected_by, "gemm_precision": gc.get_gemm_precision(),
                   "numerics": ("TF32 class (parity tol 1e-2): fp32 storage and accumulation; the "
                                "update GEMM rounds its inputs to TF32 and the dense part of the "
                                "aggregation rounds D*X to one fp16 term (the same 11-bit input "
                                "rounding); the SpMM tail gathers fp16 rows with per-row "
                                "power-of-two scales (operands above 64 MiB; the same 11-bit "
                                "rounding).  The fp32 class (tol 1e-4) is timed in 'fp32_class'.")
                   if gc.get_gemm_precision() == "tf32" else
                   "fp32 class: 3xTF32 GEMM, two-term fp16 dense aggregation operand; tol 1e-4",
                   "l2": "inputs larger than L2 (CSR 0.9 GB, H 0.24 GB at K=256); no flush",
                   "parallelism": (f"row-partition x{world} (capacity path: each rank reads its "
                                   f"rows of the .gcsr file), 1 all-gather/layer"
                                   f"{'' if args.no_overlap else ' overlapped with the owned-column SpMM'}")
                   if world > 1 else "single GPU"},
        "gpu_launches": int(launches),
        "kernel_ms": {"aggregation": spmm_ms, "gemm": gemm_ms, "hub_gemm": hub_ms,
                      "spmm_tail": tail_ms},
        "roofline": roof,
        "roofline_hub_gemm": hub_roof,
        "dense_split": {"chosen": hub.spec_label(split), "terms": hub.FORMAT_NAMES[hub.term_format()],
                        "autotune_ms": pat._plans.get(skey + ("times",))},
        "setup": setup,
    }
    result["clocks"] = clocks.summary()
    vmode = "spmmh" if uses_half(gc, pat.n_cols, K) else "spmm"
    tail_pat = hub.hub_plan(pat, split).tail if split else pat
    result["spmm_variant"] = {"mode": vmode, "chosen": tail_pat._plans.get(("variant", vmode, K)),
                              "autotune_ms": tail_pat._plans.get(("variant", vmode, K, "times"))}

    if rank == 0 and world == 1:
        parity = Parity(g.a_tilde, args.parity_rows, seed=args.seed)
        # ---- parity of the timed step on sampled rows vs the oracle -----------
        result["parity"] = parity.gcn(out, h_dev, w_dev, comp, tol_of(gc))
        # ---- e2e through the public API with host buffers ----------------------
        result["e2e"] = e2e(gc, g, spec, h_host32, args, m, n, K)
        # ---- the same step in the fp32 numerics class ------------------------------
        if not args.no_fp32_class:
            result["fp32_class"] = fp32_class(gc, g, spec, h_dev, w_dev, comp, args, m, parity)
        # ---- composition sweep ---------------------------------------------------
        if not args.no_sweep:
            result["sweep"] = sweep(gc, g, feats, args, dev, pk, parity)
            if not args.no_extra:  # GAT on the same Reddit shape (selector check)
                result["gat_reddit"] = gat_rows_reddit(gc, g.a_tilde, feats, 256, parity,
                                                       tol_of(gc), dev, selector_pick, timed_runs)
                result["epoch_reddit"] = epoch_row(gc, g, feats, "reddit", parity, tol_of(gc), dev)
        del parity
        if not args.no_extra:
            result["extra_configs"] = extra_configs(gc, args, dev, pk)
        # ---- CPU baseline: the oracle on the full graph ----------------------------
        if not args.no_cpu:
            result["cpu_baseline"] = cpu_baseline(g, args)
    if world > 1 and not args.no_extra:
        res = partitioned_products(args, rank, world, dev)
        if rank == 0:
            result["partitioned"] = res
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        line = json.dumps(result)
        print(line, flush=True)
        if args.out:
            Path(args.out).write_text(line + "\n")


def traffic_lookup(key: str, world: int):
    """ncu-measured DRAM bytes per launch of the dominant kernel for this
    exact configuration (profiles/traffic.json, written from a --set full
    capture of the same build), else None."""
    tf = ROOT / "profiles" / "traffic.json"
    if world != 1 or not tf.exists():
        return None
    v = json.loads(tf.read_text()).get(key)
    return v if isinstance(v, int) else None


def l2_lookup(key: str, world: int, kernel_ms: float | None):
    """The L2 side of the dominant kernel (the roof a gather served from L2
    meets before HBM): bytes through the L2 slices per launch from the ncu
    --set full capture of the same configuration, the rate they imply at
    the live kernel time, and ncu's L2 / L1 throughput fractions."""
    tf = ROOT / "profiles" / "traffic.json"
    if world != 1 or not tf.exists() or not kernel_ms:
        return None
    v = json.loads(tf.read_text()).get(key + "/l2")
    if not isinstance(v, dict):
        return None
    return dict(v, l2_gbs_live=round(v["l2_bytes"] / (kernel_ms * 1e-3) / 1e9, 1))


def fp32_class(gc, g, spec, h_dev, w_dev, comp, args, m, parity) -> dict:
    """The headline step in the fp32 numerics class: 3xTF32 tcgen05 GEMM and
    the two-term fp16 dense operand (its own dense-split choice); tol 1e-4."""
    import torch

    from paper_2306_15155_b200 import _native

    old = gc.get_gemm_precision()
    gc.set_gemm_precision("fp32")
    try:
        for _ in range(max(args.warmup, 1) + 1):
            out = gc.gcn_layer(g, h_dev, spec)
        torch.cuda.synchronize()
        l0 = _native.launch_count()
        e0, e1 = _events()
        e0.record()
        for _ in range(args.steps):
            out = gc.gcn_layer(g, h_dev, spec)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.steps
        launches = _native.launch_count() - l0
        from paper_2306_15155_b200 import hub

        split = g.a_tilde._plans.get(hub.split_key(args.k, spec.composition.value == "precompute"), 0)
        res = {"value": round(m / (ms * 1e-3), 1), "unit": UNIT, "ms_per_step": round(ms, 4),
               "dtype": "f32", "gemm": "3xTF32 tcgen05 (gemm_tf32x3_tcgen05)",
               "dense_split": hub.spec_label(split), "terms": hub.FORMAT_NAMES[hub.term_format()],
               "gpu_launches": int(launches)}
        res["parity"] = parity.gcn(out, h_dev, w_dev, comp, 1e-4)
        return res
    finally:
        gc.set_gemm_precision(old)


def sweep(gc, g, feats, args, dev, pk, parity) -> list[dict]:
    """BASELINE configs[1]: every GCN composition at K in {32..1024} on the
    Reddit shape (interleaved timing rounds, median), each with its
    row-sampled parity, and the selector's pick over the fastest."""
    import torch

    from paper_2306_15155_b200 import profiling, selector, sparse

    model = selector.load_b200_model("gcn")
    n, m = g.a_tilde.n_rows, g.a_tilde.nnz
    rows = []
    for K in [int(k) for k in args.sweep_ks.split(",") if k]:
        gen = torch.Generator(device=dev)
        gen.manual_seed(K)
        h = torch.rand(n, K, device=dev, generator=gen) - 0.5
        w = torch.rand(K, K, device=dev, generator=gen) - 0.5
        entry = {"K": K, "compositions": {}}
        rounds: dict = {c: [] for c in selector.B200_COMPOSITIONS["gcn"]}
        specs = {}
        for comp in selector.B200_COMPOSITIONS["gcn"]:
            base, order = comp.split(":")
            spec = gc.GcnLayerSpec(K, K, w, composition=base, order=order)
            specs[comp] = spec
            try:
                with sparse.kernel_timing("spmm") as kt:
                    med, cv = profiling.time_iterations(lambda: gc.gcn_layer(g, h, spec), 2,
                                                        args.sweep_reps)
                torch.cuda.synchronize()
                out = gc.gcn_layer(g, h, spec)
            except torch.cuda.OutOfMemoryError:
                torch.cuda.empty_cache()
                entry["compositions"][comp] = {"oom": True}
                continue
            sp = float(np.median(kt.durations_ms("spmm")))
            rounds[comp].append(med)
            dyn = base == "dynamic"
            b = spmm_alg_bytes(n, m, K, not dyn, dyn, dyn, uses_half(gc, n, K))
            entry["compositions"][comp] = {
                "ms": round(med * 1e3, 4), "edges_per_s": round(m / med, 1),
                "gflops": round(layer_flops(n, m, K, K, order) / med / 1e9, 1),
                "spmm_ms": round(sp, 4),
                "spmm_hbm_frac": round(b / (sp * 1e-3) / 1e9 / pk["hbm_gbs"], 3), "cv": round(cv, 3),
                "parity": parity.gcn(out, h, w, comp, tol_of(gc))}
            del out
        # two more interleaved rounds; the reported time is the median round
        # (a single pass in fixed order let clock / power-cap drift decide)
        for _ in range(2):
            for comp, spec in specs.items():
                if "ms" not in entry["compositions"].get(comp, {}):
                    continue
                med, _ = profiling.time_iterations(lambda: gc.gcn_layer(g, h, spec), 1,
                                                   args.sweep_reps)
                rounds[comp].append(med)
        for comp, ts in rounds.items():
            if ts and "ms" in entry["compositions"].get(comp, {}):
                med = float(np.median(ts))
                entry["compositions"][comp]["ms"] = round(med * 1e3, 4)
                entry["compositions"][comp]["edges_per_s"] = round(m / med, 1)
        ok = {c: v["ms"] for c, v in entry["compositions"].items() if "ms" in v}
        best = min(ok, key=ok.get)
        entry["fastest"] = best
        if model is not None:
            pick = selector.select(model, selector.SelectorInput(features=feats, k1=K, k2=K))
        else:
            pick = f"dynamic:{gc.ordering_heuristic(K, K).value}"
        entry["selected"] = pick
        entry["selected_over_fastest"] = round(ok[pick] / ok[best], 3) if pick in ok else None
        rows.append(entry)
        del h, w
        torch.cuda.empty_cache()
    return rows


def _time_layer(fn, reps: int) -> float:
    from paper_2306_15155_b200 import profiling

    med, _ = profiling.time_iterations(fn, 2, reps)
    return med


def cora_config(gc, args, dev) -> dict:
    """BASELINE configs[0]: 2-layer GCN 1433 -> 16 -> 7 on a Cora-shaped
    uniform graph, every composition, both numerics classes: GPU eager, GPU
    CUDA-graph replay, and the CPU oracle (reference algorithm, float64) on
    all host cores and on 1."""
    from oracle import gnn_oracle as orc
    from paper_2306_15155_b200 import graphs, profiling, selector
    from paper_2306_15155_b200.capture import GraphedForward

    import torch

    A = graphs.shape_graph("cora", seed=args.seed, device=dev)
    g = gc.NormalizedGraph.from_adjacency(A).with_precomputed()
    host = host_graph(A)
    og = orc.GcnGraph.from_adjacency(host)
    n = A.n_rows
    rng = profiling.config_rng(args.seed, "cora", 1433, 16)
    inp = profiling.draw_inputs(rng, n, 1433, 16, "gcn")
    w2 = profiling.draw_inputs(profiling.config_rng(args.seed, "cora", 16, 7), n, 16, 7, "gcn")["w"]
    h32 = inp["h"].astype(np.float32)
    w1_32, w2_32 = inp["w"].astype(np.float32), w2.astype(np.float32)
    h = torch.from_numpy(h32).to(dev)
    out = {"n": n, "m_tilde": g.a_tilde.nnz, "layers": "1433->16->7", "compositions": {}}
    old = gc.get_gemm_precision()
    for comp in selector.B200_COMPOSITIONS["gcn"]:
        base, order = comp.split(":")
        ref = orc.gcn_layer(og, orc.gcn_layer(og, h32.astype(np.float64), w1_32.astype(np.float64),
                                               base, order), w2_32.astype(np.float64), base, order)
        row = {}
        for prec in ("tf32", "fp32"):
            gc.set_gemm_precision(prec)
            specs = [gc.GcnLayerSpec(1433, 16, w1_32, composition=base, order=order),
                     gc.GcnLayerSpec(16, 7, w2_32, composition=base, order=order)]
            fwd = lambda x: gc.gcn_forward(g, x, specs)  # noqa: E731
            eager = _time_layer(lambda: fwd(h), 20)
            gf = GraphedForward(fwd, h)
            graphed = _time_layer(lambda: gf(h), 20)
            y = gf(h).cpu().numpy()
            err = orc.rel_err(y, ref)
            tol = 1e-2 if prec == "tf32" else 1e-4
            row[prec] = {"gpu_eager_ms": round(eager * 1e3, 4), "gpu_graph_ms": round(graphed * 1e3, 4),
                         "parity": {"rel_err": err, "tol": tol, "ok": bool(err <= tol)}}
        out["compositions"][comp] = row
    gc.set_gemm_precision(old)
    # the reference's own CPU path (oracle port), default composition, 1 and all threads
    for threads in (1, os.cpu_count()):
        orc.set_threads(threads)
        t = time_cpu(lambda: orc.gcn_layer(og, orc.gcn_layer(og, h32.astype(np.float64),
                                                              w1_32.astype(np.float64), "dynamic"),
                                           w2_32.astype(np.float64), "dynamic"), 3, 10)
        out[f"cpu_oracle_{threads}t_ms"] = round(t * 1e3, 3)
    return out


def selector_pick(row_comps: dict, model: str, feats, K: int, k2: int | None = None) -> dict:
    """The B200 selector's choice for this group and its time over the
    fastest composition measured (north-star target: <= 1.1)."""
    from paper_2306_15155_b200 import selector

    mdl = selector.load_b200_model(model)
    if mdl is None:
        return {}
    sel = selector.select(mdl, selector.SelectorInput(features=feats, k1=K, k2=k2 or K))
    best = min(row_comps, key=lambda c: row_comps[c]["ms"])
    out = {"fastest": best, "selected": sel}
    if sel in row_comps:
        out["selected_over_fastest"] = round(row_comps[sel]["ms"] / row_comps[best]["ms"], 3)
    return out


def timed_runs(runs: dict, rounds: int = 3, reps: int = 3) -> dict:
    """Median over interleaved rounds of each run's CUDA-event median."""
    ts = {c: [] for c in runs}
    for _ in range(rounds):
        for c, fn in runs.items():
            ts[c].append(_time_layer(fn, reps))
    return {c: float(np.median(v)) for c, v in ts.items()}


def extra_configs(gc, args, dev, pk) -> dict:
    """BASELINE configs[0] (Cora), [2] (single/4-head GAT on arxiv, SDDMM vs
    reassociated attention, reuse vs recompute, K = 32..1024) and [3] (GCN +
    GAT on products, 1 GPU): every composition timed (interleaved rounds) with
    its row-sampled parity; ms and edges/s = m / layer time."""
    import torch

    from paper_2306_15155_b200 import graphs, selector

    res = {"cora": cora_config(gc, args, dev)}
    tol = tol_of(gc)
    pick, timed = selector_pick, timed_runs

    # ---- GAT on ogbn-arxiv-shaped RMAT ---------------------------------------
    A = graphs.shape_graph("arxiv", seed=args.seed, device=dev)
    feats = gc.extract_features(A)  # raw graph, as the reference's cli.py:187
    at = gc.add_self_loops(A)
    del A
    par = Parity(at, args.parity_rows, seed=args.seed + 1)
    n, m = at.n_rows, at.nnz
    gat = []
    for heads, ks in ((1, (32, 256, 1024)), (4, (32, 256, 1024))):
        for K in ks:
            gen = torch.Generator(device=dev)
            gen.manual_seed(K + heads)
            h = torch.rand(n, K, device=dev, generator=gen) - 0.5
            w = torch.rand(K, K * heads, device=dev, generator=gen) - 0.5
            a_s = torch.rand(K * heads, device=dev, generator=gen) - 0.5
            a_d = torch.rand(K * heads, device=dev, generator=gen) - 0.5
            specs = {c: gc.GatLayerSpec(K, K, w, a_s, a_d, composition=c.split(":")[0], heads=heads,
                                        attention=c.split(":")[1])
                     for c in selector.B200_COMPOSITIONS["gat"]}
            t = timed({c: (lambda s=s: gc.gat_layer(at, h, s)) for c, s in specs.items()},
                      reps=args.sweep_reps)
            row = {"heads": heads, "k1": K, "k2": K, "compositions": {}}
            for c, s in specs.items():
                row["compositions"][c] = {"ms": round(t[c] * 1e3, 4), "edges_per_s": round(m / t[c], 1),
                                          "parity": par.gat(gc.gat_layer(at, h, s), h, w, a_s, a_d,
                                                            heads, c, tol)}
            # a multi-head layer is `heads` single-head layers (GatLayerSpec):
            # the selector is asked about one head's (k1, k2)
            row.update(pick(row["compositions"], "gat", feats, K, k2=K))
            gat.append(row)
            del h, w, specs
            torch.cuda.empty_cache()
    res["gat_arxiv"] = {"n": n, "m_tilde": m, "rows": gat}
    # GCN on the same arxiv shape (every composition, with the selector check)
    ga = gc.NormalizedGraph(a_tilde=at, d_inv_sqrt=gc.inv_sqrt_degrees(at)).with_precomputed()
    res["gcn_arxiv"] = {"n": n, "m_tilde": m,
                        "rows": gcn_rows(gc, ga, feats, (32, 256, 1024), par, tol, dev, pick, timed)}
    res["epoch_arxiv"] = epoch_row(gc, ga, feats, "arxiv", par, tol, dev, with_gat=True)
    del at, par, ga
    torch.cuda.empty_cache()
    # ---- products-shaped: GCN (4 compositions) + GAT -------------------------
    A = graphs.shape_graph("products", seed=args.seed, device=dev)
    feats = gc.extract_features(A)
    g = gc.NormalizedGraph.from_adjacency(A).with_precomputed()
    del A
    par = Parity(g.a_tilde, args.parity_rows, seed=args.seed + 2)
    n, m = g.a_tilde.n_rows, g.a_tilde.nnz
    rows = []
    for K in (32, 256, 1024):
        gen = torch.Generator(device=dev)
        gen.manual_seed(K)
        h = torch.rand(n, K, device=dev, generator=gen) - 0.5
        w = torch.rand(K, K, device=dev, generator=gen) - 0.5
        row = {"K": K, "gcn": {}, "gat": {}}
        gcn_specs = {c: gc.GcnLayerSpec(K, K, w, composition=c.split(":")[0], order=c.split(":")[1])
                     for c in selector.B200_COMPOSITIONS["gcn"]}
        t = timed({c: (lambda s=s: gc.gcn_layer(g, h, s)) for c, s in gcn_specs.items()})
        for comp, spec in gcn_specs.items():
            base = comp.split(":")[0]
            with __import__("paper_2306_15155_b200").sparse.kernel_timing("spmm") as kt:
                y = gc.gcn_layer(g, h, spec)
            torch.cuda.synchronize()
            sp = float(np.median(kt.durations_ms("spmm")))
            dyn = base == "dynamic"
            b = spmm_alg_bytes(n, m, K, not dyn, dyn, dyn, uses_half(gc, n, K))
            row["gcn"][comp] = {"ms": round(t[comp] * 1e3, 4), "edges_per_s": round(m / t[comp], 1),
                                "spmm_ms": round(sp, 4),
                                "spmm_hbm_frac": round(b / (sp * 1e-3) / 1e9 / pk["hbm_gbs"], 3),
                                "parity": par.gcn(y, h, w, comp, tol)}
            del y
        a_s = torch.rand(K, device=dev, generator=gen) - 0.5
        a_d = torch.rand(K, device=dev, generator=gen) - 0.5
        gat_specs = {c: gc.GatLayerSpec(K, K, w, a_s, a_d, composition=c.split(":")[0],
                                        attention=c.split(":")[1])
                     for c in selector.B200_COMPOSITIONS["gat"]}
        t = timed({c: (lambda s=s: gc.gat_layer(g.a_tilde, h, s)) for c, s in gat_specs.items()})
        for comp, spec in gat_specs.items():
            row["gat"][comp] = {"ms": round(t[comp] * 1e3, 4), "edges_per_s": round(m / t[comp], 1),
                                "parity": par.gat(gc.gat_layer(g.a_tilde, h, spec), h, w, a_s, a_d, 1,
                                                  comp, tol)}
        row["gcn_selection"] = pick(row["gcn"], "gcn", feats, K)
        row["gat_selection"] = pick(row["gat"], "gat", feats, K)
        rows.append(row)
        del h, w
        torch.cuda.empty_cache()
    res["products"] = {"n": n, "m_tilde": m, "rows": rows}
    res["epoch_products"] = epoch_row(gc, g, feats, "products", par, tol, dev)
    del g, par
    torch.cuda.empty_cache()
    return res


# north_star asks for layer AND epoch throughput per named shape.  One epoch
# here = a full-graph forward pass of a 2-layer model with the dataset's own
# feature and class widths (input -> 256 -> classes; the reference's own
# 2-layer model is Cora's 1433 -> 16 -> 7, timed in cora_config), each layer's
# composition picked by the B200 selector.  Training (backward) is out of
# scope in the reference itself.
EPOCH_DIMS = {"reddit": (602, 256, 41), "arxiv": (128, 256, 40), "products": (100, 256, 47)}


def _pick(model: str, feats, k1: int, k2: int) -> str:
    from paper_2306_15155_b200 import selector

    mdl = selector.load_b200_model(model)
    if mdl is None:
        return "dynamic:aggregate_first" if model == "gcn" else "reuse:reassoc"
    return selector.select(mdl, selector.SelectorInput(features=feats, k1=k1, k2=k2))


def epoch_row(gc, g, feats, shape: str, par, tol, dev, with_gat: bool = False) -> dict:
    try:
        return _epoch_row(gc, g, feats, shape, par, tol, dev, with_gat)
    except Exception as e:  # noqa: BLE001 — recorded in the line, never silently dropped
        return {"error": repr(e)[:400]}


def _epoch_row(gc, g, feats, shape: str, par, tol, dev, with_gat: bool = False) -> dict:
    """2-layer GCN (and optionally 1-head GAT) epoch on graph ``g``: ms per
    epoch (CUDA-event median of 5 after 2 warm-ups), edges/s = 2·m / t,
    GFLOP/s from the chosen orders, and each layer's row-sampled parity
    against the oracle given that layer's actual input."""
    import torch

    k0, k1, k2 = EPOCH_DIMS[shape]
    n, m = g.a_tilde.n_rows, g.a_tilde.nnz
    gen = torch.Generator(device=dev)
    gen.manual_seed(k0 * 1000 + k2)
    h = torch.rand(n, k0, device=dev, generator=gen) - 0.5
    ws = [torch.rand(a, b, device=dev, generator=gen) - 0.5 for a, b in ((k0, k1), (k1, k2))]
    dims = ((k0, k1), (k1, k2))
    comps = [_pick("gcn", feats, a, b) for a, b in dims]
    specs = [gc.GcnLayerSpec(a, b, w, composition=c.split(":")[0], order=c.split(":")[1])
             for (a, b), w, c in zip(dims, ws, comps)]
    t = _time_layer(lambda: gc.gcn_forward(g, h, specs), 5)
    y1 = gc.gcn_layer(g, h, specs[0])
    y2 = gc.gcn_layer(g, y1, specs[1])
    flops = sum(layer_flops(n, m, a, b, c.split(":")[1]) for (a, b), c in zip(dims, comps))
    out = {"dims": [k0, k1, k2], "gcn": {
        "compositions": comps, "ms": round(t * 1e3, 4), "edges_per_s": round(2 * m / t, 1),
        "gflops": round(flops / t / 1e9, 1),
        "parity": [par.gcn(y1, h, ws[0], comps[0], tol), par.gcn(y2, y1, ws[1], comps[1], tol)]}}
    del y1, y2
    if with_gat:
        att = [(torch.rand(b, device=dev, generator=gen) - 0.5,
                torch.rand(b, device=dev, generator=gen) - 0.5) for _, b in dims]
        gcomps = [_pick("gat", feats, a, b) for a, b in dims]
        gspecs = [gc.GatLayerSpec(a, b, w, s_, d_, composition=c.split(":")[0],
                                  attention=c.split(":")[1])
                  for (a, b), w, (s_, d_), c in zip(dims, ws, att, gcomps)]

        def fwd():
            x = h
            for sp in gspecs:
                x = gc.gat_layer(g.a_tilde, x, sp)
            return x

        t = _time_layer(fwd, 5)
        z1 = gc.gat_layer(g.a_tilde, h, gspecs[0])
        z2 = gc.gat_layer(g.a_tilde, z1, gspecs[1])
        out["gat"] = {"compositions": gcomps, "ms": round(t * 1e3, 4),
                      "edges_per_s": round(2 * m / t, 1),
                      "parity": [par.gat(z1, h, ws[0], *att[0], 1, gcomps[0], tol),
                                 par.gat(z2, z1, ws[1], *att[1], 1, gcomps[1], tol)]}
        del z1, z2
    del h, ws
    torch.cuda.empty_cache()
    return out


def gcn_rows(gc, g, feats, ks, par, tol, dev, pick, timed) -> list[dict]:
    """Every GCN composition at each K on graph ``g`` (interleaved timing,
    row-sampled parity) and the selector's pick over the fastest."""
    import torch

    from paper_2306_15155_b200 import selector

    n, m = g.a_tilde.n_rows, g.a_tilde.nnz
    rows = []
    for K in ks:
        gen = torch.Generator(device=dev)
        gen.manual_seed(K + 17)
        h = torch.rand(n, K, device=dev, generator=gen) - 0.5
        w = torch.rand(K, K, device=dev, generator=gen) - 0.5
        specs = {c: gc.GcnLayerSpec(K, K, w, composition=c.split(":")[0], order=c.split(":")[1])
                 for c in selector.B200_COMPOSITIONS["gcn"]}
        t = timed({c: (lambda s=s: gc.gcn_layer(g, h, s)) for c, s in specs.items()})
        row = {"K": K, "compositions": {}}
        for c, spec in specs.items():
            row["compositions"][c] = {"ms": round(t[c] * 1e3, 4), "edges_per_s": round(m / t[c], 1),
                                      "parity": par.gcn(gc.gcn_layer(g, h, spec), h, w, c, tol)}
        row.update(pick(row["compositions"], "gcn", feats, K))
        rows.append(row)
        del h, w
        torch.cuda.empty_cache()
    return rows


def gat_rows_reddit(gc, a_tilde, feats, K, par, tol, dev, pick, timed) -> dict:
    """Single-head GAT, every composition, on the Reddit shape at one K."""
    import torch

    from paper_2306_15155_b200 import selector

    n, m = a_tilde.n_rows, a_tilde.nnz
    gen = torch.Generator(device=dev)
    gen.manual_seed(K + 29)
    h = torch.rand(n, K, device=dev, generator=gen) - 0.5
    w = torch.rand(K, K, device=dev, generator=gen) - 0.5
    a_s = torch.rand(K, device=dev, generator=gen) - 0.5
    a_d = torch.rand(K, device=dev, generator=gen) - 0.5
    specs = {c: gc.GatLayerSpec(K, K, w, a_s, a_d, composition=c.split(":")[0],
                                attention=c.split(":")[1])
             for c in selector.B200_COMPOSITIONS["gat"]}
    t = timed({c: (lambda s=s: gc.gat_layer(a_tilde, h, s)) for c, s in specs.items()})
    row = {"K": K, "heads": 1, "compositions": {}}
    for c, spec in specs.items():
        row["compositions"][c] = {"ms": round(t[c] * 1e3, 4), "edges_per_s": round(m / t[c], 1),
                                  "parity": par.gat(gc.gat_layer(a_tilde, h, spec), h, w, a_s, a_d,
                                                    1, c, tol)}
    row.update(pick(row["compositions"], "gat", feats, K))
    return row


def partitioned_products(args, rank: int, world: int, dev) -> dict | None:
    """BASELINE configs[3] at N GPUs: GCN (selected composition) and GAT (all
    four compositions) on the products shape, row-partitioned through the
    capacity path; device time per layer, max over ranks."""
    import torch
    import torch.distributed as dist

    import paper_2306_15155_b200 as gc
    from paper_2306_15155_b200 import selector
    from paper_2306_15155_b200.distributed import dist_gat_layer, dist_gcn_layer

    part, d, feats, m, prep_s = load_partition(args, rank, world, dev, "products")
    nt_block = normalized_block(part, d)
    out = {"shape": "products", "m_tilde": m, "world": world, "partition_load_s": round(prep_s, 3),
           "rows": []}

    def max_ms(fn, reps=5):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = _events()
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        dist.barrier()
        t = torch.tensor([e0.elapsed_time(e1) / reps], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for K in (32, 256):
        gen = torch.Generator(device=dev)
        gen.manual_seed(K)
        h = torch.rand(part.rows, K, device=dev, generator=gen) - 0.5
        w = torch.rand(K, K, device=dev, generator=gen) - 0.5
        a_s = torch.rand(K, device=dev, generator=gen) - 0.5
        a_d = torch.rand(K, device=dev, generator=gen) - 0.5
        model = selector.load_b200_model("gcn")
        comp = selector.select(model, selector.SelectorInput(features=feats, k1=K, k2=K)) \
            if model is not None else "dynamic:aggregate_first"
        base, order = comp.split(":")
        prev = part.local
        part.local = nt_block if base == "precompute" else prev
        part._padded = part._lr = None
        row = {"K": K, "gcn": {"composition": comp}, "gat": {}}
        ms = max_ms(lambda: dist_gcn_layer(part, h, w, composition=base, order=order, d=d,
                                           overlap=True, hub_unit=True))
        row["gcn"].update({"ms": round(ms, 4), "edges_per_s": round(m / (ms * 1e-3), 1)})
        part.local = prev
        part._padded = part._lr = None
        for c in selector.B200_COMPOSITIONS["gat"]:
            spec = gc.GatLayerSpec(K, K, w, a_s, a_d, composition=c.split(":")[0],
                                   attention=c.split(":")[1])
            ms = max_ms(lambda: dist_gat_layer(part, h, spec))
            row["gat"][c] = {"ms": round(ms, 4), "edges_per_s": round(m / (ms * 1e-3), 1)}
        out["rows"].append(row)
        del h
    return out if rank == 0 else None


def cpu_baseline(g, args) -> dict:
    """The reference's CPU algorithm (oracle port, float64, all host threads)
    on the FULL graph at K in --cpu-ks: the reference default composition,
    median of 3 after 1 warm-up (1 rep at K >= 1024); nothing extrapolated."""
    from oracle import gnn_oracle as orc
    from paper_2306_15155_b200 import profiling

    threads = orc.set_threads(os.cpu_count())
    at = host_graph(g.a_tilde)
    d = orc.inv_sqrt_degrees(at)
    n, m = at.n_rows, at.nnz
    rows = []
    for K in (int(k) for k in args.cpu_ks.split(",") if k):
        inp = profiling.draw_inputs(profiling.config_rng(args.seed, args.shape, K, K), n, K, K, "gcn")
        h = inp["h"].astype(np.float32).astype(np.float64)
        w = inp["w"].astype(np.float32).astype(np.float64)
        big = K >= 1024
        t = time_cpu(lambda: cpu_oracle_layer(orc, at, d, h, w), 0 if big else 1, 1 if big else 3)
        rows.append({"K": K, "seconds_per_layer": round(t, 3), "edges_per_s": round(m / t, 1),
                     "reps": 1 if big else 3})
        del h, w
    main_row = next((r for r in rows if r["K"] == args.k), rows[-1])
    return {"value": main_row["edges_per_s"], "unit": UNIT, "cores": threads, "kind": "port",
            "cpu": cpu_model(), "sample": f"full graph (n={n}, m={m}), no sampling or "
            f"extrapolation; reference default composition (dynamic, heuristic order), float64",
            "per_k": rows, "calibration": calibration()}


def run_reference(args, rank: int, world: int) -> None:
    """The reference's CPU implementation of the path (the oracle's port of
    gnncompose, float64, all host threads — calibrated against gnncompose
    itself in profiles/data/cpu_calibration.json) on the FULL graph of the
    same workload: each step is one whole layer."""
    if rank != 0:
        return
    import torch

    from oracle import gnn_oracle as orc
    from paper_2306_15155_b200 import graphs, profiling

    # input synthesis only: the graph generator is plain torch integer ops
    # (GPU if present, else CPU); no gnnc kernel runs in this arm.
    dev = torch.device("cuda", 0) if torch.cuda.is_available() else torch.device("cpu")
    A = graphs.shape_graph(args.shape, seed=args.seed, device=dev)
    host_a = host_graph(A)
    del A
    at = orc.add_self_loops(host_a)
    d = orc.inv_sqrt_degrees(at)
    K = args.k
    n, m = at.n_rows, at.nnz
    rng = profiling.config_rng(args.seed, args.shape, K, K)
    inp = profiling.draw_inputs(rng, n, K, K, "gcn")
    h = inp["h"].astype(np.float32).astype(np.float64)
    w = inp["w"].astype(np.float32).astype(np.float64)
    threads = orc.set_threads(os.cpu_count())
    for _ in range(args.warmup):
        cpu_oracle_layer(orc, at, d, h, w)
    ts = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        cpu_oracle_layer(orc, at, d, h, w)
        ts.append(time.perf_counter() - t0)
    t = float(np.mean(ts))
    value = m / t
    sample = (f"full graph (n={n}, m={m}); each step one whole layer; reference default "
              f"composition (dynamic, heuristic order), float64")
    out = {"impl": "reference", "metric": METRIC, "value": round(value, 1), "unit": UNIT,
           "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": round(t * 1e3, 3), "higher_is_better": True, "scaling": "strong",
           "vs_baseline": None, "dtype": "f64", "data": f"synthetic RMAT {args.shape}-shaped",
           "config": {"workload": f"gcn_layer/{args.shape}/k1=k2={K}", "shape": args.shape, "n": n,
                      "m_tilde": m, "K": K, "composition": "dynamic:aggregate_first"},
           "cpu_baseline": {"value": round(value, 1), "unit": UNIT, "cores": threads, "kind": "port",
                            "sample": sample, "cpu": cpu_model(), "calibration": calibration()},
           "e2e": {"value": round(value, 1), "unit": UNIT, "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0},
           "gpu_launches": 0}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
