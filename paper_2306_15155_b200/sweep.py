"""Selector training sweep on B200 (BASELINE.json configs[4]; SENSEi stage 1).

Profiles every composition of GCN and GAT layers over uniform-random and RMAT
power-law graphs (n from 2^14 to 2^21, average degree 2..512, memory capped)
at several (k1, k2), writes NDJSON ProfileRecords, and — offline, on CPU —
trains the ranking selector on an 80/20 split by graph and reports its
quality against the per-group oracle and every static policy.

    python -m paper_2306_15155_b200.sweep profile --out records.ndjson [--quick]
    python -m paper_2306_15155_b200.sweep train --records records.ndjson
"""

from __future__ import annotations

import argparse
import json
import math
import sys
import time
import warnings
from pathlib import Path

import numpy as np

SIZES = [(32, 32), (128, 128), (512, 512), (1024, 1024), (32, 256), (256, 32), (64, 1024),
         (1024, 64)]
NS = [2 ** 14, 2 ** 16, 2 ** 18, 2 ** 20, 2 ** 21]
DEGREES = [2, 8, 32, 128, 512]
MAX_NNZ = 200_000_000
NAMED = ("arxiv", "reddit", "products")  # benchmark shapes: evaluated leave-one-shape-out
# the named shapes also run the bench's square K sweep
NAMED_SIZES = [(32, 32), (64, 64), (128, 128), (256, 256), (512, 512), (1024, 1024), (32, 256),
               (256, 32), (64, 1024), (1024, 64)]


def graph_plan(quick: bool = False) -> list[tuple[str, str, int, int]]:
    plan = []
    ns = NS[:3] if quick else NS
    for kind in ("uniform", "rmat"):
        for n in ns:
            for deg in DEGREES:
                nnz = 2 * ((n * deg) // 2)
                if nnz > MAX_NNZ or nnz // 2 > n * (n - 1) // 4:
                    continue
                plan.append((f"{kind}_n{int(math.log2(n))}_d{deg}", kind, n, nnz))
    return plan


def named_plan() -> list[tuple[str, str, int, int]]:
    """The BASELINE graph shapes themselves (arxiv, reddit, products)."""
    from .graphs import SHAPES

    return [(s.name, s.kind, s.n, s.nnz) for k, s in SHAPES.items() if k != "cora"]


def cmd_profile(args) -> None:
    import torch

    from . import graphs, profiling

    dev = torch.device("cuda", 0)
    out = Path(args.out)
    out.parent.mkdir(parents=True, exist_ok=True)
    fh = out.open("a")
    t_start = time.time()
    plan = named_plan() if args.graphs == "named" else graph_plan(args.quick)
    for gid, kind, n, nnz in plan:
        try:
            a = graphs.synthetic_graph(kind, n, nnz, seed=1 if args.graphs != "named" else 0,
                                       device=dev, max_candidates=1 << 33)
        except RuntimeError as e:  # RMAT cannot reach this density
            print(f"skip {gid}: {e}", file=sys.stderr, flush=True)
            continue
        for model in args.models.split(","):
            base = NAMED_SIZES if args.graphs == "named" else SIZES
            sizes = base if model == "gcn" else [s for s in base if s[0] <= 512 and s[1] <= 512]
            with warnings.catch_warnings():
                warnings.simplefilter("ignore")
                recs = profiling.profile([(gid, a)], sizes, model, reps=args.reps,
                                         warmup=args.warmup)
            if model == "gat" and args.graphs == "named" and args.heads > 1:
                # multi-head groups (records keyed "<shape>/h<heads>", k2 =
                # heads * k2): the bench's 4-head GAT configs
                with warnings.catch_warnings():
                    warnings.simplefilter("ignore")
                    recs += profiling.profile([(gid, a)], [(32, 32), (256, 256), (1024, 1024)],
                                              model, reps=args.reps, warmup=args.warmup,
                                              heads=args.heads)
            for r in recs:
                fh.write(json.dumps(r.to_dict()) + "\n")
            fh.flush()
            print(f"{gid} {model}: {len(recs)} records  t={time.time() - t_start:.0f}s",
                  file=sys.stderr, flush=True)
        del a
        torch.cuda.empty_cache()
    fh.close()


def evaluate(model, records, comps, detail: bool = False) -> dict:
    from .selector import SelectorInput, select

    rows = []
    groups: dict = {}
    for r in records:
        groups.setdefault((r.graph_id, r.k1, r.k2), {})[r.composition] = r
    sel, orc = [], []
    static = {c: [] for c in comps}
    for key, g in groups.items():
        if not all(c in g for c in comps):
            continue
        best = min(g[c].median_time_s for c in comps)
        r0 = next(iter(g.values()))
        pick = select(model, SelectorInput(features=r0.features, k1=r0.k1, k2=r0.k2,
                                           hw_descriptor=tuple(r0.hw_desc)))
        sel.append(g[pick].median_time_s / best)
        orc.append(1.0)
        if detail:
            fastest = min(comps, key=lambda c: g[c].median_time_s)
            rows.append({"k1": r0.k1, "k2": r0.k2, "selected": pick, "fastest": fastest,
                         "selected_over_fastest": round(sel[-1], 4)})
        for c in comps:
            static[c].append(g[c].median_time_s / best)

    def gm(x):
        return float(np.exp(np.mean(np.log(x)))) if x else float("nan")

    out = {"groups": len(sel), "selected_over_oracle_geomean": gm(sel),
           "selected_over_oracle_max": float(max(sel)) if sel else None,
           "within_1.1x": float(np.mean(np.array(sel) <= 1.1)) if sel else None,
           "static_over_oracle_geomean": {c: gm(v) for c, v in static.items()}}
    if detail:
        out["per_group"] = sorted(rows, key=lambda x: (x["k1"], x["k2"]))
    return out


def cmd_train(args) -> None:
    from .profiling import read_records
    from .selector import B200_COMPOSITIONS, MODEL_DIR, SelectorHyperparams, train

    recs = read_records(args.records)
    report = {}
    MODEL_DIR.mkdir(exist_ok=True)
    for model_tag in ("gcn", "gat"):
        comps = B200_COMPOSITIONS[model_tag]
        mine = [r for r in recs if r.model == model_tag and r.composition in comps]
        if not mine:
            continue
        graphs_ = sorted({r.graph_id for r in mine if r.graph_id.split("/")[0] not in NAMED})
        rng = np.random.default_rng(0)
        test_g = set(rng.choice(graphs_, size=max(1, len(graphs_) // 5), replace=False).tolist())
        tr = [r for r in mine if r.graph_id not in test_g]
        te = [r for r in mine if r.graph_id in test_g]
        hyper = SelectorHyperparams(n_estimators=args.trees, learning_rate=args.lr,
                                    max_depth=args.depth)
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            m = train(tr, model_tag, hyper, compositions=comps)
        rep = {"train_graphs": len({r.graph_id for r in tr}), "test_graphs": sorted(test_g),
               "hyper": vars(hyper), "train": evaluate(m, tr, comps), "test": evaluate(m, te, comps)}
        # leave-one-named-shape-out: the model never saw that benchmark shape
        # (nor the random held-out graphs); evaluated on every (k1, k2) of it
        lono = {}
        for shape in NAMED:
            held = [r for r in mine if r.graph_id.split("/")[0] == shape]
            if not held:
                continue
            with warnings.catch_warnings():
                warnings.simplefilter("ignore")
                m_s = train([r for r in tr if r.graph_id.split("/")[0] != shape], model_tag, hyper,
                            compositions=comps)
            lono[shape] = evaluate(m_s, held, comps, detail=True)
        if lono:
            rep["leave_one_named_shape_out"] = lono
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            full = train(mine, model_tag, hyper, compositions=comps)
        full.save(MODEL_DIR / f"{model_tag}_b200.json")
        rep["shipped_model_all_records"] = evaluate(full, mine, comps)
        report[model_tag] = rep
    text = json.dumps(report, indent=1)
    print(text)
    if args.report:
        Path(args.report).write_text(text + "\n")


def main(argv=None):
    p = argparse.ArgumentParser()
    sub = p.add_subparsers(dest="cmd", required=True)
    pp = sub.add_parser("profile")
    pp.add_argument("--out", required=True)
    pp.add_argument("--models", default="gcn,gat")
    pp.add_argument("--reps", type=int, default=3)
    pp.add_argument("--warmup", type=int, default=1)
    pp.add_argument("--quick", action="store_true")
    pp.add_argument("--heads", type=int, default=1,
                    help="named graphs: also profile GAT with this many heads (records keyed "
                         "'<shape>/h<heads>', k2 = heads*k2; kept out of the shipped models: "
                         "they cost held-out single-head quality, see DESIGN.md §6)")
    pp.add_argument("--graphs", choices=("sweep", "named"), default="sweep",
                    help="sweep: configs[4] uniform/RMAT grid; named: the arxiv/reddit/products shapes")
    pt = sub.add_parser("train")
    pt.add_argument("--records", required=True)
    pt.add_argument("--trees", type=int, default=300)
    pt.add_argument("--lr", type=float, default=0.05)
    pt.add_argument("--depth", type=int, default=6)
    pt.add_argument("--report", default=None)
    args = p.parse_args(argv)
    {"profile": cmd_profile, "train": cmd_train}[args.cmd](args)


if __name__ == "__main__":
    main()
