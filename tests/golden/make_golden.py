"""Generate golden fixtures by running the REFERENCE package in this container.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes tests/golden/golden.npz (arrays) and tests/golden/golden.json (strings,
stats documents, case metadata).  /root/reference does not exist on the GPU
box: the fixtures are committed and the tests read only them.  glint.cli and
glint.report are never imported (matplotlib is absent).

Models are built with THIS package's builders and handed to the reference
through its own document API (model_from_document), so the reference runs on
exactly the weights the B200 code sees; the builders' byte-compatibility with
the reference builders is itself recorded (synth section).
"""

from __future__ import annotations

import json
import pathlib
import sys

import numpy as np

HERE = pathlib.Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(ROOT))

from glint import batching as r_batching  # noqa: E402
from glint import executor as r_exec  # noqa: E402
from glint import kernels as r_k  # noqa: E402
from glint import model_ir as r_ir  # noqa: E402
from glint import reorder as r_reorder  # noqa: E402
from glint import splitter as r_split  # noqa: E402
from glint import storage as r_storage  # noqa: E402
from glint import synth as r_synth  # noqa: E402
from glint.device import DeviceBudget as RBudget  # noqa: E402

from paper_2211_15082_b200 import model_ir as my_ir  # noqa: E402
from paper_2211_15082_b200 import synth as my_synth  # noqa: E402

ARR = {}
META = {"kernels": [], "e2e": [], "schedules": {}, "orders": [], "sampling": [],
        "annotate": [], "synth": [], "batching": []}


def put(name, arr):
    assert name not in ARR, name
    ARR[name] = np.asarray(arr)
    return name


def to_ref_model(m):
    return r_ir.model_from_document(my_ir.model_document(m), my_ir.model_tensors(m))


def graphs():
    return {
        "toy": r_storage.make_graph(6, {0: [2, 3], 1: [2, 3], 2: [4, 5]}),
        "reg200": r_synth.gen_regular(200, 5, seed=1),
        "pow300": r_synth.gen_powerlaw(300, seed=2),
        "sbm160": r_synth.gen_sbm(4, 40, 0.2, 0.01, seed=3),
        "path50": r_synth.gen_path(50),
        "dup30": r_storage.make_graph(30, {v: [(v * 7) % 30, (v * 7) % 30, v, (v + 1) % 30]
                                           for v in range(0, 30, 2)}),
    }


def kernel_cases(gs):
    rng = np.random.default_rng(123)
    for gname, g in gs.items():
        for d in (1, 3, 47, 100, 128):
            if gname in ("toy", "path50") and d > 47:
                continue
            n = g.num_nodes
            x = rng.normal(size=(n, d)).astype(np.float32) * (4 if d == 3 else 1)
            for tname, targets in (("all", np.arange(n)),
                                   ("sub", np.sort(rng.choice(n, size=max(1, n // 3), replace=False))),
                                   ("perm", rng.permutation(n)[: max(1, n // 4)])):
                bc = r_k.build_batch_csc(g, targets)
                pre = f"k/{gname}/{d}/{tname}"
                case = {"graph": gname, "dim": d, "targets": put(pre + "/targets", targets),
                        "x": put(pre + "/x", x),
                        "input_ids": put(pre + "/input_ids", bc.input_ids),
                        "indptr": put(pre + "/indptr", bc.indptr),
                        "local_srcs": put(pre + "/local_srcs", bc.local_srcs),
                        "target_pos": put(pre + "/target_pos", bc.target_pos),
                        "agg_mean": put(pre + "/agg_mean", r_k.agg_mean(bc, x[bc.input_ids]))}
                if d in (3, 47) and tname != "perm":
                    heads = 2
                    w = rng.normal(size=(heads, 5, d)).astype(np.float32) / np.sqrt(d)
                    a = rng.normal(size=(heads, 10)).astype(np.float32)
                    p = r_k.AttnParams(w, a)
                    case["attn_w"] = put(pre + "/attn_w", w)
                    case["attn_a"] = put(pre + "/attn_a", a)
                    case["agg_attn"] = put(pre + "/agg_attn", r_k.agg_attn(bc, x[bc.input_ids], p))
                if tname == "all":
                    w = rng.normal(size=(7, d)).astype(np.float32)
                    b = rng.normal(size=7).astype(np.float32)
                    case["lin_w"] = put(pre + "/lin_w", w)
                    case["lin_b"] = put(pre + "/lin_b", b)
                    case["linear"] = put(pre + "/linear", r_k.linear(x, w, b))
                    for kind in ("ReLU", "LeakyReLU", "Norm", "DropoutIdentity"):
                        case["ew_" + kind] = put(pre + "/ew_" + kind, r_k.elementwise(kind, [x]))
                    case["ew_Add"] = put(pre + "/ew_Add", r_k.elementwise("Add", [x, x * 0.5, -x]))
                    case["concat"] = put(pre + "/concat", r_k.concat([x, x[:, :1], 2 * x]))
                META["kernels"].append(case)


def models():
    return {
        "gcn2": my_synth.build_gcn(8, 16, 4, 2, seed=2),
        "gcn3": my_synth.build_gcn(8, 12, 5, 3, seed=3),
        "gat2": my_synth.build_gat(8, 6, 3, 2, heads=2, seed=4),
        "gat3h4": my_synth.build_gat(8, 4, 3, 3, heads=4, seed=5),
        "jknet3": my_synth.build_jknet(8, 6, 4, 3, seed=6),
        "residual": my_synth.build_residual(8, 8, seed=7),
        "linear": my_synth.build_linear(8, 3, seed=8),
        "appnp": my_synth.build_appnp(8, 10, 4, k=3, alpha=0.1, seed=9),
    }


def e2e_cases(gs, ms):
    rng = np.random.default_rng(7)
    budgets = {"big": 1 << 30, "tight": 9000, "mid": 60_000}
    for gname in ("toy", "reg200", "pow300", "sbm160"):
        g = gs[gname]
        x = r_synth.gen_features(g.num_nodes, 8, seed=11)
        xs = r_storage.open_store(g.num_nodes, 8)
        xs.scatter(np.arange(g.num_nodes), x)
        part = np.sort(rng.choice(g.num_nodes, size=max(2, g.num_nodes // 10), replace=False))
        put(f"e/{gname}/x", x)
        put(f"e/{gname}/partial", part)
        for mname, m in ms.items():
            rm = to_ref_model(m)
            combos = [("full", "none", "big"), ("full", "rcmk", "mid"), ("partial", "none", "big"),
                      ("partial", "rcmk", "tight"), ("sampling", "random", "mid"),
                      ("full", "degree", "tight")]
            if gname == "toy":
                combos = [("full", "none", "big"), ("partial", "rcmk", "big"),
                          ("sampling", "none", "big")]
            for mode, order, bud in combos:
                name = f"e/{gname}/{mname}/{mode}/{order}/{bud}"
                kw = dict(mode=mode, order=order, seed=13, budget=RBudget(budgets[bud]),
                          executor="layerwise", thresholds=r_batching.Thresholds(64, 512))
                if mode != "full":
                    kw["targets"] = part if gname != "toy" else np.array([3, 0])
                if mode == "sampling":
                    kw["fanout"] = 3
                try:
                    res = r_exec.run_inference(rm, g, xs, **kw)
                except Exception as exc:  # record the expected error class
                    META["e2e"].append({"name": name, "graph": gname, "model": mname,
                                        "mode": mode, "order": order, "budget": budgets[bud],
                                        "error": type(exc).__name__})
                    continue
                META["e2e"].append({
                    "name": name, "graph": gname, "model": mname, "mode": mode, "order": order,
                    "budget": budgets[bud], "thresholds": [64, 512], "seed": 13,
                    "fanout": kw.get("fanout"), "targets": "partial" if mode != "full" else None,
                    "output": put(name + "/out", res.output),
                    "stats": res.stats.document(),
                })


def schedule_cases(ms):
    sys.path.insert(0, "/root/reference/pkg/tests")
    import conftest  # reference fixtures: fig a/b/c models

    extra = {"fig_a": conftest.fig_a_model(), "fig_b": conftest.fig_b_model(),
             "fig_c": conftest.fig_c_model()}
    for name, m in ms.items():
        META["schedules"][name] = r_split.format_schedule(r_split.split(to_ref_model(m)))
    for name, rm in extra.items():
        META["schedules"][name] = {"doc": r_ir.model_document(rm),
                                   "tensors": {k: v.tolist() for k, v in r_ir.model_tensors(rm).items()},
                                   "text": r_split.format_schedule(r_split.split(rm))}
    import test_splitter  # reference random layered models

    for seed in range(25):
        rm = test_splitter.random_layered_model(seed)
        META["schedules"][f"rand{seed}"] = {
            "doc": r_ir.model_document(rm),
            "tensors": {k: v.tolist() for k, v in r_ir.model_tensors(rm).items()},
            "text": r_split.format_schedule(r_split.split(rm))}


def order_cases(gs):
    for gname, g in gs.items():
        put(f"g/{gname}/indptr", g.indptr)
        put(f"g/{gname}/indices", g.indices)
        for kind in ("rcmk", "degree", "random"):
            o = r_reorder.make_order(g, kind, seed=5)
            META["orders"].append({"graph": gname, "kind": kind,
                                   "perm": put(f"o/{gname}/{kind}", o.perm)})
        g2, _ = r_reorder.apply_order(g, np.zeros((g.num_nodes, 1), np.float32),
                                      r_reorder.make_order(g, "rcmk"))
        put(f"o/{gname}/rcmk_indptr", g2.indptr)
        put(f"o/{gname}/rcmk_indices", g2.indices)
    big = r_synth.gen_powerlaw(3000, seed=4)
    put("g/pow3000/indptr", big.indptr)
    put("g/pow3000/indices", big.indices)
    META["orders"].append({"graph": "pow3000", "kind": "rcmk",
                           "perm": put("o/pow3000/rcmk", r_reorder.rcmk(big).perm)})


def sampling_cases(gs):
    for gname in ("toy", "reg200", "pow300"):
        g = gs[gname]
        for fanout, seed, layer in ((1, 9, 1), (2, 4, 2), (3, 0, 1), (50, 1, 3)):
            s = r_exec.sample_neighbors(g, np.arange(g.num_nodes), fanout, seed, layer)
            pre = f"s/{gname}/{fanout}/{seed}/{layer}"
            META["sampling"].append({"graph": gname, "fanout": fanout, "seed": seed,
                                     "layer": layer, "indptr": put(pre + "/indptr", s.indptr),
                                     "indices": put(pre + "/indices", s.indices)})
        rng = np.random.default_rng(3)
        for depth in (1, 2, 3):
            t = np.sort(rng.choice(g.num_nodes, size=3, replace=False))
            ts = r_exec.annotate(g, t, depth, "partial")
            META["annotate"].append({"graph": gname, "depth": depth, "targets": t.tolist(),
                                     "skip_from": ts.skip_from,
                                     "v": {str(k): v.tolist() for k, v in ts.v_sets.items()}})


def synth_cases():
    for name, g in (("reg", r_synth.gen_regular(120, 7, seed=5)),
                    ("pow", r_synth.gen_powerlaw(150, seed=6)),
                    ("sbm", r_synth.gen_sbm(3, 20, 0.3, 0.05, seed=7)),
                    ("path", r_synth.gen_path(9))):
        META["synth"].append({"name": name, "indptr": put(f"y/{name}/indptr", g.indptr),
                              "indices": put(f"y/{name}/indices", g.indices)})
    put("y/features", r_synth.gen_features(7, 5, seed=3))
    for name, rm in (("gcn", r_synth.build_gcn(5, 6, 3, 3, seed=2)),
                     ("gat", r_synth.build_gat(5, 4, 3, 2, heads=3, seed=2)),
                     ("jknet", r_synth.build_jknet(5, 4, 3, 3, seed=2)),
                     ("residual", r_synth.build_residual(5, 6, seed=2)),
                     ("linear", r_synth.build_linear(5, 2, seed=2))):
        for k, v in r_ir.model_tensors(rm).items():
            put(f"y/model/{name}/{k}", v)


def batching_cases():
    rng = np.random.default_rng(11)
    for case in range(6):
        degs = rng.integers(0, 40, size=400)
        prefix = np.zeros(401, dtype=np.int64)
        np.cumsum(degs, out=prefix[1:])
        cap = int(rng.integers(3000, 40000))
        c = r_batching.BatchController(r_batching.Thresholds(int(rng.integers(1, 64)),
                                                             int(rng.integers(0, 900))),
                                       RBudget(cap))
        nt0, ni0 = c.thresholds.n_t, c.thresholds.n_i
        from glint.device import BatchFootprint

        def plan_fn(s, e):
            edges = int(prefix[e] - prefix[s])
            return (s, e), BatchFootprint(0, 0, (e - s) * 13 + edges * 5 + (edges * edges) % 97, 0)

        recs = []
        for layer in (1, 2):
            recs += c.run_layer(layer, np.arange(400), prefix, plan_fn, lambda p: None)
        META["batching"].append({"degs": degs.tolist(), "cap": cap, "init": [nt0, ni0],
                                 "records": [[r.layer, r.start, r.end, r.oom_retries, r.n_t, r.n_i,
                                              r.footprint.peak] for r in recs]})


def main():
    gs = graphs()
    kernel_cases(gs)
    ms = models()
    e2e_cases(gs, ms)
    schedule_cases(ms)
    order_cases(gs)
    sampling_cases(gs)
    synth_cases()
    batching_cases()
    np.savez_compressed(HERE / "golden.npz", **ARR)
    (HERE / "golden.json").write_text(json.dumps(META, indent=0, sort_keys=True) + "\n")
    total = sum(a.nbytes for a in ARR.values())
    print(f"wrote {len(ARR)} arrays ({total / 1e6:.1f} MB raw), "
          f"{len(META['kernels'])} kernel / {len(META['e2e'])} e2e cases")


if __name__ == "__main__":
    main()
