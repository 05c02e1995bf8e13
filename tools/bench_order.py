#!/usr/bin/env python
"""cfg2/cfg3 device step on a relabelled graph: node order none vs rcmk vs degree.

SURVEY 8(d) names RCMK as cfg2's order and excludes the one-time reorder from
the timed loop.  The graph and features are relabelled once on the device
(reorder.make_order + apply_order_device); each timed step is then the same
device-resident full 3-layer pass as bench.py (run_inference, order="none", on
the relabelled inputs), CUDA-event timed after warm-up.  The relabelled rows
are checked against the unrelabelled run (within 1e-5 rel-L2: relabelling
changes the neighbour order inside each row's sum).
"""
import json
import pathlib
import sys
import time

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))


def main():
    import numpy as np
    import torch

    from paper_2211_15082_b200 import synth
    from paper_2211_15082_b200.executor import run_inference
    from paper_2211_15082_b200.reorder import apply_order_device, make_order

    model = sys.argv[1] if len(sys.argv) > 1 else "gcn3"
    n, und = synth.PRODUCTS_NODES, synth.PRODUCTS_UNDIRECTED
    m = (synth.build_gcn(100, 256, 47, 3, seed=0) if model == "gcn3"
         else synth.build_gat(100, 64, 47, 3, heads=4, seed=0))
    g = synth.gen_products_like(n, und, seed=0, device="cuda")
    x = synth.gen_features_device(n, 100, seed=0, device="cuda")
    base = None
    for kind in ("none", "rcmk", "degree"):
        t0 = time.perf_counter()
        order = make_order(g, kind)
        gi, xi = apply_order_device(g, x, order)
        torch.cuda.synchronize()
        prep = time.perf_counter() - t0
        for _ in range(3):
            run_inference(m, gi, xi, budget="device", output="device", reassociate=True)
        torch.cuda.synchronize()
        ms = []
        out = None
        for _ in range(5):
            out = None
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            out = run_inference(m, gi, xi, budget="device", output="device", reassociate=True).output
            e.record()
            torch.cuda.synchronize()
            ms.append(s.elapsed_time(e))
        inv = torch.as_tensor(np.array(order.inv), device="cuda", dtype=torch.int64)
        mine = out[inv]                         # rows back in original node order
        if base is None:
            base = mine.clone()
            err = 0.0
        else:
            err = float((mine.double() - base.double()).norm() / base.double().norm())
        print(json.dumps({"model": model, "order": kind, "prep_s": round(prep, 2),
                          "ms": [round(v, 2) for v in ms], "ms_median": float(np.median(ms)),
                          "nodes_per_s": n / (float(np.median(ms)) / 1e3),
                          "rel_l2_vs_none": err}), flush=True)
        del gi, xi, out, mine
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
