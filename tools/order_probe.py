#!/usr/bin/env python
"""Why is the cfg2 step slower on an RCMK-relabelled graph?  K1 time per order.

For each node order (none / rcmk / degree / random) the Products graph is
relabelled once on the device; then K1 (spmm_mean, the full-mode whole-layer
call the engine makes) is timed at the three cfg2 widths as the whole call,
its regular rows alone and its hub rows alone, next to the degree-schedule
build and a full engine step.  Also reported per order: how far apart in id
space a row's neighbours are (median |u - v| over edges) and how the LPT
schedule's first rows (the hub rows) spread over the id space.
"""
import json
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))


def timed(fn, reps=10):
    import torch

    fn()
    torch.cuda.synchronize()
    out = []
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        out.append(s.elapsed_time(e))
    out.sort()
    return round(out[len(out) // 2], 3), round(out[0], 3), round(out[-1], 3)


def main():
    import numpy as np
    import torch

    from paper_2211_15082_b200 import kernels, synth
    from paper_2211_15082_b200.executor import run_inference
    from paper_2211_15082_b200.reorder import apply_order_device, make_order

    orders = sys.argv[1].split(",") if len(sys.argv) > 1 else ["none", "rcmk", "degree", "random"]
    n = synth.PRODUCTS_NODES
    g0 = synth.gen_products_like(n, synth.PRODUCTS_UNDIRECTED, seed=0, device="cuda")
    x0 = synth.gen_features_device(n, 100, seed=0, device="cuda")
    m = synth.build_gcn(100, 256, 47, 3, seed=0)
    for kind in orders:
        order = make_order(g0, kind)
        g, x = apply_order_device(g0, x0, order)
        torch.cuda.synchronize()
        rec = {"order": kind}
        dst = torch.repeat_interleave(torch.arange(n, device="cuda"),
                                      g.indptr[1:] - g.indptr[:-1])
        gap = (g.indices.long() - dst).abs().float()
        rec["median_abs_gap"] = float(gap.median())
        rec["frac_gap_lt_4096"] = float((gap < 4096).float().mean())
        del dst, gap
        rec["schedule_ms"] = timed(lambda: kernels.degree_schedule(g.indptr, None, 0, n))
        sched, nh = kernels.degree_schedule(g.indptr, None, 0, n)
        nh = int(nh.item())
        hub_ids = sched[:nh].long()
        rec["hub_rows"] = nh
        rec["hub_id_span"] = [int(hub_ids.min()), int(hub_ids.max())] if nh else None
        for d in (100, 256, 48):
            h = torch.randn((n, d), device="cuda")
            out = torch.empty((n, d), device="cuda")

            def call(sch, rows, hubs):
                return lambda: kernels.spmm_mean(out, h, g.indptr, g.indices, rows,
                                                 schedule=sch, n_hub=hubs)

            rec[f"k1_d{d}"] = {"full": timed(call(sched, n, nh)),
                               "regular": timed(call(sched[nh:], n - nh, 0)),
                               "hubs": timed(call(sched[:nh], nh, nh))}
            del h, out
        for _ in range(2):
            run_inference(m, g, x, budget="device", output="device", reassociate=True)
        rec["step_ms"] = timed(lambda: run_inference(m, g, x, budget="device", output="device",
                                                     reassociate=True), reps=7)
        print(json.dumps(rec), flush=True)
        del g, x, sched
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
