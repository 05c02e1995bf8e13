#!/usr/bin/env python
"""K4 (and K1) time split: the whole call vs its regular rows alone vs its hub rows
alone, on the Products graph (how much of a call the hub rows add)."""
import json
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))


def timed(fn, reps=10):
    import torch

    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def main():
    import torch

    from paper_2211_15082_b200 import kernels, synth

    n = synth.PRODUCTS_NODES
    g = synth.gen_products_like(n, synth.PRODUCTS_UNDIRECTED, seed=0, device="cuda")
    sched, nh = kernels.degree_schedule(g.indptr, None, 0, n)
    nh = int(nh.item())
    heads = 4
    for dh in (64, 47):
        hp = kernels.head_pitch(dh)
        Z = torch.randn((n, heads * hp), device="cuda")
        s_src = torch.randn((n, heads), device="cuda")
        s_dst = torch.randn((n, heads), device="cuda")
        out = torch.empty((n, heads * dh), device="cuda")

        def call(sch, rows, hubs):
            return lambda: kernels.gat_aggregate(out, Z, s_src, s_dst, heads, dh, g.indptr,
                                                 g.indices, rows, schedule=sch, n_hub=hubs)

        full = timed(call(sched, n, nh))
        regular = timed(call(sched[nh:], n - nh, 0))
        hubs = timed(call(sched[:nh], nh, nh))
        print(json.dumps({"kernel": "gat_aggregate", "heads": heads, "head_dim": dh,
                          "hub_rows": nh, "full_ms": full, "regular_only_ms": regular,
                          "hubs_only_ms": hubs}), flush=True)
    for d in (100, 256, 48):
        h = torch.randn((n, d), device="cuda")
        out = torch.empty((n, d), device="cuda")

        def callm(sch, rows, hubs):
            return lambda: kernels.spmm_mean(out, h, g.indptr, g.indices, rows, schedule=sch,
                                             n_hub=hubs)

        print(json.dumps({"kernel": "spmm_mean", "dim": d, "full_ms": timed(callm(sched, n, nh)),
                          "regular_only_ms": timed(callm(sched[nh:], n - nh, 0)),
                          "hubs_only_ms": timed(callm(sched[:nh], nh, nh))}), flush=True)


if __name__ == "__main__":
    main()
