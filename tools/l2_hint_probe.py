#!/usr/bin/env python
"""K1 L2-policy probe (run on the B200 box): does steering L2 residency toward
high-degree source rows cut DRAM traffic of the mean aggregation?

The products-shaped graph's source ids are annotated with bit 31 = "hot"
(the top-R sources by out-degree, R = budget / row bytes); K1 then gathers hot
rows with an evict_last policy and the rest evict_first (GLINT_TUNE_L2_HINT).
Output bytes must equal the unhinted run.  One JSON line per (width, budget, mode).
"""

from __future__ import annotations

import argparse
import json
import pathlib
import sys

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def timed(fn, reps):
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

    from paper_2211_15082_b200 import _lib, kernels, synth
    from paper_2211_15082_b200.executor import agg_bytes

    ap = argparse.ArgumentParser()
    ap.add_argument("--dims", default="100,256,48")
    ap.add_argument("--budgets", default="0,20,40,60,80")
    ap.add_argument("--modes", default="1,2")
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    n = synth.PRODUCTS_NODES
    g = synth.gen_products_like(n, synth.PRODUCTS_UNDIRECTED, seed=0, device="cuda")
    deg = g.in_degrees
    hub = int(((deg + 1) >= kernels.HUB_MIN_DEGREE).sum())
    sched, _ = kernels.degree_schedule(g.indptr, None, 0, n)
    idx = g.indices
    cnt = torch.bincount(idx.long(), minlength=n)
    order = torch.argsort(cnt, descending=True)
    for d in (int(x) for x in args.dims.split(",")):
        pitch = (d + 3) // 4 * 4
        hbuf = torch.randn((n, pitch), device="cuda")
        h = hbuf[:, :d]
        out = torch.empty((n, pitch), device="cuda")[:, :d]
        _lib.call("glint_set_tuning", 11, 0)
        ms0 = timed(lambda: kernels.spmm_mean(out, h, g.indptr, idx, n, schedule=sched, n_hub=hub),
                    args.reps)
        ref = out.clone()
        nb = agg_bytes(d, g.num_edges, n)
        print(json.dumps({"dim": d, "budget_mb": 0, "mode": 0, "ms": round(ms0, 4),
                          "GBps": round(nb / ms0 / 1e6, 1)}), flush=True)
        for mb in (int(x) for x in args.budgets.split(",")):
            rows = mb * 1024 * 1024 // (pitch * 4)
            hot = torch.zeros(n, dtype=torch.bool, device="cuda")
            if rows:
                hot[order[:rows]] = True
            ann = torch.where(hot[idx.long()], idx | torch.tensor(-2 ** 31, dtype=torch.int32,
                                                                   device="cuda"), idx)
            cover = float(cnt[order[:rows]].sum()) / idx.numel() if rows else 0.0
            for mode in (int(x) for x in args.modes.split(",")):
                _lib.call("glint_set_tuning", 11, mode)
                ms = timed(lambda: kernels.spmm_mean(out, h, g.indptr, ann, n, schedule=sched,
                                                     n_hub=hub), args.reps)
                print(json.dumps({"dim": d, "budget_mb": mb, "hot_rows": rows,
                                  "gather_cover": round(cover, 3), "mode": mode, "ms": round(ms, 4),
                                  "GBps": round(nb / ms / 1e6, 1), "speedup": round(ms0 / ms, 3),
                                  "bytes_equal": bool(torch.equal(ref, out))}), flush=True)
            del ann, hot
        _lib.call("glint_set_tuning", 11, 0)
        del hbuf, out, ref


if __name__ == "__main__":
    main()
