#!/usr/bin/env python
"""Phase breakdown of the end-to-end path (pinned host buffers -> output on host).

Times, with a device synchronize after each phase: graph H2D + id narrowing,
feature H2D, the resident layer-wise engine, output gather and D2H, for the
headline workload.  Run on the B200 box; prints one JSON line.
"""

from __future__ import annotations

import json
import pathlib
import sys
import time

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import numpy as np
    import torch

    from paper_2211_15082_b200 import kernels, synth
    from paper_2211_15082_b200.batching import Thresholds
    from paper_2211_15082_b200.device import DeviceBudget
    from paper_2211_15082_b200.executor import (LayerwiseEngine, RunStats, _as_device_store,
                                                annotate, run_inference)
    from paper_2211_15082_b200.splitter import split
    from paper_2211_15082_b200.storage import CscGraph, DeviceGraph

    n, und = synth.PRODUCTS_NODES, synth.PRODUCTS_UNDIRECTED
    m = synth.build_gcn(100, 256, 47, 3, seed=0)
    g = synth.gen_products_like(n, und, seed=0, device="cuda")
    xt = synth.gen_features_device(n, 100, seed=0)
    ip = torch.empty(n + 1, dtype=torch.int64, pin_memory=True)
    ip.copy_(torch.from_numpy(g.indptr_host))
    ix = torch.empty(g.num_edges, dtype=torch.int64, pin_memory=True)
    ix.copy_(g.indices.to(torch.int64).cpu())
    xh = torch.empty((n, 100), dtype=torch.float32, pin_memory=True)
    xh.copy_(xt.cpu())
    hg = CscGraph(n, g.num_edges, ip.numpy(), ix.numpy())
    budget = DeviceBudget(160 << 30)
    out = {}

    def tick(name, t0):
        torch.cuda.synchronize()
        out[name] = (time.perf_counter() - t0) * 1e3
        return time.perf_counter()

    for rep in range(3):
        t = time.perf_counter()
        dg = DeviceGraph.from_host(hg)
        t = tick("graph_h2d_narrow_ms", t)
        x = _as_device_store(xh, dg.device)
        t = tick("features_h2d_ms", t)
        sched = split(m)
        ts = annotate(dg, np.arange(n), 3, "full")
        st = RunStats("layerwise", "full", "none", 3)
        eng = LayerwiseEngine(m, sched, dg, x, ts, budget, Thresholds(1024, 32768), st, reassociate=True)
        store = eng.run()
        t = tick("engine_ms", t)
        host = torch.empty((n, 47), dtype=torch.float32, pin_memory=True)
        host.copy_(store.view())
        t = tick("output_d2h_ms", t)
        t0 = time.perf_counter()
        res = run_inference(m, hg, xh, budget=budget, output="numpy", reassociate=True)
        torch.cuda.synchronize()
        out["run_inference_ms"] = (time.perf_counter() - t0) * 1e3
        del res, dg, x, store, eng
    print(json.dumps(out), flush=True)
    import cProfile
    import pstats

    pr = cProfile.Profile()
    pr.enable()
    res = run_inference(m, hg, xh, budget=budget, output="numpy", reassociate=True)
    torch.cuda.synchronize()
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(25)


if __name__ == "__main__":
    main()
