#!/usr/bin/env python
"""e2e A/B: run_inference from pinned host buffers, timed like bench.py's e2e."""
import json
import pathlib
import sys
import time

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))


def main():
    import os

    import torch

    from paper_2211_15082_b200 import synth
    from paper_2211_15082_b200.device import DeviceBudget
    from paper_2211_15082_b200.executor import run_inference
    from paper_2211_15082_b200.storage import CscGraph

    n, und = synth.PRODUCTS_NODES, synth.PRODUCTS_UNDIRECTED
    model = sys.argv[1] if len(sys.argv) > 1 and not sys.argv[1].startswith("--") else "gcn3"
    m = (synth.build_gcn(100, 256, 47, 3, seed=0) if model == "gcn3"
         else synth.build_gat(100, 64, 47, 3, heads=4, seed=0))
    g = synth.gen_products_like(n, und, seed=0, device="cuda")
    xt = synth.gen_features_device(n, 100, seed=0)
    ip = torch.empty(n + 1, dtype=torch.int64, pin_memory=True)
    ip.copy_(torch.from_numpy(g.indptr_host))
    ix = torch.empty(g.num_edges, dtype=torch.int64, pin_memory=True)
    ix.copy_(g.indices.to(torch.int64).cpu())
    xh = torch.empty((n, 100), dtype=torch.float32, pin_memory=True)
    xh.copy_(xt.cpu())
    hg = CscGraph(n, g.num_edges, ip.numpy(), ix.numpy())
    del g, xt
    budget = DeviceBudget(160 << 30)
    from paper_2211_15082_b200 import storage

    if "--sink-ab" in sys.argv:     # same, for the output sink's row chunks
        sys.argv[sys.argv.index("--sink-ab")] = "--fracs-ab"
        var = "GLINT_SINK_FRACS"
    else:
        var = "GLINT_UPLOAD_FRACS"
    if "--fracs-ab" in sys.argv:
        # interleaved A/B of CSR upload chunk plans (GLINT_UPLOAD_FRACS, cumulative
        # edge fractions; "" = the default geometric plan)
        plans = sys.argv[sys.argv.index("--fracs-ab") + 1].split(";")
        times = {p: [] for p in plans}

        def set_plan(p):
            if p:
                os.environ[var] = p
            else:
                os.environ.pop(var, None)

        res = None
        for p in plans:
            set_plan(p)
            res = None
            res = run_inference(m, hg, xh, budget=budget, output="numpy", reassociate=True)
        for _ in range(5):
            for p in plans:
                set_plan(p)
                res = None
                t0 = time.perf_counter()
                res = run_inference(m, hg, xh, budget=budget, output="numpy", reassociate=True)
                torch.cuda.synchronize()
                times[p].append(1e3 * (time.perf_counter() - t0))
        import numpy as np

        for p in plans:
            print(json.dumps({"model": model, "ab": f"chunk plan ({var})",
                              "fracs": p or "default plan",
                              "ms": [round(t, 1) for t in times[p]],
                              "median": float(np.median(times[p]))}), flush=True)
        return

    if "--knob-ab" in sys.argv:
        # interleaved A/B of one tuning knob: --knob-ab 20=0,1
        from paper_2211_15082_b200 import _lib
        import numpy as np

        spec = sys.argv[sys.argv.index("--knob-ab") + 1]
        key, vals = spec.split("=")
        vals = [int(v) for v in vals.split(",")]
        times = {v: [] for v in vals}
        res = None
        for v in vals:
            _lib.call("glint_set_tuning", int(key), v)
            res = None
            res = run_inference(m, hg, xh, budget=budget, output="numpy", reassociate=True)
        for _ in range(8):
            for v in vals:
                _lib.call("glint_set_tuning", int(key), v)
                res = None
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                res = run_inference(m, hg, xh, budget=budget, output="numpy", reassociate=True)
                torch.cuda.synchronize()
                times[v].append(1e3 * (time.perf_counter() - t0))
        _lib.call("glint_set_tuning", int(key), 0)
        for v in vals:
            print(json.dumps({"model": model, "ab": f"tuning knob {key}", "value": v,
                              "ms": [round(t, 1) for t in times[v]],
                              "median": float(np.median(times[v]))}), flush=True)
        return

    # --pack24-ab: alternate 24-bit packed and int32 CSR uploads in one process
    modes = (True, False) if "--pack24-ab" in sys.argv else (storage.PACK24,)
    times = {mode: [] for mode in modes}
    res = None
    for mode in modes:             # warm-up (pinned staging, allocator) per mode
        storage.PACK24 = mode
        res = None
        res = run_inference(m, hg, xh, budget=budget, output="numpy", reassociate=True)
    torch.cuda.synchronize()
    for _ in range(6 if len(modes) > 1 else 5):
        for mode in modes:
            storage.PACK24 = mode
            res = None
            t0 = time.perf_counter()
            res = run_inference(m, hg, xh, budget=budget, output="numpy", reassociate=True)
            torch.cuda.synchronize()
            times[mode].append(1e3 * (time.perf_counter() - t0))
    if len(modes) > 1:
        import numpy as np

        print(json.dumps({"model": model, "ab": "pack24 vs int32 CSR upload",
                          "pack24_ms": [round(t, 1) for t in times[True]],
                          "int32_ms": [round(t, 1) for t in times[False]],
                          "pack24_median": float(np.median(times[True])),
                          "int32_median": float(np.median(times[False]))}), flush=True)
        return
    times = times[modes[0]]
    print(json.dumps({"model": model, "sink_chunks": os.environ.get("GLINT_SINK_CHUNKS", "2"),
                      "host_narrow": os.environ.get("GLINT_HOST_NARROW", "1"),
                      "chunks": os.environ.get("GLINT_UPLOAD_CHUNKS", "default"),
                      "geometric": os.environ.get("GLINT_UPLOAD_GEOMETRIC", "0"),
                      "threads": os.environ.get("GLINT_NARROW_THREADS", "default"),
                      "ms": [round(t, 1) for t in times]}), flush=True)


if __name__ == "__main__":
    main()
