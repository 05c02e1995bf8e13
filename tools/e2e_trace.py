#!/usr/bin/env python
"""Device/host timeline of one end-to-end run_inference call (host buffers)."""

import json
import os
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))


def main():
    import torch

    from paper_2211_15082_b200 import synth
    from paper_2211_15082_b200.device import DeviceBudget
    from paper_2211_15082_b200.executor import KernelProbe, run_inference
    from paper_2211_15082_b200.storage import CscGraph

    n, und = synth.PRODUCTS_NODES, synth.PRODUCTS_UNDIRECTED
    m = (synth.build_gat(100, 64, 47, 3, heads=4, seed=0) if sys.argv[1:2] == ["gat3"]
         else synth.build_gcn(100, 256, 47, 3, seed=0))
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
    for rep in range(int(os.environ.get("GLINT_TRACE_REPS", "3"))):
        res = None
        torch.cuda.synchronize()
        probe = KernelProbe()
        res = run_inference(m, hg, xh, budget=budget, output="numpy", probe=probe, reassociate=True)
        torch.cuda.synchronize()
        probe.mark("end")
        torch.cuda.synchronize()
        print(json.dumps({"rep": rep, "timeline": probe.absolute()}), flush=True)


if __name__ == "__main__":
    main()
