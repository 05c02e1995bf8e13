#!/usr/bin/env python
"""Multi-rank functional check on one GPU box (launch with torchrun).

Every rank runs run_inference(distributed="auto") -- rows partitioned
edge-balanced, each layer's stored output exchanged -- and compares the
output bytes with its own single-rank run of the same request.  With
GLINT_DIST_BACKEND=gloo all ranks may share one GPU.  Prints one JSON line
per model from rank 0."""
import json
import os
import pathlib
import sys

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2211_15082_b200 import synth
    from paper_2211_15082_b200.device import DeviceBudget
    from paper_2211_15082_b200.executor import run_inference
    from paper_2211_15082_b200.storage import CscGraph

    world = int(os.environ["WORLD_SIZE"])
    rank = int(os.environ["RANK"])
    local = int(os.environ.get("LOCAL_RANK", "0")) % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dist.init_process_group(os.environ.get("GLINT_DIST_BACKEND", "nccl"))
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 200_000
    und = int(round(n * synth.PRODUCTS_UNDIRECTED / synth.PRODUCTS_NODES))
    g = synth.gen_products_like(n, und, seed=3, device="cuda")
    host = CscGraph(n, g.num_edges, np.asarray(g.indptr_host), g.indices.to(torch.int64).cpu().numpy())
    x = synth.gen_features_device(n, 100, seed=3, device="cuda").cpu().numpy()
    models = (("gcn3", synth.build_gcn(100, 256, 47, 3, seed=0)),
              ("gat3", synth.build_gat(100, 64, 47, 3, heads=4, seed=0)))

    def check(tag, m, hg, xx, cap, reassoc):
        kw = dict(budget=DeviceBudget(cap), reassociate=reassoc)
        ref = run_inference(m, hg, xx, distributed=False, **kw).output
        for kind in ("replicate", "halo"):
            out = run_inference(m, hg, xx, distributed="auto", exchange=kind, **kw).output
            flags = torch.tensor([1.0 if np.array_equal(ref, out) else 0.0], device="cuda")
            dist.all_reduce(flags, op=dist.ReduceOp.MIN)
            if rank == 0:
                print(json.dumps({"graph": tag, "model": name, "world": world,
                                  "nodes": hg.num_nodes, "capacity": cap, "reassociate": reassoc,
                                  "exchange": kind,
                                  "bit_identical_all_ranks": bool(flags.item() == 1.0)}), flush=True)

    for name, m in models:
        for cap in (1 << 34, 64 << 20):       # one batch per layer / many batches
            for reassoc in ((False, True) if name == "gcn3" else (False,)):
                check("products_like", m, host, x, cap, reassoc)
    # A star: every edge points into node 0, so edge-balanced ranges leave
    # ranks with no rows (those ranks must still join every
    # collective of the transform-first convs).
    from paper_2211_15082_b200.parallel import edge_balanced_ranges

    ns = 20
    star = CscGraph(ns, ns - 1, np.array([0] + [ns - 1] * ns, dtype=np.int64),
                    np.arange(1, ns, dtype=np.int64))
    xs = synth.gen_features(ns, 100, seed=1)
    cuts = edge_balanced_ranges(star.indptr, world)
    if rank == 0:
        print(json.dumps({"star_cuts": cuts.tolist(),
                          "empty_ranks": int(np.sum(np.diff(cuts) == 0))}), flush=True)
    for name, m in models:
        for reassoc in ((False, True) if name == "gcn3" else (False,)):
            check("star", m, star, xs, 1 << 34, reassoc)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
