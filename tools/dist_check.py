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
    for name, m in (("gcn3", synth.build_gcn(100, 256, 47, 3, seed=0)),
                    ("gat3", synth.build_gat(100, 64, 47, 3, heads=4, seed=0))):
        for cap in (1 << 34, 64 << 20):       # one batch per layer / many batches
            ref = run_inference(m, host, x, budget=DeviceBudget(cap), distributed=False).output
            out = run_inference(m, host, x, budget=DeviceBudget(cap), distributed="auto").output
            same = bool(np.array_equal(ref, out))
            flags = torch.tensor([1.0 if same else 0.0], device="cuda")
            dist.all_reduce(flags, op=dist.ReduceOp.MIN)
            if rank == 0:
                print(json.dumps({"model": name, "world": world, "nodes": n, "capacity": cap,
                                  "bit_identical_all_ranks": bool(flags.item() == 1.0)}), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
