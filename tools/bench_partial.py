#!/usr/bin/env python
"""cfg4 at Products scale: JKNet and APPNP partial inference on a 10% target subset.

BASELINE.json configs[3] is "JKNet / APPNP non-linear model structures with partial
inference on a 10% node subset (exercises layer partitioning and batching)".
SURVEY 8(d) fixes the setup:
* graph: the OGBN-Products-shaped graph (2,449,029 nodes, 123.7M in-edges) on the device;
* models: build_jknet(100, 256, 47, 3) and build_appnp(100, 256, 47, k=3, alpha=0.1);
* targets: sorted(rng.choice(N, N // 10, replace=False));
* order: none and rcmk.

The timed region is the public run_inference call with device-resident inputs,
after one untimed warm-up.  It covers annotate (frontier expansion plus the skip
rule), the splitter's blocks, batching and the kernels.  The RCMK relabelling is
timed as its own line.

Parity at this size uses a size-independent property, row invariance:
* order=none: the partial outputs are byte-identical to the same rows of a
  full-mode run;
* order=rcmk: they are within rel-L2 1e-5 of those rows (relabelling reorders
  each row's neighbour sums).
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

    from paper_2211_15082_b200 import _lib, synth
    from paper_2211_15082_b200.executor import run_inference

    _lib.load()
    n = int(sys.argv[1]) if len(sys.argv) > 1 else synth.PRODUCTS_NODES
    und = int(round(n * synth.PRODUCTS_UNDIRECTED / synth.PRODUCTS_NODES))
    g = synth.gen_products_like(n, und, seed=0, device="cuda")
    x = synth.gen_features_device(n, 100, seed=0, device="cuda")
    rng = np.random.default_rng(0)
    targets = np.sort(rng.choice(n, n // 10, replace=False)).astype(np.int64)
    models = {"jknet3": synth.build_jknet(100, 256, 47, 3, seed=0),
              "appnp3": synth.build_appnp(100, 256, 47, k=3, alpha=0.1, seed=0)}
    for name, m in models.items():
        full = run_inference(m, g, x, budget="device", output="device", reassociate=True).output
        want = full[torch.from_numpy(targets).cuda()]
        del full
        for order in ("none", "rcmk"):
            run_inference(m, g, x, mode="partial", targets=targets, order=order,
                          budget="device", output="device", reassociate=True)          # warm-up
            torch.cuda.synchronize()
            times = []
            res = None
            for _ in range(3):
                res = None
                t0 = time.perf_counter()
                res = run_inference(m, g, x, mode="partial", targets=targets, order=order,
                                    budget="device", output="device", reassociate=True)
                torch.cuda.synchronize()
                times.append(time.perf_counter() - t0)
            got = res.output
            st = res.stats
            if order == "none":
                parity = {"bit_identical_to_full_rows": bool(torch.equal(got, want))}
            else:
                err = float((got.double() - want.double()).norm() / want.double().norm())
                parity = {"rel_l2_vs_full_rows": err, "within_1e-5": err <= 1e-5}
            print(json.dumps({
                "workload": f"cfg4 {name} partial inference, 10% targets, OGBN-Products-shaped graph",
                "nodes": n, "in_edges": g.num_edges, "targets": len(targets), "order": order,
                "ms_median": 1e3 * float(np.median(times)), "ms_all": [1e3 * t for t in times],
                "targets_per_s": len(targets) / float(np.median(times)),
                "batches": st.batches, "layer_batches": st.layer_batches,
                "layer_aggregations": {str(k): int(v) for k, v in st.layer_aggregations.items()},
                "parity": parity, "api": "executor.run_inference (device-resident inputs)"}),
                flush=True)


if __name__ == "__main__":
    main()
