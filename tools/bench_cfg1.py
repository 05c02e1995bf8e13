"""cfg1 (BASELINE.json configs[0], the reference's CPU-runnable case) on one B200.

gen_regular(100_000, 20, seed=0), 128-d gen_features(seed=0),
build_gcn(128, 128, 128, 2, seed=0), full layer-wise inference through
run_inference with the default thresholds at a 16 GiB capacity (the capacity
tests/test_cfg1_gpu.py pins against the reference's stats document), from
host numpy inputs (graph + features uploaded, output returned to the host)
and from device-resident inputs.  BASELINE.md: the reference takes 9.35-9.82 s
for this run on the CPU.

    python tools/bench_cfg1.py > profiles/r02_cfg1.jsonl
"""

from __future__ import annotations

import json
import pathlib
import sys
import time

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))


def main():
    import numpy as np
    import torch

    from paper_2211_15082_b200 import kernels
    from paper_2211_15082_b200.batching import Thresholds
    from paper_2211_15082_b200.device import DeviceBudget
    from paper_2211_15082_b200.executor import run_inference
    from paper_2211_15082_b200.synth import build_gcn, gen_features, gen_regular

    g = gen_regular(100_000, 20, seed=0)
    x = gen_features(100_000, 128, seed=0)
    m = build_gcn(128, 128, 128, 2, seed=0)
    budget = DeviceBudget(16 << 30)
    th = Thresholds(1024, 32768)
    dg = kernels.device_graph(g)
    xd = torch.from_numpy(x).cuda()
    for inputs, name in (((g, x), "host inputs -> host output"),
                         ((dg, xd), "device-resident inputs -> device output")):
        out = "numpy" if name.startswith("host") else "device"
        for _ in range(3):
            run_inference(m, *inputs, budget=budget, thresholds=th, output=out)
        torch.cuda.synchronize()
        times = []
        res = None
        for _ in range(10):
            res = None
            t0 = time.perf_counter()
            res = run_inference(m, *inputs, budget=budget, thresholds=th, output=out)
            torch.cuda.synchronize()
            times.append(1e3 * (time.perf_counter() - t0))
        print(json.dumps({"workload": "cfg1 2-layer GCN/SAGE-mean 128->128->128, gen_regular(100k, 20)",
                          "path": name, "ms_median": round(float(np.median(times)), 3),
                          "ms_all": [round(t, 3) for t in times],
                          "nodes_per_s": 100_000 / (float(np.median(times)) / 1e3),
                          "batches": res.stats.batches,
                          "reference_cpu_s": "9.35-9.82 (BASELINE.md)"}), flush=True)


if __name__ == "__main__":
    main()
