"""Per-launch K4 times inside the cfg3 step for several hub thresholds
(kernels.GAT_HUB_MIN_DEGREE), interleaved in one process."""
import argparse
import json
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))


def main():
    import numpy as np
    import torch

    import bench
    from paper_2211_15082_b200 import kernels
    from paper_2211_15082_b200.executor import KernelProbe

    dev = torch.device("cuda", 0)
    n, und = bench.sizes(argparse.Namespace(nodes=None, undirected=None))
    g, x = bench.device_inputs(n, und, 100, dev)
    run = bench.Runner(bench.build_model("gat3"), g, x, 1, 0)
    run.step()
    res = {}
    for rep in range(4):
        for t in (512, 4096):
            kernels.GAT_HUB_MIN_DEGREE = t
            pr = KernelProbe()
            torch.cuda.synchronize()
            run.step(pr)
            torch.cuda.synchronize()
            if rep:
                res.setdefault(t, []).append([round(ms, 3) for nm, _, ms in pr.launches()
                                              if nm == "gat_aggregate"])
    for t, v in res.items():
        print(json.dumps({"gat_hub_min": t, "k4_ms_per_layer": np.median(np.asarray(v), axis=0).round(3).tolist(),
                          "all": v}))


if __name__ == "__main__":
    main()
