"""Per-launch K4 times inside the cfg3 step, interleaved in one process, for
values of one tuning knob: `python tools/gat_step_probe.py 0,5,6` sweeps the K4
launch variants (GLINT_TUNE_GAT_VARIANT = 3); `... 0,1 18` A/Bs knob 18
(GLINT_TUNE_GAT_PEAK_FIRST)."""
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
    from paper_2211_15082_b200 import _lib

    variants = [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "0,5,6,7,8,9").split(",")]
    knob = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    res, steps = {}, {}
    for rep in range(6):
        for t in variants:
            _lib.call("glint_set_tuning", knob, t)
            pr = KernelProbe()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            a.record()
            run.step(pr)
            b.record()
            torch.cuda.synchronize()
            if rep:
                steps.setdefault(t, []).append(round(a.elapsed_time(b), 3))
            if rep:
                res.setdefault(t, []).append([round(ms, 3) for nm, _, ms in pr.launches()
                                              if nm == "gat_aggregate"])
    _lib.call("glint_set_tuning", knob, 0)
    for t, v in res.items():
        print(json.dumps({"knob": knob, "value": t,
                          "k4_ms_per_layer": np.median(np.asarray(v), axis=0).round(3).tolist(),
                          "step_ms_median": float(np.median(steps[t])), "all": v}))


if __name__ == "__main__":
    main()
