"""Device/host timeline of one cfg1 run_inference call from host numpy inputs
(gen_regular(100k, 20), 128-d, build_gcn(128, 128, 128, 2), 16 GiB capacity,
default thresholds) -- where the small-graph request's time goes.

    python tools/cfg1_trace.py > profiles/r02_cfg1_trace.jsonl
"""
import json
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))


def main():
    import torch

    from paper_2211_15082_b200.batching import Thresholds
    from paper_2211_15082_b200.device import DeviceBudget
    from paper_2211_15082_b200.executor import KernelProbe, run_inference
    from paper_2211_15082_b200.synth import build_gcn, gen_features, gen_regular

    g = gen_regular(100_000, 20, seed=0)
    x = gen_features(100_000, 128, seed=0)
    m = build_gcn(128, 128, 128, 2, seed=0)
    budget = DeviceBudget(16 << 30)
    th = Thresholds(1024, 32768)
    for rep in range(4):
        probe = KernelProbe()
        torch.cuda.synchronize()
        res = run_inference(m, g, x, budget=budget, thresholds=th, output="numpy", probe=probe)
        torch.cuda.synchronize()
        probe.mark("end")
        torch.cuda.synchronize()
        if rep == 3:
            print(json.dumps({"workload": "cfg1", "timeline": probe.absolute(),
                              "batches": res.stats.batches}), flush=True)


if __name__ == "__main__":
    main()
