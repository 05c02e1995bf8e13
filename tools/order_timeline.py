#!/usr/bin/env python
"""Step-to-step spread of the cfg2 step per node order: device/host timelines.

tools/order_probe.py showed K1 is no slower on the RCMK-relabelled graph, but
the step times spread.  This runs K steps per order through run_inference
(device-resident inputs, probe attached) and prints, for the fastest and the
slowest step, every timeline marker as (device ms, host ms) since the step's
first marker, so a gap can be attributed to a host wait or to the device.
"""
import json
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))


def main():
    import torch

    from paper_2211_15082_b200 import synth
    from paper_2211_15082_b200.executor import KernelProbe, run_inference
    from paper_2211_15082_b200.reorder import apply_order_device, make_order

    orders = sys.argv[1].split(",") if len(sys.argv) > 1 else ["none", "rcmk"]
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    n = synth.PRODUCTS_NODES
    g0 = synth.gen_products_like(n, synth.PRODUCTS_UNDIRECTED, seed=0, device="cuda")
    x0 = synth.gen_features_device(n, 100, seed=0, device="cuda")
    m = synth.build_gcn(100, 256, 47, 3, seed=0)
    for kind in orders:
        g, x = apply_order_device(g0, x0, make_order(g0, kind))
        for _ in range(3):
            run_inference(m, g, x, budget="device", output="device", reassociate=True)
        torch.cuda.synchronize()
        runs = []
        for _ in range(steps):
            p = KernelProbe()
            res = run_inference(m, g, x, budget="device", output="device", reassociate=True,
                                probe=p)
            torch.cuda.synchronize()
            tl = p.absolute()
            runs.append((tl[-1][1], tl, p.summary(), list(res.stats.batch_sizes)))
            del res
        runs.sort(key=lambda r: r[0])
        for tag, r in (("fastest", runs[0]), ("slowest", runs[-1])):
            print(json.dumps({"order": kind, "which": tag, "device_ms": r[0],
                              "all_ms": [round(q[0], 2) for q in runs],
                              "kernels": {k: [c, round(t, 3)] for k, (c, _, t) in r[2].items()},
                              "batches": r[3], "timeline": r[1]}), flush=True)
        del g, x
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
