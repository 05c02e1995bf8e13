#!/usr/bin/env python
"""cProfile of the host side of run_inference on the cfg2 workload.

tools/order_timeline.py shows the device idling 3-16 ms between
run_inference's entry and the engine's first launch; this attributes that
host time (top functions by cumulative and by own time over K steps).
"""
import cProfile
import io
import pathlib
import pstats
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))


def main():
    import torch

    from paper_2211_15082_b200 import synth
    from paper_2211_15082_b200.executor import run_inference

    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    n = synth.PRODUCTS_NODES
    g = synth.gen_products_like(n, synth.PRODUCTS_UNDIRECTED, seed=0, device="cuda")
    x = synth.gen_features_device(n, 100, seed=0, device="cuda")
    m = synth.build_gcn(100, 256, 47, 3, seed=0)
    for _ in range(3):
        run_inference(m, g, x, budget="device", output="device", reassociate=True)
    torch.cuda.synchronize()
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(steps):
        res = run_inference(m, g, x, budget="device", output="device", reassociate=True)
        del res
    torch.cuda.synchronize()
    pr.disable()
    for key in ("cumulative", "tottime"):
        s = io.StringIO()
        pstats.Stats(pr, stream=s).sort_stats(key).print_stats(30)
        print(s.getvalue())


if __name__ == "__main__":
    main()
