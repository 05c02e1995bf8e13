"""K7 on one aggregate-first layer over a synthetic graph, for a grid of two
tuning knobs (default: GLINT_TUNE_FUSED_PIPE 19 x GLINT_TUNE_FUSED_VARIANT 12),
CUDA-event timed; outputs compared byte for byte with the first cell.

    python tools/k7_knob_grid.py [--graph papers|products] [--shape 128x128]
"""

from __future__ import annotations

import argparse
import json
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--graph", default="papers", choices=("papers", "products"))
    ap.add_argument("--nodes", type=int, default=None)
    ap.add_argument("--shape", default="128x128")
    ap.add_argument("--a", default="19=0,1")
    ap.add_argument("--b", default="12=0,1,2,3")
    ap.add_argument("--reps", type=int, default=15)
    args = ap.parse_args()
    import numpy as np
    import torch

    import bench
    from paper_2211_15082_b200 import _lib, kernels, synth
    from paper_2211_15082_b200.executor import conv_bytes

    dev = torch.device("cuda", 0)
    if args.graph == "papers":
        n = args.nodes or 20_000_000
        g = synth.gen_products_like(n, int(round(n * synth.PAPERS_EDGES / 2 / synth.PAPERS_NODES)),
                                    seed=0, device="cuda")
    else:
        n, und = bench.sizes(argparse.Namespace(nodes=args.nodes, undirected=None))
        g, _ = bench.device_inputs(n, und, 100, dev)
    d_in, d_out = (int(v) for v in args.shape.split("x"))
    h = torch.randn((n, d_in), device=dev)
    rng = np.random.default_rng(0)
    W = torch.from_numpy((rng.normal(size=(d_out, d_in)) / np.sqrt(d_in)).astype(np.float32)).to(dev)
    b = torch.from_numpy(rng.normal(size=d_out).astype(np.float32)).to(dev)
    sched, _ = kernels.degree_schedule(g.indptr, None, 0, n)
    out = torch.empty((n, d_out), device=dev)
    ka, va = args.a.split("=")
    kb, vb = args.b.split("=")
    ref = None
    fb = conv_bytes(d_in, d_out, g.num_edges, n)
    cells = [(int(x), int(y)) for x in va.split(",") for y in vb.split(",")]
    times = {c: [] for c in cells}
    equal = {c: True for c in cells}
    # cells interleaved round-robin so clock / power drift hits them alike
    for rep in range(args.reps + 1):
        for c in cells:
            _lib.call("glint_set_tuning", int(ka), c[0])
            _lib.call("glint_set_tuning", int(kb), c[1])
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            kernels.conv_mean(out, h, W, b, _lib.ACT_RELU, g.indptr, g.indices, n, schedule=sched)
            e1.record()
            torch.cuda.synchronize()
            if ref is None:
                ref = out.clone()
            equal[c] = equal[c] and bool(torch.equal(out, ref))
            if rep:
                times[c].append(e0.elapsed_time(e1))
    for c in cells:
        ms = float(np.median(times[c]))
        print(json.dumps({"graph": args.graph, "nodes": n, "edges": g.num_edges, "shape": args.shape,
                          f"knob{ka}": c[0], f"knob{kb}": c[1], "ms": round(ms, 3),
                          "gbs": round(fb / (ms / 1e3) / 1e9, 1), "reps": args.reps,
                          "min_ms": round(min(times[c]), 3), "bytes_equal": equal[c]}), flush=True)
    _lib.call("glint_set_tuning", int(ka), 0)
    _lib.call("glint_set_tuning", int(kb), 0)


if __name__ == "__main__":
    main()
