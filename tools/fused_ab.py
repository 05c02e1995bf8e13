"""A/B of K7 (fused aggregate -> transform) against K1 + K2 on the cfg2 graph.

Part 1, one aggregate-first ConvMean over every node (layer 1: 100 -> 256 and
a 128 -> 256 / 128 -> 128 variant on 128-wide features), CUDA-event timed,
interleaved, with the outputs compared byte for byte.  Part 2, the whole
3-layer cfg2 step through the engine with K7 on and off (interleaved).

    python tools/fused_ab.py [--nodes N] [--reps 5] > profiles/r02_fused_ab.jsonl
"""

from __future__ import annotations

import argparse
import json
import pathlib
import sys

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nodes", type=int, default=None)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--no-step", action="store_true")
    ap.add_argument("--variants", default="0", help="GLINT_TUNE_FUSED_VARIANT values (comma list)")
    ap.add_argument("--knob", type=int, default=12,
                    help="tuning knob --variants sweeps (12 FUSED_VARIANT, 19 FUSED_PIPE)")
    ap.add_argument("--shapes", default="100x256,128x256,128x128,100x47")
    ap.add_argument("--graph", default="products", choices=("products", "papers"),
                    help="papers: gen_products_like at cfg5's average degree (--nodes, "
                         "default 20M), features 128-wide")
    args = ap.parse_args()
    import numpy as np
    import torch

    import bench
    from paper_2211_15082_b200 import _lib, kernels
    from paper_2211_15082_b200.executor import agg_bytes, conv_bytes
    from paper_2211_15082_b200.storage import pitch_of

    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    if args.graph == "papers":
        from paper_2211_15082_b200 import synth

        n = args.nodes or 20_000_000
        und = int(round(n * synth.PAPERS_EDGES / 2 / synth.PAPERS_NODES))
        g = synth.gen_products_like(n, und, seed=0, device="cuda")
        x100 = torch.randn((n, 100), device=dev)
        args.no_step = True
    else:
        n, und = bench.sizes(argparse.Namespace(nodes=args.nodes, undirected=None))
        g, x100 = bench.device_inputs(n, und, 100, dev)
    E = g.num_edges
    sched, n_hub = kernels.degree_schedule(g.indptr, None, 0, n)
    n_hub = int(n_hub.item())
    rng = np.random.default_rng(0)

    def ev():
        return torch.cuda.Event(enable_timing=True)

    import ctypes

    lib = _lib.load()
    shapes = [tuple(int(v) for v in sh.split("x")) for sh in args.shapes.split(",")]
    tt = []
    for rep in range(6):
        a0, a1, a2 = ev(), ev(), ev()
        a0.record()
        sc2, nh2 = kernels.degree_schedule(g.indptr, None, 0, n)
        a1.record()
        torch.arange(0, n, device=dev, dtype=torch.int64)
        a2.record()
        torch.cuda.synchronize()
        tt.append((round(a0.elapsed_time(a1), 4), round(a1.elapsed_time(a2), 4)))
    print(json.dumps({"part": "schedule", "ms_sched_arange": tt,
                      "equal": bool(torch.equal(sc2, sched))}), flush=True)
    for (d_in, d_out), var in [(sh, int(v)) for sh in shapes for v in args.variants.split(",")]:
        lib.glint_set_tuning(args.knob, var)
        h = x100 if d_in == 100 else torch.randn((n, d_in), device=dev)
        W = torch.from_numpy((rng.normal(size=(d_out, d_in)) / np.sqrt(d_in)).astype(np.float32)).to(dev)
        b = torch.from_numpy(rng.normal(size=d_out).astype(np.float32)).to(dev)
        agg = torch.empty((n, pitch_of(d_in)), device=dev)[:, :d_in]
        o1 = torch.empty((n, pitch_of(d_out)), device=dev)[:, :d_out]
        o2 = torch.empty((n, pitch_of(d_out)), device=dev)[:, :d_out]
        t_un, t_k1, t_fu = [], [], []
        for rep in range(args.reps + 1):
            a0, a1, a2, b0, b1 = ev(), ev(), ev(), ev(), ev()
            a0.record()
            kernels.spmm_mean(agg, h, g.indptr, g.indices, n, schedule=sched, n_hub=n_hub)
            a1.record()
            kernels.linear_into(o1, agg, W, b, _lib.ACT_RELU, precision=_lib.PREC_3XTF32)
            a2.record()
            b0.record()
            kernels.conv_mean(o2, h, W, b, _lib.ACT_RELU, g.indptr, g.indices, n, schedule=sched)
            b1.record()
            torch.cuda.synchronize()
            if rep:
                t_k1.append(a0.elapsed_time(a1))
                t_un.append(a0.elapsed_time(a2))
                t_fu.append(b0.elapsed_time(b1))
        equal = bool(torch.equal(o1.contiguous().view(torch.int32), o2.contiguous().view(torch.int32)))
        # one more launch with the phase counters on
        lib.glint_set_tuning(13, 1)
        cnt = (ctypes.c_uint64 * 8)()
        lib.glint_debug_counters(1, cnt, 0, 1)
        kernels.conv_mean(o2, h, W, b, _lib.ACT_RELU, g.indptr, g.indices, n, schedule=sched)
        torch.cuda.synchronize()
        lib.glint_debug_counters(1, cnt, 8, 1)
        lib.glint_set_tuning(13, 0)
        loop = max(cnt[0], 1)
        prof = {"stage_wait_frac": round(cnt[1] / loop, 4), "tile_wait_frac": round(cnt[2] / loop, 4),
                "rows": int(cnt[3]), "tiles": int(cnt[4])}
        fb = conv_bytes(d_in, d_out, E, n)
        print(json.dumps({
            "part": "layer", "knob": args.knob, "variant": var, "d_in": d_in, "d_out": d_out, "nodes": n, "edges": E,
            "prof": prof,
            "unfused_ms": round(float(np.median(t_un)), 4), "k1_ms": round(float(np.median(t_k1)), 4),
            "fused_ms": round(float(np.median(t_fu)), 4),
            "fused_all_ms": [round(t, 3) for t in t_fu], "unfused_all_ms": [round(t, 3) for t in t_un],
            "bytes_equal": equal, "fused_algorithmic_bytes": fb,
            "fused_gbs": round(fb / (float(np.median(t_fu)) / 1e3) / 1e9, 1),
            "k1_gbs": round(agg_bytes(d_in, E, n) / (float(np.median(t_k1)) / 1e3) / 1e9, 1)}),
            flush=True)
        del agg, o1, o2
        torch.cuda.empty_cache()

    lib.glint_set_tuning(args.knob, 0)
    if args.no_step:
        return
    m = bench.build_model("gcn3")
    run = bench.Runner(m, g, x100, 1, 0)
    outs = {}
    for fuse in (True, False):
        kernels.FUSE_CONV = fuse
        outs[fuse] = run.step().data.clone()
    times = {True: [], False: []}
    for rep in range(args.reps + 1):
        for fuse in (True, False):
            kernels.FUSE_CONV = fuse
            torch.cuda.synchronize()
            a, b2 = ev(), ev()
            a.record()
            run.step()
            b2.record()
            torch.cuda.synchronize()
            if rep:
                times[fuse].append(a.elapsed_time(b2))
    from paper_2211_15082_b200.executor import KernelProbe

    import os

    for reserve in (4, 8, 16):
        os.environ["GLINT_FUSED_RESERVE_SMS"] = str(reserve)
        tt = []
        for rep in range(args.reps + 1):
            torch.cuda.synchronize()
            a, b2 = ev(), ev()
            a.record()
            run.step()
            b2.record()
            torch.cuda.synchronize()
            if rep:
                tt.append(a.elapsed_time(b2))
        print(json.dumps({"part": "reserve", "reserve_sms": reserve,
                          "ms": round(float(np.median(tt)), 3), "all_ms": [round(t, 3) for t in tt]}),
              flush=True)
    os.environ["GLINT_FUSED_RESERVE_SMS"] = "8"
    probes = {}
    for fuse in (True, False, True, False):
        kernels.FUSE_CONV = fuse
        pr = KernelProbe()
        torch.cuda.synchronize()
        run.step(pr)
        torch.cuda.synchronize()
        probes[fuse] = {"launches": [(nm, round(ms, 3)) for nm, _, ms in pr.launches()],
                        "timeline": [(nm, round(ms, 3)) for nm, ms in pr.timeline()]}
    for fuse in (True, False):
        print(json.dumps({"part": "step_probe", "fused": fuse, **probes[fuse]}), flush=True)
    kernels.FUSE_CONV = True
    print(json.dumps({
        "part": "step", "model": "gcn3", "nodes": n,
        "fused_ms": round(float(np.median(times[True])), 3),
        "unfused_ms": round(float(np.median(times[False])), 3),
        "fused_all_ms": [round(t, 3) for t in times[True]],
        "unfused_all_ms": [round(t, 3) for t in times[False]],
        "output_bytes_equal": bool(torch.equal(outs[True], outs[False]))}), flush=True)


if __name__ == "__main__":
    main()
