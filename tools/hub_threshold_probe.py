"""How many leading schedule rows should go to the hub kernels?  K1 and K4
whole-layer launches on the cfg2/cfg3 graph with the hub count taken at
deg+1 >= T for T in 512 ... 65536 (the schedule is longest-first, so every
T is a prefix of the same order), CUDA-event timed, interleaved, bytes
compared with T = 512.

    python tools/hub_threshold_probe.py > profiles/r02_hub_threshold.jsonl
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
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    import numpy as np
    import torch

    import bench
    from paper_2211_15082_b200 import kernels

    dev = torch.device("cuda", 0)
    n, und = bench.sizes(argparse.Namespace(nodes=None, undirected=None))
    g, _x = bench.device_inputs(n, und, 100, dev)
    del _x
    degs = np.diff(g.indptr_host)
    sched, _ = kernels.degree_schedule(g.indptr, None, 0, n)
    thresholds = (512, 1024, 2048, 4096, 8192, 65536)
    hubs = {t: int((degs + 1 >= t).sum()) for t in thresholds}
    # the schedule buckets by floor(log2(deg+1)), so the rows with deg+1 >= T
    # (T a power of two) are exactly its first hubs[T] entries

    def ev():
        return torch.cuda.Event(enable_timing=True)

    cases = [("k1", 256), ("k1", 48), ("k4", 64), ("k4", 47)]
    for kind, width in cases:
        if kind == "k1":
            h = torch.randn((n, width), device=dev)
            out = torch.empty((n, width), device=dev)
            heads = None
        else:
            heads, dh = 4, width
            hp = kernels.head_pitch(dh)
            h = torch.randn((n, heads * hp), device=dev)
            h.view(n, heads, hp)[:, :, dh:] = 0
            s_src = torch.randn((n, heads), device=dev)
            s_dst = torch.randn((n, heads), device=dev)
            out = torch.empty((n, heads * dh), device=dev)

        def run(nh):
            if kind == "k1":
                kernels.spmm_mean(out, h, g.indptr, g.indices, n, schedule=sched, n_hub=nh)
            else:
                kernels.gat_aggregate(out, h, s_src, s_dst, heads, dh, g.indptr, g.indices, n,
                                      schedule=sched, n_hub=nh, act=1)

        ref = None
        times = {t: [] for t in thresholds}
        for rep in range(args.reps + 1):
            for t in thresholds:
                a, b = ev(), ev()
                a.record()
                run(hubs[t])
                b.record()
                torch.cuda.synchronize()
                if rep:
                    times[t].append(a.elapsed_time(b))
                if ref is None:
                    ref = out.clone()
                elif rep == 0:
                    assert torch.equal(out, ref), (kind, width, t)
        print(json.dumps({"kernel": kind, "width": width, "hub_rows": hubs,
                          "ms": {t: round(float(np.median(v)), 3) for t, v in times.items()},
                          "bytes_equal": True}), flush=True)
        del h, out
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
