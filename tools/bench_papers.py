#!/usr/bin/env python
"""cfg5 on ONE B200: full 3-layer GCN inference on a Papers100M-shaped graph.

BASELINE.json configs[4] has N = 111,059,956 nodes, E = 1,615,685,872 in-edges,
128-dim fp32 features and build_gcn(128, 128, 172, 3).  The paper splits this
graph across 8 GPUs; here it runs on a single 180 GB B200.  The graph is
generated on the device (synth.gen_products_like: seeded Chung-Lu, symmetric,
heavy-tailed).  The CSR is int64 indptr 0.9 GB plus int32 indices 6.5 GB.

Per step, untimed: the features are drawn again (57 GB).
Per step, timed (CUDA events): one full layer-wise pass.  The engine owns x and
frees it after layer 1, so the peak is layer 3's H2 (57 GB) + output (76 GB) +
CSR + one batch.  Every other step keeps x resident, which would need 199 GB.

Output: one JSON line with nodes/s, the aggregation's achieved GB/s over
SURVEY 8d algorithmic bytes, per-layer times, batches and peak memory.

    python tools/bench_papers.py [--nodes N] [--steps K] [--warmup W] [--capacity-gib C]
"""

from __future__ import annotations

import argparse
import json
import pathlib
import sys
import time

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def run(nodes=None, steps=2, warmup=1, capacity_gib=64.0, keep_cache=True):
    """The cfg5 measurement as a dict (bench.py's cfg5 secondary calls this)."""
    import numpy as np
    import torch

    from paper_2211_15082_b200 import _lib, synth
    from paper_2211_15082_b200.batching import Thresholds
    from paper_2211_15082_b200.device import DeviceBudget
    from paper_2211_15082_b200.executor import (KernelProbe, LayerwiseEngine, RunStats,
                                                _as_device_store, annotate)
    from paper_2211_15082_b200.splitter import split

    _lib.load()
    dev = torch.device("cuda", 0)
    n = nodes or synth.PAPERS_NODES
    und = int(round(n * synth.PAPERS_EDGES / 2 / synth.PAPERS_NODES))
    t0 = time.perf_counter()
    g = synth.gen_products_like(n, und, seed=0, device="cuda")
    torch.cuda.synchronize()
    gen_s = time.perf_counter() - t0
    torch.cuda.empty_cache()
    m = synth.build_gcn(128, 128, 172, 3, seed=0)
    schedule = split(m)
    tsets = annotate(g, np.arange(0), m.depth, "full")
    budget = DeviceBudget(int(capacity_gib * (1 << 30)))
    th0 = Thresholds(1024, 32768)
    per_step = []
    summ = None
    for i in range(warmup + steps):
        x = _as_device_store(synth.gen_features_device(n, 128, seed=i, device="cuda"), dev)
        torch.cuda.synchronize()
        torch.cuda.reset_peak_memory_stats()
        stats = RunStats("layerwise", "full", "none", m.depth, (th0.n_t, th0.n_i))
        eng = LayerwiseEngine(m, schedule, g, x, tsets, budget, th0, stats, release_input=True,
                              reassociate=True)
        del x
        probe = KernelProbe()
        eng.probe = probe
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        out = eng.run()
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e)
        if i >= warmup:
            summ = probe.summary()
            per_step.append({"ms": ms, "layers": [(nm, round(t, 2)) for nm, t in probe.timeline()],
                             "batches": stats.batches, "layer_batches": stats.layer_batches,
                             "peak_alloc_gib": torch.cuda.max_memory_allocated() / 2 ** 30})
        del out, eng
        if not keep_cache:
            torch.cuda.empty_cache()
    n_edges = int(g.num_edges)
    del g
    torch.cuda.empty_cache()
    ms = float(np.mean([st["ms"] for st in per_step]))
    per = [summ.get(k, (0, 0, 0.0)) for k in ("spmm_mean", "conv_mean")]
    cnt, nbytes, agg_ms = (sum(v[i] for v in per) for i in range(3))
    lin = summ.get("linear", (0, 0, 0.0))
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) \
        if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    peak = peaks.get("hbm_gbs", 6650.0)
    return {
        "workload": "cfg5 3-layer GCN (ConvMean 128->128->128->172, ReLU) full inference, "
                    "OGBN-Papers100M-shaped graph, 1 B200",
        "nodes": n, "in_edges": n_edges,
        "graph_gen_s": round(gen_s, 1),
        "value": n / (ms / 1e3), "unit": "nodes/s", "ms_per_step": ms, "steps": steps,
        "warmup": warmup,
        "aggregation": {"kernels": {k: v for k, v in summ.items() if k != "linear"},
                        "launches": cnt, "algorithmic_bytes": nbytes, "ms": agg_ms,
                        "achieved_gbs": nbytes / (agg_ms / 1e3) / 1e9 if agg_ms else None,
                        "frac_of_peak": (nbytes / (agg_ms / 1e3) / 1e9 / peak) if agg_ms else None,
                        "peak_gbs": peak},
        "gemm": {"ms": lin[2], "tflops": lin[1] / (lin[2] / 1e3) / 1e12 if lin[2] else None},
        "capacity_gib": capacity_gib, "per_step": per_step,
        "allocator": ("caching allocator kept between steps (steady state)" if keep_cache
                      else "empty_cache between steps (every step allocates its stores)"),
        "data": "synthetic (device generator, random-init weights)"}


def main():
    from paper_2211_15082_b200 import synth

    ap = argparse.ArgumentParser()
    ap.add_argument("--nodes", type=int, default=synth.PAPERS_NODES)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--warmup", type=int, default=1)
    ap.add_argument("--capacity-gib", type=float, default=64.0,
                    help="batch footprint capacity (the batch controller's budget)")
    ap.add_argument("--empty-cache", action="store_true",
                    help="release the caching allocator's blocks between steps, so every "
                         "step pays cudaMalloc of its 57-76 GB stores (tools/cfg5_cache_ab.sh)")
    args = ap.parse_args()
    print(json.dumps(run(args.nodes, args.steps, args.warmup, args.capacity_gib, not args.empty_cache)),
          flush=True)


if __name__ == "__main__":
    main()
