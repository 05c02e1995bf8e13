#!/usr/bin/env python
"""Benchmark: full-graph layer-wise GNN inference on B200 (BASELINE.json metric).

Workload (BASELINE.json configs[1], "cfg2"): 3-layer GCN -- ConvMean
100 -> 256 -> 256 -> 47 with ReLU between layers (glint build_gcn) -- full
inference over an OGBN-Products-shaped synthetic graph: 2,449,029 nodes,
61,859,140 undirected edges stored both ways = 123,718,280 in-edges,
heavy-tailed degrees (synth.gen_products_like), N(0,1) fp32 features,
random-init weights.  A "step" is one complete inference pass (all three
layers, all batches, batch planning included).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

value  = nodes/s of the device-resident step (graph, features, weights already
         in HBM; max over ranks of the CUDA-event time of K steps).
e2e    = the same metric through the public API run_inference() from pinned
         host buffers: H2D of graph + features and D2H of the output inside
         the timed region.
roofline = the dominant kernel (mean aggregation), achieved algorithmic bytes
         (SURVEY §8d B_agg per launch) / measured launch time vs the measured
         HBM copy peak (MEASURED_PEAKS.json).
cpu_baseline / --impl reference = the CPU oracle (numpy restatement of the
         reference hot path, single-threaded like the reference) timed on a
         bounded sample of the same workload on this host.
Multi-GPU (torchrun): nodes are row-partitioned edge-balanced, each layer's
stored output is exchanged over NCCL (strong scaling: total work fixed).
"""

from __future__ import annotations

import argparse
import json
import os
import pathlib
import statistics
import sys
import threading
import time

ROOT = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "full-graph layer-wise inference nodes/s; aggregation HBM GB/s vs peak"
UNIT = "nodes/s"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", choices=["b200", "reference"], default="b200")
    p.add_argument("--model", choices=["gcn3", "gat3"], default="gcn3")
    p.add_argument("--nodes", type=int, default=None)
    p.add_argument("--undirected", type=int, default=None)
    p.add_argument("--precision", choices=["fp32", "3xtf32"], default=None)
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--cpu-sample", type=int, default=None, help="target nodes per layer")
    p.add_argument("--tune", action="append", default=[],
                   help="diagnostics: glint_set_tuning KEY=VALUE (performance knobs only)")
    p.add_argument("--timeline", action="store_true",
                   help="diagnostics: add per-batch GPU timeline of the last timed step")
    return p.parse_args()


# ------------------------------------------------------------------ setup --


def dist_setup(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # GLINT_DIST_BACKEND=gloo runs several ranks on one GPU (NCCL refuses
    # duplicate devices): a functional check of the multi-rank path on a
    # 1-GPU box, not a performance configuration.
    backend = os.environ.get("GLINT_DIST_BACKEND") or ("nccl" if torch.cuda.is_available() else "gloo")
    if torch.cuda.is_available():
        local = local % torch.cuda.device_count()
        torch.cuda.set_device(local)
    if world > 1 and not dist.is_initialized():
        dist.init_process_group(backend)
    return rank, world, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def max_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([float(x)], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def workload(args):
    from paper_2211_15082_b200 import synth

    n = args.nodes or synth.PRODUCTS_NODES
    und = args.undirected or (synth.PRODUCTS_UNDIRECTED if args.nodes is None
                              else int(round(n * synth.PRODUCTS_UNDIRECTED / synth.PRODUCTS_NODES)))
    if args.model == "gcn3":
        m = synth.build_gcn(100, 256, 47, 3, seed=0)
        desc = "3-layer GCN (ConvMean 100->256->256->47, ReLU)"
    else:
        m = synth.build_gat(100, 64, 47, 3, heads=4, seed=0)
        desc = "3-layer GAT, 4 heads (ConvAttn 100->4x64->4x64->4x47, ReLU)"
    return n, und, m, desc


def make_graph_and_features(n, und, dim):
    from paper_2211_15082_b200 import synth

    g = synth.gen_products_like(n, und, seed=0, device="cuda")
    x = synth.gen_features_device(n, dim, seed=0, device="cuda")
    return g, x


# ----------------------------------------------------------------- clocks --


class ClockSampler:
    """nvidia-smi style sampling of SM clock and throttle reasons via NVML."""

    REASONS = {
        "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4,
        "hw_slowdown": 0x8, "sync_boost": 0x10, "sw_thermal_slowdown": 0x20,
        "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80,
        "display_clock_setting": 0x100,
    }

    def __init__(self, index, period=0.05):
        self.index, self.period = index, period
        self.samples, self.reasons = [], set()
        self._stop = threading.Event()
        self._t = None
        self.max_mhz = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:  # noqa: BLE001 - clocks are best effort
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                mask = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for name, bit in self.REASONS.items():
                    if mask & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:  # noqa: BLE001
                pass
            self._stop.wait(self.period)

    def __enter__(self):
        if self.nv is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._t is not None:
            self._t.join()

    def report(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ------------------------------------------------------------ CPU oracle --


def cpu_sample_rate(indptr, indices, m, sample_nodes, seed=0):
    """Time the oracle (reference algorithm, numpy, 1 thread) on a contiguous
    sample of targets per layer; returns (nodes/s, seconds, description)."""
    import numpy as np

    from oracle import glint_oracle as orc

    n = len(indptr) - 1
    convs = [m.operators[o] for o in m.topo_order if m.operators[o].is_conv]
    rng = np.random.default_rng(seed)
    lo = n // 2
    targets = np.arange(lo, min(n, lo + sample_nodes), dtype=np.int64)
    per_layer = []
    stores = {}
    for op in convs:
        d_in = (op.params["weight"].shape[1] if op.kind == "ConvMean"
                else op.params["weight"].shape[2])
        if d_in not in stores:      # a full-size host embedding store (random rows, tiled)
            block = rng.standard_normal((1 << 16, d_in), dtype=np.float32)
            stores[d_in] = np.resize(block, (n, d_in))
        h_store = stores[d_in]
        t0 = time.perf_counter()
        bc = orc.build_batch_csc(indptr, indices, targets)          # plan (kernels.py:71-77)
        h = h_store[bc.input_ids]                                    # store gather (executor.py:353)
        if op.kind == "ConvMean":
            out = orc.linear(orc.agg_mean(bc, h), op.params["weight"], op.params.get("bias"))
        else:
            out = orc.agg_attn(bc, h, op.params["weight"], op.params["attn"])
        out = orc.elementwise("ReLU", [out])
        per_layer.append(time.perf_counter() - t0)
    total = sum(per_layer)
    rate = len(targets) / total
    desc = (f"{len(targets)} contiguous targets [{lo}, {lo + len(targets)}) per layer, all "
            f"{len(convs)} layers (build_batch_csc + gather + aggregate + transform + ReLU); "
            f"per-layer s {['%.2f' % t for t in per_layer]}")
    return rate, total, desc


def host_csc(g):
    import numpy as np

    return g.indptr_host, g.indices.cpu().numpy().astype(np.int64)


# ------------------------------------------------------------- reference --


def run_reference(args, rank, world):
    if rank != 0:
        return
    import numpy as np

    n, und, m, desc = workload(args)
    g, _x = make_graph_and_features(n, und, m.input_dim)
    indptr, indices = host_csc(g)
    del g, _x
    sample = args.cpu_sample or 4096
    for _ in range(max(args.warmup, 0)):
        cpu_sample_rate(indptr, indices, m, min(sample, 1024))
    rates, secs = [], []
    for k in range(args.steps):
        r, s, sdesc = cpu_sample_rate(indptr, indices, m, sample, seed=k)
        rates.append(r)
        secs.append(s)
    value = len(rates) / sum(1.0 / r for r in rates)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000 * statistics.mean(secs), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "impl": "reference",
        "config": config_block(args, n, und, desc, world),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "port",
                         "sample": sdesc},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def config_block(args, n, und, desc, world):
    # cfg5 (Papers100M-shaped, 1.6B edges) runs in tools/bench_papers.py: its
    # features cannot stay resident next to the layer-3 output on one GPU.
    cfg = "cfg2" if args.model == "gcn3" else "cfg3"
    din, dh = 100, 256
    return {"workload": f"{cfg} {desc} full inference, OGBN-Products-shaped graph",
            "nodes": n, "in_edges": 2 * und, "gnn": args.model, "mode": "full",
            "order": "none", "budget": "device (free HBM after resident stores)",
            "l2": "inputs larger than L2 (features %.2f GB, hidden %.2f GB per layer)"
                  % (n * din * 4 / 1e9, n * dh * 4 / 1e9),
            "parallelism": f"row-partition x{world}" + (" + NCCL per-layer exchange"
                                                        if world > 1 else "")}


# -------------------------------------------------------------------- b200 --


def main():
    args = parse()
    rank, world, local = dist_setup(args)
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    import numpy as np
    import torch

    from paper_2211_15082_b200 import _lib, kernels
    from paper_2211_15082_b200.batching import Thresholds
    from paper_2211_15082_b200.device import DeviceBudget
    from paper_2211_15082_b200.executor import (KernelProbe, LayerwiseEngine, RunStats,
                                                _as_device_store, _resident_bytes, annotate)
    from paper_2211_15082_b200.parallel import RowExchange, edge_balanced_ranges
    from paper_2211_15082_b200.splitter import split

    _lib.load()
    if args.precision:
        kernels.PRECISION = _lib.PREC_3XTF32 if args.precision == "3xtf32" else _lib.PREC_FP32
    for kv in args.tune:
        k, v = kv.split("=")
        _lib.call("glint_set_tuning", int(k), int(v))
    dev = torch.device("cuda", local)
    n, und, m, desc = workload(args)
    g, xt = make_graph_and_features(n, und, m.input_dim)
    x = _as_device_store(xt, dev)
    schedule = split(m)
    tsets = annotate(g, np.arange(0), m.depth, "full")
    resident = _resident_bytes(m, schedule, tsets, g)
    budget = DeviceBudget.from_device(reserve_bytes=resident + (2 << 30))
    budget = DeviceBudget(int(min_over_ranks(budget.capacity, world)))
    th0 = Thresholds(1024, 32768)
    cuts = edge_balanced_ranges(g.indptr_host, world)
    ex = RowExchange(cuts, rank, world) if world > 1 else None
    state = {"thresholds": th0}

    def step(probe=None):
        stats = RunStats("layerwise", "full", "none", m.depth, (th0.n_t, th0.n_i))
        eng = LayerwiseEngine(m, schedule, g, x, tsets, budget, th0, stats,
                              row_range=ex.row_range if ex else None)
        eng.probe = probe
        out = eng.run(exchange=ex)
        state["stats"] = stats
        return out

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    probe = KernelProbe()
    launches0 = _lib.LAUNCHES[0]
    barrier(world)
    torch.cuda.synchronize()
    with ClockSampler(local) as clocks:
        t_start = torch.cuda.Event(enable_timing=True)
        t_end = torch.cuda.Event(enable_timing=True)
        t_start.record()
        step_events = []
        for _ in range(args.steps):
            step(probe)
            ev = torch.cuda.Event(enable_timing=True)
            ev.record()
            step_events.append(ev)
        t_end.record()
        torch.cuda.synchronize()
        barrier(world)
    step_ms = [t_start.elapsed_time(step_events[0])] + [
        a.elapsed_time(b) for a, b in zip(step_events, step_events[1:])]
    launches = (_lib.LAUNCHES[0] - launches0) // max(args.steps, 1)
    ms = t_start.elapsed_time(t_end) / args.steps
    ms = max_over_ranks(ms, world)
    value = n / (ms / 1e3)

    summ = probe.summary()
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) \
        if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    agg_name = "spmm_mean" if args.model == "gcn3" else "gat_aggregate"
    cnt, nbytes, agg_ms = summ.get(agg_name, (0, 0, 0.0))
    achieved = (nbytes / (agg_ms / 1e3) / 1e9) if agg_ms else None
    lin = summ.get("linear", (0, 0, 0.0))
    roofline = {
        "kernel": agg_name, "bound": "hbm", "achieved": achieved, "peak": hbm_peak,
        "unit": "GB/s", "frac": (achieved / hbm_peak) if achieved else None,
        "traffic": traffic_from_profiles(agg_name),
        "traffic_basis": "DRAM read+write bytes per aggregation launch (regular + hub kernels), "
                         "ncu launch list of this bench step (profiles/ncu_traffic.json); "
                         "compare with algorithmic_bytes_per_launch",
        "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback 6.65 TB/s",
        "achieved_basis": "sum of SURVEY 8d B_agg over the step's aggregation launches / sum of "
                          "their CUDA-event durations (same stream)",
        "launches_per_step": cnt // max(args.steps, 1),
        "algorithmic_bytes_per_launch": nbytes // max(cnt, 1),
        "algorithmic_bytes_per_step": nbytes // max(args.steps, 1),
        "kernel_ms_per_step": agg_ms / max(args.steps, 1),
        "kernel_share_of_step": (agg_ms / args.steps) / ms if ms else None,
        "gemm_ms_per_step": lin[2] / max(args.steps, 1),
        "gemm_tflops": (lin[1] / (lin[2] / 1e3) / 1e12) if lin[2] else None,
    }
    st = state["stats"]
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": config_block(args, n, und, desc, world),
        "batches_per_step": st.batches,
        "layer_batches": st.layer_batches,
        "roofline": roofline, "gpu_launches": launches, "clocks": clocks.report(),
        "step_ms": [round(t, 3) for t in step_ms],
        **({"tuning": args.tune} if args.tune else {}),
        **({"timeline_ms": [(n, round(t, 3)) for n, t in probe.timeline()],
            "launch_ms": [(n, round(t, 4), round(b / t / 1e6, 1) if n != "linear"
                           else round(b / t / 1e9, 1)) for n, b, t in probe.launches()]}
           if args.timeline else {}),
    }
    line["config"]["capacity_bytes"] = budget.capacity
    line["config"]["gemm_precision"] = "3xtf32" if kernels.PRECISION == _lib.PREC_3XTF32 else "fp32"
    if not args.no_e2e:
        line["e2e"] = run_e2e(args, m, g, xt, budget, world, rank, ex)
    del x
    if rank == 0 and world == 1 and not args.no_cpu:
        indptr, indices = host_csc(g)
        sample = args.cpu_sample or 32768      # ~10 s of single-core CPU work
        rate, secs, sdesc = cpu_sample_rate(indptr, indices, m, sample)
        line["cpu_baseline"] = {"value": rate, "unit": UNIT, "cores": 1, "kind": "port",
                                "sample": sdesc, "seconds": secs,
                                "host_cpus": os.cpu_count()}
    if rank == 0:
        print(json.dumps(line), flush=True)
    barrier(world)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


def min_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([float(x)], device="cuda", dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    return t.item()


def traffic_from_profiles(kernel):
    """DRAM bytes per launch from the committed ncu capture summary, if any."""
    p = ROOT / "profiles" / "ncu_traffic.json"
    if not p.exists():
        return None
    try:
        return json.loads(p.read_text()).get(kernel, {}).get("dram_bytes_per_launch")
    except Exception:  # noqa: BLE001
        return None


def run_e2e(args, m, g, xt, budget, world, rank, ex):
    """Same metric through the public API run_inference from pinned host buffers."""
    import torch

    from paper_2211_15082_b200.executor import run_inference
    from paper_2211_15082_b200.storage import CscGraph

    n = g.num_nodes
    ip = torch.empty(n + 1, dtype=torch.int64, pin_memory=True)
    ip.copy_(torch.from_numpy(g.indptr_host))
    ix = torch.empty(g.num_edges, dtype=torch.int64, pin_memory=True)
    ix.copy_(g.indices.to(torch.int64).cpu())
    xh = torch.empty(tuple(xt.shape), dtype=torch.float32, pin_memory=True)
    xh.copy_(xt.cpu())
    host_graph = CscGraph(n, g.num_edges, ip.numpy(), ix.numpy())
    h2d = ip.numel() * 8 + ix.numel() * 8 + xh.numel() * 4
    d2h = n * m.output_dim * 4
    steps = max(1, min(args.steps, 3))
    for _ in range(1):
        run_inference(m, host_graph, xh, budget=budget, output="numpy")
    barrier(world)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = None
    for _ in range(steps):
        res = None      # the caller is done with the previous result (recycles pinned staging)
        res = run_inference(m, host_graph, xh, budget=budget, output="numpy")
    torch.cuda.synchronize()
    barrier(world)
    dt = (time.perf_counter() - t0) / steps
    dt = max_over_ranks(dt, world)
    assert res.output.shape == (n, m.output_dim)
    return {"value": n / dt, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "ms_per_step": dt * 1e3, "steps": steps, "api": "executor.run_inference",
            "host_buffers": "pinned torch CPU tensors (graph int64 CSC, fp32 features)"}


if __name__ == "__main__":
    main()
