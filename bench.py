#!/usr/bin/env python
"""Benchmark: full-graph layer-wise GNN inference on B200 (BASELINE.json metric).

Workload (BASELINE.json configs[1], "cfg2"): 3-layer GCN -- ConvMean
100 -> 256 -> 256 -> 47 with ReLU between layers (glint build_gcn) -- full
inference over an OGBN-Products-shaped synthetic graph: 2,449,029 nodes,
61,859,140 undirected edges stored in both directions = 123,718,280 in-edges,
heavy-tailed degrees, N(0,1) fp32 features, random-init weights.  The inputs
come from workload.py, which both arms share and which never touches the
product package.  A "step" is one complete inference pass: all three layers,
all batches, and the batch planning.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

value  = nodes/s of the device-resident step: graph, features and weights
         are already in HBM; max over ranks of the CUDA-event time of K steps.
e2e    = the same metric through the public API run_inference(), from pinned
         host buffers.  The H2D of graph + features and the D2H of the output
         are inside the timed region.
roofline = the dominant kernel (the aggregation): achieved algorithmic bytes
         (SURVEY 8d B_agg per launch) / measured launch time, against the
         measured HBM copy peak (MEASURED_PEAKS.json).
parity = outside the timed region: each layer of one more step is checked
         against the CPU oracle on >= 4096 random targets plus the top-50 hub
         rows, fed with the device's own H^{l-1}.  K1 bytes must be equal, the
         conv rows are compared by rel-L2, and the batch records are compared
         with a plan-only replay of the reference controller at the same
         capacity.
secondary (N=1) = cfg3 (3-layer GAT, 4 heads) measured the same way, and
         cfg2 on the RCMK-relabelled graph (the relabelling is one-time and
         outside the timed region).
cpu_baseline / --impl reference = the CPU oracle (the numpy restatement of the
         reference hot path, single-threaded like the reference) timed on a
         bounded sample of the same workload on this host.  The reference arm
         imports neither the product package nor its library.
Multi-GPU (torchrun): nodes are row-partitioned edge-balanced, and each
layer's stored output is exchanged over NCCL.  This is strong scaling: the
total work is fixed.
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

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "full-graph layer-wise inference nodes/s; aggregation HBM GB/s vs peak"
UNIT = "nodes/s"
DATA = "synthetic (workload.py: the same graph, features and weights in both arms)"


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
    p.add_argument("--no-parity", action="store_true")
    p.add_argument("--no-secondary", action="store_true")
    p.add_argument("--no-cfg5", action="store_true", help="skip the 1.6B-edge cfg5 secondary")
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


def _reduce(x, world, op, dtype):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([float(x)], device="cuda" if torch.cuda.is_available() else "cpu",
                     dtype=dtype)
    dist.all_reduce(t, op=op)
    return t.item()


def max_over_ranks(x, world):
    import torch
    import torch.distributed as dist

    return _reduce(x, world, dist.ReduceOp.MAX if world > 1 else None, torch.float64)


def min_over_ranks(x, world):
    import torch
    import torch.distributed as dist

    return _reduce(x, world, dist.ReduceOp.MIN if world > 1 else None, torch.float64)


# --------------------------------------------------------------- workload --


def sizes(args):
    import workload

    n = args.nodes or workload.PRODUCTS_NODES
    und = args.undirected or (workload.PRODUCTS_UNDIRECTED if args.nodes is None else int(
        round(n * workload.PRODUCTS_UNDIRECTED / workload.PRODUCTS_NODES)))
    return n, und


MODEL_DESC = {"gcn3": "3-layer GCN (ConvMean 100->256->256->47, ReLU)",
              "gat3": "3-layer GAT, 4 heads (ConvAttn 100->4x64->4x64->4x47, ReLU)"}


def layer_specs(model):
    """Package-free description of the model's convs (workload.py weights)."""
    import workload

    if model == "gcn3":
        ps = workload.gcn_params(100, 256, 47, 3, seed=0)
        return [{"kind": "ConvMean", "weight": w, "bias": b, "relu": i < len(ps) - 1}
                for i, (w, b) in enumerate(ps)]
    ps = workload.gat_params(100, 64, 47, 3, heads=4, seed=0)
    return [{"kind": "ConvAttn", "weight": w, "attn": a, "relu": i < len(ps) - 1}
            for i, (w, a) in enumerate(ps)]


def config_block(model, n, und, world, order="none"):
    """Identical in both arms (the driver compares them)."""
    cfg = "cfg2" if model == "gcn3" else "cfg3"
    din, dh = 100, 256
    return {"workload": f"{cfg} {MODEL_DESC[model]} full inference, OGBN-Products-shaped graph",
            "nodes": n, "in_edges": 2 * und, "gnn": model, "mode": "full", "order": order,
            "graph": "workload.products_like_csc(seed=0): Chung-Lu alpha 0.45, symmetric, "
                     "slices ascending",
            "features": "workload.features(seed=0): N(0,1) fp32",
            "l2": "inputs larger than L2 (features %.2f GB, hidden %.2f GB per layer)"
                  % (n * din * 4 / 1e9, n * dh * 4 / 1e9),
            "parallelism": f"row-partition x{world}" + (" + NCCL per-layer exchange"
                                                        if world > 1 else "")}


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


_CPU_CTX = {}


def _cpu_block_layers(bounds):
    """One worker: targets [lo, hi) through every layer of the sample (the
    reference's per-batch work, glint/executor.py:351-384).  Returns per-layer
    seconds."""
    import contextlib

    from oracle import glint_oracle as orc

    try:
        from threadpoolctl import threadpool_limits
        one_blas_thread = threadpool_limits(1)   # one BLAS thread per worker process
    except Exception:  # noqa: BLE001
        one_blas_thread = contextlib.nullcontext()
    c = _CPU_CTX
    targets = np.arange(bounds[0], bounds[1], dtype=np.int64)
    per_layer = []
    with one_blas_thread:
        for i, spec in enumerate(c["layers"]):
            h_store = c["x"] if i == 0 else c["stores"][spec["weight"].shape[-1]]
            t0 = time.perf_counter()
            bc = orc.build_batch_csc(c["indptr"], c["indices"], targets)   # kernels.py:71-77
            h = h_store[bc.input_ids]                                        # executor.py:353
            if spec["kind"] == "ConvMean":
                out = orc.linear(orc.agg_mean(bc, h), spec["weight"], spec.get("bias"))
            else:
                out = orc.agg_attn(bc, h, spec["weight"], spec["attn"])
            if spec["relu"]:
                out = orc.elementwise("ReLU", [out])
            per_layer.append(time.perf_counter() - t0)
    return per_layer


def cpu_sample_rate(indptr, indices, x_host, layers, per_worker, seed=0, workers=1):
    """Time the oracle (the reference algorithm, numpy) on contiguous blocks of
    targets, one block per worker process (`workers` host cores, forked, one
    BLAS thread each), every block through all layers the way the reference
    executes one batch.  Returns (nodes/s over the wall time, seconds,
    description).

    Layer 1 reads the real features.  Layers 2-3 read a full-size store of
    seeded random rows, because computing the true H^1 for every node is the
    whole CPU run this sample bounds."""
    import multiprocessing as mp

    n = len(indptr) - 1
    rng = np.random.default_rng(seed)
    lo = n // 2 - (workers * per_worker) // 2
    lo = max(0, lo)
    hi = min(n, lo + workers * per_worker)
    stores = {}
    for i, spec in enumerate(layers):
        d_in = spec["weight"].shape[-1]
        if i > 0 and d_in not in stores:      # full-size store of random rows (tiled)
            block = rng.standard_normal((1 << 16, d_in), dtype=np.float32)
            stores[d_in] = np.resize(block, (n, d_in))
    _CPU_CTX.update(indptr=indptr, indices=indices, x=x_host, layers=layers, stores=stores)
    cuts = np.linspace(lo, hi, workers + 1).astype(np.int64)
    blocks = [(int(cuts[k]), int(cuts[k + 1])) for k in range(workers)]
    if workers == 1:
        t0 = time.perf_counter()
        per = [_cpu_block_layers(blocks[0])]
        total = time.perf_counter() - t0
    else:
        with mp.get_context("fork").Pool(workers) as pool:   # forked before the clock starts
            pool.map(_cpu_block_layers, [(b[0], b[0] + 1) for b in blocks])   # warm the workers
            t0 = time.perf_counter()
            per = pool.map(_cpu_block_layers, blocks, chunksize=1)
            total = time.perf_counter() - t0
    _CPU_CTX.clear()
    rate = (hi - lo) / total
    layer_s = np.max(np.asarray(per), axis=0)
    desc = (f"{hi - lo} contiguous targets [{lo}, {hi}) in {workers} blocks of ~{per_worker}, "
            f"one forked worker process per host core, all {len(layers)} layers (build_batch_csc + "
            f"gather + aggregate + transform + ReLU); slowest worker's per-layer s "
            f"{['%.2f' % t for t in layer_s]}")
    return rate, total, desc


def cpu_workers() -> int:
    """Host cores the CPU arm uses: all of them (GLINT_CPU_WORKERS overrides)."""
    return max(1, int(os.environ.get("GLINT_CPU_WORKERS", os.cpu_count() or 1)))


def host_inputs(n, und, dim):
    """Host numpy (indptr, indices int64, features) from workload.py; drawn
    on the GPU when there is one (the same bytes the B200 arm uses)."""
    import torch

    import workload

    dev = "cuda" if torch.cuda.is_available() else "cpu"
    indptr, src = workload.products_like_csc(n, und, seed=0, device=dev)
    x = workload.features(n, dim, seed=0, device=dev)
    out = indptr.cpu().numpy(), src.cpu().numpy(), x.cpu().numpy()
    del indptr, src, x
    if dev == "cuda":
        torch.cuda.empty_cache()
    return out


def cpu_block(value, cores, sample, seconds=None):
    import workload

    return {"value": value, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample,
            **({"seconds": seconds} if seconds is not None else {}),
            "cpu_model": workload.cpu_model_name(), "host_cpus": os.cpu_count(),
            "threads_note": "the reference's hot ops (np.add.at, einsum, np.unique) are "
                            "single-threaded numpy; the arm runs one worker process per "
                            "host core on disjoint target blocks (the reference's batches "
                            "are independent), one BLAS thread each"}


# ------------------------------------------------------------- reference --


def run_reference(args, rank, world):
    """The CPU arm: oracle only -- no import of paper_2211_15082_b200."""
    if rank != 0:
        return
    n, und = sizes(args)
    layers = layer_specs(args.model)
    indptr, indices, x = host_inputs(n, und, 100)
    sample = args.cpu_sample or 4096          # targets per worker per step
    workers = cpu_workers()
    for _ in range(max(args.warmup, 0)):
        cpu_sample_rate(indptr, indices, x, layers, min(sample, 1024), workers=workers)
    rates, secs = [], []
    sdesc = ""
    for k in range(args.steps):
        r, s, sdesc = cpu_sample_rate(indptr, indices, x, layers, sample, seed=k, workers=workers)
        rates.append(r)
        secs.append(s)
    value = len(rates) / sum(1.0 / r for r in rates)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000 * statistics.mean(secs), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": DATA,
        "impl": "reference",
        "config": config_block(args.model, n, und, world),
        "cpu_baseline": cpu_block(value, workers, sdesc),
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# -------------------------------------------------------------------- b200 --


def device_inputs(n, und, dim, dev):
    """workload.py's graph and features, kept on the device."""
    import torch

    import workload
    from paper_2211_15082_b200 import kernels
    from paper_2211_15082_b200.storage import DeviceGraph

    indptr, src = workload.products_like_csc(n, und, seed=0, device=dev)
    indices = kernels.narrow_ids(src, n)
    del src
    g = DeviceGraph(n, int(indptr[-1].item()), indptr, indices, indptr.cpu().numpy())
    x = workload.features(n, dim, seed=0, device=dev)
    torch.cuda.empty_cache()
    return g, x


def build_model(model):
    from paper_2211_15082_b200 import synth

    if model == "gcn3":
        return synth.build_gcn(100, 256, 47, 3, seed=0)
    return synth.build_gat(100, 64, 47, 3, heads=4, seed=0)


class Runner:
    """The device-resident step of one (model, graph) and its measurements."""

    def __init__(self, m, g, x, world, local, ex=None):
        import numpy as np

        from paper_2211_15082_b200.batching import Thresholds
        from paper_2211_15082_b200.device import DeviceBudget
        from paper_2211_15082_b200.executor import _as_device_store, _resident_bytes, annotate
        from paper_2211_15082_b200.splitter import split

        self.m, self.g, self.world, self.local, self.ex = m, g, world, local, ex
        self.x = _as_device_store(x, g.indptr.device)
        self.schedule = split(m)
        self.tsets = annotate(g, np.arange(0), m.depth, "full")
        resident = _resident_bytes(m, self.schedule, self.tsets, g, reassociate=True)
        budget = DeviceBudget.from_device(reserve_bytes=resident + (2 << 30))
        self.budget = DeviceBudget(int(min_over_ranks(budget.capacity, world)))
        self.th0 = Thresholds(1024, 32768)
        self.stats = None

    def engine(self, probe=None):
        from paper_2211_15082_b200.executor import LayerwiseEngine, RunStats

        stats = RunStats("layerwise", "full", "none", self.m.depth, (self.th0.n_t, self.th0.n_i))
        eng = LayerwiseEngine(self.m, self.schedule, self.g, self.x, self.tsets, self.budget,
                              self.th0, stats, row_range=self.ex.row_range if self.ex else None,
                              reassociate=True)
        eng.probe = probe
        self.stats = stats
        return eng

    def step(self, probe=None):
        return self.engine(probe).run(exchange=self.ex)

    def measure(self, steps, warmup, agg_name, clocks=False):
        import torch

        from paper_2211_15082_b200 import _lib
        from paper_2211_15082_b200.executor import KernelProbe

        for _ in range(warmup):
            self.step()
        torch.cuda.synchronize()
        probe = KernelProbe()
        launches0 = _lib.LAUNCHES[0]
        barrier(self.world)
        torch.cuda.synchronize()
        sampler = ClockSampler(self.local) if clocks else None
        if sampler:
            sampler.__enter__()
        t_start = torch.cuda.Event(enable_timing=True)
        t_end = torch.cuda.Event(enable_timing=True)
        t_start.record()
        step_events = []
        for _ in range(steps):
            self.step(probe)
            ev = torch.cuda.Event(enable_timing=True)
            ev.record()
            step_events.append(ev)
        t_end.record()
        torch.cuda.synchronize()
        barrier(self.world)
        if sampler:
            sampler.__exit__(None, None, None)
        step_ms = [t_start.elapsed_time(step_events[0])] + [
            a.elapsed_time(b) for a, b in zip(step_events, step_events[1:])]
        ms = max_over_ranks(t_start.elapsed_time(t_end) / steps, self.world)
        out = {"value": self.g.num_nodes / (ms / 1e3), "ms_per_step": ms,
               "step_ms": [round(t, 3) for t in step_ms],
               # our kernels launched inside the timed region (all steps); the
               # ncu launch list of the same command is profiles/r02_launches_gcn3.csv
               "gpu_launches": _lib.LAUNCHES[0] - launches0,
               "gpu_launches_per_step": (_lib.LAUNCHES[0] - launches0) / max(steps, 1),
               "roofline": roofline(probe.summary(), agg_name, steps, ms),
               "batches_per_step": self.stats.batches,
               "layer_batches": self.stats.layer_batches,
               "capacity_bytes": self.budget.capacity}
        if sampler:
            out["clocks"] = sampler.report()
        self.probe = probe
        return out


def roofline(summ, agg_name, steps, ms):
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) \
        if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    # aggregation launches: K1 (spmm_mean) or K4 (gat_aggregate), plus K7
    # (conv_mean: an aggregate-first ConvMean's aggregation fused with its
    # transform; its bytes are B_agg plus the output rows)
    names = [agg_name] + (["conv_mean"] if agg_name == "spmm_mean" else [])
    per = {nm: summ[nm] for nm in names if nm in summ}
    cnt = sum(v[0] for v in per.values())
    nbytes = sum(v[1] for v in per.values())
    agg_ms = sum(v[2] for v in per.values())
    achieved = (nbytes / (agg_ms / 1e3) / 1e9) if agg_ms else None
    lin = summ.get("linear", (0, 0, 0.0))
    k = max(steps, 1)
    return {
        "kernel": "+".join(per) or agg_name, "bound": "hbm", "achieved": achieved, "peak": hbm_peak,
        "per_kernel": {nm: {"launches_per_step": v[0] // k, "bytes_per_step": v[1] // k,
                            "ms_per_step": v[2] / k,
                            "gbs": (v[1] / (v[2] / 1e3) / 1e9) if v[2] else None}
                       for nm, v in per.items()},
        "unit": "GB/s", "frac": (achieved / hbm_peak) if achieved else None,
        "traffic": traffic_from_profiles(agg_name),
        "traffic_kernel": agg_name,
        "traffic_basis": "DRAM read+write bytes per aggregation launch (regular + hub kernels), "
                         "ncu launch list of this bench step (profiles/ncu_traffic.json); "
                         "compare with algorithmic_bytes_per_launch",
        "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback 6.65 TB/s",
        "achieved_basis": "sum of SURVEY 8d B_agg over the step's aggregation launches (K7: "
                          "B_agg + its output rows) / sum of their CUDA-event durations "
                          "(same stream)",
        "launches_per_step": cnt // k,
        "algorithmic_bytes_per_launch": nbytes // max(cnt, 1),
        "algorithmic_bytes_per_step": nbytes // k,
        "kernel_ms_per_step": agg_ms / k,
        "kernel_share_of_step": (agg_ms / k) / ms if ms else None,
        "gemm_ms_per_step": lin[2] / k,
        "gemm_tflops": (lin[1] / (lin[2] / 1e3) / 1e12) if lin[2] else None,
    }


def traffic_from_profiles(kernel):
    """DRAM bytes per launch from the committed ncu capture summary, if any."""
    p = ROOT / "profiles" / "ncu_traffic.json"
    if not p.exists():
        return None
    try:
        return json.loads(p.read_text()).get(kernel, {}).get("dram_bytes_per_launch")
    except Exception:  # noqa: BLE001
        return None


# ------------------------------------------------------------------ parity --


def parity_check(runner, specs, host_csr, n_random=4096, n_hubs=50):
    """One more step with every layer's store kept; each layer is checked on
    the sample against the oracle fed with the device's own H^{l-1}.
    Outside the timed region."""
    import numpy as np
    import torch

    from oracle import parity
    from paper_2211_15082_b200 import _lib, kernels
    from paper_2211_15082_b200.executor import _dims_table
    from paper_2211_15082_b200.splitter import TensorRef

    t0 = time.perf_counter()
    indptr, indices = host_csr
    g, m = runner.g, runner.m
    dev = g.indptr.device
    eng = runner.engine()
    eng.retain_stores = True
    eng.run()
    torch.cuda.synchronize()
    stats = runner.stats
    targets = parity.spot_targets(indptr, n_random, n_hubs)
    bc = parity.batch_for(indptr, indices, targets)
    ids_dev = torch.from_numpy(bc.input_ids).to(dev)
    tg_dev = torch.from_numpy(targets).to(dev)
    n = g.num_nodes
    sched, nh = kernels.degree_schedule(g.indptr, None, 0, n)
    nh = int(nh.item())
    layers = []
    for blk, spec in zip(runner.schedule.blocks, specs):
        in_key = blk.input_keys()[0]
        h = eng.stores[in_key].view()
        got = eng.stores[TensorRef(blk.block_id, blk.outputs[0]).key].view()
        h_rows = h.index_select(0, ids_dev).cpu().numpy()
        got_rows = got.index_select(0, tg_dev).cpu().numpy()
        rec = {"layer": blk.layer, "kind": spec["kind"], "width_in": int(h.shape[1])}
        agg_dev = None
        if spec["kind"] == "ConvMean":
            conv = next(o for o in blk.op_ids if blk.kinds[o] == "ConvMean")
            # K1 exactly as the engine launches it: one whole-layer call with the
            # LPT schedule and the hub rows on the side stream
            if eng._reassociate(conv):
                w = eng.params.w[conv]
                d_out = int(w.shape[0])
                zfull = torch.empty((n, (d_out + 3) // 4 * 4), device=dev)
                z = zfull[:, :d_out]
                kernels.linear_into(z, h, w, None, _lib.ACT_NONE, precision=eng.precision)
                agg = torch.empty_like(zfull)[:, :d_out]
                kernels.spmm_mean(agg, z, g.indptr, g.indices, n, schedule=sched, n_hub=nh)
                z_rows = z.index_select(0, ids_dev).cpu().numpy()
                rec["k1_bytes_equal"] = parity.agg_check(
                    bc, z_rows, agg.index_select(0, tg_dev).cpu().numpy())
                rec["k1_operand"] = f"z = H W^T ({d_out} cols, reassociated layer)"
                del zfull, z, agg
            else:
                d = int(h.shape[1])
                agg = torch.empty((n, (d + 3) // 4 * 4), device=dev)[:, :d]
                kernels.spmm_mean(agg, h, g.indptr, g.indices, n, schedule=sched, n_hub=nh)
                agg_dev = agg.index_select(0, tg_dev).cpu().numpy()
                rec["k1_operand"] = f"H^{blk.layer - 1} ({d} cols)"
                del agg
        chk = parity.conv_check(bc, h_rows, spec, got_rows, agg_dev)
        if chk["agg_bytes_equal"] is not None:
            rec["k1_bytes_equal"] = chk["agg_bytes_equal"]
        rec["rel_l2"] = chk["rel_l2"]
        rec["max_abs"] = chk["max_abs"]
        layers.append(rec)
    # batch records: plan-only replay of the reference controller
    dims = _dims_table(m, runner.schedule)
    blocks = [{"layer": b.layer, "has_conv": b.has_conv,
               "input_widths": [dims[k] for k in b.input_keys()],
               "ops": [(dom, dims[o]) for o, kind, dom in b.iter_ops()
                       if kind not in ("Input", "Output")],
               "output_widths": [dims[o] for o in b.output_ids()]} for b in runner.schedule.blocks]
    want = parity.replay_layers(indptr, indices, runner.budget.capacity, runner.th0.n_t,
                                runner.th0.n_i, blocks)
    got = [(l, t, p, a, b) for l, t, p, (_, a, b) in zip(
        stats.batch_layers, stats.batch_sizes, stats.batch_footprints, stats.trajectory)]
    records_equal = (got == [w[:5] for w in want]
                     and stats.oom_retries == sum(w[5] for w in want))
    for st in list(eng.stores):
        eng.stores.pop(st, None)
    del eng
    torch.cuda.empty_cache()
    k1 = [r["k1_bytes_equal"] for r in layers if "k1_bytes_equal" in r]
    return {"k1_bytes_equal": all(k1) if k1 else None,
            "conv_rel_l2_max": max(r["rel_l2"] for r in layers),
            "final_rel_l2": layers[-1]["rel_l2"],
            "records_equal": bool(records_equal),
            "tolerance": "K1 bytes equal; conv rows rel-L2 <= 1e-4 (3xTF32 GEMM, reassociated "
                         "layer 3 ~1e-7); batch records byte-equal",
            "pass": bool((all(k1) if k1 else True) and records_equal
                         and max(r["rel_l2"] for r in layers) <= 1e-4),
            "sample": f"{len(targets)} targets: {n_random} seeded random + the {n_hubs} largest "
                      f"in-degree rows + nodes 0 and N-1; {len(bc.local_srcs)} edges, "
                      f"{len(bc.input_ids)} input rows; oracle fed with the device's H^(l-1)",
            "records": {"batches": len(want), "layer1_targets": [w[1] for w in want
                                                                 if w[0] == 1]},
            "layers": layers, "seconds": round(time.perf_counter() - t0, 1)}


# -------------------------------------------------------------------- e2e --


def run_e2e(m, g, xt, budget, world, steps):
    """Same metric through the public API run_inference from pinned host buffers."""
    import torch

    from paper_2211_15082_b200.executor import run_inference
    from paper_2211_15082_b200.storage import PACK24, CscGraph

    n = g.num_nodes
    ip = torch.empty(n + 1, dtype=torch.int64, pin_memory=True)
    ip.copy_(torch.from_numpy(g.indptr_host))
    ix = torch.empty(g.num_edges, dtype=torch.int64, pin_memory=True)
    ix.copy_(g.indices.to(torch.int64).cpu())
    xh = torch.empty(tuple(xt.shape), dtype=torch.float32, pin_memory=True)
    xh.copy_(xt.cpu())
    host_graph = CscGraph(n, g.num_edges, ip.numpy(), ix.numpy())
    id_bytes = 3 if (PACK24 and n <= (1 << 24)) else 4
    h2d = ip.numel() * 8 + ix.numel() * id_bytes + xh.numel() * 4
    d2h = n * m.output_dim * 4
    run_inference(m, host_graph, xh, budget=budget, output="numpy", reassociate=True)
    barrier(world)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = None
    for _ in range(steps):
        res = None      # the caller is done with the previous result (recycles pinned staging)
        res = run_inference(m, host_graph, xh, budget=budget, output="numpy", reassociate=True)
    torch.cuda.synchronize()
    barrier(world)
    dt = max_over_ranks((time.perf_counter() - t0) / steps, world)
    assert res.output.shape == (n, m.output_dim)
    return {"value": n / dt, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "ms_per_step": dt * 1e3, "steps": steps, "api": "executor.run_inference",
            "host_buffers": "pinned torch CPU tensors (graph int64 CSC, fp32 features)",
            "h2d_basis": f"bytes that cross PCIe: int64 indptr, {id_bytes}-byte packed ids "
                         f"(the API takes int64; the uploader narrows on host threads), "
                         f"fp32 features",
            "caller_host_bytes": ip.numel() * 8 + ix.numel() * 8 + xh.numel() * 4}


# ------------------------------------------------------------------- main --


def main():
    args = parse()
    rank, world, local = dist_setup(args)
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    import torch

    from paper_2211_15082_b200 import _lib, kernels
    from paper_2211_15082_b200.parallel import RowExchange, edge_balanced_ranges

    _lib.load()
    if args.precision:
        kernels.PRECISION = _lib.PREC_3XTF32 if args.precision == "3xtf32" else _lib.PREC_FP32
    for kv in args.tune:
        k, v = kv.split("=")
        _lib.call("glint_set_tuning", int(k), int(v))
    dev = torch.device("cuda", local)
    n, und = sizes(args)
    g, xt = device_inputs(n, und, 100, dev)
    cuts = edge_balanced_ranges(g.indptr_host, world)
    ex = RowExchange(cuts, rank, world) if world > 1 else None
    agg_of = {"gcn3": "spmm_mean", "gat3": "gat_aggregate"}

    m = build_model(args.model)
    run = Runner(m, g, xt, world, local, ex)
    meas = run.measure(args.steps, args.warmup, agg_of[args.model], clocks=True)
    line = {
        "metric": METRIC, "value": meas["value"], "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": meas["ms_per_step"],
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": DATA,
        "config": config_block(args.model, n, und, world),
        "engine": {"capacity_bytes": meas["capacity_bytes"],
                   "gemm_precision": "3xtf32" if kernels.PRECISION == _lib.PREC_3XTF32 else "fp32",
                   "reassociate": True},
        "batches_per_step": meas["batches_per_step"], "layer_batches": meas["layer_batches"],
        "roofline": meas["roofline"], "gpu_launches": meas["gpu_launches"],
        "gpu_launches_per_step": meas["gpu_launches_per_step"],
        "clocks": meas["clocks"], "step_ms": meas["step_ms"],
        **({"tuning": args.tune} if args.tune else {}),
    }
    if args.timeline:
        line["timeline_ms"] = [(nm, round(t, 3)) for nm, t in run.probe.timeline()]
    if not args.no_e2e:
        line["e2e"] = run_e2e(m, g, xt, run.budget, world, max(1, min(args.steps, 3)))
    host_csr = None
    if rank == 0 and world == 1 and not (args.no_parity and args.no_cpu):
        host_csr = (g.indptr_host, g.indices.to(torch.int64).cpu().numpy())
    if host_csr is not None and not args.no_parity:
        line["parity"] = parity_check(run, layer_specs(args.model), host_csr)
    del run
    torch.cuda.empty_cache()

    if world == 1 and not args.no_secondary:
        sec = {}
        other = "gat3" if args.model == "gcn3" else "gcn3"
        m2 = build_model(other)
        run2 = Runner(m2, g, xt, world, local)
        meas2 = run2.measure(max(3, min(args.steps, 8)), 3, agg_of[other])
        sec["cfg3" if other == "gat3" else "cfg2"] = {
            "config": config_block(other, n, und, world),
            **{k: meas2[k] for k in ("value", "ms_per_step", "step_ms", "roofline",
                                     "gpu_launches", "layer_batches")},
            **({"e2e": run_e2e(m2, g, xt, run2.budget, world, 2)} if not args.no_e2e else {}),
            **({"parity": parity_check(run2, layer_specs(other), host_csr)}
               if host_csr is not None and not args.no_parity else {}),
        }
        del run2
        torch.cuda.empty_cache()
        sec[f"{'cfg2' if args.model == 'gcn3' else 'cfg3'}_rcmk"] = order_secondary(
            args, m, g, xt, world, local, agg_of[args.model])
        # the other BASELINE configs, measured in the same driver run; a failure
        # here is recorded, never allowed to lose the headline line
        for key, fn in (("cfg4", lambda: cfg4_secondary(g, xt)),
                        ("cfg5", lambda: None if (args.no_cfg5 or args.nodes) else cfg5_secondary())):
            try:
                r = fn()
                if r is not None:
                    sec[key] = r
            except Exception as exc:  # noqa: BLE001
                sec[key] = {"error": f"{type(exc).__name__}: {exc}"[:300]}
            torch.cuda.empty_cache()
        line["secondary"] = sec
    if rank == 0 and world == 1 and not args.no_cpu:
        sample = args.cpu_sample or 4096       # per worker: ~16 workers x 1.5 s of CPU work
        workers = cpu_workers()
        x_host = xt.cpu().numpy()
        rate, secs, sdesc = cpu_sample_rate(host_csr[0], host_csr[1], x_host,
                                            layer_specs(args.model), sample, workers=workers)
        line["cpu_baseline"] = cpu_block(rate, workers, sdesc, secs)
    if rank == 0:
        print(json.dumps(line), flush=True)
    barrier(world)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


def order_secondary(args, m, g, xt, world, local, agg_name):
    """The same step on the RCMK-relabelled graph (cfg2's order).
    The relabelling (RCMK permutation + device relabel of CSR and features)
    is one-time and outside the timed region."""
    import torch

    from paper_2211_15082_b200.reorder import apply_order_device, make_order

    t0 = time.perf_counter()
    order = make_order(g, "rcmk")
    gi, xi = apply_order_device(g, xt, order)
    torch.cuda.synchronize()
    prep = time.perf_counter() - t0
    run = Runner(m, gi, xi, world, local)
    meas = run.measure(max(3, min(args.steps, 10)), 3, agg_name)
    out = {"config": config_block(args.model, g.num_nodes, g.num_edges // 2, world, "rcmk"),
           "reorder_s": round(prep, 2),
           **{k: meas[k] for k in ("value", "ms_per_step", "step_ms", "roofline")}}
    del run, gi, xi
    torch.cuda.empty_cache()
    return out


def cfg4_secondary(g, xt, reps=3):
    """BASELINE configs[3]: JKNet and APPNP partial inference on a 10% target
    subset of the same graph, through run_inference with device-resident inputs
    (median of `reps` calls after one warm-up), each checked byte-for-byte
    against the same rows of a full-mode run (row invariance)."""
    import torch

    from paper_2211_15082_b200 import synth
    from paper_2211_15082_b200.executor import run_inference

    n = g.num_nodes
    targets = np.sort(np.random.default_rng(0).choice(n, n // 10, replace=False)).astype(np.int64)
    out = {"workload": "cfg4 JKNet / APPNP (100->256->256->47) partial inference, 10% targets",
           "targets": len(targets)}
    for name, m in (("jknet3", synth.build_jknet(100, 256, 47, 3, seed=0)),
                    ("appnp3", synth.build_appnp(100, 256, 47, k=3, alpha=0.1, seed=0))):
        kw = dict(budget="device", output="device", reassociate=True)
        want = run_inference(m, g, xt, **kw).output[torch.from_numpy(targets).cuda()]
        run_inference(m, g, xt, mode="partial", targets=targets, **kw)
        torch.cuda.synchronize()
        times, res = [], None
        for _ in range(reps):
            res = None
            t0 = time.perf_counter()
            res = run_inference(m, g, xt, mode="partial", targets=targets, **kw)
            torch.cuda.synchronize()
            times.append(1e3 * (time.perf_counter() - t0))
        ms = float(np.median(times))
        out[name] = {"ms_per_call": round(ms, 3), "targets_per_s": len(targets) / (ms / 1e3),
                     "all_ms": [round(t, 3) for t in times],
                     "bit_identical_to_full_rows": bool(torch.equal(res.output, want)),
                     "layer_batches": res.stats.layer_batches}
        del want, res
        torch.cuda.empty_cache()
    return out


def cfg5_secondary(steps=2, warmup=1, capacity_gib=64.0):
    """BASELINE configs[4] on ONE B200 (tools/bench_papers.py): a 111M-node,
    1.6B-edge Papers100M-shaped graph, 3-layer GCN 128->128->128->172, full
    inference at a 64 GiB batch capacity, the engine owning (and freeing) x,
    the caching allocator's blocks kept between steps."""
    import torch

    sys.path.insert(0, str(ROOT / "tools"))
    import bench_papers

    torch.cuda.empty_cache()
    res = bench_papers.run(steps=steps, warmup=warmup, capacity_gib=capacity_gib)
    torch.cuda.empty_cache()
    return {k: res[k] for k in ("workload", "nodes", "in_edges", "value", "unit", "ms_per_step",
                                "aggregation", "gemm", "capacity_gib", "allocator")} | {
        "step_ms": [round(st["ms"], 1) for st in res["per_step"]],
        "layer_batches": res["per_step"][-1]["layer_batches"],
        "peak_alloc_gib": round(res["per_step"][-1]["peak_alloc_gib"], 1)}


if __name__ == "__main__":
    main()
