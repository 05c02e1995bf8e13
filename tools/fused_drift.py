"""Per-launch time and SM clock of K7 vs K1 + K2 over back-to-back blocks of
launches (layer 1 of cfg2, 100 -> 256): does K7 slow down as it repeats, and is
it the clock (power cap) or the kernel?

    python tools/fused_drift.py > profiles/r02_fused_drift.jsonl
"""

from __future__ import annotations

import argparse
import json
import pathlib
import sys
import threading
import time

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


class Clocks(threading.Thread):
    def __init__(self):
        super().__init__(daemon=True)
        import pynvml

        pynvml.nvmlInit()
        self.nv = pynvml
        self.h = pynvml.nvmlDeviceGetHandleByIndex(0)
        self.samples = []
        self.stop = False

    def run(self):
        while not self.stop:
            self.samples.append((time.perf_counter(),
                                 self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM),
                                 self.nv.nvmlDeviceGetPowerUsage(self.h) / 1000.0))
            time.sleep(0.005)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--block", type=int, default=12)
    ap.add_argument("--rounds", type=int, default=3)
    args = ap.parse_args()
    import numpy as np
    import torch

    import bench
    from paper_2211_15082_b200 import _lib, kernels

    dev = torch.device("cuda", 0)
    n, und = bench.sizes(argparse.Namespace(nodes=None, undirected=None))
    g, h = bench.device_inputs(n, und, 100, dev)
    sched, n_hub = kernels.degree_schedule(g.indptr, None, 0, n)
    n_hub = int(n_hub.item())
    rng = np.random.default_rng(0)
    W = torch.from_numpy((rng.normal(size=(256, 100)) / 10).astype(np.float32)).to(dev)
    b = torch.from_numpy(rng.normal(size=256).astype(np.float32)).to(dev)
    agg = torch.empty((n, 100), device=dev)
    out = torch.empty((n, 256), device=dev)
    clk = Clocks()
    clk.start()

    def fused():
        kernels.conv_mean(out, h, W, b, _lib.ACT_RELU, g.indptr, g.indices, n, schedule=sched)

    def unfused():
        kernels.spmm_mean(agg, h, g.indptr, g.indices, n, schedule=sched, n_hub=n_hub)
        kernels.linear_into(out, agg, W, b, _lib.ACT_RELU, precision=_lib.PREC_3XTF32)

    def k1():
        kernels.spmm_mean(agg, h, g.indptr, g.indices, n, schedule=sched, n_hub=n_hub)

    for rnd in range(args.rounds):
        for name, fn in (("fused", fused), ("unfused", unfused), ("k1", k1)):
            torch.cuda.synchronize()
            time.sleep(0.5)
            evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.block + 1)]
            t0 = time.perf_counter()
            evs[0].record()
            for i in range(args.block):
                fn()
                evs[i + 1].record()
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            ms = [round(evs[i].elapsed_time(evs[i + 1]), 3) for i in range(args.block)]
            s = [x for x in clk.samples if t0 <= x[0] <= t1]
            print(json.dumps({"round": rnd, "kernel": name, "ms": ms,
                              "sm_mhz": [x[1] for x in s][::max(1, len(s) // 12)],
                              "power_w": [round(x[2]) for x in s][::max(1, len(s) // 12)]}),
                  flush=True)
    clk.stop = True


if __name__ == "__main__":
    main()
