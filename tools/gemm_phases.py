#!/usr/bin/env python
"""Phase-cycle breakdown of the tcgen05 3xTF32 GEMM (GLINT_TUNE_GEMM_PROF)."""

from __future__ import annotations

import ctypes
import json
import pathlib
import sys

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import torch

    from paper_2211_15082_b200 import _lib, kernels

    n = int(sys.argv[1]) if len(sys.argv) > 1 else 2_449_029
    names = ["prod_wait_empty", "prod_work", "mma_wait_full", "mma_wait_tmem_empty",
             "epi_wait_tmem_full", "epi_work", "kernel_cycles", "tiles"]
    for K, N in ((256, 256), (100, 256), (256, 48)):
        a = torch.randn((n, K), device="cuda")
        w = torch.randn((N, K), device="cuda") / K ** 0.5
        c = torch.empty((n, N), device="cuda")
        _lib.call("glint_set_tuning", 1, 0)
        kernels.linear_into(c, a, w, None, 0, precision=1)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        kernels.linear_into(c, a, w, None, 0, precision=1)
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e)
        buf = (ctypes.c_uint64 * 8)()
        _lib.call("glint_debug_counters", 0, ctypes.addressof(buf), 8, 1)
        _lib.call("glint_set_tuning", 1, 1)
        kernels.linear_into(c, a, w, None, 0, precision=1)
        torch.cuda.synchronize()
        _lib.call("glint_debug_counters", 0, ctypes.addressof(buf), 8, 1)
        _lib.call("glint_set_tuning", 1, 0)
        vals = dict(zip(names, list(buf)))
        ctas = min(148, -(-n // 256))
        tiles = max(vals["tiles"], 1)
        per_tile = {k: vals[k] / tiles for k in names[:6]}
        # producer counters are summed over 8 warps, epilogue over 4
        per_tile["prod_wait_empty"] /= 8
        per_tile["prod_work"] /= 8
        per_tile["epi_wait_tmem_full"] /= 4
        per_tile["epi_work"] /= 4
        print(json.dumps({"K": K, "N": N, "ms_unprofiled": ms, "ctas": ctas,
                          "kernel_cycles_per_cta": vals["kernel_cycles"] / ctas,
                          "cycles_per_tile": {k: round(v) for k, v in per_tile.items()},
                          "tiles": tiles}), flush=True)


if __name__ == "__main__":
    main()
