#!/usr/bin/env python
"""Host int64 -> int32 narrowing throughput (glint_narrow_ids_host) vs threads,
and the pinned H2D rate of int32 vs int64 CSR chunks."""
import json
import os
import pathlib
import sys
import time

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))


def main():
    import ctypes

    import numpy as np
    import torch

    from paper_2211_15082_b200 import _lib

    lib = _lib.load()
    m = 123_718_280
    src = torch.empty(m, dtype=torch.int64, pin_memory=True)
    src.copy_(torch.randint(0, 2_449_029, (m,), dtype=torch.int64))
    dst = torch.empty(m, dtype=torch.int32, pin_memory=True)
    print(json.dumps({"cpus": os.cpu_count()}), flush=True)
    for t in (1, 2, 4, 8, 16):
        best = 1e9
        for _ in range(3):
            t0 = time.perf_counter()
            bad = lib.glint_narrow_ids_host(ctypes.c_void_p(src.data_ptr()),
                                            ctypes.c_void_p(dst.data_ptr()), m, t)
            best = min(best, time.perf_counter() - t0)
        ok = bool(torch.equal(dst[:1000].to(torch.int64), src[:1000]))
        print(json.dumps({"threads": t, "ms": 1e3 * best, "GBps_read": m * 8 / best / 1e9,
                          "bad": int(bad), "ok": ok}), flush=True)
    dev = torch.device("cuda", 0)
    d64 = torch.empty(m, dtype=torch.int64, device=dev)
    d32 = torch.empty(m, dtype=torch.int32, device=dev)
    for name, h, d in (("int64", src, d64), ("int32", dst, d32)):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        d.copy_(h, non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        print(json.dumps({"h2d": name, "ms": 1e3 * dt, "GBps": h.numel() * h.element_size() / dt / 1e9}),
              flush=True)


if __name__ == "__main__":
    main()
