"""Is the e2e CSR preparation bound by host memory bandwidth?  Times, on the
GPU box: the host int64->int32 narrowing of the Products CSR ids on T threads
alone, a 0.98 GB pinned H2D copy (the features) alone, and both at once.

    python tools/host_bw_probe.py > profiles/r02_host_bw_probe.jsonl
"""
import ctypes
import json
import pathlib
import sys
import threading
import time

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))


def main():
    import numpy as np
    import torch

    from paper_2211_15082_b200 import _lib

    lib = _lib.load()
    E = 123_718_280
    rng = np.random.default_rng(0)
    src = torch.empty(E, dtype=torch.int64, pin_memory=True)
    src.numpy()[:] = rng.integers(0, 2_449_029, size=E)
    dst = torch.empty(E, dtype=torch.int32, pin_memory=True)
    feats = torch.empty((2_449_029, 100), dtype=torch.float32, pin_memory=True)
    dev = torch.empty_like(feats, device="cuda")
    s = torch.cuda.Stream()

    def narrow(threads):
        t0 = time.perf_counter()
        bad = lib.glint_narrow_ids_host(ctypes.c_void_p(src.data_ptr()), ctypes.c_void_p(dst.data_ptr()),
                                        E, threads)
        return time.perf_counter() - t0, bad

    def copy():
        t0 = time.perf_counter()
        with torch.cuda.stream(s):
            dev.copy_(feats, non_blocking=True)
        s.synchronize()
        return time.perf_counter() - t0

    for rep in range(3):
        for threads in (6, 12, 16):
            tn, _ = narrow(threads)
            print(json.dumps({"rep": rep, "what": "narrow alone", "threads": threads,
                              "ms": round(tn * 1e3, 2), "read_gbs": round(E * 8 / tn / 1e9, 1)}), flush=True)
        tc = copy()
        print(json.dumps({"rep": rep, "what": "H2D 0.98 GB alone", "ms": round(tc * 1e3, 2),
                          "gbs": round(feats.numel() * 4 / tc / 1e9, 1)}), flush=True)
        res = {}
        th = threading.Thread(target=lambda: res.setdefault("c", copy()))
        th.start()
        tn, _ = narrow(12)
        th.join()
        print(json.dumps({"rep": rep, "what": "both", "narrow_ms": round(tn * 1e3, 2),
                          "copy_ms": round(res["c"] * 1e3, 2)}), flush=True)


if __name__ == "__main__":
    main()
