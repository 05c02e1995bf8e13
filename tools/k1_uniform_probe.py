"""K1 (spmm_mean) on the same synthetic shape as tools/probes/bulk_gather_probe.cu:
2,449,029 rows of exactly 50 uniform random in-neighbours, 192-byte (d=48) and
768-byte (d=192) rows.  Prints gathered GB/s (rows * 50 * row bytes / time) so
the two gather engines compare directly.

    python tools/k1_uniform_probe.py
"""

from __future__ import annotations

import json
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))


def main():
    import numpy as np
    import torch

    from paper_2211_15082_b200 import kernels

    dev = torch.device("cuda", 0)
    n, deg = 2449029, 50
    rng = np.random.default_rng(0)
    indptr = torch.arange(0, (n + 1) * deg, deg, dtype=torch.int64, device=dev)
    indices = torch.from_numpy(rng.integers(0, n, size=n * deg, dtype=np.int32)).to(dev)
    for d in (48, 192):
        h = torch.zeros((n, d), device=dev)
        out = torch.empty((n, d), device=dev)
        sched, n_hub = kernels.degree_schedule(indptr, None, 0, n)
        n_hub = int(n_hub.item())
        for _ in range(2):
            kernels.spmm_mean(out, h, indptr, indices, n, schedule=sched, n_hub=n_hub)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(5):
            kernels.spmm_mean(out, h, indptr, indices, n, schedule=sched, n_hub=n_hub)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 5
        print(json.dumps({"kernel": "k1_spmm_mean", "row_bytes": 4 * d, "rows": n, "deg": deg,
                          "ms": round(ms, 4),
                          "gathered_gbs": round(n * deg * 4 * d / ms / 1e6, 1)}), flush=True)


if __name__ == "__main__":
    main()
