#!/usr/bin/env python
"""Where does a layer-1 bootstrap batch's K1 time go?  Splits one contiguous
batch of the headline graph into its hub rows and its regular rows and times
each part alone (CUDA events, same stream), with the batch's degree profile."""

from __future__ import annotations

import json
import pathlib
import sys

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import torch

    from paper_2211_15082_b200 import _lib, kernels, synth
    from tools.sweep_kernels import timed

    n = synth.PRODUCTS_NODES
    g = synth.gen_products_like(n, synth.PRODUCTS_UNDIRECTED, seed=0, device="cuda")
    deg = g.in_degrees
    d = int(sys.argv[1]) if len(sys.argv) > 1 else 100
    h = torch.randn((n, d), device="cuda")
    out = torch.empty((n, d), device="cuda")
    pos = 0
    for size in (1024, 4096, 16384, 65536, 262144):
        dg = deg[pos:pos + size]
        sch, nh = kernels.degree_schedule(g.indptr, None, pos, size)
        nh = int(nh.item())
        o2 = out[pos:pos + size]
        full = timed(lambda: kernels.spmm_mean(o2, h, g.indptr, g.indices, size, row_base=pos,
                                               schedule=sch, n_hub=nh))
        hubs = timed(lambda: kernels.spmm_mean(o2, h, g.indptr, g.indices, nh, row_base=pos,
                                               schedule=sch, n_hub=nh)) if nh else 0.0
        reg_s = sch[nh:]
        reg = timed(lambda: kernels.spmm_mean(o2, h, g.indptr, g.indices, size - nh,
                                              row_base=pos, schedule=reg_s, n_hub=0))
        top = sorted(dg.tolist(), reverse=True)[:5]
        print(json.dumps({"rows": size, "base": pos, "dim": d, "hubs": nh, "edges": int(dg.sum()),
                          "top_deg": top, "ms_full": full, "ms_hubs_only": hubs,
                          "ms_regular_only": reg}), flush=True)
        pos += size


if __name__ == "__main__":
    main()
