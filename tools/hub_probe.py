#!/usr/bin/env python
"""One hubs-only K1 launch of the 65536-row layer-1 batch (for ncu)."""
import pathlib
import sys

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import torch

    from paper_2211_15082_b200 import kernels, synth

    n = synth.PRODUCTS_NODES
    g = synth.gen_products_like(n, synth.PRODUCTS_UNDIRECTED, seed=0, device="cuda")
    d = int(sys.argv[1]) if len(sys.argv) > 1 else 100
    h = torch.randn((n, d), device="cuda")
    out = torch.empty((n, d), device="cuda")
    pos, size = 21504, 65536
    sch, nh = kernels.degree_schedule(g.indptr, None, pos, size)
    nh = int(nh.item())
    for _ in range(2):
        kernels.spmm_mean(out[pos:pos + size], h, g.indptr, g.indices, nh, row_base=pos,
                          schedule=sch, n_hub=nh)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
