#!/usr/bin/env python
"""Is the chunked CSR upload asynchronous for numpy views of pinned memory?"""

import pathlib
import sys
import time

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))


def main():
    import torch

    from paper_2211_15082_b200 import synth
    from paper_2211_15082_b200.executor import _copy_stream
    from paper_2211_15082_b200.storage import CscGraph, DeviceGraph

    n, und = synth.PRODUCTS_NODES, synth.PRODUCTS_UNDIRECTED
    g = synth.gen_products_like(n, und, seed=0, device="cuda")
    ip = torch.empty(n + 1, dtype=torch.int64, pin_memory=True)
    ip.copy_(torch.from_numpy(g.indptr_host))
    ix = torch.empty(g.num_edges, dtype=torch.int64, pin_memory=True)
    ix.copy_(g.indices.to(torch.int64).cpu())
    hg = CscGraph(n, g.num_edges, ip.numpy(), ix.numpy())
    t = torch.from_numpy(hg.indices)
    print("pinned tensor:", ix.is_pinned(), "numpy view re-wrapped:", t.is_pinned(),
          "slice:", t[5:100].is_pinned(), "same ptr:", t.data_ptr() == ix.data_ptr())
    dev = torch.device("cuda", 0)
    for rep in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        dg = DeviceGraph.upload_async(hg, dev, _copy_stream(dev))
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        print(f"upload_async host {1e3 * (t1 - t0):.2f} ms, until done {1e3 * (t2 - t0):.2f} ms")
        del dg


if __name__ == "__main__":
    main()
