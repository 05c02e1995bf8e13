"""The NCCL code path of the row exchange on ONE GPU: a 1-rank NCCL process
group drives RowExchange (grouped broadcasts through the coalescing manager,
and the halo all-to-all) inside the engine exactly as a multi-GPU run does,
plus the direct tensor exchanges.  Outputs must be bit-identical to the
engine without an exchange.  This pool has one GPU per call, so this is the
only place the NCCL calls themselves execute before a multi-GPU run.

    python tools/nccl_single_check.py [nodes]
"""

from __future__ import annotations

import argparse
import json
import os
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))


def main():
    import numpy as np
    import torch
    import torch.distributed as dist

    import bench
    from paper_2211_15082_b200.parallel import HaloPlan, RowExchange

    n_nodes = int(sys.argv[1]) if len(sys.argv) > 1 else 30000
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29561")
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1)
    dev = torch.device("cuda", 0)
    n, und = bench.sizes(argparse.Namespace(nodes=n_nodes, undirected=None))
    g, x = bench.device_inputs(n, und, 100, dev)
    cuts = np.array([0, n], dtype=np.int64)
    for model in ("gcn3", "gat3"):
        m = bench.build_model(model)
        want = bench.Runner(m, g, x, 1, 0).step().data.clone()
        for kind in ("replicate", "halo"):
            halo = HaloPlan(g.indptr_host, g.indices, cuts, 0) if kind == "halo" else None
            ex = RowExchange(cuts, 0, 1, halo=halo)
            got = bench.Runner(m, g, x, 1, 0, ex=ex).step().data
            print(json.dumps({"model": model, "exchange": kind, "backend": dist.get_backend(),
                              "bit_identical": bool(torch.equal(got, want)),
                              "bytes_sent": ex.bytes_sent}), flush=True)
            assert torch.equal(got, want), (model, kind)
    # direct tensor exchanges (transform-first pieces, model output)
    t = torch.randn((n, 48), device=dev)
    ref = t.clone()
    for kind in ("replicate", "halo"):
        halo = HaloPlan(g.indptr_host, g.indices, cuts, 0) if kind == "halo" else None
        ex = RowExchange(cuts, 0, 1, halo=halo)
        ex.exchange_tensors((t,))
        ex.replicate_tensor(t)
        assert torch.equal(t, ref), kind
    print(json.dumps({"direct_exchanges": "ok"}), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
