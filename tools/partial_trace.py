"""Device/host timeline and kernel summary of one cfg4 partial call (JKNet or
APPNP, 10% targets, Products-shaped graph) -- where a partial call's time goes.
`gcn3-sampling` traces a sampling-mode call (fanout 10, all nodes) of the cfg2 GCN.

    python tools/partial_trace.py [jknet3|appnp3|gcn3-sampling] > profiles/r02_cfg4_trace.jsonl
"""
import json
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))


def main():
    import numpy as np
    import torch

    from paper_2211_15082_b200 import synth
    from paper_2211_15082_b200.executor import KernelProbe, run_inference

    name = sys.argv[1] if len(sys.argv) > 1 else "jknet3"
    n, und = synth.PRODUCTS_NODES, synth.PRODUCTS_UNDIRECTED
    g = synth.gen_products_like(n, und, seed=0, device="cuda")
    x = synth.gen_features_device(n, 100, seed=0, device="cuda")
    targets = np.sort(np.random.default_rng(0).choice(n, n // 10, replace=False)).astype(np.int64)
    if name == "gcn3-sampling":
        m = synth.build_gcn(100, 256, 47, 3, seed=0)
        kw = dict(mode="sampling", fanout=10, seed=1)
    else:
        m = (synth.build_jknet(100, 256, 47, 3, seed=0) if name == "jknet3"
             else synth.build_appnp(100, 256, 47, k=3, alpha=0.1, seed=0))
        kw = dict(mode="partial", targets=targets)
    for rep in range(3):
        probe = KernelProbe()
        torch.cuda.synchronize()
        res = run_inference(m, g, x, budget="device", output="device", reassociate=True,
                            probe=probe, **kw)
        torch.cuda.synchronize()
        probe.mark("end")
        torch.cuda.synchronize()
        if rep == 2:
            print(json.dumps({"model": name, "timeline": probe.absolute(),
                              "kernels": {k: [v[0], round(v[2], 3)] for k, v in probe.summary().items()},
                              "layer_batches": res.stats.layer_batches}), flush=True)


if __name__ == "__main__":
    main()
