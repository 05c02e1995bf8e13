import cProfile, pstats, sys, time, json
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from paper_2211_15082_b200 import synth
from paper_2211_15082_b200.executor import run_inference, KernelProbe
n, und = synth.PRODUCTS_NODES, synth.PRODUCTS_UNDIRECTED
g = synth.gen_products_like(n, und, seed=0, device="cuda")
x = synth.gen_features_device(n, 100, seed=0, device="cuda")
targets = np.sort(np.random.default_rng(0).choice(n, n // 10, replace=False)).astype(np.int64)
m = synth.build_appnp(100, 256, 47, k=3, alpha=0.1, seed=0)
kw = dict(mode="partial", targets=targets)
for _ in range(2):
    run_inference(m, g, x, budget="device", output="device", reassociate=True, **kw)
torch.cuda.synchronize()
pr = cProfile.Profile()
starts = []
for rep in range(8):
    probe = KernelProbe()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    pr.enable()
    res = run_inference(m, g, x, budget="device", output="device", reassociate=True, probe=probe, **kw)
    pr.disable()
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    tl = dict((a, b) for a, b, c in probe.absolute())
    starts.append((round((t1 - t0) * 1e3, 2), round(tl["start"], 2)))
print("per-rep (call ms, start ms)", starts)
pstats.Stats(pr).sort_stats("cumtime").print_stats(35)
