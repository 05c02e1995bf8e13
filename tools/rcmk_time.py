import sys, time, ctypes
sys.path.insert(0, '.')
import numpy as np, torch
import bench
from paper_2211_15082_b200 import reorder, _lib
from paper_2211_15082_b200.reorder import _sorted_adjacency_device, NodeOrder
import argparse
n, und = bench.sizes(argparse.Namespace(nodes=None, undirected=None))
g, x = bench.device_inputs(n, und, 100, torch.device('cuda', 0))
for rep in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    ptr, adj = _sorted_adjacency_device(g)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    perm = np.empty(n, dtype=np.int64)
    rc = _lib.load().glint_rcmk_sorted_host(n, ptr.ctypes.data_as(ctypes.c_void_p), adj.ctypes.data_as(ctypes.c_void_p), perm.ctypes.data_as(ctypes.c_void_p))
    t2 = time.perf_counter()
    o = NodeOrder(perm)
    t3 = time.perf_counter()
    g2, x2 = reorder.apply_order_device(g, x, o)
    torch.cuda.synchronize(); t4 = time.perf_counter()
    print(dict(adj_device=round(t1-t0,3), host_bfs=round(t2-t1,3), nodeorder=round(t3-t2,3), apply=round(t4-t3,3), nnz=len(adj)))
