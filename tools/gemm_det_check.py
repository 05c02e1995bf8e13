#!/usr/bin/env python
"""v3 GEMM determinism + agreement with v2 at the workload's M (run on the B200
box): three v3 runs per shape must equal each other and the v2 bytes; a
mismatch prints its row/column pattern (whole tiles wrong = a pipeline race).
This caught the two-converter-group parity ambiguity."""
import sys, json, torch
sys.path.insert(0, '/root/repo')
from paper_2211_15082_b200 import _lib, kernels
torch.manual_seed(0)
M = 2449029
for K in (100, 128, 256):
    x = torch.randn((M, K), device='cuda')
    for N in (47, 64, 128, 172, 192, 256):
        w = torch.randn((N, K), device='cuda') / K ** 0.5
        outs = []
        for r in range(3):
            o = torch.empty((M, N), device='cuda')
            kernels.linear_into(o, x, w, None, 0, precision=_lib.PREC_3XTF32)
            outs.append(o)
        _lib.call("glint_set_tuning", 9, 1)
        ref = torch.empty((M, N), device='cuda')
        kernels.linear_into(ref, x, w, None, 0, precision=_lib.PREC_3XTF32)
        _lib.call("glint_set_tuning", 9, 0)
        for r, o in enumerate(outs):
            bad = (o != ref)
            nb = int(bad.sum())
            rec = {"K": K, "N": N, "run": r, "mismatch": nb}
            if nb:
                idx = bad.nonzero()
                rows, cols = idx[:, 0], idx[:, 1]
                rec.update(rows_unique=int(rows.unique().numel()), cols=sorted(set(cols.tolist()))[:12],
                           row_mod256=sorted(set((rows % 256).tolist()))[:12], first_rows=rows[:5].tolist(),
                           maxdiff=float((o - ref).abs().max()))
            print(json.dumps(rec), flush=True)
