#!/usr/bin/env python
"""Halo size of the row-partitioned exchange on the cfg5 (Papers100M-shaped)
graph (run on the B200 box; the graph is generated on the device).

For P ranks with edge-balanced contiguous ranges [p_k, p_{k+1}), rank j's
aggregation reads the source rows of its CSR slice.  Full replication ships
every rank (P-1)/P of all rows per exchange; a halo exchange ships only the
remote rows rank j's slice references.  Prints, per (order, P), the halo rows
per rank as a fraction of the remote rows (mean and max over ranks), i.e. the
fraction of full-replication exchange bytes the halo exchange moves.
"""

from __future__ import annotations

import argparse
import json
import pathlib
import sys
import time

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def halo_stats(indptr, indices, n, parts):
    import numpy as np
    import torch

    from paper_2211_15082_b200.parallel import edge_balanced_ranges

    cuts = edge_balanced_ranges(indptr.cpu().numpy(), parts)
    fr, rows = [], []
    for j in range(parts):
        lo, hi = int(cuts[j]), int(cuts[j + 1])
        e0, e1 = int(indptr[lo]), int(indptr[hi])
        src = torch.unique(indices[e0:e1])
        remote = int(((src < lo) | (src >= hi)).sum())
        fr.append(remote / max(1, n - (hi - lo)))
        rows.append(remote)
        del src
    return {"parts": parts, "halo_frac_mean": float(np.mean(fr)), "halo_frac_max": float(np.max(fr)),
            "halo_rows_mean": float(np.mean(rows)), "cuts": [int(c) for c in cuts]}


def main():
    import torch

    from paper_2211_15082_b200 import synth

    ap = argparse.ArgumentParser()
    ap.add_argument("--nodes", type=int, default=synth.PAPERS_NODES)
    ap.add_argument("--edges", type=int, default=synth.PAPERS_EDGES)
    ap.add_argument("--parts", default="2,4,8")
    ap.add_argument("--orders", default="none,degree")
    args = ap.parse_args()
    t = time.time()
    g = synth.gen_products_like(args.nodes, args.edges // 2, seed=0, device="cuda")
    n = g.num_nodes
    print(json.dumps({"graph": {"nodes": n, "edges": g.num_edges, "gen_s": round(time.time() - t, 1)}}),
          flush=True)
    indptr, indices = g.indptr, g.indices
    for order in args.orders.split(","):
        if order == "degree":
            # relabel by descending degree (ties by id): new id = rank in that order
            deg = indptr[1:] - indptr[:-1]
            perm = torch.argsort(-deg * (n + 1) + torch.arange(n, device="cuda"))
            inv = torch.empty_like(perm)
            inv[perm] = torch.arange(n, device="cuda")
            new_deg = deg[perm]
            new_indptr = torch.zeros(n + 1, dtype=torch.int64, device="cuda")
            torch.cumsum(new_deg, 0, out=new_indptr[1:])
            # rows in new order; sources renamed (slice order within a row is kept)
            dst_new = torch.repeat_interleave(torch.arange(n, device="cuda"), new_deg)
            src_pos = (indptr[perm][dst_new] + (torch.arange(dst_new.numel(), device="cuda")
                                                 - new_indptr[dst_new]))
            del dst_new
            new_indices = inv[indices[src_pos].long()].to(torch.int32)
            del src_pos
            ip, ix = new_indptr, new_indices
        else:
            ip, ix = indptr, indices
        for p in (int(x) for x in args.parts.split(",")):
            rec = halo_stats(ip, ix, n, p)
            rec.update(order=order)
            rec.pop("cuts")
            print(json.dumps(rec), flush=True)
        if order == "degree":
            del ip, ix, new_indptr, new_indices, perm, inv


if __name__ == "__main__":
    main()
