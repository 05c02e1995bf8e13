"""Multi-GPU full-graph inference: edge-balanced row partition + per-layer exchange.

One process per GPU (torchrun), NCCL over NVLink/NVSwitch through
``torch.distributed``.  Within a layer every target row is independent
(batch invariance, glint/kernels.py:1-8), so rank k computes the contiguous
node range [p_k, p_{k+1}) of every full-mode layer and the only data-path
communication is one exchange per stored layer output that a later layer
reads: each rank broadcasts its row slice to all ranks (uneven slices, so P
root broadcasts rather than a padded all-gather).  The model output is never
exchanged; rows are gathered to the host once.

Split points balance aggregation bytes, not node counts: the cost of a row is
proportional to deg + 1 (its gathered rows), so p_k is the first node whose
prefix of (deg + 1) reaches k/P of the total.

Outputs are bit-identical for every P (tests/test_parallel_cpu.py checks the
partition and exchange logic on gloo; the GPU engine is the same code path
with a row range).
"""

from __future__ import annotations

import numpy as np


def edge_balanced_ranges(indptr_host, parts) -> np.ndarray:
    """P+1 split points over [0, N) balancing sum(deg+1) per part."""
    indptr_host = np.asarray(indptr_host, dtype=np.int64)
    n = len(indptr_host) - 1
    parts = int(parts)
    if parts < 1:
        raise ValueError("parts must be >= 1")
    cost = indptr_host + np.arange(n + 1, dtype=np.int64)     # prefix of (deg + 1)
    total = int(cost[-1])
    goals = (np.arange(parts + 1, dtype=np.float64) * total / parts)
    cuts = np.searchsorted(cost, goals, side="left").astype(np.int64)
    cuts[0], cuts[-1] = 0, n
    return np.maximum.accumulate(np.minimum(cuts, n))


class RowExchange:
    """After a block: broadcast each rank's slice of every store read later."""

    def __init__(self, cuts, rank, world, group=None):
        self.cuts = np.asarray(cuts, dtype=np.int64)
        self.rank, self.world, self.group = int(rank), int(world), group
        self.bytes_sent = 0

    @property
    def row_range(self):
        return int(self.cuts[self.rank]), int(self.cuts[self.rank + 1])

    def exchange_tensor(self, data):
        """In place: rows [cuts[k], cuts[k+1]) of `data` come from rank k."""
        import torch.distributed as dist

        works = []
        for k in range(self.world):
            lo, hi = int(self.cuts[k]), int(self.cuts[k + 1])
            if hi <= lo:
                continue
            part = data[lo:hi]
            if k == self.rank:
                self.bytes_sent += part.numel() * part.element_size()
            works.append(dist.broadcast(part, src=k, group=self.group, async_op=True))
        for w in works:
            w.wait()

    def __call__(self, engine, blk):
        """Hook for LayerwiseEngine.run: exchange outputs later blocks read.

        A store whose every later reader transforms its source rows first
        (reassociated ConvMean, ConvAttn) is skipped: those convs transform only
        the rank's own rows and exchange the result, which is narrower (layer 3:
        47 vs 256 columns) and spares every rank the other ranks' transforms."""
        from .splitter import TensorRef

        for o in blk.outputs:
            key = TensorRef(blk.block_id, o).key
            if key == engine.schedule.model_output.key:
                continue
            if engine.schedule.drop_after.get(key, blk.block_id) <= blk.block_id:
                continue
            readers = [c for c in engine.users.get(o, ()) if c not in blk.op_ids]
            if readers and all(engine.transform_first(c) for c in readers):
                continue
            self.exchange_tensor(engine.stores[key].data)
