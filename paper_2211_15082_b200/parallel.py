"""Multi-GPU full-graph inference: edge-balanced row partition + per-layer exchange.

One process per GPU (torchrun), NCCL over NVLink/NVSwitch through
``torch.distributed``.  Within a layer every target row is independent
(batch invariance, glint/kernels.py:1-8), so rank k computes the contiguous
node range [p_k, p_{k+1}) of every full-mode layer and the only data-path
communication is one exchange per stored layer output that a later layer
reads: each rank broadcasts its row slice to all ranks.  The slices are
uneven, so this is P root broadcasts rather than a padded all-gather, issued
as ONE grouped NCCL collective (ncclGroupStart/End through torch's coalescing
manager) per exchanged piece.  The model output is never
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
    """Broadcast each rank's slice of every store read later.

    Overlapped with the block: each rank range is cut into `chunks` pieces;
    after every batch the engine reports how far its rows are done
    (progress), and each fully computed piece is posted at once -- P root
    broadcasts per piece, in the same (piece, root, store) order on every rank
    -- on the collective stream, while the next batches compute.  The block
    end posts whatever is left and waits."""

    def __init__(self, cuts, rank, world, group=None, chunks=4):
        self.cuts = np.asarray(cuts, dtype=np.int64)
        self.rank, self.world, self.group = int(rank), int(world), group
        self.chunks = max(1, int(chunks))
        self.bytes_sent = 0
        self._blk = None
        self._posted = 0
        self._works = []

    def _piece(self, k, c):
        lo, hi = int(self.cuts[k]), int(self.cuts[k + 1])
        return lo + (hi - lo) * c // self.chunks, lo + (hi - lo) * (c + 1) // self.chunks

    def _keys(self, engine, blk):
        from .splitter import TensorRef

        keys = []
        for o in blk.outputs:
            key = TensorRef(blk.block_id, o).key
            if key == engine.schedule.model_output.key:
                continue
            if engine.schedule.drop_after.get(key, blk.block_id) <= blk.block_id:
                continue
            readers = [c for c in engine.users.get(o, ()) if c not in blk.op_ids]
            if readers and all(engine.transform_first(c) for c in readers):
                continue
            keys.append(key)
        return keys

    def _group_device(self):
        """The CUDA device to coalesce on (NCCL), or None (gloo: serial)."""
        import torch
        import torch.distributed as dist

        if dist.get_backend(self.group) != "nccl":
            return None
        return torch.device("cuda", torch.cuda.current_device())

    def _broadcasts(self, parts):
        """[(tensor, root)] as ONE grouped collective on NCCL (ncclGroupStart /
        ncclGroupEnd around the P root broadcasts: the transfers run concurrently
        instead of one root after another); serial async broadcasts on gloo.
        Returns the work handles."""
        import torch.distributed as dist

        parts = [(t, k) for t, k in parts if t.numel()]
        if not parts:
            return []
        dev = self._group_device()
        if dev is None:
            return [dist.broadcast(t, src=k, group=self.group, async_op=True) for t, k in parts]
        with dist._coalescing_manager(group=self.group, device=dev, async_ops=True) as cm:
            for t, k in parts:
                dist.broadcast(t, src=k, group=self.group, async_op=True)
        return [cm]

    def _post(self, engine, keys, upto):
        while self._posted < upto:
            c = self._posted
            parts = []
            for k in range(self.world):
                lo, hi = self._piece(k, c)
                if hi <= lo:
                    continue
                for key in keys:
                    part = engine.stores[key].data[lo:hi]
                    if k == self.rank:
                        self.bytes_sent += part.numel() * part.element_size()
                    parts.append((part, k))
            self._works += self._broadcasts(parts)
            self._posted += 1

    def piece_bounds(self):
        """Row bounds of this rank's pieces: the engine cuts its launches there,
        so each finished piece is broadcast while the next one computes (one
        whole-layer launch would leave nothing to overlap)."""
        return [self._piece(self.rank, c)[1] for c in range(self.chunks)]

    def progress(self, engine, blk, done_hi):
        """Rows [.., done_hi) of this rank's range are computed for `blk`."""
        if self._blk is not blk:
            self._blk, self._posted, self._works = blk, 0, []
            self._keys_cache = self._keys(engine, blk)
        if not self._keys_cache:
            return
        ready = 0
        while ready < self.chunks and self._piece(self.rank, ready)[1] <= done_hi:
            ready += 1
        self._post(engine, self._keys_cache, ready)

    @property
    def row_range(self):
        return int(self.cuts[self.rank]), int(self.cuts[self.rank + 1])

    def exchange_tensor(self, data):
        """In place: rows [cuts[k], cuts[k+1]) of `data` come from rank k."""
        self.exchange_tensors((data,))

    def exchange_tensors(self, tensors):
        """exchange_tensor over several row-aligned tensors in one grouped collective."""
        parts = []
        for k in range(self.world):
            lo, hi = int(self.cuts[k]), int(self.cuts[k + 1])
            if hi <= lo:
                continue
            for data in tensors:
                part = data[lo:hi]
                if k == self.rank:
                    self.bytes_sent += part.numel() * part.element_size()
                parts.append((part, k))
        for w in self._broadcasts(parts):
            w.wait()

    def __call__(self, engine, blk):
        """Hook for LayerwiseEngine.run at the end of a block: post the pieces
        not yet sent and wait for all of them.

        A store whose every later reader transforms its source rows first
        (reassociated ConvMean, ConvAttn) is skipped: those convs transform only
        the rank's own rows and exchange the result, which is narrower (layer 3:
        47 vs 256 columns) and spares every rank the other ranks' transforms."""
        if self._blk is not blk:
            self._blk, self._posted, self._works = blk, 0, []
            self._keys_cache = self._keys(engine, blk)
        self._post(engine, self._keys_cache, self.chunks)
        for w in self._works:
            w.wait()
        self._blk, self._posted, self._works = None, 0, []
