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

Halo option (``kind="halo"``): a rank's aggregation reads only its own rows
and the source rows its CSR slice references, so instead of replicating every
slice everywhere each rank ships rank j exactly the rows of its range that j's
slice reads -- one all-to-all (variable splits) per exchanged store.  Every
rank holds the full CSR, so each computes every pair's row lists locally
(HaloPlan, once per run).  Rows nobody references are never sent; their
stale values are never read.  The model output is still replicated in full.
Measured halo sizes on the cfg5 graph: tools/halo_fraction.py.

Outputs are bit-identical for every P (tests/test_parallel_cpu.py checks the
partition and both exchanges on gloo; the GPU engine is the same code path
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


class HaloPlan:
    """Per-pair row lists of the halo exchange for `rank`.

    recv[k]: ascending global ids in rank k's range that this rank's CSR slice
    reads (received from k); send[j]: ids in this rank's range that rank j's
    slice reads (sent to j).  Self entries are empty.  Built from the full CSR
    (indptr on the host, indices on any device) with one unique() per slice."""

    def __init__(self, indptr_host, indices, cuts, rank):
        import torch

        self.cuts = np.asarray(cuts, dtype=np.int64)
        self.rank = int(rank)
        world = len(self.cuts) - 1
        indptr_host = np.asarray(indptr_host, dtype=np.int64)
        dev = indices.device
        need = []                     # need[j][k]: rows of k's range read by j's slice
        for j in range(world):
            lo, hi = int(self.cuts[j]), int(self.cuts[j + 1])
            src = torch.unique(indices[int(indptr_host[lo]):int(indptr_host[hi])].to(torch.int64))
            bounds = torch.searchsorted(src, torch.as_tensor(self.cuts, device=dev))
            row = []
            for k in range(world):
                if k == j:
                    row.append(src[:0])
                else:
                    row.append(src[int(bounds[k]):int(bounds[k + 1])])
            need.append(row)
        self.recv = [need[self.rank][k] for k in range(world)]
        self.send = [need[j][self.rank] for j in range(world)]
        self.recv_rows = torch.cat(self.recv) if world else indices.new_zeros(0, dtype=torch.int64)
        self.send_rows = torch.cat(self.send) if world else indices.new_zeros(0, dtype=torch.int64)
        self.recv_counts = [int(t.numel()) for t in self.recv]
        self.send_counts = [int(t.numel()) for t in self.send]

    def fraction(self, num_nodes):
        """Rows received / rows a full replication would receive."""
        own = int(self.cuts[self.rank + 1] - self.cuts[self.rank])
        return sum(self.recv_counts) / max(1, int(num_nodes) - own)


def _take_rows(data, rows):
    """data[rows] into a dense buffer: the glint row-copy kernel on CUDA; host
    tensors (the gloo logic tests) use torch indexing."""
    import torch

    out = torch.empty((rows.numel(), data.shape[1]), dtype=data.dtype, device=data.device)
    if rows.numel() == 0:
        return out
    if data.is_cuda:
        from . import kernels

        kernels.copy_rows(out, data, src_rows=rows)
    else:
        out.copy_(data[rows])
    return out


def _put_rows(data, rows, buf):
    if rows.numel() == 0:
        return
    if data.is_cuda:
        from . import kernels

        kernels.copy_rows(data, buf, dst_rows=rows)
    else:
        data[rows] = buf


class RowExchange:
    """Broadcast each rank's slice of every store read later.

    Overlapped with the block: each rank range is cut into `chunks` pieces;
    after every batch the engine reports how far its rows are done
    (progress), and each fully computed piece is posted at once -- P root
    broadcasts per piece, in the same (piece, root, store) order on every rank
    -- on the collective stream, while the next batches compute.  The block
    end posts whatever is left and waits."""

    def __init__(self, cuts, rank, world, group=None, chunks=4, halo=None):
        self.cuts = np.asarray(cuts, dtype=np.int64)
        self.rank, self.world, self.group = int(rank), int(world), group
        self.halo = halo                # HaloPlan: ship only the rows other ranks read
        # the halo exchange runs once per store at the block end (its rows are
        # scattered, not contiguous pieces)
        self.chunks = 1 if halo is not None else max(1, int(chunks))
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

    def _halo_exchange(self, data):
        """One all-to-all: this rank's rows that rank j reads go to j; the rows
        this rank reads from rank k arrive from k and are scattered in place."""
        import torch.distributed as dist

        plan = self.halo
        send = _take_rows(data, plan.send_rows)
        recv = data.new_empty((plan.recv_rows.numel(), data.shape[1]))
        self.bytes_sent += send.numel() * send.element_size()
        dist.all_to_all_single(recv, send, output_split_sizes=plan.recv_counts,
                               input_split_sizes=plan.send_counts, group=self.group)
        _put_rows(data, plan.recv_rows, recv)

    def _post(self, engine, keys, upto):
        if self.halo is not None:
            if self._posted < upto:
                for key in keys:
                    data = engine.stores[key].data
                    # the store may be wider than its pitch view: exchange the
                    # underlying row-major rows
                    self._halo_exchange(data)
                self._posted = upto
            return
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
        """exchange_tensor over several row-aligned tensors in one grouped
        collective (halo mode: only the rows other ranks' slices read)."""
        if self.halo is not None:
            for data in tensors:
                self._halo_exchange(data)
            return
        self.replicate_tensors(tensors)

    def replicate_tensor(self, data):
        """Every rank gets every row (the model output), whatever the mode."""
        self.replicate_tensors((data,))

    def replicate_tensors(self, tensors):
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
