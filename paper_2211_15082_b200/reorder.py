"""Node orders and physical relabelling (behaviour of glint/reorder.py).

* ``rcmk`` -- reverse Cuthill-McKee with the reference's tie rules
  (glint/reorder.py:72-123), computed by the native host routine
  ``glint_rcmk_host`` in libglint_b200.so (O(E log d) instead of a Python BFS
  at ~65 us/node).  Byte-identical permutation (tests/golden).
* ``degree_sort`` (stable ascending in-degree), ``random_order``
  (numpy default_rng(seed).permutation) -- host numpy, as in the reference.
* ``apply_order`` -- relabels the CSC on the DEVICE (glint_relabel_csc: each
  slice mapped elementwise through inv, stored order preserved, which keeps
  every aggregation's summation order and hence the output bytes) and permutes
  feature rows with glint_copy_rows_f32.
"""

from __future__ import annotations

import ctypes
import struct
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import FormatError
from .storage import CscGraph

PERM_MAGIC = b"DGIP"


@dataclass(frozen=True)
class NodeOrder:
    """perm[new position] = old id; inv[old id] = new position."""

    perm: np.ndarray

    def __post_init__(self):
        from .storage import arange_ids

        perm = np.ascontiguousarray(self.perm, dtype=np.int64)
        n = len(perm)
        if perm is arange_ids(n):          # cached identity: nothing to check or invert
            object.__setattr__(self, "perm", perm)
            object.__setattr__(self, "_inv", perm)
            return
        if n and not (perm[0] == 0 and perm[-1] == n - 1 and np.all(np.diff(perm) == 1)):
            seen = np.zeros(n, dtype=bool)
            ok = perm.min() >= 0 and perm.max() < n
            if ok:
                seen[perm] = True
            if not ok or not seen.all():
                raise ValueError("perm is not a permutation")
        inv = np.empty(n, dtype=np.int64)
        inv[perm] = np.arange(n, dtype=np.int64)
        object.__setattr__(self, "perm", perm)
        object.__setattr__(self, "_inv", inv)

    @property
    def inv(self) -> np.ndarray:
        return self._inv

    @property
    def num_nodes(self) -> int:
        return len(self.perm)

    def is_identity(self) -> bool:
        from .storage import arange_ids

        if self.perm is arange_ids(self.num_nodes):
            return True
        return bool(np.array_equal(self.perm, np.arange(self.num_nodes)))


def identity_order(g) -> NodeOrder:
    from .storage import arange_ids

    return NodeOrder(arange_ids(g.num_nodes))


def _host_csc(g):
    if isinstance(g, CscGraph):
        return g.indptr, g.indices
    return g.indptr_host, g.indices.cpu().numpy().astype(np.int64)


def _sorted_adjacency_device(dg):
    """Symmetrised adjacency of a DeviceGraph with every row deduplicated, free
    of self loops and ordered by (degree, id) -- the order the RCMK BFS visits
    candidates in (reorder.py:89-99).  Two device sorts: (row, col) to merge
    duplicates and count degrees, then (row, rank of col by (degree, id)).
    Returns device (ptr int64 [n+1], adj int32 [nnz], rank int64 [n]: each
    node's position in the (degree, id) order)."""
    import torch

    n = int(dg.num_nodes)
    dev = dg.indptr.device
    deg_in = dg.indptr[1:] - dg.indptr[:-1]
    dst = torch.repeat_interleave(torch.arange(n, device=dev), deg_in)
    src = dg.indices.to(torch.int64)
    keep = src != dst
    src, dst = src[keep], dst[keep]
    key = torch.unique(torch.cat([src * n + dst, dst * n + src]))   # sorted, deduplicated
    del src, dst, keep
    row = key // n
    col = key - row * n
    del key
    deg = torch.bincount(row, minlength=n)
    order = torch.sort(deg * n + torch.arange(n, device=dev)).indices     # by (degree, id)
    rank = torch.empty_like(order)
    rank[order] = torch.arange(n, device=dev)
    key2 = torch.sort(row * n + rank[col]).values
    del row, col
    adj = order[key2 % n].to(torch.int32)
    ptr = torch.zeros(n + 1, dtype=torch.int64, device=dev)
    torch.cumsum(deg, 0, out=ptr[1:])
    return ptr, adj, rank


# Level cap of the device BFS: path-like graphs with thousands of BFS levels
# are faster on the host's linear queue than one device round trip per level.
RCMK_MAX_DEVICE_LEVELS = 4096


def _rcmk_device(dg):
    """RCMK on the device, the same permutation as the sequential reference
    (reorder.py:72-123): components by union-find, starts = each component's
    minimum (degree, id) member, components in ascending start order, then a
    level-synchronous BFS over every component at once in which a node's
    parent is its first neighbour in the previous level's sequence and each
    level is ordered by (parent index, (degree, id) rank) -- exactly the order
    the sequential queue appends nodes in.  Returns perm (host int64), or None
    past RCMK_MAX_DEVICE_LEVELS levels."""
    import torch

    from . import kernels

    n = int(dg.num_nodes)
    dev = dg.indptr.device
    ptr, adj, rank = _sorted_adjacency_device(dg)
    st = kernels.stream_handle()
    comp = torch.empty(n, dtype=torch.int32, device=dev)
    _lib.call("glint_rcmk_components", n, kernels.ptr(ptr), kernels.ptr(adj), kernels.ptr(comp), st)
    start_key = torch.empty(n, dtype=torch.int64, device=dev)
    _lib.call("glint_rcmk_starts", n, kernels.ptr(ptr), kernels.ptr(comp), kernels.ptr(start_key), st)
    ids = torch.arange(n, device=dev, dtype=torch.int64)
    roots = torch.nonzero(comp.to(torch.int64) == ids).flatten()
    starts = torch.sort(start_key[roots] & 0xFFFFFFFF).values          # component order
    comp_rank = torch.empty(n, dtype=torch.int64, device=dev)
    comp_rank[comp[starts].to(torch.int64)] = torch.arange(len(starts), device=dev)
    level = torch.full((n,), -1, dtype=torch.int32, device=dev)
    gidx = torch.empty(n, dtype=torch.int64, device=dev)
    best = torch.full((n,), torch.iinfo(torch.int64).max, dtype=torch.int64, device=dev)
    none = torch.iinfo(torch.int64).max
    frontier = starts.to(torch.int32)
    level[starts] = 0
    gidx[starts] = torch.arange(len(starts), device=dev)
    depth = 0
    while len(frontier):
        if depth >= RCMK_MAX_DEVICE_LEVELS:
            return None
        _lib.call("glint_rcmk_expand", len(frontier), kernels.ptr(frontier), kernels.ptr(ptr),
                  kernels.ptr(adj), kernels.ptr(level), kernels.ptr(best), st)
        cand = torch.nonzero(best != none).flatten()
        if len(cand) == 0:
            break
        order = torch.sort(best[cand] * n + rank[cand]).indices
        nxt = cand[order]
        best[cand] = none
        depth += 1
        level[nxt] = depth
        gidx[nxt] = torch.arange(len(nxt), device=dev)
        frontier = nxt.to(torch.int32)
    # sequence = (component, level, index in level); RCMK reverses it
    seq = torch.sort(gidx, stable=True).indices
    key1 = comp_rank[comp[seq].to(torch.int64)] * (depth + 1) + level[seq].to(torch.int64)
    seq = seq[torch.sort(key1, stable=True).indices]
    return seq.flip(0).cpu().numpy().astype(np.int64)


def rcmk(g) -> NodeOrder:
    """Reverse Cuthill-McKee over in- plus out-edges.

    A DeviceGraph runs entirely on the device (_rcmk_device: union-find
    components and a level-synchronous BFS; a linear native BFS on the host for
    graphs deeper than RCMK_MAX_DEVICE_LEVELS); a host CscGraph runs the
    all-host native version (same tie rules, same permutation).
    """
    from .storage import DeviceGraph

    if isinstance(g, DeviceGraph) and int(g.num_nodes) > 0:
        # a pure function of the (immutable) graph: computed once per DeviceGraph
        hit = g._cache.get("rcmk_order")
        if hit is not None:
            return hit
        perm = _rcmk_device(g)
        if perm is not None:
            order = g._cache["rcmk_order"] = NodeOrder(perm)
            return order
        ptr, adj, _ = _sorted_adjacency_device(g)      # deep BFS: the host's queue
        ptr, adj = ptr.cpu().numpy(), adj.cpu().numpy()
        n = int(g.num_nodes)
        perm = np.empty(n, dtype=np.int64)
        rc = _lib.load().glint_rcmk_sorted_host(n, ptr.ctypes.data_as(ctypes.c_void_p),
                                                adj.ctypes.data_as(ctypes.c_void_p),
                                                perm.ctypes.data_as(ctypes.c_void_p))
        if rc != 0:
            raise ValueError(f"rcmk failed with status {rc}")
        return NodeOrder(perm)
    indptr, indices = _host_csc(g)
    indptr = np.ascontiguousarray(indptr, dtype=np.int64)
    indices = np.ascontiguousarray(indices, dtype=np.int64)
    n = int(g.num_nodes)
    perm = np.empty(n, dtype=np.int64)
    rc = _lib.load().glint_rcmk_host(n, indptr.ctypes.data_as(ctypes.c_void_p),
                                     indices.ctypes.data_as(ctypes.c_void_p),
                                     perm.ctypes.data_as(ctypes.c_void_p))
    if rc != 0:
        raise ValueError(f"rcmk failed with status {rc}")
    return NodeOrder(perm)


def degree_sort(g) -> NodeOrder:
    degs = g.in_degrees if isinstance(g, CscGraph) else np.diff(g.indptr_host)
    return NodeOrder(np.argsort(degs, kind="stable").astype(np.int64))


def random_order(g, seed) -> NodeOrder:
    return NodeOrder(np.random.default_rng(seed).permutation(g.num_nodes).astype(np.int64))


def make_order(g, kind, seed=0) -> NodeOrder:
    makers = {"none": lambda: identity_order(g), "rcmk": lambda: rcmk(g),
              "degree": lambda: degree_sort(g), "random": lambda: random_order(g, seed)}
    if kind not in makers:
        raise ValueError(f"unknown order kind {kind!r}")
    return makers[kind]()


def apply_order(g, x, order: NodeOrder):
    """Relabel graph + permute feature rows under `order` (glint/reorder.py:149-181).

    The work runs on the GPU; the result has the same kind as the inputs
    (CscGraph / numpy / EmbeddingStore in -> host out, DeviceGraph / CUDA
    tensor in -> device out).
    """
    from .storage import CscGraph, EmbeddingStore

    if order.num_nodes != g.num_nodes:
        raise ValueError(f"order over {order.num_nodes} nodes, graph has {g.num_nodes}")
    if order.is_identity():
        return g, x
    g2, x2 = apply_order_device(g, x, order)
    if isinstance(g, CscGraph):
        g2 = g2.to_host()
    if isinstance(x, EmbeddingStore):
        st = EmbeddingStore(x.num_rows, x.dim)
        st._data = x2.cpu().numpy()
        x2 = st
    elif isinstance(x, np.ndarray):
        x2 = x2.cpu().numpy()
    return g2, x2


def apply_order_device(g, x, order: NodeOrder):
    """Device relabel; always returns (DeviceGraph, device features or None)."""
    import torch

    from . import kernels
    from .storage import DeviceGraph, DeviceStore

    if order.num_nodes != g.num_nodes:
        raise ValueError(f"order over {order.num_nodes} nodes, graph has {g.num_nodes}")
    dg = kernels.device_graph(g)
    if order.is_identity():
        return dg, x
    dev = dg.indptr.device
    hit = dg._cache.get("relabelled")
    if hit is not None and hit[0] is order:       # same graph, same order: same CSC
        perm, g2 = hit[1], hit[2]
    else:
        perm = torch.from_numpy(order.perm).to(dev)
        inv = torch.from_numpy(order.inv).to(dev)
        new_indptr = kernels.degree_prefix_dev(dg, perm)
        new_indices = torch.empty_like(dg.indices)
        _lib.call("glint_relabel_csc", dg.num_nodes, kernels.ptr(dg.indptr),
                  kernels.ptr(dg.indices), kernels.ptr(perm), kernels.ptr(inv),
                  kernels.ptr(new_indptr), kernels.ptr(new_indices), kernels.stream_handle())
        host_ptr = np.zeros(dg.num_nodes + 1, dtype=np.int64)
        np.cumsum(np.diff(dg.indptr_host)[order.perm], out=host_ptr[1:])
        g2 = DeviceGraph(dg.num_nodes, dg.num_edges, new_indptr, new_indices, host_ptr)
        if dg is g:               # a caller's DeviceGraph (not a fresh upload): keep it
            dg._cache["relabelled"] = (order, perm, g2)
    if x is None:
        return g2, None
    if isinstance(x, DeviceStore):
        x2 = DeviceStore(x.num_rows, x.dim, dev)
        kernels.copy_rows(x2.view(), x.view(), src_rows=perm)
        return g2, x2
    xd = kernels.to_device(x.to_array() if hasattr(x, "to_array") else x, torch.float32)
    if xd.shape[0] != g.num_nodes:
        raise ValueError(f"feature rows {xd.shape[0]} != num_nodes {g.num_nodes}")
    out = torch.empty_like(xd)
    kernels.copy_rows(out, xd, src_rows=perm)
    return g2, out


def bandwidth(g) -> int:
    indptr, indices = _host_csc(g)
    if len(indices) == 0:
        return 0
    dst = np.repeat(np.arange(g.num_nodes, dtype=np.int64), np.diff(indptr))
    return int(np.max(np.abs(indices - dst)))


def save_order(order: NodeOrder, path):
    with open(path, "wb") as f:
        f.write(PERM_MAGIC + struct.pack("<Q", order.num_nodes))
        f.write(order.perm.astype("<u8").tobytes())


def load_order(path) -> NodeOrder:
    with open(path, "rb") as f:
        if f.read(4) != PERM_MAGIC:
            raise FormatError("bad permutation magic at offset 0")
        (n,) = struct.unpack("<Q", f.read(8))
        perm = np.frombuffer(f.read(8 * n), dtype="<u8")
        if len(perm) != n:
            raise FormatError("truncated permutation file")
    return NodeOrder(perm.astype(np.int64))
