"""Drop-in device kernels for glint/kernels.py, running on the sm_100a library.

Signatures, argument meaning and errors follow the reference module
(glint/kernels.py:28-239): ``agg_mean(bc, h_in)``, ``agg_attn(bc, h_in,
params)``, ``linear(x, weight, bias)``, ``elementwise(kind, inputs)``,
``concat(parts)``, ``build_batch_csc(graph, targets)``,
``gather_slices(graph, targets)``, ``trivial_batch_csc(targets)``.
Shape errors raise ``ValueError`` as in the reference.

Arrays may be numpy (copied to the GPU, result copied back as numpy) or CUDA
torch tensors (results stay on the device).  Every numeric result is produced
by a kernel in ``libglint_b200.so``; torch only allocates memory and supplies
streams.  There is no CPU path: without a CUDA device every call raises.

Numerics: ``agg_mean`` is byte-identical to the reference (sequential fp32
adds in stored order, self last, IEEE division).  ``linear`` / the attention
projection accumulate in fp32 (or split-TF32 on tensor cores) in a fixed
order per row, so results are row/batch invariant but not bitwise equal to
numpy's einsum; they agree within the stated tolerance (tests use rel-L2 <=
1e-5 per kernel, 1e-4 end to end).
"""

from __future__ import annotations

import os

from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import InternalError

LEAKY_SLOPE = np.float32(0.2)
NORM_EPS = np.float32(1e-12)
ELEMENTWISE_KINDS = ("ReLU", "LeakyReLU", "Add", "Norm", "DropoutIdentity")

# Degree threshold (deg + 1, power of two) above which a row is aggregated by a
# whole CTA instead of one warp (see csrc/aggregate.cu).
HUB_MIN_DEGREE = 512

# GEMM precision used by linear / attention projection: split-TF32 on the
# tcgen05 tensor cores (~1e-6 rel-L2 vs fp64); PREC_FP32 selects the CUDA-core
# fp32 FMA-chain kernel.
PRECISION = _lib.PREC_3XTF32
# K7 fused aggregate->transform for aggregate-first ConvMeans (GLINT_FUSE_CONV=0: K1 + K2)
FUSE_CONV = os.environ.get("GLINT_FUSE_CONV", "1") == "1"


def _torch():
    import torch

    return torch


def cuda_device(device=None):
    torch = _torch()
    if not torch.cuda.is_available():
        raise InternalError("no CUDA device visible: the B200 kernels have no CPU fallback")
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    dev = torch.device(device)
    if dev.type != "cuda":
        raise InternalError(f"device {dev} is not a CUDA device")
    return dev if dev.index is not None else torch.device("cuda", torch.cuda.current_device())


def stream_handle():
    return _torch().cuda.current_stream().cuda_stream


def ptr(t):
    return None if t is None else t.data_ptr()


def ld(t) -> int:
    if t.dim() != 2 or (t.shape[1] > 1 and t.stride(1) != 1):
        raise ValueError("matrix operands must be 2-D with unit column stride")
    return max(int(t.stride(0)), int(t.shape[1]))


def to_device(x, dtype=None, device=None):
    """numpy / torch -> contiguous-rows CUDA tensor (no copy when already there)."""
    torch = _torch()
    dev = cuda_device(device)
    if isinstance(x, torch.Tensor):
        t = x
        if dtype is not None and t.dtype != dtype:
            t = t.to(dtype)
        if t.device != dev:
            t = t.to(dev)
        if t.dim() == 2 and t.shape[1] > 1 and t.stride(1) != 1:
            t = t.contiguous()
        return t
    arr = np.asarray(x)
    if dtype is None:
        dtype = torch.float32 if arr.dtype.kind == "f" else torch.int64
    np_dtype = {torch.float32: np.float32, torch.int64: np.int64, torch.int32: np.int32}[dtype]
    arr = np.ascontiguousarray(arr, dtype=np_dtype)
    if arr.nbytes >= PAGEABLE_STAGED_MIN:
        # large host arrays: the library's multi-threaded pinned staging
        # (glint_h2d_pageable) instead of the driver's ~10 GB/s pageable path
        out = torch.empty(arr.shape, dtype=dtype, device=dev)
        _lib.call("glint_h2d_pageable", out.data_ptr(), arr.ctypes.data, arr.nbytes,
                  PAGEABLE_THREADS, stream_handle())
        return out
    return torch.from_numpy(arr).to(dev)


# numpy arrays at least this large go through glint_h2d_pageable
PAGEABLE_STAGED_MIN = int(os.environ.get("GLINT_PAGEABLE_STAGED_MIN", 8 << 20))
PAGEABLE_THREADS = int(os.environ.get("GLINT_PAGEABLE_THREADS", 8))


def _f32(x):
    return to_device(x, _torch().float32)


def _i64(x):
    return to_device(x, _torch().int64)


def _is_host(*xs) -> bool:
    torch = _torch()
    return any(not isinstance(x, torch.Tensor) for x in xs if x is not None)


def _ret(t, host):
    return t.cpu().numpy() if host else t


def narrow_ids_into(out32, idx64, limit, bad):
    """int64 -> int32 into `out32` on the current stream; bad (device int64[1])
    receives the count of ids outside [0, limit) -- no host sync."""
    _lib.call("glint_narrow_ids", idx64.shape[0], ptr(idx64), ptr(out32), int(limit), ptr(bad),
              stream_handle())
    return out32


def narrow_ids(idx64, limit):
    """int64 -> int32 device ids, raising if any id is outside [0, limit)."""
    torch = _torch()
    out = torch.empty(idx64.shape[0], dtype=torch.int32, device=idx64.device)
    bad = torch.empty(1, dtype=torch.int64, device=idx64.device)
    _lib.call("glint_narrow_ids", idx64.shape[0], ptr(idx64), ptr(out), int(limit), ptr(bad),
              stream_handle())
    if int(bad.item()):
        raise ValueError(f"{int(bad.item())} node ids outside [0, {limit})")
    return out


# ------------------------------------------------------------------ graphs --


def device_graph(graph, device=None):
    """CscGraph / DeviceGraph -> DeviceGraph (a host graph is uploaded on every call)."""
    from .storage import CscGraph, DeviceGraph

    if isinstance(graph, DeviceGraph):
        return graph
    if isinstance(graph, CscGraph):
        return DeviceGraph.from_host(graph, device)
    raise TypeError(f"expected a CscGraph or DeviceGraph, got {type(graph).__name__}")


class IdSet:
    """Sorted node-id set over [0, N) held as a device bitmap + rank prefix."""

    def __init__(self, num_nodes, device=None):
        torch = _torch()
        self.n = int(num_nodes)
        nbytes = _lib.query("glint_idset_workspace_bytes", self.n)
        self.ws = torch.empty((nbytes + 7) // 8, dtype=torch.int64, device=cuda_device(device))
        self.count_dev = torch.zeros(1, dtype=torch.int64, device=self.ws.device)
        _lib.call("glint_idset_clear", ptr(self.ws), self.n, stream_handle())

    def add_ids(self, ids=None, base=0, n=0):
        if ids is not None:
            n = ids.shape[0]
        _lib.call("glint_idset_add_ids", ptr(self.ws), self.n, ptr(ids), int(base), int(n),
                  stream_handle())
        return self

    def add_neighbors(self, g, targets=None, base=0, n=0):
        if targets is not None:
            n = targets.shape[0]
        _lib.call("glint_idset_add_neighbors", ptr(self.ws), self.n, ptr(g.indptr),
                  ptr(g.indices), ptr(targets), int(base), int(n), stream_handle())
        return self

    def finalize(self):
        _lib.call("glint_idset_finalize", ptr(self.ws), self.n, ptr(self.count_dev),
                  stream_handle())
        return self

    def count(self) -> int:
        return int(self.count_dev.item())

    def extract(self, count=None):
        torch = _torch()
        count = self.count() if count is None else count
        out = torch.empty(count, dtype=torch.int64, device=self.ws.device)
        if count:
            _lib.call("glint_idset_extract", ptr(self.ws), self.n, ptr(out), stream_handle())
        return out

    def lookup(self, ids=None, ids32=None, want64=True, want32=False):
        torch = _torch()
        n = (ids if ids is not None else ids32).shape[0]
        p64 = torch.empty(n, dtype=torch.int64, device=self.ws.device) if want64 else None
        p32 = torch.empty(n, dtype=torch.int32, device=self.ws.device) if want32 else None
        _lib.call("glint_idset_lookup", ptr(self.ws), self.n, ptr(ids), ptr(ids32), n, ptr(p64),
                  ptr(p32), stream_handle())
        return p64, p32

    def rank_map(self):
        torch = _torch()
        out = torch.empty(self.n, dtype=torch.int32, device=self.ws.device)
        _lib.call("glint_idset_rank_map", ptr(self.ws), self.n, ptr(out), stream_handle())
        return out


def degree_prefix_dev(g, targets=None, base=0, n=0):
    """Device exclusive prefix of in-degrees over targets (n+1 entries)."""
    torch = _torch()
    if targets is not None:
        n = targets.shape[0]
    out = torch.empty(n + 1, dtype=torch.int64, device=g.indptr.device)
    wsb = _lib.query("glint_scan_workspace_bytes", n)
    ws = torch.empty((wsb + 7) // 8, dtype=torch.int64, device=g.indptr.device)
    _lib.call("glint_degree_prefix", ptr(g.indptr), ptr(targets), int(base), int(n), ptr(out),
              ptr(ws), wsb, stream_handle())
    return out


def hub_prefix_dev(g, targets=None, base=0, n=0, hub_min=None):
    """Device exclusive prefix of hub flags (deg+1 >= HUB_MIN_DEGREE) over targets."""
    torch = _torch()
    hub_min = HUB_MIN_DEGREE if hub_min is None else hub_min
    if targets is not None:
        n = targets.shape[0]
    out = torch.empty(n + 1, dtype=torch.int64, device=g.indptr.device)
    wsb = _lib.query("glint_scan_workspace_bytes", n)
    ws = torch.empty((wsb + 7) // 8, dtype=torch.int64, device=g.indptr.device)
    _lib.call("glint_hub_prefix", ptr(g.indptr), ptr(targets), int(base), int(n), int(hub_min),
              ptr(out), ptr(ws), wsb, stream_handle())
    return out


def degree_schedule(indptr, row_ids=None, row_base=0, n_rows=0, hub_min=None):
    """Longest-first row order (int32) and hub count, computed on the device.

    Returns (schedule tensor, n_hub device tensor).  The host count of hubs is
    available from the host degrees without a sync (see executor).
    """
    torch = _torch()
    hub_min = HUB_MIN_DEGREE if hub_min is None else hub_min
    if row_ids is not None:
        n_rows = row_ids.shape[0]
    sched = torch.empty(max(n_rows, 1), dtype=torch.int32, device=indptr.device)
    n_hub = torch.zeros(1, dtype=torch.int64, device=indptr.device)
    wsb = _lib.query("glint_degree_schedule_workspace_bytes")
    ws = torch.empty((wsb + 7) // 8, dtype=torch.int64, device=indptr.device)
    _lib.call("glint_degree_schedule", int(n_rows), ptr(indptr), ptr(row_ids), int(row_base),
              int(hub_min), ptr(sched), ptr(n_hub), ptr(ws), wsb, stream_handle())
    return sched, n_hub


def sample_neighbors_dev(dg, nodes, fanout, seed, layer):
    """Device neighbour sampling (glint/executor.py:74-115) -> DeviceGraph.

    nodes: sorted unique host int64 ids (or None = every node).  The segment
    offsets come from the host indptr (no device sync); draws, selection and
    the ascending sort of each kept slice run in glint_sample_neighbors.
    """
    import numpy as np

    from .storage import DeviceGraph

    torch = _torch()
    n = int(dg.num_nodes)
    dev = dg.indptr.device
    ip_h = np.asarray(dg.indptr_host, dtype=np.int64)
    select = int(fanout) <= 32 and int(_lib.query("glint_get_tuning", 15)) == 0
    if nodes is None:
        # offsets of an all-node draw depend only on (graph, fanout): cached,
        # so a sampling run's 3 draws and every later run skip the host scans
        key = ("sample_offsets", int(fanout))
        hit = dg._cache.get(key)
        if hit is None:
            kept = np.minimum(np.diff(ip_h), int(fanout))
            full_ptr = np.zeros(n + 1, dtype=np.int64)
            np.cumsum(kept, out=full_ptr[1:])
            hit = dg._cache[key] = (full_ptr, torch.from_numpy(full_ptr).to(dev))
        full_ptr, oo = hit
        n_sel, e_sel, e_out = n, int(ip_h[-1]), int(full_ptr[-1])
        nodes_dev, lo, local_off = None, dg.indptr, ip_h
    else:
        nodes = np.asarray(nodes, dtype=np.int64)
        degs = np.diff(ip_h)[nodes]
        nodes_dev = torch.from_numpy(nodes).to(dev)
        kept = np.minimum(degs, int(fanout))
        local_off = np.zeros(len(degs) + 1, dtype=np.int64)
        np.cumsum(degs, out=local_off[1:])
        out_off = np.zeros(len(degs) + 1, dtype=np.int64)
        np.cumsum(kept, out=out_off[1:])
        n_sel, e_sel, e_out = len(degs), int(local_off[-1]), int(out_off[-1])
        full_ptr = np.zeros(n + 1, dtype=np.int64)
        full_ptr[nodes + 1] = kept
        np.cumsum(full_ptr, out=full_ptr)
        lo = None if select else torch.from_numpy(local_off).to(dev)
        oo = torch.from_numpy(out_off).to(dev)
    out_idx = torch.empty(max(e_out, 1), dtype=torch.int32, device=dev)[:e_out]
    if e_out:
        dg.wait_rows()
        wsb = 0 if select else _lib.query("glint_sample_workspace_bytes", n_sel, e_sel, e_out)
        ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device=dev) if wsb else None
        _lib.call("glint_sample_neighbors", ptr(dg.indptr), ptr(dg.indices), ptr(nodes_dev),
                  n_sel, ptr(lo), e_sel, ptr(oo), e_out, int(fanout), int(seed), int(layer),
                  ptr(out_idx), ptr(ws), wsb, stream_handle())
    dev_ptr = oo if nodes is None else torch.from_numpy(full_ptr).to(dev)
    return DeviceGraph(n, e_out, dev_ptr, out_idx, full_ptr)


# -------------------------------------------------------------- batch CSC --


@dataclass(frozen=True)
class BatchCsc:
    """Local adjacency of one batch (glint/kernels.py:28-53), arrays on device.

    ``local32`` is the int32 copy of ``local_srcs`` the kernels consume.
    """

    targets: object
    input_ids: object
    indptr: object
    local_srcs: object
    target_pos: object
    local32: object = None

    @property
    def num_targets(self) -> int:
        return int(self.targets.shape[0])

    @property
    def num_inputs(self) -> int:
        return int(self.input_ids.shape[0])

    @property
    def num_edges(self) -> int:
        return int(self.local_srcs.shape[0])


def gather_slices(graph, targets):
    """(srcs, local indptr) of the targets' in-neighbour slices (glint/kernels.py:56-68)."""
    host = _is_host(targets)
    g = device_graph(graph)
    t = _i64(targets)
    indptr = degree_prefix_dev(g, t)
    total = int(indptr[-1].item())
    torch = _torch()
    srcs = torch.empty(total, dtype=torch.int64, device=g.indptr.device)
    if total:
        _lib.call("glint_gather_slices", ptr(g.indptr), ptr(g.indices), ptr(t), 0, t.shape[0],
                  ptr(indptr), ptr(srcs), None, None, g.num_nodes, None, None, stream_handle())
    return _ret(srcs, host), _ret(indptr, host)


def build_batch_csc(graph, targets) -> BatchCsc:
    """input_ids = unique(targets u srcs); local positions by rank (glint/kernels.py:71-77)."""
    torch = _torch()
    g = device_graph(graph)
    t = _i64(targets)
    nt = t.shape[0]
    ids = IdSet(g.num_nodes, g.indptr.device)
    if nt:
        ids.add_ids(t).add_neighbors(g, t)
    ids.finalize()
    indptr = degree_prefix_dev(g, t)
    counts = torch.stack([ids.count_dev[0], indptr[-1]]).cpu()
    n_in, n_e = int(counts[0]), int(counts[1])
    input_ids = ids.extract(n_in) if nt else t.clone()
    local64 = torch.empty(n_e, dtype=torch.int64, device=t.device)
    local32 = torch.empty(n_e, dtype=torch.int32, device=t.device)
    if n_e:
        _lib.call("glint_gather_slices", ptr(g.indptr), ptr(g.indices), ptr(t), 0, nt,
                  ptr(indptr), None, None, ptr(ids.ws), g.num_nodes, ptr(local64), ptr(local32),
                  stream_handle())
    target_pos = ids.lookup(t)[0] if nt else t.clone()
    return BatchCsc(t, input_ids, indptr, local64, target_pos, local32)


def trivial_batch_csc(targets) -> BatchCsc:
    """Conv-less block batch: inputs are exactly the (stably sorted) targets."""
    torch = _torch()
    t = _i64(targets)
    order = torch.sort(t, stable=True).indices
    input_ids = t[order]
    target_pos = torch.searchsorted(input_ids, t)
    empty = torch.zeros(0, dtype=torch.int64, device=t.device)
    return BatchCsc(t, input_ids, torch.zeros(t.shape[0] + 1, dtype=torch.int64, device=t.device),
                    empty, target_pos, torch.zeros(0, dtype=torch.int32, device=t.device))


# ------------------------------------------------------------- aggregation --


def spmm_mean(out, h, indptr, indices, n_rows, row_ids=None, row_base=0, self_rows=None,
              col_map=None, schedule=None, n_hub=0, bias=None, act=0):
    """Raw K1 launch on device tensors (see glint_spmm_mean_f32)."""
    dim = int(out.shape[1])
    _lib.call("glint_spmm_mean_f32", int(n_rows), dim, ptr(indptr), ptr(indices), ptr(row_ids),
              int(row_base), ptr(self_rows), ptr(col_map), ptr(h), ld(h), ptr(out), ld(out),
              ptr(schedule), int(n_hub), ptr(bias), int(act), stream_handle())
    if int(n_hub) > 0:              # the hub-row kernel beside the regular rows
        _lib.LAUNCHES[0] += 1
    return out


# L2 steering of K1's widest gathers: the source ids of the most-read rows
# (highest out-degree, as many as fit GLINT_K1_HOT_MB of L2) carry bit 31 in a
# per-graph annotated copy of `indices`, and K1 loads them evict_last and the
# rest evict_first (GLINT_TUNE_L2_HINT = 1).  Only rows of >= HOT_MIN_ROW_BYTES:
# profiles/r02_l2_hint_probe.jsonl measured up to 3.6% at d=256 and nothing at
# d=48 / d=100.  0 disables.
HOT_MB = int(os.environ.get("GLINT_K1_HOT_MB", "80"))
HOT_MIN_ROW_BYTES = 1024


def hot_indices(dg, row_bytes, reserve=0):
    """The DeviceGraph's indices with bit 31 set on ids of its hottest source
    rows (cached per graph and row count), or None when steering is off.
    `reserve` bytes of the HOT_MB budget are already held by other evict_last
    data (K4's score table)."""
    torch = _torch()
    budget = (HOT_MB << 20) - int(reserve)
    if HOT_MB <= 0 or budget <= 0 or row_bytes < HOT_MIN_ROW_BYTES or dg.num_edges == 0:
        return None
    rows = min(int(dg.num_nodes), budget // int(row_bytes))
    key = ("hot_indices", rows)
    hit = dg._cache.get(key)
    if hit is None:
        # built on the graph's second request: the annotation pass (~1 ms on
        # the Products graph) outweighs its gain for a graph used once (an e2e
        # call uploads a fresh DeviceGraph each time)
        seen = dg._cache.get(("hot_requests", rows), 0)
        dg._cache[("hot_requests", rows)] = seen + 1
        if seen < 1:
            return None
        # the copy is outside the batch budget: only with ample free HBM
        free, _total = torch.cuda.mem_get_info(dg.indices.device)
        if free < 4 * dg.indices.numel() * dg.indices.element_size():
            return None
        idx = dg.indices
        cnt = torch.bincount(idx.long(), minlength=int(dg.num_nodes))
        hot = torch.zeros(int(dg.num_nodes), dtype=torch.bool, device=idx.device)
        hot[torch.topk(cnt, rows).indices] = True
        flag = torch.tensor(-2 ** 31, dtype=torch.int32, device=idx.device)
        hit = dg._cache[key] = torch.where(hot[idx.long()], idx | flag, idx)
    return hit


def spmm_mean_hot(out, h, dg, n_rows, **kw):
    """K1 with the hot-row L2 policy when it applies (same bytes as spmm_mean)."""
    ann = hot_indices(dg, ld(h) * 4) if kw.get("col_map") is None else None
    if ann is None:
        return spmm_mean(out, h, dg.indptr, dg.indices, n_rows, **kw)
    _lib.call("glint_set_tuning", 11, 1)
    try:
        return spmm_mean(out, h, dg.indptr, ann, n_rows, **kw)
    finally:
        _lib.call("glint_set_tuning", 11, 0)


_SMS = {}


def fused_ctas_beside_planning() -> int:
    """K7 grid while the batch planner's counting kernels run beside it: all SMs
    but GLINT_FUSED_RESERVE_SMS (default 8).  K7 holds a whole SM per CTA, so
    without a reserve the planner's kernels wait for it to finish."""
    torch = _torch()
    dev = torch.cuda.current_device()
    if dev not in _SMS:
        _SMS[dev] = torch.cuda.get_device_properties(dev).multi_processor_count
    reserve = int(os.environ.get("GLINT_FUSED_RESERVE_SMS", "8"))
    return max(1, _SMS[dev] - reserve) if reserve > 0 else 0


def conv_mean_supported(h, d_out, precision=None) -> bool:
    """Whether K7 (the fused aggregate->transform) takes this ConvMean: 3xTF32,
    d_in <= 128 on a 16-byte row pitch, d_out <= 256."""
    prec = PRECISION if precision is None else precision
    d_in = int(h.shape[1])
    return (prec == _lib.PREC_3XTF32 and FUSE_CONV and bool(_lib.query(
        "glint_conv_mean_supported", d_in, int(d_out))) and ld(h) % 4 == 0
        and ptr(h) % 16 == 0)


def conv_mean(out, h, weight, bias, act, indptr, indices, n_rows, row_ids=None, row_base=0,
              self_rows=None, col_map=None, schedule=None, max_ctas=0):
    """K7 launch: out = act(mean(h) W^T + b) in one kernel (glint_conv_mean_f32),
    the composition of spmm_mean and linear_into without the B x d_in aggregate
    in HBM (model_ir.py:336-338)."""
    torch = _torch()
    d_in, d_out = int(h.shape[1]), int(out.shape[1])
    nbytes = int(_lib.query("glint_conv_mean_workspace_bytes", d_in, d_out))
    ws = torch.empty(nbytes, dtype=torch.uint8, device=out.device)
    _lib.call("glint_conv_mean_f32", int(n_rows), d_in, d_out, ptr(indptr), ptr(indices),
              ptr(row_ids), int(row_base), ptr(self_rows), ptr(col_map), ptr(h), ld(h),
              ptr(weight), ld(weight), ptr(bias), int(act), ptr(out), ld(out), ptr(schedule),
              int(max_ctas), ptr(ws), nbytes, stream_handle())
    return out


def _local_schedule(indptr, n_rows):
    """LPT schedule + hub count for a local (batch) CSC; syncs for the count."""
    sched, n_hub = degree_schedule(indptr, None, 0, n_rows)
    return sched, int(n_hub.item())


def agg_mean(bc: BatchCsc, h_in):
    """Mean over in-neighbours plus self, byte-identical to glint/kernels.py:122-135."""
    host = _is_host(h_in)
    h = _f32(h_in)
    if h.dim() != 2 or h.shape[0] != bc.num_inputs:
        raise ValueError(f"h_in has {h.shape[0] if h.dim() else 0} rows, expected {bc.num_inputs}")
    torch = _torch()
    out = torch.empty((bc.num_targets, h.shape[1]), dtype=torch.float32, device=h.device)
    if bc.num_targets:
        local32 = bc.local32 if bc.local32 is not None else bc.local_srcs.to(torch.int32)
        sched, n_hub = _local_schedule(bc.indptr, bc.num_targets)
        spmm_mean(out, h, bc.indptr, local32, bc.num_targets, self_rows=bc.target_pos,
                  schedule=sched, n_hub=n_hub)
    return _ret(out, host)


def leaky_relu(x, slope=LEAKY_SLOPE):
    if float(slope) != float(LEAKY_SLOPE):
        raise ValueError("only the reference slope 0.2 is supported on device")
    return elementwise("LeakyReLU", [x])


@dataclass(frozen=True)
class AttnParams:
    """weight (heads, head_dim, in_dim); attn (heads, 2*head_dim): [src | dst]."""

    weight: object
    attn: object

    @property
    def num_heads(self) -> int:
        return int(self.weight.shape[0])

    @property
    def head_dim(self) -> int:
        return int(self.weight.shape[1])

    def validate(self):
        if len(self.weight.shape) != 3:
            raise ValueError(f"attention weight must be rank 3, got {tuple(self.weight.shape)}")
        if tuple(self.attn.shape) != (self.num_heads, 2 * self.head_dim):
            raise ValueError(f"attention vector shape {tuple(self.attn.shape)} != "
                             f"({self.num_heads}, {2 * self.head_dim})")


def head_pitch(head_dim) -> int:
    return (int(head_dim) + 3) // 4 * 4


def padded_head_weight(weight, device=None):
    """(H, dh, K) -> (H * pitch, K) device matrix with zero pad rows per head."""
    torch = _torch()
    w = _f32(weight)
    H, dh, K = (int(s) for s in w.shape)
    hp = head_pitch(dh)
    out = torch.zeros((H, hp, K), dtype=torch.float32, device=w.device)
    out[:, :dh, :] = w
    return out.reshape(H * hp, K)


def attn_project(h, w_pad, attn, heads, head_dim, precision=None, out=None):
    """Z = h W_pad^T (head-padded) and the per-head scores s_src / s_dst
    (into `out` = (Z, s_src, s_dst) row views when given)."""
    torch = _torch()
    hp = head_pitch(head_dim)
    M = h.shape[0]
    if out is not None:
        Z, s_src, s_dst = out
    else:
        Z = torch.empty((M, heads * hp), dtype=torch.float32, device=h.device)
        s_src = torch.empty((M, heads), dtype=torch.float32, device=h.device)
        s_dst = torch.empty((M, heads), dtype=torch.float32, device=h.device)
    a = _f32(attn).contiguous()
    prec = PRECISION if precision is None else precision
    _lib.call("glint_gat_project_f32", M, heads, head_dim, hp, int(w_pad.shape[1]), ptr(h), ld(h),
              None, ptr(w_pad), ld(w_pad), ptr(a), ptr(Z), ld(Z), ptr(s_src), ptr(s_dst),
              int(prec), stream_handle())
    return Z, s_src, s_dst


GAT_TWO_PHASE = True    # honoured when a caller passes edge_range (measured slower: profiles/r01_gat_sweep_two_phase.jsonl)


def gat_aggregate(out, Z, s_src, s_dst, heads, head_dim, indptr, indices, n_rows, row_ids=None,
                  row_base=0, self_rows=None, col_map=None, schedule=None, n_hub=0,
                  act=0, edge_range=None):
    """K4.  edge_range=(base, span) covering every row's edges of indptr selects
    the two-phase path (glint_gat_aggregate_ws_f32, same bytes)."""
    if edge_range is not None and GAT_TWO_PHASE and int(n_rows) > 0:
        base, span = (int(v) for v in edge_range)
        torch = _torch()
        wsb = _lib.query("glint_gat_aggregate_workspace_bytes", int(n_rows), span, heads)
        ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device=Z.device)
        _lib.call("glint_gat_aggregate_ws_f32", int(n_rows), heads, head_dim,
                  head_pitch(head_dim), ptr(indptr), ptr(indices), ptr(row_ids), int(row_base),
                  ptr(self_rows), ptr(col_map), ptr(Z), ld(Z), ptr(s_src), ptr(s_dst),
                  float(LEAKY_SLOPE), ptr(out), ld(out), ptr(schedule), int(n_hub), int(act),
                  base, span, ptr(ws), wsb, stream_handle())
        return out
    if int(n_hub) > 0:              # the hub-row kernel beside the regular rows
        _lib.LAUNCHES[0] += 1
    _lib.call("glint_gat_aggregate_f32", int(n_rows), heads, head_dim, head_pitch(head_dim),
              ptr(indptr), ptr(indices), ptr(row_ids), int(row_base), ptr(self_rows),
              ptr(col_map), ptr(Z), ld(Z), ptr(s_src), ptr(s_dst), float(LEAKY_SLOPE), ptr(out),
              ld(out), ptr(schedule), int(n_hub), int(act), stream_handle())
    return out


def agg_attn(bc: BatchCsc, h_in, params: AttnParams):
    """Multi-head additive attention over N(v) u {v} (glint/kernels.py:170-203)."""
    params.validate()
    host = _is_host(h_in)
    h = _f32(h_in)
    if h.dim() != 2 or h.shape[0] != bc.num_inputs:
        raise ValueError(f"h_in has {h.shape[0] if h.dim() else 0} rows, expected {bc.num_inputs}")
    torch = _torch()
    H, dh = params.num_heads, params.head_dim
    if int(params.weight.shape[2]) != h.shape[1]:
        raise ValueError(f"linear shape mismatch: x {tuple(h.shape)} vs weight "
                         f"{tuple(params.weight.shape[1:])}")
    Z, s_src, s_dst = attn_project(h, padded_head_weight(params.weight), params.attn, H, dh)
    out = torch.empty((bc.num_targets, H * dh), dtype=torch.float32, device=h.device)
    if bc.num_targets:
        local32 = bc.local32 if bc.local32 is not None else bc.local_srcs.to(torch.int32)
        sched, n_hub = _local_schedule(bc.indptr, bc.num_targets)
        gat_aggregate(out, Z, s_src, s_dst, H, dh, bc.indptr, local32, bc.num_targets,
                      self_rows=bc.target_pos, schedule=sched, n_hub=n_hub)
    return _ret(out, host)


# ------------------------------------------------------------- dense + rows --


def linear_into(C, x, w, bias, act, a_rows=None, precision=None):
    prec = PRECISION if precision is None else precision
    M = int(a_rows.shape[0]) if a_rows is not None else int(x.shape[0])
    _lib.call("glint_linear_f32", M, int(w.shape[0]), int(w.shape[1]), ptr(x), ld(x),
              ptr(a_rows), ptr(w), ld(w), ptr(bias), int(act), ptr(C), ld(C), int(prec),
              stream_handle())
    return C


def linear(x, weight, bias=None):
    """out[i] = weight @ x[i] (+ bias) (glint/kernels.py:95-107)."""
    host = _is_host(x)     # the container kind follows the data, not the parameters
    xd, wd = _f32(x), _f32(weight)
    if xd.dim() != 2 or wd.dim() != 2 or xd.shape[1] != wd.shape[1]:
        raise ValueError(f"linear shape mismatch: x {tuple(xd.shape)} vs weight {tuple(wd.shape)}")
    bd = None
    if bias is not None:
        bd = _f32(bias).contiguous()
        if tuple(bd.shape) != (wd.shape[0],):
            raise ValueError(f"bias shape {tuple(bd.shape)} != ({wd.shape[0]},)")
    torch = _torch()
    out = torch.empty((xd.shape[0], wd.shape[0]), dtype=torch.float32, device=xd.device)
    if xd.shape[0]:
        linear_into(out, xd, wd.contiguous(), bd, _lib.ACT_NONE)
    return _ret(out, host)


def elementwise_into(out, kind, mats, rows=None):
    import ctypes

    n = len(mats)
    ptrs = (ctypes.c_void_p * n)(*[m.data_ptr() for m in mats])
    lds = (ctypes.c_int64 * n)(*[ld(m) for m in mats])
    rws = (ctypes.c_void_p * n)(*[(r.data_ptr() if r is not None else None)
                                  for r in (rows or [None] * n)])
    _lib.call("glint_elementwise_f32", _lib.EW_KINDS[kind], int(out.shape[0]), int(out.shape[1]),
              n, ptrs, lds, rws, ptr(out), ld(out), stream_handle())
    return out


def elementwise(kind, inputs):
    """ReLU / LeakyReLU / Add / Norm / DropoutIdentity (glint/kernels.py:206-231)."""
    if kind not in _lib.EW_KINDS:
        raise ValueError(f"unknown elementwise kind {kind!r}")
    host = _is_host(*inputs)
    mats = [_f32(m) for m in inputs]
    if kind == "Add":
        if len(mats) < 2:
            raise ValueError("Add needs at least two operands")
        for m in mats[1:]:
            if tuple(m.shape) != tuple(mats[0].shape):
                raise ValueError(f"Add shape mismatch: {tuple(mats[0].shape)} vs {tuple(m.shape)}")
    elif len(mats) != 1:
        raise ValueError(f"{kind} takes exactly one operand")
    torch = _torch()
    out = torch.empty(tuple(mats[0].shape), dtype=torch.float32, device=mats[0].device)
    if out.numel():
        # Add over more than 8 operands chains launches: ((a+b)+...)+z keeps the order.
        acc = mats[0]
        rest = mats[1:]
        first = True
        while first or rest:
            take = rest[:7] if kind == "Add" else []
            rest = rest[7:] if kind == "Add" else []
            elementwise_into(out, kind, [acc] + take)
            acc, first = out, False
    return _ret(out, host)


def copy_rows(dst, src, src_rows=None, dst_rows=None, n_rows=None):
    if n_rows is None:
        n_rows = (src_rows.shape[0] if src_rows is not None else
                  dst_rows.shape[0] if dst_rows is not None else src.shape[0])
    _lib.call("glint_copy_rows_f32", int(n_rows), int(src.shape[1]), ptr(src), ld(src),
              ptr(src_rows), ptr(dst), ld(dst), ptr(dst_rows), stream_handle())
    return dst


def concat(parts):
    """Column concatenation (glint/kernels.py:234-239)."""
    host = _is_host(*parts)
    mats = [_f32(p) for p in parts]
    rows = {int(m.shape[0]) for m in mats}
    if len(rows) > 1:
        raise ValueError(f"concat row mismatch: {sorted(rows)}")
    torch = _torch()
    width = sum(int(m.shape[1]) for m in mats)
    out = torch.empty((mats[0].shape[0], width), dtype=torch.float32, device=mats[0].device)
    col = 0
    for m in mats:
        if m.shape[1] and m.shape[0]:
            copy_rows(out[:, col:col + m.shape[1]], m)
        col += int(m.shape[1])
    return _ret(out, host)
