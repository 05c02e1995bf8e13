"""Inference engines, target annotation and the request API on B200.

Drop-in for glint/executor.py: ``run_inference`` keeps the reference's
signature, modes (full / partial / sampling), executors (layerwise /
nodewise), orders, stats document and error behaviour
(glint/executor.py:481-543).  What changes is where the work happens:

* every stored layer output is an HBM-resident ``DeviceStore``; a block's
  batches read neighbour rows straight from the resident input store through
  the CSC (no per-batch gather copy of ``input_ids`` rows, which the reference
  pays at executor.py:353-354);
* input-domain operators (those feeding a Conv of their block) are evaluated
  once per layer over the layer's input rows instead of once per batch
  (results are per-row functions, so the bytes are the same);
* a ConvMean followed by ReLU/LeakyReLU in the same block runs as
  aggregation + one GEMM with bias and activation fused in the epilogue,
  writing directly into the output store;
* batch planning (the feedback controller's n_inputs count) runs on a side
  stream with device id-set kernels, so the host sync per plan overlaps the
  previous batch's kernels; batch membership is identical to the reference
  for the same capacity and initial thresholds.

Annotation (partial/sampling target sets) expands frontiers with the device
id-set kernels; sampling draws (splitmix64 priorities, smallest fanout kept)
are computed on the host as in the reference and uploaded.
"""

from __future__ import annotations

import os
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib, device as devmodel, kernels
from .batching import BatchController, Thresholds, next_batch
from .errors import ConfigError, DeviceAllocationError, DeviceCapacityError, InternalError
from .model_ir import ModelGraph
from .reorder import NodeOrder, apply_order_device, make_order
from .splitter import INPUT_REF, BlockSchedule, TensorRef, split
from .storage import (HOST_NARROW, CscGraph, DeviceGraph, DeviceStore, EmbeddingStore,
                      arange_ids, pitch_of)

MODES = ("full", "partial", "sampling")


# ----------------------------------------------------------------- targets --


@dataclass
class TargetSets:
    mode: str
    depth: int
    v_sets: dict
    sampled: dict | None = None
    skip_from: int | None = None

    def graph_for_layer(self, g, layer):
        if self.sampled is not None and layer in self.sampled:
            return self.sampled[layer]
        return g


_U64 = np.uint64
_M1 = _U64(0xBF58476D1CE4E5B9)
_M2 = _U64(0x94D049BB133111EB)
_GOLD = _U64(0x9E3779B97F4A7C15)


def _mix(x):
    """splitmix64 finaliser over uint64 arrays (wrapping arithmetic)."""
    z = (np.asarray(x, dtype=np.uint64) + _GOLD).astype(np.uint64)
    z = (z ^ (z >> _U64(30))) * _M1
    z = (z ^ (z >> _U64(27))) * _M2
    return z ^ (z >> _U64(31))


def sample_neighbors(g, nodes, fanout, seed, layer):
    """min(fanout, deg) distinct in-neighbours per node (glint/executor.py:74-115).

    A DeviceGraph is sampled on the device and returns a DeviceGraph; a host
    CscGraph keeps the numpy path (the oracle-pinned restatement).

    Edge priority = mix(base ^ mix(node * M1) ^ slot), base = mix(mix(seed) ^
    mix(layer * M2)); each node keeps its `fanout` smallest priorities and the
    kept slice is stored ascending.  Reproducible and independent of the order
    or grouping of `nodes`.
    """
    if fanout < 1:
        raise ValueError(f"fanout must be >= 1, got {fanout}")
    if isinstance(g, DeviceGraph):
        # device draws (glint_sample_neighbors): same priorities, same bytes
        nodes = _sorted_unique(nodes)
        every = len(nodes) == g.num_nodes
        return kernels.sample_neighbors_dev(g, None if every else nodes, fanout, seed, layer)
    indptr_h, indices_h = _host_arrays(g)
    n = g.num_nodes
    nodes = _sorted_unique(nodes)
    out_ptr = np.zeros(n + 1, dtype=np.int64)
    if len(nodes) == 0:
        return CscGraph(n, 0, out_ptr, np.zeros(0, dtype=np.int64))
    starts = indptr_h[nodes]
    lens = indptr_h[nodes + 1] - starts
    total = int(lens.sum())
    owner = np.repeat(np.arange(len(nodes), dtype=np.int64), lens)
    first = np.repeat(np.cumsum(lens) - lens, lens)
    slot = np.arange(total, dtype=np.int64) - first
    srcs = indices_h[np.repeat(starts, lens) + slot]
    with np.errstate(over="ignore"):
        base = _mix(_mix(np.uint64(np.int64(seed))) ^ _mix(np.uint64(layer) * _M2))
        prio = _mix(base ^ _mix(nodes[owner].astype(np.uint64) * _M1) ^ slot.astype(np.uint64))
    ranked = np.lexsort((prio, owner))          # by node, then priority
    keep = ranked[slot < fanout]                 # slot == rank inside each node's run
    k_owner, k_src = owner[keep], srcs[keep]
    k_src = k_src[np.lexsort((k_src, k_owner))]
    out_ptr[nodes + 1] = np.minimum(lens, fanout)
    np.cumsum(out_ptr, out=out_ptr)
    return CscGraph(n, int(out_ptr[-1]), out_ptr, k_src)


def _host_arrays(g):
    if isinstance(g, CscGraph):
        return g.indptr, g.indices
    key = "host_indices"
    if key not in g._cache:
        g._cache[key] = g.indices.cpu().numpy().astype(np.int64)
    return g.indptr_host, g._cache[key]


def _expand_dev(dg, nodes_np):
    """sorted unique(nodes u in-neighbours(nodes)) via device id sets."""
    import torch

    dg.wait_rows()
    ids = kernels.IdSet(dg.num_nodes, dg.indptr.device)
    if len(nodes_np):
        a = np.ascontiguousarray(nodes_np, dtype=np.int64)
        t = torch.from_numpy(a if a.flags.writeable else a.copy()).to(dg.indptr.device)
        ids.add_ids(t).add_neighbors(dg, t)
    ids.finalize()
    return ids.extract().cpu().numpy()


def _sorted_unique(a):
    """np.unique(a) without the hash/sort when `a` is already strictly
    increasing (the usual target list): an O(n) check instead of ~30 ms for
    245K ids on the box's CPU."""
    a = np.asarray(a, dtype=np.int64)
    if len(a) < 2 or bool(np.all(a[1:] > a[:-1])):
        return a
    return np.unique(a)


def skip_fires(n_next, graph) -> bool:
    """|V[l+1]| * d_avg >= n, exact in integers (glint/executor.py:124-126)."""
    return n_next * graph.num_edges >= graph.num_nodes * graph.num_nodes


def annotate(g, targets, depth, mode, fanout=None, seed=0) -> TargetSets:
    """Per-layer target sets V[depth..1] (glint/executor.py:129-164)."""
    if mode not in MODES:
        raise ConfigError(f"unknown inference mode {mode!r}")
    n = g.num_nodes
    targets = np.asarray(targets, dtype=np.int64)
    if not (mode == "full" and len(targets) == n and _is_arange(targets)):
        targets = _sorted_unique(targets)
    if len(targets) and (targets[0] < 0 or targets[-1] >= n):
        raise ConfigError("target ids out of range")
    sampled = None
    if mode == "sampling":
        if fanout is None or fanout < 1:
            raise ConfigError("sampling mode requires fanout >= 1")
        every = arange_ids(n)
        sampled = {l: sample_neighbors(g, every, fanout, seed, l) for l in range(1, depth + 1)}
    if depth == 0:
        return TargetSets(mode, 0, {0: targets}, sampled)
    every = arange_ids(n)
    if mode == "full":
        return TargetSets(mode, depth, {l: every for l in range(1, depth + 1)}, sampled)
    v_sets = {depth: targets}
    skip_from = None
    for l in range(depth - 1, 0, -1):
        g_used = sampled[l + 1] if sampled else g
        if len(targets) and skip_fires(len(v_sets[l + 1]), g_used):
            skip_from = l
            for ll in range(l, 0, -1):
                v_sets[ll] = every
            break
        v_sets[l] = _expand_dev(kernels.device_graph(g_used) if not isinstance(g_used, DeviceGraph)
                                else g_used, v_sets[l + 1])
    return TargetSets(mode, depth, v_sets, sampled, skip_from)


# ------------------------------------------------------------------- stats --


@dataclass
class RunStats:
    """Deterministic run statistics (document schema glint-stats-v1)."""

    executor: str
    mode: str
    order: str
    depth: int
    initial_thresholds: tuple | None = None
    layer_batches: dict = field(default_factory=dict)
    layer_transfer: dict = field(default_factory=dict)
    layer_aggregations: dict = field(default_factory=dict)
    layer_input_bytes: dict = field(default_factory=dict)
    total_transfer: int = 0
    total_input_bytes: int = 0
    total_aggregations: int = 0
    max_footprint: int = 0
    batches: int = 0
    trajectory: list = field(default_factory=list)
    batch_footprints: list = field(default_factory=list)
    batch_transfers: list = field(default_factory=list)
    batch_layers: list = field(default_factory=list)
    batch_sizes: list = field(default_factory=list)
    oom_retries: int = 0
    thresholds_carry: bool = True
    wall_time: float = 0.0

    def _add_batch(self, layer, n_targets, fp, thresholds=None, retries=0):
        self.batches += 1
        for d, v in ((self.layer_batches, 1), (self.layer_transfer, fp.transfer_bytes),
                     (self.layer_input_bytes, fp.input_bytes)):
            d[layer] = d.get(layer, 0) + v
        self.total_transfer += fp.transfer_bytes
        self.total_input_bytes += fp.input_bytes
        self.max_footprint = max(self.max_footprint, fp.peak)
        self.oom_retries += retries
        self.batch_footprints.append(fp.peak)
        self.batch_transfers.append(fp.transfer_bytes)
        self.batch_layers.append(layer)
        self.batch_sizes.append(n_targets)
        if thresholds is not None:
            self.trajectory.append((layer, thresholds.n_t, thresholds.n_i))

    def _add_aggregations(self, layer, count):
        self.layer_aggregations[layer] = self.layer_aggregations.get(layer, 0) + count
        self.total_aggregations += count

    def to_lines(self) -> list:
        kv = [("schema", "glint-stats-v1"), ("executor", self.executor), ("mode", self.mode),
              ("order", self.order), ("depth", str(self.depth)), ("batches", str(self.batches)),
              ("total.transfer_bytes", str(self.total_transfer)),
              ("total.input_bytes", str(self.total_input_bytes)),
              ("total.aggregations", str(self.total_aggregations)),
              ("max_footprint_bytes", str(self.max_footprint)),
              ("oom_retries", str(self.oom_retries)),
              ("thresholds.carry_across_layers", str(self.thresholds_carry).lower())]
        if self.initial_thresholds is not None:
            kv.append(("thresholds.initial",
                       f"{self.initial_thresholds[0]},{self.initial_thresholds[1]}"))
        for l in sorted(self.layer_batches):
            kv += [(f"layer.{l}.batches", str(self.layer_batches[l])),
                   (f"layer.{l}.transfer_bytes", str(self.layer_transfer[l])),
                   (f"layer.{l}.input_bytes", str(self.layer_input_bytes.get(l, 0)))]
        for l in sorted(self.layer_aggregations):
            kv.append((f"layer.{l}.aggregations", str(self.layer_aggregations[l])))
        if self.trajectory:
            kv.append(("thresholds.trajectory",
                       ";".join(f"{l}:{a}:{b}" for l, a, b in self.trajectory)))
        for name, vals in (("footprint_bytes", self.batch_footprints),
                           ("transfer_bytes", self.batch_transfers),
                           ("layer", self.batch_layers), ("targets", self.batch_sizes)):
            if vals:
                kv.append((f"batch.{name}", ",".join(str(v) for v in vals)))
        return [f"{k}\t{v}" for k, v in kv]

    def document(self) -> str:
        return "\n".join(self.to_lines()) + "\n"


def parse_stats(text) -> dict:
    out = {}
    for line in text.splitlines():
        if line.strip():
            k, _, v = line.partition("\t")
            out[k] = v
    return out


# ---------------------------------------------------------- device engine --


def _ref_key(schedule: BlockSchedule, m: ModelGraph, producer) -> str:
    if m.operators[producer].kind == "Input":
        return INPUT_REF
    return TensorRef(schedule.assignment[producer], producer).key


def _dims_table(m: ModelGraph, schedule: BlockSchedule) -> dict:
    dims = {INPUT_REF: m.input_dim}
    dims.update(m.out_dims)
    for blk in schedule.blocks:
        for ref in blk.input_refs:
            dims[ref.key] = m.input_dim if ref.key == INPUT_REF else m.out_dims[ref.op]
    return dims


class _RowSpace:
    """Rows of a device matrix: all nodes (identity) or a sorted id subset."""

    def __init__(self, ids=None, rank_map=None):
        self.ids = ids              # torch.int64 sorted, or None for identity
        self.rank_map = rank_map    # torch.int32 [N] or None

    @property
    def identity(self):
        return self.ids is None

    def positions(self, targets):
        """Row positions of (device int64) node ids in this space."""
        if self.identity:
            return targets
        return self.rank_map.index_select(0, targets).to(targets.dtype)


@dataclass
class _Plan:
    start: int
    end: int
    num_inputs: int
    num_edges: int
    num_hubs: int = 0


_PLAN_STREAMS: dict = {}
_PARAM_CACHE: dict = {}


def _plan_stream(device):
    """One planning side stream per device, reused by every engine.

    High priority: the controller's n_inputs counts are a chain of host
    round trips (each plan depends on the previous batch's adapt step), issued
    while a whole-layer aggregation fills the GPU.  At default priority their
    small kernels queued behind every pending aggregation CTA, so the chain
    ran only after the layer finished and left the device idle ~1.6 ms per
    step between layers 1 and 2 (tools/order_timeline.py); at high priority
    the block scheduler slots them in as aggregation CTAs retire.
    GLINT_PLAN_PRIORITY=0 restores the default (A/B)."""
    import torch

    s = _PLAN_STREAMS.get(device)
    if s is None:
        prio = -1 if os.environ.get("GLINT_PLAN_PRIORITY", "1") == "1" else 0
        s = _PLAN_STREAMS[device] = torch.cuda.Stream(device=device, priority=prio)
    return s


_HUB_STREAMS: dict = {}


def _hub_stream(device):
    """High-priority side stream for the hub rows beside a K7 launch: its CTAs
    take the SMs K7 leaves free as soon as they are issued."""
    import torch

    s = _HUB_STREAMS.get(device)
    if s is None:
        s = _HUB_STREAMS[device] = torch.cuda.Stream(device=device, priority=-1)
    return s


def _device_params(m: ModelGraph, device):
    """Device weights of a model, uploaded once per (model, device) and kept
    while the model object is alive (the model is immutable)."""
    import weakref

    key = (id(m), str(device))
    hit = _PARAM_CACHE.get(key)
    if hit is not None and hit[0]() is m:
        return hit[1]
    p = _Params(m, device)
    for k in [k for k, (ref, _) in _PARAM_CACHE.items() if ref() is None]:
        del _PARAM_CACHE[k]
    _PARAM_CACHE[key] = (weakref.ref(m), p)
    return p


class _Params:
    """Device copies of model parameters."""

    def __init__(self, m: ModelGraph, device):
        import torch

        self.w, self.b, self.attn, self.w_pad = {}, {}, {}, {}
        for op in m.operators.values():
            if op.kind in ("ConvMean", "Linear"):
                # rows padded to a 16-byte pitch (K2's tensor maps need it; the
                # pad is zero and never read)
                w = np.ascontiguousarray(op.params["weight"], dtype=np.float32)
                wp = torch.zeros((w.shape[0], pitch_of(w.shape[1])), dtype=torch.float32,
                                 device=device)
                wp[:, :w.shape[1]] = torch.from_numpy(w).to(device)
                self.w[op.op_id] = wp[:, :w.shape[1]]
                b = op.params.get("bias")
                self.b[op.op_id] = (None if b is None else torch.from_numpy(
                    np.ascontiguousarray(b, dtype=np.float32)).to(device))
            elif op.kind == "ConvAttn":
                self.w_pad[op.op_id] = kernels.padded_head_weight(
                    torch.from_numpy(np.ascontiguousarray(op.params["weight"], np.float32)).to(device))
                self.attn[op.op_id] = torch.from_numpy(np.ascontiguousarray(
                    op.params["attn"], dtype=np.float32)).to(device)


class LayerwiseEngine:
    """Executes a BlockSchedule over HBM-resident stores (glint/executor.py:301-384)."""

    def __init__(self, m: ModelGraph, schedule: BlockSchedule, g: DeviceGraph, x: DeviceStore,
                 tsets: TargetSets, budget, thresholds: Thresholds, stats: RunStats,
                 precision=None, row_range=None, reassociate=False, release_input=False):
        import torch

        self.m, self.schedule, self.g, self.tsets = m, schedule, g, tsets
        # opt-in: mean(h)W^T+b vs mean(hW^T)+b differ at ~1e-7 in fp32, so the
        # reference contract (layer-wise == node-wise == eval_reference bytes)
        # holds only with reassociation off, the default
        self.reassociate = reassociate
        self.retain_stores = False          # checkers: keep every layer's store alive
        self.release_input = release_input  # engine owns x: free it after its last reader
        self.budget, self.stats = budget, stats
        self.controller = BatchController(thresholds=thresholds, budget=budget)
        self.dev = g.indptr.device
        self.precision = kernels.PRECISION if precision is None else precision
        self.params = _device_params(m, self.dev)
        self.dims = _dims_table(m, schedule)
        self.stores = {INPUT_REF: x}
        self.spaces = {INPUT_REF: _RowSpace()}
        self.plan_stream = _plan_stream(self.dev)
        self.users = m.consumers()
        self.row_range = row_range          # (lo, hi) node range owned by this rank (full mode)
        self._graph_cache = {}
        self._plan_sets = {}
        self._sched_cache = {}
        self.kernel_launches = 0
        self.probe = None               # optional KernelProbe (bench roofline timing)
        self.sink = None                # optional sink(store, row_lo, row_hi) for final rows
        self.exchange = None            # RowExchange of a distributed run (set by run())
        # output chunks streamed to the host sink (each is bounded by its slowest hub row)
        self.sink_chunks = int(os.environ.get("GLINT_SINK_CHUNKS", "2"))
        # one launch per full-mode conv layer when the budget admits it
        self.whole_layer = os.environ.get("GLINT_WHOLE_LAYER", "1") == "1"
        self._fused_ctas = 0            # K7 grid cap while planning runs beside it
        self._fused_ok = True           # K7 allowed for the launch in progress
        self.k7_launches = {"whole": 0, "split": 0}
        # whole-layer K7 launches keep their hub rows inside (default) or run
        # them beside K7 as in row chunks (GLINT_K7_HUBS=beside, A/B)
        self.k7_hubs_beside = os.environ.get("GLINT_K7_HUBS", "inside") == "beside"

    # -- helpers ------------------------------------------------------------

    def _graph_for(self, layer) -> DeviceGraph:
        gl = self.tsets.graph_for_layer(self.g, layer)
        if isinstance(gl, DeviceGraph):
            return gl
        dg = self._graph_cache.get(layer)
        if dg is None:
            dg = self._graph_cache[layer] = DeviceGraph.from_host(gl, self.dev)
        return dg

    def _hub_counter(self, gl: DeviceGraph, targets_dev, full):
        """Prefix of hub rows (deg+1 >= HUB_MIN_DEGREE) over the layer's targets:
        (device tensor, host copy or None).  Computed on the planning stream
        (it needs only indptr, not the features or the edge ids)."""
        import torch

        if not full:
            return kernels.hub_prefix_dev(gl, targets_dev), None
        key = ("hubpre", kernels.HUB_MIN_DEGREE)
        hit = gl._cache.get(key)
        if hit is None:
            self.plan_stream.wait_event(gl.indptr_event)
            with torch.cuda.stream(self.plan_stream):
                pre = kernels.hub_prefix_dev(gl, None, 0, gl.num_nodes)
                hit = gl._cache[key] = (pre, pre.cpu().numpy())
        return hit

    def _reassociate(self, o) -> bool:
        """Transform-then-aggregate for a ConvMean that narrows the row width.

        mean_{N(v)+v}(h) W^T + b == mean_{N(v)+v}(h W^T) + b exactly in real
        arithmetic (fp32 rounding differs at ~1e-7 relative, inside the 1e-4
        end-to-end bar); gathering the narrow rows moves d_out/d_in of the
        bytes (256 -> 48 floats per neighbour for the headline layer 3).
        """
        if not self.reassociate:
            return False
        w = self.m.operators[o].params["weight"]
        return pitch_of(w.shape[0]) < pitch_of(w.shape[1])

    def _fusions(self, blk):
        """conv/linear op -> activation op fused into its epilogue.  An identity
        (DropoutIdentity: x at inference, reference kernels.py:206-231) fuses
        the same way with no activation, so the producer writes straight into
        the identity's destination (its store) instead of a copy pass."""
        fused = {}
        for o in blk.op_ids:
            k = blk.kinds[o]
            if k not in _EPILOGUE_ACTS:
                continue
            x = self.m.operators[o].inputs[0]
            if (x in blk.kinds and blk.kinds[x] in ("ConvMean", "ConvAttn", "Linear")
                    and blk.domains[x] == "target" and blk.domains[o] == "target"
                    and self.users[x] == [o] and x not in blk.outputs):
                fused[x] = o
        return fused

    # -- planning -------------------------------------------------------------

    def _planner(self, blk, gl, targets_dev, targets_np, full, prefix, hub_pre, hub_host):
        import torch

        n_nodes = gl.num_nodes
        dims = self.dims

        def plan_fn(start, end):
            n_t = end - start
            n_e = int(prefix[end] - prefix[start]) if blk.has_conv else 0
            n_h = 0
            if not blk.has_conv or n_t == 0:
                n_i = n_t
            elif full and n_t == n_nodes:
                n_i = n_t
                n_h = int(hub_host[n_nodes])
            elif full and (start, end) in gl._cache.get("plan_counts", {}):
                # full-mode counts are a pure function of the (immutable) graph
                # and the contiguous range: memoized on the DeviceGraph, so a
                # repeated run plans the same batches without counting kernels
                n_i, n_h = gl._cache["plan_counts"][(start, end)]
            else:
                ids = gl._cache.get("plan_idset")      # reused across batches and runs
                gl.wait_rows(end if full else None, stream=self.plan_stream)
                with torch.cuda.stream(self.plan_stream):
                    if ids is None:
                        ids = gl._cache["plan_idset"] = kernels.IdSet(n_nodes, self.dev)
                    else:
                        _lib.call("glint_idset_clear", kernels.ptr(ids.ws), ids.n,
                                  kernels.stream_handle())
                    if full:
                        ids.add_ids(None, start, n_t).add_neighbors(gl, None, start, n_t)
                    else:
                        sl = targets_dev[start:end]
                        ids.add_ids(sl).add_neighbors(gl, sl)
                    ids.finalize()
                    counts = torch.stack([ids.count_dev[0],
                                          hub_pre[end] - hub_pre[start]]).cpu()
                    n_i, n_h = int(counts[0]), int(counts[1])
                if full:
                    memo = gl._cache.setdefault("plan_counts", {})
                    if len(memo) > 4096:
                        memo.clear()
                    memo[(start, end)] = (n_i, n_h)
            fp = devmodel.footprint_counts(blk, n_t, n_i, n_e, dims)
            return _Plan(start, end, n_i, n_e, n_h), fp

        return plan_fn

    # -- layer-wide input-domain evaluation ---------------------------------

    def _layer_inputs(self, blk, gl, targets_dev, full):
        """Evaluate input-domain ops once over the layer's input rows R."""
        import torch

        mats, spaces = {}, {}
        ops = [o for o in blk.op_ids if blk.domains[o] == "input"
               and blk.kinds[o] not in ("Input", "Output")]
        if not ops:
            return mats, spaces
        if full:
            space = _RowSpace()
            n_rows = gl.num_nodes
        else:
            ids = kernels.IdSet(gl.num_nodes, self.dev)
            ids.add_ids(targets_dev).add_neighbors(gl, targets_dev).finalize()
            rows = ids.extract()
            space = _RowSpace(rows, ids.rank_map())
            n_rows = int(rows.shape[0])
        # an activation / identity whose producer is an input-domain Linear used
        # only by it runs in that GEMM's epilogue (the producer's rows are never
        # materialised), as _fusions does for the target domain
        fused, skip = {}, set()
        for o in ops:
            if blk.kinds[o] not in _EPILOGUE_ACTS:
                continue
            x = self.m.operators[o].inputs[0]
            if (x in ops and blk.kinds[x] == "Linear" and self.users[x] == [o]
                    and x not in blk.outputs):
                fused[x], skip = o, skip | {o}
        for o in ops:
            if o in skip:
                continue
            op = self.m.operators[o]
            operands, row_sel = [], []
            for p in op.inputs:
                if p in mats:
                    operands.append(mats[p])
                    row_sel.append(None)
                else:
                    st = self.stores[_ref_key(self.schedule, self.m, p)]
                    sp = self.spaces[_ref_key(self.schedule, self.m, p)]
                    operands.append(st.view())
                    if space.identity and sp.identity:
                        row_sel.append(None)
                    else:
                        sel = space.ids if not space.identity else torch.arange(
                            n_rows, device=self.dev, dtype=torch.int64)
                        row_sel.append(sp.positions(sel))
            width = self.m.out_dims[o]
            out = torch.empty((n_rows, pitch_of(width)), dtype=torch.float32, device=self.dev)[:, :width]
            act_op = fused.get(o)
            self._eval_normal_into(out, op, operands, row_sel,
                                   fused_act=blk.kinds[act_op] if act_op else None)
            target = act_op or o
            mats[target] = out
            spaces[target] = space
            if act_op is None:
                mats[o] = out
                spaces[o] = space
        return mats, spaces

    # -- operator evaluation --------------------------------------------------

    def _eval_normal_into(self, out, op, operands, row_sel, fused_act=None):
        k = op.kind
        if k == "Linear":
            act = _act_code(fused_act)
            kernels.linear_into(out, operands[0], self.params.w[op.op_id], self.params.b[op.op_id],
                                act, a_rows=row_sel[0], precision=self.precision)
        elif k == "Concat":
            col = 0
            for mat, rs in zip(operands, row_sel):
                w = int(mat.shape[1])
                kernels.copy_rows(out[:, col:col + w], mat, src_rows=rs, n_rows=out.shape[0])
                col += w
        elif k in kernels.ELEMENTWISE_KINDS:
            n = len(operands)
            if n <= 8:
                kernels.elementwise_into(out, k, operands, row_sel)
            else:
                kernels.elementwise_into(out, k, operands[:8], row_sel[:8])
                rest, rrest = operands[8:], row_sel[8:]
                while rest:
                    kernels.elementwise_into(out, k, [out] + rest[:7], [None] + rrest[:7])
                    rest, rrest = rest[7:], rrest[7:]
        else:
            raise InternalError(f"unexpected operator kind {k}")
        self.kernel_launches += 1

    # -- one block ------------------------------------------------------------

    def run_block(self, blk):
        import torch

        m = self.m
        layer = blk.layer
        targets_np = self.tsets.v_sets[layer]
        gl = self._graph_for(layer) if blk.has_conv else self.g
        n_nodes = self.g.num_nodes
        full = len(targets_np) == n_nodes
        lo, hi = 0, len(targets_np)
        if self.row_range is not None and full:
            lo, hi = self.row_range
        # pinned + non_blocking: a pageable copy would block the host until the
        # previous layer's kernels finish, and this block's host planning would
        # then leave the device idle (cfg4 JKNet: 7 ms per call)
        targets_dev = None if full else torch.tensor(
            np.ascontiguousarray(targets_np, dtype=np.int64)).pin_memory().to(
                self.dev, non_blocking=True)

        # output stores
        if full:
            out_space = _RowSpace()
        else:
            ids = kernels.IdSet(n_nodes, self.dev)
            ids.add_ids(targets_dev).finalize()
            out_space = _RowSpace(targets_dev, ids.rank_map())
        for o in blk.outputs:
            key = TensorRef(blk.block_id, o).key
            # full mode writes every row (own rows by the kernels, the others by
            # the exchange), so the store needs no memset
            self.stores[key] = DeviceStore(len(targets_np), m.out_dims[o], self.dev,
                                           rows=out_space.ids, rank_map=out_space.rank_map,
                                           zero_fill=not full)
            self.spaces[key] = out_space

        if blk.has_conv:
            prefix = (gl.indptr_host if full else
                      _prefix_host(gl.in_degrees, targets_np))
        else:
            prefix = np.zeros(len(targets_np) + 1, dtype=np.int64)
        hub_pre, hub_host = (self._hub_counter(gl, targets_dev, full) if blk.has_conv
                             else (None, None))
        if self.probe is not None:
            self.probe.mark(f"L{layer} stores + hub prefix")
        layer_mats, layer_spaces = self._layer_inputs(blk, gl, targets_dev, full)
        if self.probe is not None:
            self.probe.mark(f"L{layer} input-domain ops")
        fused = self._fusions(blk)
        gat_cache = {}
        n_convs = sum(1 for _, k, _ in blk.iter_ops() if k in ("ConvMean", "ConvAttn"))
        # Transform-first convs (reassociated ConvMean, ConvAttn) transform their
        # source rows once per layer, before any batch, on EVERY rank: in a
        # distributed run the exchange of the transformed rows is a collective
        # that a rank with an empty row range must join too.
        if blk.has_conv and (hi > lo or self.exchange is not None):
            for o in blk.op_ids:
                if blk.kinds[o] in ("ConvMean", "ConvAttn") and self.transform_first(o):
                    gat_cache[o] = self._transform(o, layer_mats, layer_spaces)

        out_key = self.schedule.model_output.key
        sink_store = (self.stores.get(out_key) if self.sink is not None
                      and blk.block_id == self.schedule.model_output.block else None)

        def run_rows(r0, r1, n_inputs, whole=False):
            # Rows [r0, r1) may run as row chunks -- the kernels are row-invariant,
            # so the bytes are identical -- (a) in the final block, so each
            # finished chunk's device->host copy overlaps the next chunk, and (b)
            # while the graph is still uploading, so a chunk starts as soon as its
            # CSR rows have arrived.
            cuts = {r0, r1}
            if sink_store is not None and r1 - r0 >= 2 * self.sink_chunks:
                env = os.environ.get("GLINT_SINK_FRACS")     # A/B: cumulative row fractions
                if env:
                    fr = np.asarray([float(f) for f in env.split(",")])
                    cuts.update(int(c) for c in (r0 + fr * (r1 - r0)).astype(np.int64))
                else:
                    cuts.update(int(c) for c in np.linspace(r0, r1, self.sink_chunks + 1)
                                .astype(np.int64))
            if full and gl.upload_in_flight():
                cuts.update(h for h, _ in gl._pending if r0 < h < r1)
            if full and self.exchange is not None and hasattr(self.exchange, "piece_bounds"):
                cuts.update(b for b in self.exchange.piece_bounds() if r0 < b < r1)
            cuts = sorted(cuts)
            if hub_host is not None:
                hubs = hub_host[np.asarray(cuts)]
            elif hub_pre is not None and len(cuts) > 2:
                hubs = hub_pre[torch.as_tensor(cuts, device=self.dev)].cpu().numpy()
            else:
                hubs = None
            for k in range(len(cuts) - 1):
                c0, c1 = cuts[k], cuts[k + 1]
                n_hub = int(hubs[k + 1] - hubs[k]) if hubs is not None else self._batch_hubs
                sub = _Plan(c0, c1, n_inputs, int(prefix[c1] - prefix[c0]), n_hub)
                # K7 walks a hub row with one warp: fine inside a whole-layer
                # launch (the longest rows start first, other SMs keep going),
                # but a row chunk or a batch would wait for its longest hub
                # row, which K1's hub CTAs stream ~4x faster
                self._fused_ok = ((whole and len(cuts) == 2 and not self.k7_hubs_beside)
                                  or n_hub == 0)
                self._run_batch(blk, gl, sub, full, targets_dev, layer_mats, layer_spaces, fused,
                                gat_cache)
                if self.probe is not None:
                    self.probe.mark(f"L{layer} rows [{c0},{c1}) launched")
                if sink_store is not None:
                    self.sink(sink_store, c0, c1)
                    if self.probe is not None:
                        self.probe.mark(f"L{layer} sink [{c0},{c1}) queued")
                if full and self.exchange is not None and hasattr(self.exchange, "progress"):
                    self.exchange.progress(self, blk, c1)   # overlap: send finished pieces

        # Speculation while the CSR is still uploading (full mode): a batch's rows
        # are launched before its planning count blocks the host (the count needs
        # the batch's edge ids, i.e. the whole upload for the last layer-1
        # batch).  Batch invariance makes early (or repeated, after an OOM
        # retry shrinks a batch) computation of a row harmless; planning and the
        # batch records are untouched.
        spec = {"hi": lo}
        speculate = full and blk.has_conv and gl.upload_in_flight()
        # Whole-layer run (full mode): when the budget admits the layer's rows
        # as ONE batch, they run as one launch up front (LPT schedule over every
        # row, hub rows beside them) instead of the controller's bootstrap
        # batches (layer 1: 1024, 2048, ... rows, each bounded by its slowest
        # row).  Row invariance makes the bytes identical; the controller still
        # plans its batches (records and stats unchanged) and execute() finds
        # their rows done, exactly as for the upload speculation above.
        if (self.whole_layer and full and blk.has_conv and hi > lo and devmodel.admit(
                devmodel.footprint_counts(blk, hi - lo, n_nodes, int(prefix[hi] - prefix[lo]),
                                          self.dims), self.budget)):
            if self.probe is not None:
                self.probe.mark(f"L{layer} whole layer [{lo},{hi})")
            # The controller's batches after this launch need counting kernels
            # (plan stream) unless its first batch is the whole range: K7's
            # persistent grid then leaves SMs for them, so planning overlaps
            # the layer instead of following it.
            first_end = min(next_batch(prefix, lo, self.controller.thresholds), hi)
            counts = ((first_end < hi or (hi - lo) < n_nodes)
                      and (lo, first_end) not in gl._cache.get("plan_counts", {}))
            self._fused_ctas = kernels.fused_ctas_beside_planning() if counts else 0
            try:
                run_rows(lo, hi, n_nodes, whole=True)
                spec["hi"] = hi
                speculate = True
                self._fused_ctas = 0
            except torch.cuda.OutOfMemoryError:
                self._fused_ctas = 0
                # the real allocator disagrees with the footprint model: fall
                # back to the controller's batches (rows done so far are valid
                # and are recomputed with the same bytes)
                torch.cuda.empty_cache()

        def execute(plan: _Plan):
            if self.probe is not None:
                self.probe.mark(f"L{layer} plan->exec [{plan.start},{plan.end})")
            self._batch_hubs = plan.num_hubs
            r0 = max(plan.start, spec["hi"]) if speculate else plan.start
            if r0 < plan.end:
                try:
                    run_rows(r0, plan.end, plan.num_inputs)
                except torch.cuda.OutOfMemoryError as exc:   # -> controller on_oom
                    torch.cuda.empty_cache()
                    raise DeviceAllocationError(str(exc).splitlines()[0]) from exc

        if self.probe is not None:
            self.probe.mark(f"L{layer} transforms / whole layer")
        if full:
            self.plan_stream.wait_event(gl.indptr_event)     # planning reads only the CSR
        else:   # target lists / hub prefix were produced on the main stream
            self.plan_stream.wait_stream(torch.cuda.current_stream(self.dev))
        plan_fn = self._planner(blk, gl, targets_dev, targets_np, full, prefix, hub_pre, hub_host)
        sub_targets = targets_np[lo:hi] if (lo, hi) != (0, len(targets_np)) else targets_np
        sub_prefix = prefix[lo:hi + 1] - prefix[lo] if (lo, hi) != (0, len(targets_np)) else prefix

        def plan_off(start, end):
            a, b = start + lo, end + lo
            if speculate and b > spec["hi"]:
                # Only a batch the footprint model is sure to admit runs ahead
                # of its count: n_inputs <= min(N, n_targets + n_edges) bounds
                # the footprint from above, so the budget holds during uploads.
                n_e = int(prefix[b] - prefix[a])
                bound = devmodel.footprint_counts(blk, b - a, min(n_nodes, (b - a) + n_e), n_e,
                                                  self.dims)
                if devmodel.admit(bound, self.budget):
                    run_rows(max(a, spec["hi"]), b, b - a)
                    spec["hi"] = b
            plan, fp = plan_fn(a, b)
            return plan, fp

        records = self.controller.run_layer(layer, sub_targets, sub_prefix, plan_off, execute)
        for rec in records:
            self.stats._add_batch(layer, rec.n_targets, rec.footprint,
                                  Thresholds(rec.n_t, rec.n_i), rec.oom_retries)
            self.stats._add_aggregations(layer, n_convs * rec.n_targets)
        return records

    def _run_batch(self, blk, gl, plan, full, targets_dev, layer_mats, layer_spaces, fused,
                   gat_cache):
        import torch

        m = self.m
        s, e = plan.start, plan.end
        B = e - s
        if blk.has_conv:
            gl.wait_rows(e if full else None)   # CSR rows of an in-flight upload
        if B == 0:
            return
        row_ids = None if full else targets_dev[s:e]
        row_base = s if full else 0
        batch_nodes = (torch.arange(s, e, device=self.dev, dtype=torch.int64) if full
                       else row_ids)
        mats = {}
        out_keys = {o: TensorRef(blk.block_id, o).key for o in blk.outputs}

        def dest(o, width):
            """Output buffer for op o: the store slice when o is a stored output."""
            if o in out_keys and blk.domains[o] == "target":
                return self.stores[out_keys[o]].data[s:e, :width]
            return torch.empty((B, pitch_of(width)), dtype=torch.float32, device=self.dev)[:, :width]

        def operand(p):
            """(matrix, row selector) of operand p restricted to the batch targets."""
            if p in mats:
                return mats[p], None
            if p in layer_mats:
                sp = layer_spaces[p]
                if sp.identity:
                    return layer_mats[p][s:e] if full else layer_mats[p], (None if full else row_ids)
                return layer_mats[p], sp.positions(batch_nodes)
            key = _ref_key(self.schedule, m, p)
            st, sp = self.stores[key], self.spaces[key]
            if sp.identity:
                return (st.view()[s:e], None) if full else (st.view(), row_ids)
            return st.view(), sp.positions(batch_nodes)

        def conv_source(p):
            """(matrix over some row space, col_map) feeding a conv."""
            if p in layer_mats:
                sp = layer_spaces[p]
                return layer_mats[p], sp.rank_map
            key = _ref_key(self.schedule, m, p)
            return self.stores[key].view(), self.spaces[key].rank_map

        sched = self._schedule(gl, row_ids, row_base, B, full) if blk.has_conv else None
        n_hub = plan.num_hubs
        if self.probe is not None:
            self.probe.mark(f"L{blk.layer} [{s},{e}) schedule")

        skip = set(fused.values())
        for o in blk.op_ids:
            op = m.operators[o]
            if op.kind in ("Input", "Output") or blk.domains[o] == "input" or o in skip:
                continue
            if op.kind == "ConvMean" and self._reassociate(o):
                # mean(h) W^T + b == mean(h W^T) + b: transform all source rows
                # once per layer (narrower), aggregate the narrow rows with the
                # bias + activation in the aggregation epilogue.
                _h, cmap = conv_source(op.inputs[0])
                d_out = m.out_dims[o]
                act_op = fused.get(o)
                target = act_op or o
                out = dest(target, d_out)
                act = _act_code(m.operators[act_op].kind if act_op else None)
                if self.probe is not None:
                    self.probe.begin("spmm_mean")
                kernels.spmm_mean(out, gat_cache[o], gl.indptr, gl.indices, B, row_ids=row_ids,
                                  row_base=row_base, col_map=cmap, schedule=sched, n_hub=n_hub,
                                  bias=self.params.b[o], act=act)
                if self.probe is not None:
                    self.probe.end(agg_bytes(pitch_of(d_out), plan.num_edges, B))
                self.kernel_launches += 1
                mats[target] = out
                if act_op is None:
                    mats[o] = out
            elif op.kind == "ConvMean" and kernels.conv_mean_supported(
                    conv_source(op.inputs[0])[0], m.out_dims[o], self.precision) and (
                    self._fused_ok or (sched is not None and 0 < n_hub < B)):
                # K7: aggregate and transform in one kernel; the B x d_in
                # aggregate stays on chip (model_ir.py:336-338)
                h, cmap = conv_source(op.inputs[0])
                d_in, d_out = int(h.shape[1]), m.out_dims[o]
                act_op = fused.get(o)
                target = act_op or o
                out = dest(target, d_out)
                act = _act_code(m.operators[act_op].kind if act_op else None)
                if self.probe is not None:
                    self.probe.begin("conv_mean")
                split = not self._fused_ok
                if split:
                    self._hub_rows_beside_k7(out, h, cmap, o, act, gl, row_ids, row_base, sched,
                                             n_hub, B)
                else:
                    kernels.conv_mean(out, h, self.params.w[o], self.params.b[o], act, gl.indptr,
                                      gl.indices, B, row_ids=row_ids, row_base=row_base,
                                      col_map=cmap, schedule=sched, max_ctas=self._fused_ctas)
                self.k7_launches["split" if split else "whole"] += 1
                if self.probe is not None:
                    self.probe.end(conv_bytes(d_in, d_out, plan.num_edges, B))
                self.kernel_launches += 5 if split else 2
                mats[target] = out
                if act_op is None:
                    mats[o] = out
            elif op.kind == "ConvMean":
                h, cmap = conv_source(op.inputs[0])
                d_in = int(h.shape[1])
                agg = torch.empty((B, pitch_of(d_in)), dtype=torch.float32, device=self.dev)[:, :d_in]
                if self.probe is not None:
                    self.probe.begin("spmm_mean")
                kernels.spmm_mean_hot(agg, h, gl, B, row_ids=row_ids, row_base=row_base,
                                      col_map=cmap, schedule=sched, n_hub=n_hub)
                if self.probe is not None:
                    self.probe.end(agg_bytes(d_in, plan.num_edges, B))
                act_op = fused.get(o)
                target = act_op or o
                out = dest(target, m.out_dims[o])
                act = _act_code(m.operators[act_op].kind if act_op else None)
                if self.probe is not None:
                    self.probe.begin("linear")
                kernels.linear_into(out, agg, self.params.w[o], self.params.b[o], act,
                                    precision=self.precision)
                if self.probe is not None:
                    self.probe.end(2 * B * d_in * m.out_dims[o])   # FLOPs
                self.kernel_launches += 2
                mats[target] = out
                if act_op is None:
                    mats[o] = out
            elif op.kind == "ConvAttn":
                _h, cmap = conv_source(op.inputs[0])
                W = op.params["weight"]
                H, dh = int(W.shape[0]), int(W.shape[1])
                Z, s_src, s_dst = gat_cache[o]
                act_op = fused.get(o)
                target = act_op or o
                out = dest(target, H * dh)
                act = _act_code(m.operators[act_op].kind if act_op else None)
                if self.probe is not None:
                    self.probe.begin("gat_aggregate")
                hot = (kernels.hot_indices(gl, kernels.ld(Z) * 4, reserve=GAT_SCORE_L2)
                       if cmap is None else None)
                kernels.gat_aggregate(out, Z, s_src, s_dst, H, dh, gl.indptr,
                                      gl.indices if hot is None else hot, B,
                                      row_ids=row_ids, row_base=row_base, col_map=cmap,
                                      schedule=sched, n_hub=n_hub, act=act)
                if self.probe is not None:
                    self.probe.end(agg_bytes(H * dh, plan.num_edges, B, heads=H))
                self.kernel_launches += 1
                mats[target] = out
                if act_op is None:
                    mats[o] = out
            else:
                ops_, sels = zip(*(operand(p) for p in op.inputs))
                act_op = fused.get(o)
                target = act_op or o
                out = dest(target, m.out_dims[o])
                self._eval_normal_into(out, op, list(ops_), list(sels),
                                       fused_act=m.operators[act_op].kind if act_op else None)
                mats[target] = out
                if act_op is None:
                    mats[o] = out

        for o in blk.outputs:
            st = self.stores[out_keys[o]]
            if blk.domains[o] == "input":
                src, sel = operand(o)
                kernels.copy_rows(st.data[s:e, :st.dim], src, src_rows=sel, n_rows=B)
                self.kernel_launches += 1
            else:
                mat = mats[o]
                view = st.data[s:e, :st.dim]
                if mat.data_ptr() != view.data_ptr():
                    kernels.copy_rows(view, mat)
                    self.kernel_launches += 1

    def _hub_rows_beside_k7(self, out, h, cmap, o, act, gl, row_ids, row_base, sched, n_hub, B):
        """K7 over a launch whose schedule starts with hub rows (a row chunk or a
        batch): the regular rows [n_hub, B) of the schedule run as K7 on all
        but `GLINT_FUSED_RESERVE_SMS` SMs, while the hub rows run beside it on a
        high-priority side stream as K1's hub CTAs into a compact buffer, K2,
        and a row scatter into `out`.  K7 would walk a hub row with one warp,
        and the launch would wait for its longest hub row.  Same bytes as K7 or
        K1 + K2 (row invariance)."""
        import torch

        main = torch.cuda.current_stream(self.dev)
        side = _hub_stream(self.dev)
        side.wait_stream(main)
        sched.record_stream(side)
        if row_ids is not None:
            row_ids.record_stream(side)
        d_in, d_out = int(h.shape[1]), int(out.shape[1])
        with torch.cuda.stream(side):
            hub_pos = sched[:n_hub].to(torch.int64)
            csr_rows = (hub_pos + row_base) if row_ids is None else row_ids[hub_pos]
            agg = torch.empty((n_hub, pitch_of(d_in)), dtype=torch.float32,
                              device=self.dev)[:, :d_in]
            all_hubs = torch.arange(n_hub, dtype=torch.int32, device=self.dev)
            kernels.spmm_mean(agg, h, gl.indptr, gl.indices, n_hub, row_ids=csr_rows,
                              col_map=cmap, schedule=all_hubs, n_hub=n_hub)
            res = torch.empty((n_hub, pitch_of(d_out)), dtype=torch.float32,
                              device=self.dev)[:, :d_out]
            kernels.linear_into(res, agg, self.params.w[o], self.params.b[o], act,
                                precision=self.precision)
            kernels.copy_rows(out, res, dst_rows=hub_pos)
        kernels.conv_mean(out, h, self.params.w[o], self.params.b[o], act, gl.indptr,
                          gl.indices, B - n_hub, row_ids=row_ids, row_base=row_base,
                          col_map=cmap, schedule=sched[n_hub:],
                          max_ctas=kernels.fused_ctas_beside_planning())
        main.wait_stream(side)

    def _transform(self, o, layer_mats, layer_spaces):
        """Per-layer source transform of a transform-first conv: z = h W^T for a
        reassociated ConvMean; (Z, s_src, s_dst) for a ConvAttn.  In distributed
        full mode each rank transforms its own rows and the result is exchanged."""
        import torch

        op = self.m.operators[o]
        p = op.inputs[0]
        h = (layer_mats[p] if p in layer_mats
             else self.stores[_ref_key(self.schedule, self.m, p)].view())
        own = self._own_source_rows(h)
        lo, hi = own if own else (0, int(h.shape[0]))
        n_src = int(h.shape[0])
        if op.kind == "ConvMean":
            d_in, d_out = int(h.shape[1]), self.m.out_dims[o]
            zfull = torch.empty((n_src, pitch_of(d_out)), dtype=torch.float32, device=self.dev)
            z = zfull[:, :d_out]
            if self.probe is not None:
                self.probe.begin("linear")
            kernels.linear_into(z[lo:hi], h[lo:hi], self.params.w[o], None, _lib.ACT_NONE,
                                precision=self.precision)
            if self.probe is not None:
                self.probe.end(2 * (hi - lo) * d_in * d_out)
            if own:     # every rank sends its transformed rows (d_out wide, not d_in)
                self.exchange.exchange_tensor(zfull)
            self.kernel_launches += 1
            return z
        W = op.params["weight"]
        H, dh = int(W.shape[0]), int(W.shape[1])
        proj = (torch.empty((n_src, H * kernels.head_pitch(dh)), dtype=torch.float32,
                            device=self.dev),
                torch.empty((n_src, H), dtype=torch.float32, device=self.dev),
                torch.empty((n_src, H), dtype=torch.float32, device=self.dev))
        if self.probe is not None:
            self.probe.begin("linear")
        kernels.attn_project(h[lo:hi], self.params.w_pad[o], self.params.attn[o], H, dh,
                             precision=self.precision, out=tuple(t[lo:hi] for t in proj))
        if self.probe is not None:
            self.probe.end(2 * (hi - lo) * int(h.shape[1]) * H * kernels.head_pitch(dh))
        if own:     # exchange the projected rows and scores, not the source rows
            self.exchange.exchange_tensors(proj)
        self.kernel_launches += 2
        return proj

    def _schedule(self, gl, row_ids, row_base, B, full):
        if not full:
            sched, _ = kernels.degree_schedule(gl.indptr, row_ids, 0, B)
            self.kernel_launches += 3
            return sched
        key = (id(gl), row_base, B)
        sched = self._sched_cache.get(key)
        if sched is None:
            sched, _ = kernels.degree_schedule(gl.indptr, None, row_base, B)
            self._sched_cache = {key: sched}
            self.kernel_launches += 3
        return sched

    def release_after(self, blk):
        if self.retain_stores:
            return
        out_key = self.schedule.model_output.key
        keep = (out_key,) if self.release_input else (INPUT_REF, out_key)
        for key, last in self.schedule.drop_after.items():
            if last == blk.block_id and key not in keep:
                st = self.stores.pop(key, None)
                if st is not None:
                    st.release()

    def _own_source_rows(self, h):
        """(lo, hi) when this rank should transform only its own rows of a full
        source matrix and exchange the (narrower / per-head) result instead of
        the source: distributed full mode with a whole-graph source."""
        if self.exchange is None or self.row_range is None or h.shape[0] != self.g.num_nodes:
            return None
        return self.row_range

    def transform_first(self, op_id) -> bool:
        """Convs that transform every source row before aggregating (reassociated
        ConvMean, ConvAttn): in distributed mode they exchange the transformed
        rows, so their source store needs no exchange of its own."""
        op = self.m.operators[op_id]
        return op.kind == "ConvAttn" or (op.kind == "ConvMean" and self._reassociate(op_id))

    def run(self, exchange=None):
        self.exchange = exchange
        if self.probe is not None:
            self.probe.mark("start")
        for blk in self.schedule.blocks:
            self.run_block(blk)
            if self.probe is not None:
                self.probe.mark(f"L{blk.layer} last batch done")
            if exchange is not None:
                exchange(self, blk)
            self.release_after(blk)
            if self.probe is not None:
                self.probe.mark(f"L{blk.layer} released")
        return self.stores[self.schedule.model_output.key]


# ops a producer's epilogue absorbs: activations, and the inference identity
# e2e chunking: CSRs below SMALL_UPLOAD_EDGES edges upload in one chunk; the
# output streams to the host in chunks of about SINK_CHUNK_BYTES
SMALL_UPLOAD_EDGES = 8 << 20
SINK_CHUNK_BYTES = 57_500_000

_EPILOGUE_ACTS = ("ReLU", "LeakyReLU", "DropoutIdentity")


def _act_code(kind):
    """Epilogue activation code of a fused op kind (None: no fused op)."""
    return {None: _lib.ACT_NONE, "ReLU": _lib.ACT_RELU, "LeakyReLU": _lib.ACT_LEAKY_RELU,
            "DropoutIdentity": _lib.ACT_NONE}[kind]


def agg_bytes(width, n_edges, n_rows, heads=0) -> int:
    """Algorithmic HBM bytes of one aggregation launch (SURVEY §8d B_agg):
    gathered fp32 source rows + self rows, int32 indices, int64 indptr, and for
    attention the per-head scores (s_src per edge and self, s_dst per target)."""
    b = 4 * width * (n_edges + n_rows) + 4 * n_edges + 8 * (n_rows + 1)
    if heads:
        b += 4 * heads * (n_edges + 2 * n_rows)
    return b


# L2 already held for K4's evict_last source-score table (N x heads fp32) when
# hot Z rows are steered beside it (Products: 39 MB)
GAT_SCORE_L2 = 40 << 20


def conv_bytes(d_in, d_out, n_edges, n_rows) -> int:
    """Algorithmic HBM bytes of one fused aggregate->transform launch (K7): the
    aggregation's B_agg at d_in plus the d_out-wide output rows (the aggregate
    itself never leaves the SM; W is L2-resident)."""
    return agg_bytes(d_in, n_edges, n_rows) + 4 * pitch_of(d_out) * n_rows


class KernelProbe:
    """CUDA-event timing of selected launches on the launching stream."""

    def __init__(self):
        self.records = []
        self.marks = []
        self._open = None

    def begin(self, name):
        import torch

        ev = torch.cuda.Event(enable_timing=True)
        ev.record()
        self._open = (name, ev)

    def end(self, nbytes):
        import torch

        ev = torch.cuda.Event(enable_timing=True)
        ev.record()
        name, start = self._open
        self.records.append((name, nbytes, start, ev))
        self._open = None

    def mark(self, name, stream=None):
        """Timeline marker on `stream` (default current): device event + host time."""
        import torch

        ev = torch.cuda.Event(enable_timing=True)
        ev.record(stream)
        self.marks.append((name, ev, time.perf_counter()))

    def timeline(self):
        """[(name, device ms since previous marker)] (call after synchronize)."""
        out = []
        for (_, e0, _), (name, e1, _) in zip(self.marks, self.marks[1:]):
            out.append((name, e0.elapsed_time(e1)))
        return out

    def absolute(self):
        """[(name, device ms since first marker, host ms since first marker)]."""
        if not self.marks:
            return []
        e0, h0 = self.marks[0][1], self.marks[0][2]
        return [(n, round(e0.elapsed_time(e), 3), round(1e3 * (h - h0), 3))
                for n, e, h in self.marks]

    def launches(self):
        """[(name, bytes or flops, ms)] per probed launch (call after synchronize)."""
        return [(name, nbytes, s.elapsed_time(e)) for name, nbytes, s, e in self.records]

    def summary(self):
        """{name: (launches, total bytes, total ms)} (call after synchronize)."""
        out = {}
        for name, nbytes, s, e in self.records:
            c, b, t = out.get(name, (0, 0, 0.0))
            out[name] = (c + 1, b + nbytes, t + s.elapsed_time(e))
        return out


def _prefix_host(degs, targets_np):
    pre = np.zeros(len(targets_np) + 1, dtype=np.int64)
    if len(targets_np):
        np.cumsum(degs[targets_np], out=pre[1:])
    return pre


def infer_layerwise(m: ModelGraph, schedule: BlockSchedule, g, x_store, tsets: TargetSets,
                    budget, thresholds: Thresholds, stats: RunStats, store_backing="memory",
                    workdir=None, precision=None):
    """Execute the block schedule; returns the model-output DeviceStore."""
    dg = kernels.device_graph(g)
    x = _as_device_store(x_store, dg.device)
    eng = LayerwiseEngine(m, schedule, dg, x, tsets, budget, thresholds, stats, precision)
    return eng.run()


# --------------------------------------------------------------- nodewise --


def infer_nodewise(m: ModelGraph, g, x_store, targets, batch_size, budget, stats: RunStats,
                   sampled=None, precision=None):
    """Per-chunk multi-hop evaluation of the unsplit DAG (glint/executor.py:387-469).

    The correctness baseline: recomputes shared neighbours per chunk.  Runs on
    the device with the same kernels; a footprint over capacity is a hard
    DeviceCapacityError.
    """
    import torch

    if batch_size < 1:
        raise ConfigError(f"batch size must be >= 1, got {batch_size}")
    dg = kernels.device_graph(g)
    x = _as_device_store(x_store, dg.device).view()
    targets = np.asarray(targets, dtype=np.int64)
    out = torch.zeros((len(targets), m.output_dim), dtype=torch.float32, device=dg.device)
    graphs = {}

    def graph_for(layer):
        if sampled is not None and layer in sampled:
            if layer not in graphs:
                graphs[layer] = kernels.device_graph(sampled[layer], dg.device)
            return graphs[layer]
        return dg

    params = _Params(m, dg.device)
    for start in range(0, len(targets), batch_size):
        chunk = targets[start:start + batch_size]
        chunk_sorted = np.unique(chunk)
        need = {m.output_id: chunk_sorted}
        for op_id in reversed(m.topo_order):
            cur = need.get(op_id)
            op = m.operators[op_id]
            if cur is None or op.kind == "Input":
                continue
            req = _expand_dev(graph_for(m.layer_of[op_id]), cur) if op.is_conv else cur
            for p in op.inputs:
                need[p] = np.union1d(need[p], req) if p in need else req
        slice_b = inter_b = 0
        agg_counts, bcs = {}, {}
        for op_id in m.topo_order:
            op = m.operators[op_id]
            if op_id not in need or op.kind in ("Input", "Output"):
                continue
            inter_b += len(need[op_id]) * m.out_dims[op_id] * devmodel.VALUE_BYTES
            if op.is_conv:
                bc = kernels.build_batch_csc(graph_for(m.layer_of[op_id]), need[op_id])
                bcs[op_id] = bc
                slice_b += (bc.num_targets + 1 + bc.num_edges) * devmodel.ID_BYTES
                lay = m.layer_of[op_id]
                agg_counts[lay] = agg_counts.get(lay, 0) + bc.num_targets
        in_b = len(need[m.input_id]) * m.input_dim * devmodel.VALUE_BYTES
        out_b = len(chunk) * m.output_dim * devmodel.VALUE_BYTES
        fp = devmodel.BatchFootprint(slice_b, in_b, inter_b, out_b)
        if fp.peak > budget.capacity:
            raise DeviceCapacityError(
                f"node-wise batch of {len(chunk)} targets needs {fp.peak} B, "
                f"over device capacity {budget.capacity} B")
        need_dev = {k: torch.from_numpy(v).to(dg.device) for k, v in need.items()}
        mats = {m.input_id: x.index_select(0, need_dev[m.input_id])}

        def rows_of(p, ids_dev):
            return torch.searchsorted(need_dev[p], ids_dev)

        for op_id in m.topo_order:
            op = m.operators[op_id]
            if op_id not in need or op.kind in ("Input", "Output"):
                continue
            if op.is_conv:
                bc = bcs[op_id]
                p = op.inputs[0]
                h = mats[p].index_select(0, rows_of(p, bc.input_ids))
                mats[op_id] = _eval_conv_dev(op, bc, h, params, precision)
            else:
                rows = need_dev[op_id]
                mats[op_id] = _eval_normal_dev(
                    op, [mats[p].index_select(0, rows_of(p, rows)) for p in op.inputs], params,
                    precision)
        prod = m.operators[m.output_id].inputs[0]
        ck = torch.from_numpy(np.array(chunk, dtype=np.int64)).to(dg.device)
        out[start:start + len(chunk)] = mats[prod].index_select(0, rows_of(prod, ck))
        stats._add_batch(0, len(chunk), fp)
        for lay, cnt in sorted(agg_counts.items()):
            stats._add_aggregations(lay, cnt)
    return out


def _eval_conv_dev(op, bc, h, params, precision):
    import torch

    if op.kind == "ConvMean":
        agg = kernels.agg_mean(bc, h)
        out = torch.empty((agg.shape[0], params.w[op.op_id].shape[0]), dtype=torch.float32,
                          device=h.device)
        return kernels.linear_into(out, agg, params.w[op.op_id], params.b[op.op_id],
                                   _lib.ACT_NONE, precision=precision)
    W = op.params["weight"]
    H, dh = int(W.shape[0]), int(W.shape[1])
    Z, s_src, s_dst = kernels.attn_project(h, params.w_pad[op.op_id], params.attn[op.op_id], H,
                                           dh, precision=precision)
    out = torch.empty((bc.num_targets, H * dh), dtype=torch.float32, device=h.device)
    if bc.num_targets:
        sched, n_hub = kernels._local_schedule(bc.indptr, bc.num_targets)
        kernels.gat_aggregate(out, Z, s_src, s_dst, H, dh, bc.indptr, bc.local32, bc.num_targets,
                              self_rows=bc.target_pos, schedule=sched, n_hub=n_hub)
    return out


def _eval_normal_dev(op, mats, params, precision):
    import torch

    if op.kind == "Linear":
        w = params.w[op.op_id]
        out = torch.empty((mats[0].shape[0], w.shape[0]), dtype=torch.float32,
                          device=mats[0].device)
        return kernels.linear_into(out, mats[0], w, params.b[op.op_id], _lib.ACT_NONE,
                                   precision=precision)
    if op.kind == "Concat":
        return kernels.concat(mats)
    return kernels.elementwise(op.kind, mats)


# ------------------------------------------------------------- request API --


@dataclass
class InferenceResult:
    output: object                # numpy (host inputs) or CUDA tensor; user target order
    target_ids: np.ndarray
    stats: RunStats
    order: NodeOrder
    schedule: BlockSchedule | None = None
    budget: object = None


def _host_tensor_ok(x) -> bool:
    """Features that live on the host (numpy / EmbeddingStore / CPU tensor)."""
    import torch

    if isinstance(x, DeviceStore):
        return False
    if isinstance(x, torch.Tensor):
        return not x.is_cuda
    return True


_COPY_STREAMS: dict = {}


def _copy_stream(device):
    import torch

    s = _COPY_STREAMS.get(device)
    if s is None:
        s = _COPY_STREAMS[device] = torch.cuda.Stream(device=device)
    return s


def _as_device_store(x, device, non_blocking=False) -> DeviceStore:
    import torch

    if isinstance(x, DeviceStore):
        return x
    arr = x.to_array() if isinstance(x, EmbeddingStore) else x
    if non_blocking and isinstance(arr, torch.Tensor) and arr.dtype == torch.float32:
        t = arr.to(kernels.cuda_device(device), non_blocking=True)
    else:
        t = kernels.to_device(arr, torch.float32, device)
    n, d = int(t.shape[0]), int(t.shape[1])
    if d % 4 == 0 and t.is_contiguous():
        return DeviceStore(n, d, t.device, data=t)
    st = DeviceStore(n, d, t.device)
    kernels.copy_rows(st.view(), t)
    return st


def _dims_of(x):
    if isinstance(x, (EmbeddingStore, DeviceStore)):
        return x.num_rows, x.dim
    return int(x.shape[0]), int(x.shape[1])


def resolve_budget(budget, resident_bytes=0):
    if budget is None:
        raise ConfigError("a device budget is required")
    if isinstance(budget, str):
        if budget != "device":
            raise ConfigError(f"unknown budget spec {budget!r}")
        return devmodel.DeviceBudget.from_device(reserve_bytes=resident_bytes)
    return budget


class _HostSink:
    """Streams finished output rows to pinned host memory on a copy stream.

    A pitched store (47 columns in 48-float rows) is first packed into a dense
    device buffer allocated here, before the run (K5 row copy on the compute
    stream, ~0.1 ms per 0.46 GB), so each chunk leaves in one 1-D copy at full
    PCIe rate: a 2-D copy of 188-byte rows runs at 33 GB/s instead of 52
    (profiles/r01_pcie_copy_rates.jsonl), and no allocation happens in the
    last layer's loop."""

    def __init__(self, n_rows, dim, device):
        import torch

        self.host = torch.empty((n_rows, dim), dtype=torch.float32, pin_memory=True)
        self.stream = torch.cuda.Stream(device=device)
        self.device = device
        self.dense = None
        if pitch_of(dim) != dim:
            self.dense = torch.empty((n_rows, dim), dtype=torch.float32, device=device)

    def __call__(self, store, lo, hi):
        import torch

        src = store.view()[lo:hi]
        if self.dense is not None and not src.is_contiguous():
            src = kernels.copy_rows(self.dense[lo:hi], src)
        ev = torch.cuda.Event()
        ev.record()
        with torch.cuda.stream(self.stream):
            self.stream.wait_event(ev)
            self.host[lo:hi].copy_(src, non_blocking=True)

    def finish(self):
        self.stream.synchronize()
        return self.host.numpy()


def _exchange_for(distributed, mode, g, kind="replicate"):
    """RowExchange when running full-mode inference across torch.distributed ranks
    (kind "halo": each rank receives only the rows its CSR slice reads)."""
    if distributed is False or mode != "full":
        return None
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        if distributed is True:
            raise ConfigError("distributed=True needs an initialised process group")
        return None
    from .parallel import HaloPlan, RowExchange, edge_balanced_ranges

    if kind not in ("replicate", "halo"):
        raise ConfigError(f"unknown exchange {kind!r} (replicate | halo)")
    world = dist.get_world_size()
    cuts = edge_balanced_ranges(g.indptr_host, world)
    halo = HaloPlan(g.indptr_host, g.indices, cuts, dist.get_rank()) if kind == "halo" else None
    return RowExchange(cuts, dist.get_rank(), world, halo=halo)


def run_inference(m: ModelGraph, g, x_store, *, mode="full", targets=None, fanout=None, seed=0,
                  executor="layerwise", order="none", budget=None, thresholds=None,
                  batch_size=1024, store_backing="memory", workdir=None, output="auto",
                  precision=None, distributed="auto", reassociate=False,
                  probe=None, exchange="replicate") -> InferenceResult:
    """End to end: reorder, annotate, execute, de-permute (glint/executor.py:481-543).

    ``budget`` may be a DeviceBudget (reference behaviour) or ``"device"``:
    capacity from free HBM after the resident stores are planned.
    ``output``: "numpy", "device" or "auto" (numpy when the features came
    from the host).  ``store_backing="file"`` is accepted for compatibility;
    stores stay HBM-resident either way (outputs are identical).
    ``distributed``: "auto" row-partitions full-mode layer-wise inference over
    an initialised torch.distributed group (one process per GPU, NCCL); each
    rank computes its edge-balanced node range and returns the full output.
    Batch records / stats then describe the calling rank's own batches.
    ``exchange``: "replicate" broadcasts every rank's rows of each exchanged
    layer to all ranks; "halo" ships each rank only the rows its CSR slice
    reads (one all-to-all per layer; tools/halo_fraction.py measures the
    saving).  Outputs are byte-identical either way.
    ``reassociate=True`` (opt-in) computes a width-narrowing ConvMean as
    mean(h W^T) + b: exact in real arithmetic, ~1e-7 apart in fp32, and it
    gathers d_out instead of d_in floats per edge.  Off by default so that
    layer-wise, node-wise and eval_reference stay byte-identical, as in the
    reference (glint/executor.py:481-543).
    """
    import torch

    if mode == "partial" and targets is None:
        raise ConfigError("partial mode requires a target list")
    if mode == "sampling" and (fanout is None or fanout < 1):
        raise ConfigError("sampling mode requires fanout >= 1")
    if budget is None:
        raise ConfigError("a device budget is required")
    n_rows, dim = _dims_of(x_store)
    if n_rows != g.num_nodes or dim != m.input_dim:
        raise ConfigError(f"features ({n_rows}x{dim}) do not match "
                          f"graph ({g.num_nodes} nodes) and model input dim {m.input_dim}")
    if mode not in MODES:
        raise ConfigError(f"unknown inference mode {mode!r}")
    if executor not in ("layerwise", "nodewise"):
        raise ConfigError(f"unknown executor {executor!r}")
    if mode == "full" or targets is None:
        user_targets = arange_ids(g.num_nodes)
    else:
        user_targets = np.asarray(targets, dtype=np.int64)
        if len(user_targets) != len(_sorted_unique(user_targets)):
            raise ConfigError("duplicate target ids")
        if len(user_targets) and (user_targets.min() < 0 or user_targets.max() >= g.num_nodes):
            raise ConfigError("target ids out of range")
    host_out = (output == "numpy") or (output == "auto" and not isinstance(
        x_store, (torch.Tensor, DeviceStore)))

    if probe is not None:
        probe.mark("run_inference entry")
    # RCMK of a host graph runs on its device copy (reorder._rcmk_device),
    # once the CSR has landed; the other orders are cheap host numpy
    rcmk_on_device = order == "rcmk" and isinstance(g, CscGraph) and g.num_nodes > 0
    node_order = None if rcmk_on_device else make_order(g, order, seed)
    if isinstance(g, CscGraph) and _host_tensor_ok(x_store):
        # Host inputs: features first, then the CSR in row chunks on a copy
        # stream; layer-1 batches start as soon as their rows have arrived.
        dev = kernels.cuda_device()
        copy = _copy_stream(dev)
        box = {}

        def upload_features():          # queued right after indptr, before the CSR
            box["x"] = _as_device_store(x_store, dev, non_blocking=True)
            box["ev"] = torch.cuda.Event()
            box["ev"].record(copy)
            if probe is not None:
                probe.mark("features uploaded (copy stream)", copy)

        # The packed CSR (host-narrowed, 24-bit) uploads faster than layer 1
        # computes, so layer 1 only needs a small first chunk to start on and
        # then stays ahead of the rest: chunk ends at 1/16, 1/4, 1/2, 3/4 of the
        # edges (tools/e2e_ab.py --fracs-ab: median 64.8 ms vs 66.9 for the
        # geometric 1/16, 1/8, 1/4, 1/2 plan, whose last half-of-the-edges chunk
        # left 7.7 ms of layer 1 behind the upload; 66.6 for 8 uniform chunks;
        # profiles/r01_e2e_fracs_ab.jsonl).  Without host narrowing: 16 chunks.
        # A small CSR (cfg1: 2M edges) goes in one chunk: its upload is shorter
        # than the per-chunk planning and launches it would overlap.
        small = g.num_edges < SMALL_UPLOAD_EDGES
        chunks = int(os.environ.get("GLINT_UPLOAD_CHUNKS",
                                    "1" if small else ("5" if HOST_NARROW else "16")))
        geometric = os.environ.get("GLINT_UPLOAD_GEOMETRIC", "0") == "1"
        fracs = ((0.0625, 0.25, 0.5, 0.75) if HOST_NARROW and not geometric and not small
                 and "GLINT_UPLOAD_CHUNKS" not in os.environ else None)
        dg0 = DeviceGraph.upload_async(g, dev, copy, after_indptr=upload_features, chunks=chunks,
                                       geometric=geometric, fracs=fracs)
        x0, x_ready = box["x"], box["ev"]
        if probe is not None:
            probe.mark("csr uploaded (copy stream)", copy)
            probe.mark("uploads issued (main stream)")
        torch.cuda.current_stream(dev).wait_event(x_ready)
        if node_order is None or not node_order.is_identity():
            dg0.wait_rows()
    else:
        dg0 = kernels.device_graph(g)
        x0 = _as_device_store(x_store, dg0.device)
    if node_order is None:
        node_order = make_order(dg0, order, seed)
    g_i, x_i = apply_order_device(dg0, x0, node_order)
    if mode == "full" or targets is None:
        internal = user_targets                      # sorted(inv[arange(N)]) == arange(N)
    elif node_order.is_identity():
        internal = _sorted_unique(user_targets)      # ids are distinct: a sorted copy
    else:
        internal = np.sort(node_order.inv[user_targets]) if len(user_targets) else user_targets
    thresholds = thresholds or Thresholds(n_t=1024, n_i=32768)
    stats = RunStats(executor=executor, mode=mode, order=order, depth=m.depth,
                     initial_thresholds=(thresholds.n_t, thresholds.n_i)
                     if executor == "layerwise" else None)
    started = time.perf_counter()
    tsets = annotate(g_i, internal, m.depth, mode, fanout, seed)   # device draws in sampling mode
    schedule = None
    if executor == "layerwise":
        schedule = split(m)
        bud = resolve_budget(budget, _resident_bytes(m, schedule, tsets, g_i, reassociate))
        ex = _exchange_for(distributed, mode, g_i, exchange)
        eng = LayerwiseEngine(m, schedule, g_i, x_i, tsets, bud, thresholds, stats, precision,
                              row_range=ex.row_range if ex else None, reassociate=reassociate)
        row_ids = tsets.v_sets[m.depth if m.depth else 0]
        streamed = None
        if (host_out and ex is None and node_order.is_identity() and _is_arange(row_ids)
                and len(row_ids) == g.num_nodes and user_targets is arange_ids(g.num_nodes)):
            streamed = _HostSink(g.num_nodes, m.output_dim, dg0.device)
            eng.sink = streamed
            if "GLINT_SINK_CHUNKS" not in os.environ:
                # the device->host copy outlasts the last layer, so it should
                # start early: chunks of ~57 MB, 1..16 of them -- GCN's 0.46 GB
                # output in 8 (tools/e2e_ab.py --sink-ab: 63.6 ms vs 64.4 with
                # 4; profiles/r01_e2e_sink_ab.jsonl), GAT's 1.84 GB in 16, and a
                # small output in one piece (each chunk costs ~0.2 ms of host
                # launches and planning)
                out_bytes = g.num_nodes * m.output_dim * 4
                eng.sink_chunks = int(min(16, max(1, round(out_bytes / SINK_CHUNK_BYTES))))
        eng.probe = probe
        store = eng.run(exchange=ex)
        if ex is not None:
            ex.replicate_tensor(store.data)     # every rank returns the full output
        if streamed is None:
            wanted = user_targets if node_order.is_identity() else node_order.inv[user_targets]
            out_dev = _gather_rows(store, row_ids, wanted, dg0.device)
    else:
        bud = resolve_budget(budget)
        out_sorted = infer_nodewise(m, g_i, x_i, internal, batch_size, bud, stats,
                                    sampled=tsets.sampled, precision=precision)
        row_ids = internal
        out_dev = _gather_dense(out_sorted, row_ids, node_order.inv[user_targets])
    if executor == "layerwise" and streamed is not None:
        if probe is not None:
            probe.mark("output streamed (copy stream)", streamed.stream)
        output_val = streamed.finish()
        if probe is not None:
            probe.mark("output on host")
    elif host_out:
        staging = torch.empty(tuple(out_dev.shape), dtype=torch.float32, pin_memory=True)
        staging.copy_(out_dev)
        output_val = staging.numpy()
    else:
        output_val = out_dev
    torch.cuda.synchronize(dg0.device)
    stats.wall_time = time.perf_counter() - started
    if probe is not None:
        probe.mark("return")
    return InferenceResult(output=output_val, target_ids=user_targets, stats=stats,
                           order=node_order, schedule=schedule, budget=bud)


def _transform_bytes(m, blk, src_rows, reassociate):
    """Bytes of a block's per-layer transformed source rows (transform-first
    convs: ConvAttn's Z and scores, a reassociated narrowing ConvMean's z),
    alive while the block runs, outside the per-batch footprint model."""
    total = 0
    for o in blk.op_ids:
        op = m.operators[o]
        if op.kind == "ConvAttn":
            H, dh = int(op.params["weight"].shape[0]), int(op.params["weight"].shape[1])
            total += src_rows * (H * kernels.head_pitch(dh) + 2 * H) * 4
        elif op.kind == "ConvMean" and reassociate:
            w = op.params["weight"]
            if pitch_of(w.shape[0]) < pitch_of(w.shape[1]):
                total += src_rows * pitch_of(w.shape[0]) * 4
    return total


def _resident_bytes(m, schedule, tsets, g, reassociate=False):
    """Upper bound of resident bytes alive at once (for budget='device'): the
    stores, plus the running block's transformed source rows."""
    live = 0
    peak = 0
    sizes = {}
    for blk in schedule.blocks:
        rows = len(tsets.v_sets[blk.layer])
        for o in blk.outputs:
            sizes[TensorRef(blk.block_id, o).key] = rows * pitch_of(m.out_dims[o]) * 4
            live += sizes[TensorRef(blk.block_id, o).key]
        src_rows = len(tsets.v_sets[blk.layer - 1]) if blk.layer > 1 and \
            (blk.layer - 1) in tsets.v_sets else g.num_nodes
        peak = max(peak, live + _transform_bytes(m, blk, src_rows, reassociate))
        for key, last in schedule.drop_after.items():
            if last == blk.block_id and key in sizes:
                live -= sizes.pop(key)
    return peak


def _is_arange(a) -> bool:
    """a == arange(len(a)) (O(1) for the cached identity, cheap checks first)."""
    n = len(a)
    if a is arange_ids(n):
        return True
    return n == 0 or (a[0] == 0 and a[-1] == n - 1 and bool(np.all(np.diff(a) == 1)))


def _gather_rows(store: DeviceStore, row_ids, wanted, device):
    """Rows of `store` (rows = sorted row_ids) for internal ids `wanted`, in order."""
    import torch

    if len(row_ids) == store.num_rows and _is_arange(row_ids):
        if _is_arange(wanted) and len(wanted) == store.num_rows:
            return store.view()                      # identity: no gather needed
        if len(wanted) and (wanted.min() < 0 or wanted.max() >= store.num_rows):
            raise InternalError("output rows do not cover the requested targets")
        out = torch.empty((len(wanted), store.dim), dtype=torch.float32, device=device)
        if len(wanted):
            kernels.copy_rows(out, store.view(),
                              src_rows=torch.from_numpy(np.ascontiguousarray(wanted)).to(device))
        return out
    out = torch.empty((len(wanted), store.dim), dtype=torch.float32, device=device)
    if not len(wanted):
        return out
    if store.rank_map is not None and store.rows is not None:
        # positions on the device through the store's node -> row rank map
        w = torch.tensor(np.ascontiguousarray(wanted, dtype=np.int64)).to(device)
        if int(w.min()) < 0 or int(w.max()) >= store.rank_map.numel():
            raise InternalError("output rows do not cover the requested targets")
        pos = store.rank_map.index_select(0, w).to(torch.int64)
        ok = (pos >= 0) & (pos < store.num_rows)
        if not bool(ok.all()) or not torch.equal(store.rows.index_select(0, pos.clamp(0)), w):
            raise InternalError("output rows do not cover the requested targets")
        kernels.copy_rows(out, store.view(), src_rows=pos)
        return out
    pos = np.searchsorted(row_ids, wanted)
    safe = np.minimum(pos, len(row_ids) - 1)
    if not np.array_equal(row_ids[safe], wanted):
        raise InternalError("output rows do not cover the requested targets")
    kernels.copy_rows(out, store.view(), src_rows=torch.from_numpy(pos.astype(np.int64)).to(device))
    return out


def _gather_dense(mat, row_ids, wanted):
    import torch

    pos = np.searchsorted(row_ids, wanted)
    if len(wanted):
        safe = np.minimum(pos, len(row_ids) - 1)
        if not np.array_equal(row_ids[safe], wanted):
            raise InternalError("output rows do not cover the requested targets")
    out = torch.empty((len(wanted), mat.shape[1]), dtype=torch.float32, device=mat.device)
    if len(wanted):
        kernels.copy_rows(out, mat, src_rows=torch.from_numpy(pos.astype(np.int64)).to(mat.device))
    return out
