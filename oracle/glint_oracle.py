"""CPU ORACLE -- test infrastructure only.

A plain numpy restatement of the reference `glint` hot path (arXiv 2211.15082,
pkg/src/glint/*.py), used as the CHECKER for the B200 implementation.  Only
tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
leg may import it; the product package never does (it has no CPU fallback).

Pinning: every function here is checked against golden vectors produced by
running the reference itself in the build container (tests/golden/
make_golden.py -> tests/golden/*.npz, tests/test_oracle_golden.py).

Each function cites the reference file:line it restates.  The numerics use
the same numpy primitives as the reference (np.add.at accumulation in edge
order, einsum for dense transforms), so this oracle is byte-identical to the
reference on the same inputs, and equally single-threaded.
"""

from __future__ import annotations

from collections import namedtuple

import numpy as np

LEAKY_SLOPE = np.float32(0.2)      # kernels.py:22
NORM_EPS = np.float32(1e-12)       # kernels.py:23

Batch = namedtuple("Batch", "targets input_ids indptr local_srcs target_pos")


# -- batch structure: kernels.py:56-88 ------------------------------------------


def gather_slices(indptr, indices, targets):
    """kernels.py:56-68: concatenated in-neighbour slices + local offsets."""
    targets = np.asarray(targets, dtype=np.int64)
    lo = indptr[targets]
    cnt = indptr[targets + 1] - lo
    local = np.zeros(len(targets) + 1, dtype=np.int64)
    np.cumsum(cnt, out=local[1:])
    n = int(local[-1])
    if n == 0:
        return np.zeros(0, dtype=np.int64), local
    src_pos = np.repeat(lo - local[:-1], cnt) + np.arange(n, dtype=np.int64)
    return np.asarray(indices, dtype=np.int64)[src_pos], local


def build_batch_csc(indptr, indices, targets) -> Batch:
    """kernels.py:71-77: input_ids = unique(targets u srcs); searchsorted positions."""
    targets = np.asarray(targets, dtype=np.int64)
    srcs, local = gather_slices(indptr, indices, targets)
    ids = np.unique(np.concatenate([targets, srcs])) if len(targets) else targets
    return Batch(targets, ids, local, np.searchsorted(ids, srcs), np.searchsorted(ids, targets))


def prefix_for_targets(indptr, targets):
    """storage.py:159-165."""
    targets = np.asarray(targets, dtype=np.int64)
    out = np.zeros(len(targets) + 1, dtype=np.int64)
    if len(targets):
        np.cumsum(indptr[targets + 1] - indptr[targets], out=out[1:])
    return out


# -- numerics: kernels.py:95-239 ---------------------------------------------------


def linear(x, w, b=None):
    """kernels.py:95-107 (einsum, fp32)."""
    out = np.einsum("ij,kj->ik", np.asarray(x, np.float32), np.asarray(w, np.float32))
    return out if b is None else out + np.asarray(b, np.float32)


def _seg_sum(vals, seg, n):
    """kernels.py:110-115: np.add.at accumulates strictly in element order."""
    out = np.zeros((n,) + vals.shape[1:], dtype=np.float32)
    if len(seg):
        np.add.at(out, seg, vals)
    return out


def _edge_owner(bc):
    """kernels.py:118-119."""
    return np.repeat(np.arange(len(bc.targets), dtype=np.int64), np.diff(bc.indptr))


def agg_mean(bc, h):
    """kernels.py:122-135: (sum of neighbours in stored order + self) / (deg+1)."""
    h = np.asarray(h, np.float32)
    s = _seg_sum(h[bc.local_srcs], _edge_owner(bc), len(bc.targets))
    s += h[bc.target_pos]
    return s / (np.diff(bc.indptr) + 1).astype(np.float32)[:, None]


def leaky_relu(x):
    """kernels.py:138-140."""
    x = np.asarray(x, np.float32)
    return np.where(x >= 0, x, LEAKY_SLOPE * x)


def agg_attn(bc, h, weight, attn):
    """kernels.py:170-203: per-head additive attention, heads concatenated."""
    h = np.asarray(h, np.float32)
    seg = _edge_owner(bc)
    outs = []
    heads, dh = weight.shape[0], weight.shape[1]
    for k in range(heads):
        z = linear(h, weight[k])
        s_src = np.einsum("ij,j->i", z, np.asarray(attn[k, :dh], np.float32))
        s_dst = np.einsum("ij,j->i", z, np.asarray(attn[k, dh:], np.float32))
        sd = s_dst[bc.target_pos]
        self_logit = leaky_relu(s_src[bc.target_pos] + sd)
        edge_logit = leaky_relu(s_src[bc.local_srcs] + sd[seg])
        peak = self_logit.copy()
        if len(seg):
            np.maximum.at(peak, seg, edge_logit)
        w_e = np.exp(edge_logit - peak[seg])
        w_s = np.exp(self_logit - peak)
        den = _seg_sum(w_e, seg, len(bc.targets)) + w_s
        num = _seg_sum(w_e[:, None] * z[bc.local_srcs], seg, len(bc.targets))
        num += w_s[:, None] * z[bc.target_pos]
        outs.append(num / den[:, None])
    return np.concatenate(outs, axis=1)


def elementwise(kind, mats):
    """kernels.py:206-231."""
    mats = [np.asarray(m, np.float32) for m in mats]
    if kind == "ReLU":
        return np.maximum(mats[0], np.float32(0))
    if kind == "LeakyReLU":
        return leaky_relu(mats[0])
    if kind == "DropoutIdentity":
        return mats[0].copy()
    if kind == "Add":
        acc = mats[0].copy()
        for m in mats[1:]:
            acc += m
        return acc
    if kind == "Norm":
        x = mats[0]
        return x / np.sqrt(np.sum(x * x, axis=1) + NORM_EPS)[:, None]
    raise ValueError(kind)


def concat(mats):
    """kernels.py:234-239."""
    return np.concatenate([np.asarray(m, np.float32) for m in mats], axis=1)


# -- whole-graph model evaluation: model_ir.py:334-372 -----------------------------

OpSpec = namedtuple("OpSpec", "op_id kind inputs params")


def model_spec(m):
    """Duck-typed (op list in topological order, input id, output id) of a model."""
    ops = [OpSpec(o, m.operators[o].kind, tuple(m.operators[o].inputs),
                  dict(m.operators[o].params)) for o in m.topo_order]
    return ops, m.input_id, m.output_id


def eval_model(spec, indptr, indices, x):
    """model_ir.py:354-372: one batch holding the whole graph, topological order."""
    ops, _in_id, out_id = spec
    n = len(indptr) - 1
    bc = build_batch_csc(indptr, indices, np.arange(n, dtype=np.int64))
    mats = {}
    for op in ops:
        if op.kind == "Input":
            mats[op.op_id] = np.asarray(x, np.float32)
        elif op.kind == "Output":
            mats[op.op_id] = mats[op.inputs[0]]
        elif op.kind == "ConvMean":                       # model_ir.py:336-338
            mats[op.op_id] = linear(agg_mean(bc, mats[op.inputs[0]]), op.params["weight"],
                                    op.params.get("bias"))
        elif op.kind == "ConvAttn":                       # model_ir.py:339-340
            mats[op.op_id] = agg_attn(bc, mats[op.inputs[0]], op.params["weight"],
                                      op.params["attn"])
        elif op.kind == "Linear":                         # model_ir.py:345-346
            mats[op.op_id] = linear(mats[op.inputs[0]], op.params["weight"],
                                    op.params.get("bias"))
        elif op.kind == "Concat":
            mats[op.op_id] = concat([mats[p] for p in op.inputs])
        else:
            mats[op.op_id] = elementwise(op.kind, [mats[p] for p in op.inputs])
    return mats[out_id]


def conv_rows(indptr, indices, h_in, targets, op):
    """One conv for a target subset (executor.py:351-384 on a single batch).

    By batch invariance (kernels.py:1-14) these rows equal the whole-graph
    rows, so large runs are spot-checked on a sample of targets.  Returns
    (aggregated rows or None, conv output rows)."""
    bc = build_batch_csc(indptr, indices, targets)
    hh = np.asarray(h_in, np.float32)[bc.input_ids]
    if op.kind == "ConvMean":
        agg = agg_mean(bc, hh)
        return agg, linear(agg, op.params["weight"], op.params.get("bias"))
    return None, agg_attn(bc, hh, op.params["weight"], op.params["attn"])


# -- batch controller replay: batching.py:40-124 -----------------------------------


def next_batch(prefix, pos, n_t, n_i):
    """batching.py:40-53."""
    n = len(prefix) - 1
    j = min(pos + n_t, n, int(np.searchsorted(prefix, prefix[pos] + n_i, side="right")) - 1)
    return max(j, pos + 1)


def replay_batches(prefix, capacity, n_t, n_i, peak_fn):
    """batching.py:90-124 with admit (device.py:84-86) and adapt/on_oom
    (batching.py:56-65).  peak_fn(start, end) -> accounted peak bytes.
    Returns [(start, end, retries, n_t_after, n_i_after, peak)] and the final
    thresholds (they carry across layers)."""
    target = int(0.9 * capacity)                          # device.py:36-37
    out = []
    pos, n = 0, len(prefix) - 1
    while pos < n:
        retries = 0
        while True:
            end = next_batch(prefix, pos, n_t, n_i)
            peak = peak_fn(pos, end)
            if peak <= capacity:
                break
            if end - pos == 1:
                raise MemoryError(f"node at {pos} alone needs {peak} B")
            n_t, n_i = max(1, n_t // 2), n_i // 2
            retries += 1
        if peak > 0:
            r = min(4.0, max(0.5, target / peak))
            n_t, n_i = max(1, round(r * n_t)), max(0, round(r * n_i))
        out.append((pos, end, retries, n_t, n_i, peak))
        pos = end
    return out, (n_t, n_i)


# -- reverse Cuthill-McKee: reorder.py:55-123 ---------------------------------------


def rcmk(indptr, indices):
    """reorder.py:72-123 (pure Python BFS; desk scale only)."""
    n = len(indptr) - 1
    dst = np.repeat(np.arange(n, dtype=np.int64), np.diff(indptr))
    src = np.asarray(indices, dtype=np.int64)
    keep = src != dst
    a = np.concatenate([src[keep], dst[keep]])
    b = np.concatenate([dst[keep], src[keep]])
    ptr = np.zeros(n + 1, dtype=np.int64)
    nb = np.zeros(0, dtype=np.int64)
    if len(a):
        key = np.unique(a * n + b)
        ua, nb = key // n, key % n
        np.add.at(ptr[1:], ua, 1)
        np.cumsum(ptr, out=ptr)
    deg = np.diff(ptr)
    comp = np.full(n, -1, dtype=np.int64)
    starts = []
    for s in range(n):
        if comp[s] >= 0:
            continue
        c = len(starts)
        comp[s] = c
        stack, members = [s], [s]
        while stack:
            u = stack.pop()
            for v in nb[ptr[u]:ptr[u + 1]]:
                if comp[v] < 0:
                    comp[v] = c
                    stack.append(v)
                    members.append(v)
        mem = np.array(members, dtype=np.int64)
        starts.append(int(mem[np.lexsort((mem, deg[mem]))[0]]))
    starts.sort()
    seen = np.zeros(n, dtype=bool)
    seq = []
    for s in starts:
        seen[s] = True
        q = [s]
        head = 0
        while head < len(q):
            u = q[head]
            head += 1
            cand = nb[ptr[u]:ptr[u + 1]]
            cand = cand[~seen[cand]]
            if len(cand):
                cand = cand[np.lexsort((cand, deg[cand]))]
                seen[cand] = True
                q.extend(cand.tolist())
        seq.extend(q)
    return np.array(seq[::-1], dtype=np.int64)
