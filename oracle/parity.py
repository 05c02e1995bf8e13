"""CPU ORACLE (checker) -- parity at the bench's own scale.  Test infrastructure only.

Used by bench.py OUTSIDE its timed region and by tests/ to check a full-size
B200 run against the reference algorithm without running the whole reference
(a 2.45M-node, 124M-edge layer takes the numpy reference minutes):

* ``spot_targets`` -- a seeded random sample of targets plus the highest
  in-degree rows (the hub rows the B200 path sends to its side-stream kernels).
* ``conv_check`` -- by batch invariance (glint/kernels.py:1-14) one conv's rows
  for a target subset equal its whole-graph rows, so the oracle recomputes
  the sampled rows from the device run's own H^{l-1} rows (build_batch_csc +
  gather + agg_mean/agg_attn + linear, glint/executor.py:351-384) and compares.
* ``footprint_peak`` / ``replay_layers`` -- the batch controller replayed
  plan-only (glint/batching.py:90-124 with glint/device.py:61-86), n_inputs
  counted with a host bitmap, so the device run's batch records can be
  compared byte-for-byte at the device's capacity.

Nothing here is on the product path; the package never imports it.
"""

from __future__ import annotations

import numpy as np

from . import glint_oracle as orc

ID_BYTES = 8        # glint/device.py:21
VALUE_BYTES = 4     # glint/device.py:22


def spot_targets(indptr, n_random=4096, n_hubs=50, seed=1234):
    """Sorted unique: n_random uniform node ids, the n_hubs largest in-degree
    rows, and the first and last node."""
    n = len(indptr) - 1
    rng = np.random.default_rng(seed)
    rnd = rng.choice(n, size=min(n_random, n), replace=False)
    deg = np.diff(indptr)
    hubs = np.argpartition(deg, -min(n_hubs, n))[-min(n_hubs, n):] if n else deg[:0]
    return np.unique(np.concatenate([rnd, hubs, [0, n - 1]]).astype(np.int64))


def batch_for(indptr, indices, targets):
    """orc.build_batch_csc over a (possibly huge) host CSC."""
    return orc.build_batch_csc(indptr, indices, targets)


def rel_l2(got, want) -> float:
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    den = float(np.linalg.norm(want))
    return float(np.linalg.norm(got - want)) / (den if den > 0 else 1.0)


def conv_check(bc, h_rows, layer_spec, got_rows, agg_dev_rows=None):
    """One conv of a sequential model on the sample batch `bc`.

    h_rows: the device run's H^{l-1} at bc.input_ids (host fp32).
    layer_spec: {"kind": "ConvMean", "weight", "bias", "relu"} or
                {"kind": "ConvAttn", "weight", "attn", "relu"}.
    got_rows: the device run's H^l at bc.targets.
    agg_dev_rows: optionally the device's own aggregation (K1) of the same
                  rows, checked byte-for-byte against agg_mean (kernels.py:122-135).
    Returns {"rel_l2": ..., "agg_bytes_equal": bool|None, "max_abs": ...}."""
    out = {"agg_bytes_equal": None}
    if layer_spec["kind"] == "ConvMean":
        agg = orc.agg_mean(bc, h_rows)
        if agg_dev_rows is not None:
            out["agg_bytes_equal"] = bool(np.asarray(agg_dev_rows, np.float32).tobytes()
                                          == agg.tobytes())
        want = orc.linear(agg, layer_spec["weight"], layer_spec.get("bias"))
    else:
        want = orc.agg_attn(bc, h_rows, layer_spec["weight"], layer_spec["attn"])
    if layer_spec.get("relu"):
        want = orc.elementwise("ReLU", [want])
    out["rel_l2"] = rel_l2(got_rows, want)
    out["max_abs"] = float(np.max(np.abs(np.asarray(got_rows, np.float64) - want))) \
        if want.size else 0.0
    return out


def agg_check(bc, h_rows, agg_dev_rows) -> bool:
    """K1 bytes == agg_mean bytes (kernels.py:122-135) on the sample batch."""
    return bool(np.asarray(agg_dev_rows, np.float32).tobytes()
                == orc.agg_mean(bc, h_rows).tobytes())


# -- plan-only replay of the batch controller ---------------------------------------


def footprint_peak(n_t, n_i, n_e, block) -> int:
    """glint/device.py:61-81.  `block` = {"has_conv": bool, "input_widths": [...],
    "ops": [(domain, width), ...] (non-marker ops), "output_widths": [...]}."""
    if n_t == 0:
        return 0
    peak = (n_t + 1 + n_e) * ID_BYTES if block["has_conv"] else 0
    peak += sum(n_i * w * VALUE_BYTES for w in block["input_widths"])
    for domain, w in block["ops"]:
        peak += (n_i if domain == "input" else n_t) * w * VALUE_BYTES
    peak += sum(n_t * w * VALUE_BYTES for w in block["output_widths"])
    return peak


class InputCounter:
    """|unique(targets u in-neighbours)| of a contiguous full-mode batch
    [start, end) (= BatchCsc.num_inputs, kernels.py:71-77), by a host bitmap."""

    def __init__(self, indptr, indices):
        self.indptr, self.indices = indptr, indices
        self.mark = np.zeros(len(indptr) - 1, dtype=bool)

    def __call__(self, start, end) -> int:
        n = len(self.mark)
        if start == 0 and end == n:
            return n
        self.mark[:] = False
        self.mark[start:end] = True
        self.mark[self.indices[self.indptr[start]:self.indptr[end]]] = True
        return int(np.count_nonzero(self.mark))


def replay_layers(indptr, indices, capacity, n_t, n_i, blocks):
    """Full-mode plan-only replay of every block (thresholds carry across
    layers, glint/executor.py:329-347).  Returns per batch
    (layer, n_targets, peak, n_t_after, n_i_after, retries)."""
    count = InputCounter(indptr, indices)
    out = []
    for blk in blocks:
        def peak_fn(a, b, blk=blk):
            n_e = int(indptr[b] - indptr[a]) if blk["has_conv"] else 0
            ni = count(a, b) if blk["has_conv"] else b - a
            return footprint_peak(b - a, ni, n_e, blk)

        prefix = indptr if blk["has_conv"] else np.zeros(len(indptr), dtype=np.int64)
        recs, (n_t, n_i) = orc.replay_batches(prefix, capacity, n_t, n_i, peak_fn)
        for start, end, retries, t_after, i_after, peak in recs:
            out.append((blk["layer"], end - start, peak, t_after, i_after, retries))
    return out
