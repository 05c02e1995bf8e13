"""Batch memory accounting: the feedback signal of the batch controller.

Same deterministic model as the reference (glint/device.py:1-90) so that batch
membership is bit-identical for the same capacity and initial thresholds:

* graph slice (conv blocks only): (n_targets + 1 + n_edges) * 8 B
* each input tensor of the block: n_inputs * width * 4 B
* each non-marker operator output: rows * width * 4 B, rows = n_inputs for
  input-domain operators, n_targets otherwise
* each stored block output: n_targets * width * 4 B

What is new on B200 is where ``capacity`` comes from: ``DeviceBudget.from_device``
derives it from the free HBM reported by the driver (cudaMemGetInfo through the
C ABI) after the resident embedding stores are accounted for, instead of a
host-side constant.  The model stays conservative with respect to what the
resident executor actually allocates per batch (it never materialises the
gathered input copies the model charges for).
"""

from __future__ import annotations

from dataclasses import dataclass

ID_BYTES = 8
VALUE_BYTES = 4

# Setpoint fraction of capacity (glint/device.py:36-37).
SETPOINT_FRACTION = 0.9


@dataclass(frozen=True)
class DeviceBudget:
    """Capacity in bytes; the controller steers batch peaks toward 90% of it."""

    capacity: int

    def __post_init__(self):
        t = self.target
        if t <= 0 or t >= self.capacity:
            raise ValueError(f"capacity {self.capacity} leaves no valid setpoint")

    @property
    def target(self) -> int:
        return int(SETPOINT_FRACTION * self.capacity)

    @classmethod
    def from_device(cls, device=None, reserve_bytes=0, fraction=1.0) -> "DeviceBudget":
        """Capacity = free HBM on `device` minus `reserve_bytes`, times `fraction`."""
        free, _total = device_memory(device)
        cap = int((free - int(reserve_bytes)) * fraction)
        if cap <= 16:
            raise ValueError(f"no free device memory left for batches (free={free})")
        return cls(cap)


# cudaMemGetInfo costs ~1-2 ms per call on the B200 boxes and now and then tens
# of ms (tools/partial_host_profile.py: one call of eight took ~45 ms), so a
# query is reused for MEMINFO_TTL_S: in between, free HBM moves by what this
# process's caching allocator reserved or released since the query.
MEMINFO_TTL_S = 2.0
_MEMINFO = {}


def device_memory(device=None, max_age_s=None):
    """(free, total) bytes of a CUDA device: the driver's numbers, at most
    `max_age_s` (default MEMINFO_TTL_S) old, corrected for this process's
    reservations since (torch.cuda.memory_reserved)."""
    import ctypes
    import time

    import torch

    from . import _lib

    dev = torch.cuda.current_device() if device is None else torch.device(device).index or 0
    ttl = MEMINFO_TTL_S if max_age_s is None else max_age_s
    now = time.monotonic()
    reserved = torch.cuda.memory_reserved(dev)
    hit = _MEMINFO.get(dev)
    if hit is not None and now - hit[0] <= ttl:
        _t, free_q, total, reserved_q = hit
        return max(0, free_q - (reserved - reserved_q)), total
    free = ctypes.c_size_t(0)
    total = ctypes.c_size_t(0)
    _lib.call("glint_device_info", int(dev), None, None, None,
              ctypes.addressof(free), ctypes.addressof(total))
    _MEMINFO[dev] = (now, int(free.value), int(total.value), reserved)
    return int(free.value), int(total.value)


@dataclass(frozen=True)
class BatchFootprint:
    graph_slice_bytes: int
    input_bytes: int
    intermediate_bytes: int
    output_bytes: int

    @property
    def peak(self) -> int:
        return (self.graph_slice_bytes + self.input_bytes
                + self.intermediate_bytes + self.output_bytes)

    @property
    def transfer_bytes(self) -> int:
        """Bytes that would cross host<->device; intermediates stay on device."""
        return self.graph_slice_bytes + self.input_bytes + self.output_bytes


ZERO_FOOTPRINT = BatchFootprint(0, 0, 0, 0)


def footprint_counts(block, n_targets, n_inputs, n_edges, dims) -> BatchFootprint:
    """Footprint from the three batch counts (no BatchCsc needed)."""
    if n_targets == 0:
        return ZERO_FOOTPRINT
    slice_bytes = (n_targets + 1 + n_edges) * ID_BYTES if block.has_conv else 0
    input_bytes = 0
    for key in block.input_keys():
        input_bytes += n_inputs * dims[key] * VALUE_BYTES
    inter = 0
    for op_id, kind, domain in block.iter_ops():
        if kind in ("Input", "Output"):
            continue
        inter += (n_inputs if domain == "input" else n_targets) * dims[op_id] * VALUE_BYTES
    out_bytes = 0
    for op_id in block.output_ids():
        out_bytes += n_targets * dims[op_id] * VALUE_BYTES
    return BatchFootprint(slice_bytes, input_bytes, inter, out_bytes)


def footprint(block, bc, dims) -> BatchFootprint:
    """glint/device.py:61-81 signature: footprint of `block` on BatchCsc `bc`."""
    return footprint_counts(block, bc.num_targets, bc.num_inputs, bc.num_edges, dims)


def admit(fp: BatchFootprint, budget: DeviceBudget) -> bool:
    """A batch whose peak equals the capacity is still admitted."""
    return fp.peak <= budget.capacity


def meter_transfer(fp: BatchFootprint) -> int:
    return fp.transfer_bytes
