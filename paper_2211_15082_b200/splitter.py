"""Split a model DAG into per-layer ConvBlocks (behaviour of glint/splitter.py).

The schedule decides which tensors are stored between layers and therefore
which HBM-resident stores the B200 executor allocates; it must match the
reference exactly (golden strings, tests/golden).  Rules (glint/splitter.py:1-22):

* every Conv sits in the block of its layer counter;
* a normal operator may move between the highest Conv-ancestor layer (>= 1)
  and the lowest Conv-descendant layer; with no Conv descendant (and the
  Output marker) it joins the last block;
* among edge-monotone placements pick the lexicographic minimum of
  (stored-input counts of blocks 2..L, -#ops at or above each boundary,
  sorted ids below each boundary), enumerating placements in
  itertools.product order so ties resolve identically;
* operators feeding a Conv of their own block are input-domain.

Planning runs once per model on the host (microseconds to milliseconds).
"""

from __future__ import annotations

import itertools
import logging
from dataclasses import dataclass, field

from .errors import InternalError
from .model_ir import ModelGraph

log = logging.getLogger(__name__)

INPUT_REF = "input"
MAX_ASSIGNMENTS = 2_000_000


@dataclass(frozen=True)
class TensorRef:
    block: int
    op: str

    @property
    def key(self) -> str:
        return INPUT_REF if self.block == 0 else f"b{self.block}.{self.op}"


@dataclass
class ConvBlock:
    block_id: int
    layer: int
    op_ids: list
    kinds: dict
    domains: dict
    input_refs: list
    outputs: list

    @property
    def has_conv(self) -> bool:
        return any(k in ("ConvMean", "ConvAttn") for k in self.kinds.values())

    def iter_ops(self):
        for op_id in self.op_ids:
            yield op_id, self.kinds[op_id], self.domains[op_id]

    def input_keys(self):
        return [r.key for r in self.input_refs]

    def output_ids(self):
        return list(self.outputs)


@dataclass
class BlockSchedule:
    blocks: list
    schema: dict
    drop_after: dict
    model_output: TensorRef
    depth: int
    assignment: dict = field(default_factory=dict)

    def block_input_counts(self) -> dict:
        return {b.block_id: len(b.input_refs) for b in self.blocks}


def _conv_bounds(m: ModelGraph):
    """(highest Conv-ancestor layer or 0, lowest Conv-descendant layer or None)."""
    above = {}
    for op_id in m.topo_order:
        best = 0
        for p in m.operators[op_id].inputs:
            best = max(best, m.layer_of[p] if m.operators[p].is_conv else above[p])
        above[op_id] = best
    below = {}
    users = m.consumers()
    for op_id in reversed(m.topo_order):
        lows = [m.layer_of[c] if m.operators[c].is_conv else below[c] for c in users[op_id]]
        lows = [x for x in lows if x is not None]
        below[op_id] = min(lows) if lows else None
    return above, below


def feasible_blocks(m: ModelGraph) -> dict:
    above, below = _conv_bounds(m)
    out = {}
    for op_id in m.topo_order:
        op = m.operators[op_id]
        if op.kind == "Input":
            continue
        if op.is_conv:
            out[op_id] = (m.layer_of[op_id],) * 2
        elif m.depth == 0:
            out[op_id] = (0, 0)
        elif op.kind == "Output" or below[op_id] is None:
            out[op_id] = (m.depth, m.depth)
        else:
            out[op_id] = (max(1, above[op_id]), below[op_id])
    return out


def _home(m, assignment, op_id):
    return 0 if m.operators[op_id].kind == "Input" else assignment[op_id]


def _reads(m: ModelGraph, assignment) -> dict:
    """block -> set of (producer block, producer key) read from outside the block."""
    reads = {b: set() for b in set(assignment.values())}
    for op_id, b in assignment.items():
        for p in m.operators[op_id].inputs:
            pb = _home(m, assignment, p)
            if pb != b:
                reads[b].add((pb, p if pb else INPUT_REF))
    return reads


def _score(m: ModelGraph, assignment, movable):
    reads = _reads(m, assignment)
    counts = tuple(len(reads.get(b, ())) for b in range(2, m.depth + 1))
    above, beneath = [], []
    for cut in range(1, m.depth):
        above.append(-sum(1 for o in movable if assignment[o] <= cut))
        beneath.append(tuple(sorted(o for o in movable if assignment[o] > cut)))
    return counts, tuple(above), tuple(beneath)


def _placements(m: ModelGraph, ranges, movable):
    pinned = {o: lo for o, (lo, hi) in ranges.items() if lo == hi}
    if not movable:
        yield dict(pinned)
        return
    choices = [range(ranges[o][0], ranges[o][1] + 1) for o in movable]
    size = 1
    for c in choices:
        size *= len(c)
        if size > MAX_ASSIGNMENTS:
            raise InternalError(f"cut search space exceeds {MAX_ASSIGNMENTS} assignments")
    producers = {o: [p for p in m.operators[o].inputs if m.operators[p].kind != "Input"]
                 for o in m.operators}
    users = m.consumers()
    for pick in itertools.product(*choices):
        a = dict(pinned)
        a.update(zip(movable, pick))
        if all(all(a[p] <= a[o] for p in producers[o])
               and all(a[c] >= a[o] for c in users[o] if c in a) for o in movable):
            yield a


def _best_placement(m: ModelGraph, ranges) -> dict:
    movable = sorted(o for o, (lo, hi) in ranges.items() if lo != hi)
    best, best_score = None, None
    for a in _placements(m, ranges, movable):
        s = _score(m, a, movable)
        if best_score is None or s < best_score:
            best, best_score = a, s
    if best is None:
        raise InternalError("no valid operator-to-block assignment found")
    return best


def _domains(m: ModelGraph, ops, kinds) -> dict:
    member = set(ops)
    users = m.consumers()
    feeds = set()
    for op_id in reversed([o for o in m.topo_order if o in member]):
        if kinds[op_id] in ("ConvMean", "ConvAttn"):
            continue
        if any(c in member and (kinds[c] in ("ConvMean", "ConvAttn") or c in feeds)
               for c in users[op_id]):
            feeds.add(op_id)
    return {o: ("input" if o in feeds else "target") for o in ops}


def split(m: ModelGraph) -> BlockSchedule:
    ranges = feasible_blocks(m)
    assignment = _best_placement(m, ranges)
    depth = m.depth
    if depth == 0:
        assignment = {o: 1 for o in assignment}
    block_ids = list(range(1, depth + 1)) if depth else [1]
    members = {b: [] for b in block_ids}
    for op_id in m.topo_order:
        if m.operators[op_id].kind != "Input":
            members[assignment[op_id]].append(op_id)
    users = m.consumers()
    reads = _reads(m, assignment)
    out_producer = m.operators[m.output_id].inputs[0]
    blocks = []
    for b in block_ids:
        ops = members[b]
        kinds = {o: m.operators[o].kind for o in ops}
        refs = sorted((TensorRef(pb, p) for pb, p in reads.get(b, ())), key=lambda r: r.key)
        stored = []
        for o in ops:
            if kinds[o] in ("Input", "Output"):
                continue
            later = any(_home(m, assignment, c) > b for c in users[o])
            if later or (o == out_producer and b == block_ids[-1]):
                stored.append(o)
            if not users[o]:
                log.warning("operator %r has no consumer; its output is dropped "
                            "immediately after block %d", o, b)
        blocks.append(ConvBlock(block_id=b, layer=b if depth else 0, op_ids=ops, kinds=kinds,
                                domains=_domains(m, ops, kinds), input_refs=refs,
                                outputs=stored))
    schema = {blk.block_id: list(blk.input_refs) for blk in blocks}
    return BlockSchedule(blocks=blocks, schema=schema, drop_after=plan_lifetimes(blocks, schema),
                         model_output=TensorRef(assignment[out_producer], out_producer),
                         depth=depth, assignment=assignment)


def plan_lifetimes(blocks, schema) -> dict:
    """Stored tensor key -> id of the last block that reads it (or its own block)."""
    last = {}
    for blk in blocks:
        for ref in schema[blk.block_id]:
            last[ref.key] = max(last.get(ref.key, blk.block_id), blk.block_id)
    for blk in blocks:
        for o in blk.outputs:
            last.setdefault(TensorRef(blk.block_id, o).key, blk.block_id)
    return last


def enumerate_cuts(m: ModelGraph, l) -> list:
    """Brute force of boundary l|l+1 (glint/splitter.py:290-331), for tests."""
    if not 1 <= l < max(m.depth, 1):
        raise ValueError(f"boundary {l} out of range for depth {m.depth}")
    ranges = feasible_blocks(m)
    movable = sorted(o for o, (lo, hi) in ranges.items() if lo <= l < hi)
    base = {o: lo for o, (lo, hi) in ranges.items()}
    producers = {o: [p for p in m.operators[o].inputs if m.operators[p].kind != "Input"]
                 for o in m.operators}
    found = []
    for k in range(len(movable) + 1):
        for down in itertools.combinations(movable, k):
            down_set = set(down)
            a = dict(base)
            for o in movable:
                a[o] = l + 1 if o in down_set else min(l, ranges[o][1])
            if any(a[p] > a[o] for o in m.operators if m.operators[o].kind != "Input"
                   for p in producers[o]):
                continue
            crossing = set()
            for o, b in a.items():
                if b == l + 1:
                    for p in m.operators[o].inputs:
                        pb = _home(m, a, p)
                        if pb != l + 1:
                            crossing.add((pb, p))
            found.append((tuple(sorted(down_set)), len(crossing), len(movable) - len(down_set)))
    return found


def format_schedule(schedule: BlockSchedule) -> str:
    head = (f"schedule blocks={len(schedule.blocks)} depth={schedule.depth} "
            f"output={schedule.model_output.key}")
    lines = [head]
    for blk in schedule.blocks:
        ops = ",".join(f"{o}:{blk.domains[o][0]}" for o in blk.op_ids)
        drops = ",".join(sorted(k for k, b in schedule.drop_after.items()
                                if b == blk.block_id and k not in (INPUT_REF,
                                                                   schedule.model_output.key)))
        lines.append(f"block {blk.block_id} layer={blk.layer} ops=[{ops}] "
                     f"inputs=[{','.join(blk.input_keys())}] outputs=[{','.join(blk.outputs)}] "
                     f"drop=[{drops}]")
    return "\n".join(lines)
