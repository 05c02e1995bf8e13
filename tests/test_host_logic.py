"""Host-side logic of the package against the reference's golden outputs (CPU only).

Covers the pieces that decide WHAT the device computes: model IR and its file
formats, the block splitter, node orders (native RCMK), neighbour sampling,
the batch controller and the seeded generators / model builders.
"""

import numpy as np
import pytest

from conftest import golden_graph
from paper_2211_15082_b200 import batching, model_ir, reorder, splitter, synth
from paper_2211_15082_b200.device import BatchFootprint, DeviceBudget, footprint_counts
from paper_2211_15082_b200.errors import ConfigError, DeviceCapacityError, FormatError
from paper_2211_15082_b200.executor import RunStats, parse_stats, sample_neighbors, skip_fires


def golden_models():
    """The exact models tests/golden/make_golden.py handed to the reference."""
    return {
        "gcn2": synth.build_gcn(8, 16, 4, 2, seed=2),
        "gcn3": synth.build_gcn(8, 12, 5, 3, seed=3),
        "gat2": synth.build_gat(8, 6, 3, 2, heads=2, seed=4),
        "gat3h4": synth.build_gat(8, 4, 3, 3, heads=4, seed=5),
        "jknet3": synth.build_jknet(8, 6, 4, 3, seed=6),
        "residual": synth.build_residual(8, 8, seed=7),
        "linear": synth.build_linear(8, 3, seed=8),
        "appnp": synth.build_appnp(8, 10, 4, k=3, alpha=0.1, seed=9),
    }


def _doc_model(entry):
    tensors = {k: np.asarray(v, dtype=np.float32) for k, v in entry["tensors"].items()}
    return model_ir.model_from_document(entry["doc"], tensors)


# -- splitter ------------------------------------------------------------------


def test_schedules_match_reference(golden):
    _, meta = golden
    ms = golden_models()
    for name, want in meta["schedules"].items():
        if isinstance(want, str):
            got = splitter.format_schedule(splitter.split(ms[name]))
            assert got == want, name
        else:
            got = splitter.format_schedule(splitter.split(_doc_model(want)))
            assert got == want["text"], name


def test_jknet_lifetimes():
    s = splitter.split(synth.build_jknet(4, 4, 3, layers=3, seed=0))
    assert [len(s.schema[b]) for b in (1, 2, 3, 4)] == [1, 1, 1, 3]
    assert s.drop_after["b1.drop1"] == 4 and s.drop_after["b3.drop3"] == 4


def test_enumerate_cuts_matches_split_minimum(golden):
    _, meta = golden
    for name, entry in meta["schedules"].items():
        if not name.startswith("rand"):
            continue
        m = _doc_model(entry)
        s = splitter.split(m)
        for l in range(1, m.depth):
            best = min(c[1] for c in splitter.enumerate_cuts(m, l))
            assert len(s.schema[l + 1]) == best, (name, l)


# -- model IR ----------------------------------------------------------------------


def test_model_roundtrip(tmp_path):
    for m in golden_models().values():
        mp, pp = tmp_path / "m.json", tmp_path / "m.dgiw"
        model_ir.save_model(m, mp, pp)
        m2 = model_ir.parse_model(mp, pp)
        assert m2.topo_order == m.topo_order and m2.layer_of == m.layer_of
        assert m2.out_dims == m.out_dims
        for o in m.operators:
            for k, v in m.operators[o].params.items():
                assert m2.operators[o].params[k].tobytes() == v.tobytes()


def test_model_errors():
    ops = {"x": model_ir.Operator("x", "Input", ()),
           "a": model_ir.Operator("a", "ReLU", ("b",)),
           "b": model_ir.Operator("b", "ReLU", ("a",)),
           "out": model_ir.Operator("out", "Output", ("a",))}
    with pytest.raises(FormatError, match="cycle"):
        model_ir.build_model(ops, 2, "out")
    with pytest.raises(FormatError, match="dimension mismatch"):
        model_ir.build_model({"x": model_ir.Operator("x", "Input", ()),
                              "l": model_ir.Operator("l", "Linear", ("x",),
                                                     {"weight": np.zeros((2, 3), np.float32)}),
                              "out": model_ir.Operator("out", "Output", ("l",))}, 2, "out")


def test_jknet_depth_is_four():
    assert synth.build_jknet(4, 4, 3, 3).depth == 4


# -- orders --------------------------------------------------------------------------


def test_native_rcmk_and_orders_match_reference(golden):
    arrs, meta = golden
    for c in meta["orders"]:
        g = golden_graph(arrs, c["graph"])
        got = reorder.make_order(g, c["kind"], seed=5).perm
        assert np.array_equal(got, arrs[c["perm"]]), (c["graph"], c["kind"])


def _sym(n, edges):
    from paper_2211_15082_b200.storage import make_graph

    sl = {v: [] for v in range(n)}
    for u, v in edges:
        sl[u].append(v)
        sl[v].append(u)
    return make_graph(n, {v: sorted(s) for v, s in sl.items()})


def test_rcmk_known_answers():
    # reference test_reorder.py:21-31: path 0-2-1-3 -> [3,1,2,0]; no edges -> reversed ids
    assert reorder.rcmk(_sym(4, [(0, 2), (2, 1), (1, 3)])).perm.tolist() == [3, 1, 2, 0]
    from paper_2211_15082_b200.storage import make_graph

    assert reorder.rcmk(make_graph(5, {})).perm.tolist() == [4, 3, 2, 1, 0]


def test_degree_sort_toy(golden):
    arrs, _ = golden
    assert reorder.degree_sort(golden_graph(arrs, "toy")).perm.tolist() == [3, 4, 5, 0, 1, 2]


# -- sampling / annotation helpers ---------------------------------------------------


def test_sample_neighbors_matches_reference(golden):
    arrs, meta = golden
    for c in meta["sampling"]:
        g = golden_graph(arrs, c["graph"])
        s = sample_neighbors(g, np.arange(g.num_nodes), c["fanout"], c["seed"], c["layer"])
        assert np.array_equal(s.indptr, arrs[c["indptr"]])
        assert np.array_equal(s.indices, arrs[c["indices"]])


def test_skip_rule_integer_exact(golden):
    arrs, _ = golden
    g = golden_graph(arrs, "toy")
    assert skip_fires(6, g) and not skip_fires(5, g)


# -- batching ------------------------------------------------------------------------


@pytest.mark.parametrize("case", range(6))
def test_controller_matches_reference(golden, case):
    _, meta = golden
    c = meta["batching"][case]
    degs = np.asarray(c["degs"], dtype=np.int64)
    prefix = np.zeros(len(degs) + 1, dtype=np.int64)
    np.cumsum(degs, out=prefix[1:])
    ctl = batching.BatchController(batching.Thresholds(*c["init"]), DeviceBudget(c["cap"]))

    def plan_fn(s, e):
        edges = int(prefix[e] - prefix[s])
        return (s, e), BatchFootprint(0, 0, (e - s) * 13 + edges * 5 + (edges * edges) % 97, 0)

    got = []
    for layer in (1, 2):
        for r in ctl.run_layer(layer, np.arange(len(degs)), prefix, plan_fn, lambda p: None):
            got.append([r.layer, r.start, r.end, r.oom_retries, r.n_t, r.n_i, r.footprint.peak])
    assert got == c["records"]


def test_controller_unrecoverable_singleton():
    ctl = batching.BatchController(batching.Thresholds(4, 100), DeviceBudget(25))
    prefix = np.array([0, 20, 21, 22])
    with pytest.raises(DeviceCapacityError, match="node 0"):
        ctl.run_layer(1, np.arange(3), prefix,
                      lambda s, e: ((s, e), BatchFootprint(0, 0, (e - s) * 10 + 2 * int(prefix[e] - prefix[s]), 0)),
                      lambda p: None)


def test_controller_real_allocation_failure_halves_and_retries():
    """A DeviceAllocationError while an admitted batch executes is on_oom: the
    thresholds halve, the same cursor is re-planned, the retry is recorded."""
    from paper_2211_15082_b200.errors import DeviceAllocationError

    ctl = batching.BatchController(batching.Thresholds(8, 10 ** 6), DeviceBudget(10 ** 9))
    prefix = np.arange(33, dtype=np.int64)
    ran = []

    def execute(plan):
        s, e = plan
        if e - s > 2:                      # the device refuses anything above 2 rows
            raise DeviceAllocationError("cudaErrorMemoryAllocation")
        ran.append(plan)

    recs = ctl.run_layer(1, np.arange(32), prefix,
                         lambda s, e: ((s, e), BatchFootprint(0, 0, 1, 0)), execute)
    assert recs[0].start == 0 and recs[0].end == 2 and recs[0].oom_retries == 2
    assert [(r.start, r.end) for r in recs] == ran
    assert sum(r.n_targets for r in recs) == 32
    with pytest.raises(DeviceCapacityError):
        ctl2 = batching.BatchController(batching.Thresholds(1, 10), DeviceBudget(10 ** 9))
        ctl2.run_layer(1, np.arange(3), np.arange(4),
                       lambda s, e: ((s, e), BatchFootprint(0, 0, 1, 0)),
                       lambda p: (_ for _ in ()).throw(DeviceAllocationError("oom")))


def test_adapt_half_even_rounding():
    t = batching.adapt(batching.Thresholds(5, 5), 900, 1800)  # r = 0.5 -> round(2.5) = 2
    assert (t.n_t, t.n_i) == (2, 2)


def test_footprint_kat():
    # reference test_device.py:38-45: toy target A -> 1 target, 3 inputs, 2 edges,
    # width 1: slice 32 + inputs 12 + conv output 4 + stored output 4 = 52 B
    blk = splitter.split(synth.build_gcn(1, 1, 1, 1)).blocks[0]
    fp = footprint_counts(blk, 1, 3, 2, {"input": 1, "conv1": 1, "out": 1})
    assert fp.graph_slice_bytes == (1 + 1 + 2) * 8
    assert (fp.input_bytes, fp.intermediate_bytes, fp.output_bytes) == (12, 4, 4)
    assert fp.peak == 52
    assert footprint_counts(blk, 0, 0, 0, {"input": 1, "conv1": 1}).peak == 0


def test_budget_setpoint():
    assert DeviceBudget(1000).target == 900
    with pytest.raises(ValueError):
        DeviceBudget(1)


# -- synth ---------------------------------------------------------------------------


def test_generators_match_reference_bytes(golden):
    arrs, meta = golden
    mine = {"reg": synth.gen_regular(120, 7, seed=5), "pow": synth.gen_powerlaw(150, seed=6),
            "sbm": synth.gen_sbm(3, 20, 0.3, 0.05, seed=7), "path": synth.gen_path(9)}
    for c in meta["synth"]:
        g = mine[c["name"]]
        assert np.array_equal(g.indptr, arrs[c["indptr"]]), c["name"]
        assert np.array_equal(g.indices, arrs[c["indices"]]), c["name"]
    assert synth.gen_features(7, 5, seed=3).tobytes() == arrs["y/features"].tobytes()


def test_model_builders_match_reference_weights(golden):
    arrs, _ = golden
    mine = {"gcn": synth.build_gcn(5, 6, 3, 3, seed=2),
            "gat": synth.build_gat(5, 4, 3, 2, heads=3, seed=2),
            "jknet": synth.build_jknet(5, 4, 3, 3, seed=2),
            "residual": synth.build_residual(5, 6, seed=2),
            "linear": synth.build_linear(5, 2, seed=2)}
    for name, m in mine.items():
        for k, v in model_ir.model_tensors(m).items():
            assert v.tobytes() == arrs[f"y/model/{name}/{k}"].tobytes(), (name, k)


def test_stats_document_roundtrip():
    st = RunStats(executor="layerwise", mode="full", order="none", depth=2,
                  initial_thresholds=(1024, 32768))
    st._add_batch(1, 3, BatchFootprint(8, 4, 4, 4), batching.Thresholds(4, 9), 1)
    st._add_aggregations(1, 3)
    doc = parse_stats(st.document())
    assert doc["schema"] == "glint-stats-v1" and doc["batch.targets"] == "3"
    assert doc["thresholds.trajectory"] == "1:4:9" and doc["oom_retries"] == "1"


def test_run_inference_config_errors():
    from paper_2211_15082_b200.executor import run_inference

    g = synth.gen_regular(10, 2, 0)
    m = synth.build_gcn(3, 4, 2, 2)
    x = synth.gen_features(10, 3, 0)
    with pytest.raises(ConfigError):
        run_inference(m, g, x, mode="partial", budget=DeviceBudget(1 << 20))
    with pytest.raises(ConfigError):
        run_inference(m, g, x, mode="sampling", budget=DeviceBudget(1 << 20))
    with pytest.raises(ConfigError):
        run_inference(m, g, synth.gen_features(10, 4, 0), budget=DeviceBudget(1 << 20))
    with pytest.raises(ConfigError):
        run_inference(m, g, x, budget=None)
