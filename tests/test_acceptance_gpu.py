"""The reference's acceptance properties and dispatch KATs, on the device path.

* C1 (reference test_acceptance.py:63-101): layer-wise == node-wise output
  bytes across models x graphs x modes x orders x batch regimes, with the
  drop-in API's default settings.
* C5 (test_acceptance.py:173-199): dynamic batch control -- every batch fits
  the capacity, steady-state batches reach 70% of the setpoint, a too-small
  bootstrap recovers by halving, output byte-equal to node-wise.
* C6 (test_acceptance.py:202-220): RCMK moves >= 10% fewer transfer bytes than
  the mean of random orders on the community-structured SBM graph.
* a9 dispatch (model_ir.py:334-372; test_model_ir.py:164-195): eval_conv /
  eval_normal / eval_reference on the device, against the reference KATs and
  golden whole-graph outputs; eval_reference == layer-wise bytes.
* f2 annotation (executor.py:129-164): the device annotate() target sets equal
  the reference's golden sets.
"""

import zlib

import numpy as np
import pytest

from conftest import golden_graph, rel_l2

pytestmark = pytest.mark.gpu

BIG = 1 << 30


def _budget(cap=BIG):
    from paper_2211_15082_b200.device import DeviceBudget

    return DeviceBudget(cap)


def test_c1_layerwise_equals_nodewise_matrix(cuda):
    from paper_2211_15082_b200.batching import Thresholds
    from paper_2211_15082_b200.executor import run_inference
    from paper_2211_15082_b200.synth import (build_gat, build_gcn, build_jknet, build_residual,
                                             gen_features, gen_path, gen_powerlaw, gen_regular,
                                             gen_sbm)

    graphs = {"path": gen_path(64), "regular1k": gen_regular(1000, 4, seed=3),
              "powerlaw2k": gen_powerlaw(2000, seed=4), "sbm1k": gen_sbm(20, 50, 0.1, 0.002, seed=5)}
    models = {"gcn2": build_gcn(4, 4, 3, layers=2, seed=1), "gcn3": build_gcn(4, 4, 3, layers=3, seed=2),
              "gat2": build_gat(4, 3, 2, layers=2, heads=2, seed=3),
              "jknet3": build_jknet(4, 4, 3, layers=3, seed=4), "residual": build_residual(4, 4, seed=5)}
    cells = 0
    for gname, g in graphs.items():
        n = g.num_nodes
        x = gen_features(n, 4, seed=9)
        rng = np.random.default_rng(zlib.crc32(gname.encode()))
        mode_cases = [("full", None, None),
                      ("partial", np.sort(rng.choice(n, size=max(1, n // 100), replace=False)), None),
                      ("partial", np.sort(rng.choice(n, size=max(1, n // 10), replace=False)), None),
                      ("sampling", None, 2), ("sampling", None, 10)]
        for mname, m in models.items():
            for mode, targets, fanout in mode_cases:
                nt = n if targets is None else len(targets)
                regimes = [(Thresholds(10 ** 6, 10 ** 9), nt),
                           (Thresholds(max(1, nt // 4), 10 ** 9), max(1, nt // 4)),
                           (Thresholds(max(1, nt // 16), 10 ** 9), max(1, nt // 16))]
                for order in ("none", "rcmk", "random"):
                    for th, bs in regimes:
                        common = dict(mode=mode, targets=targets, fanout=fanout, seed=17,
                                      order=order, budget=_budget())
                        lw = run_inference(m, g, x, executor="layerwise", thresholds=th, **common)
                        nw = run_inference(m, g, x, executor="nodewise", batch_size=bs, **common)
                        assert lw.output.tobytes() == nw.output.tobytes(), \
                            (gname, mname, mode, fanout, order, bs)
                        cells += 1
    assert cells == 4 * 5 * 5 * 3 * 3


def test_c5_dynamic_batch_control(cuda):
    from paper_2211_15082_b200.batching import Thresholds
    from paper_2211_15082_b200.executor import run_inference
    from paper_2211_15082_b200.synth import build_gcn, gen_features, gen_regular

    g = gen_regular(5000, 8, seed=42)
    x = gen_features(5000, 4, seed=1)
    m = build_gcn(4, 4, 3, layers=2, seed=6)
    budget = _budget(60_000)
    lw = run_inference(m, g, x, executor="layerwise", budget=budget,
                       thresholds=Thresholds(1024, 32768))
    st = lw.stats
    assert 20 <= st.batches <= 60, st.batches
    assert st.oom_retries > 0
    assert max(st.batch_footprints) <= budget.capacity
    tail = {i for i in range(st.batches)
            if i + 1 == st.batches or st.batch_layers[i + 1] != st.batch_layers[i]}
    steady = [p for i, p in enumerate(st.batch_footprints) if i >= 5 and i not in tail]
    assert steady and all(p >= 0.7 * budget.target for p in steady)
    nw = run_inference(m, g, x, executor="nodewise", budget=_budget(), batch_size=512)
    assert lw.output.tobytes() == nw.output.tobytes()


def test_c6_rcmk_saves_transfer(cuda):
    from paper_2211_15082_b200.batching import Thresholds
    from paper_2211_15082_b200.executor import run_inference
    from paper_2211_15082_b200.synth import build_gcn, gen_features, gen_sbm

    g = gen_sbm(20, 50, 0.1, 0.002, seed=3)
    x = gen_features(1000, 16, seed=2)
    m = build_gcn(16, 16, 8, layers=2, seed=6)

    def transfer(order, seed=0):
        return run_inference(m, g, x, executor="layerwise", budget=_budget(100_000),
                             thresholds=Thresholds(64, 2048), order=order,
                             seed=seed).stats.total_transfer

    rc = transfer("rcmk")
    mean_rnd = sum(transfer("random", k) for k in range(5)) / 5
    assert rc <= 0.9 * mean_rnd, (rc, mean_rnd)


# -- a9: operator dispatch on the device ---------------------------------------------


def _toy():
    from paper_2211_15082_b200.storage import make_graph

    return make_graph(6, {0: [2, 3], 1: [2, 3], 2: [4, 5]})


def _identity_conv(op_id, inputs, dim):
    from paper_2211_15082_b200.model_ir import Operator

    return Operator(op_id, "ConvMean", inputs, {"weight": np.eye(dim, dtype=np.float32),
                                                "bias": np.zeros(dim, np.float32)})


def test_eval_reference_kats(cuda):
    """test_model_ir.py:164-195 on the device."""
    from paper_2211_15082_b200 import _lib, kernels
    from paper_2211_15082_b200.model_ir import Operator, build_model, eval_reference
    from paper_2211_15082_b200.synth import build_linear

    g = _toy()
    ops = {"x": Operator("x", "Input", ()), "conv": _identity_conv("conv", ("x",), 1),
           "out": Operator("out", "Output", ("conv",))}
    m = build_model(ops, 1, "out")
    prev = kernels.PRECISION
    kernels.PRECISION = _lib.PREC_FP32      # identity weights: the GEMM is exact in fp32
    try:
        x = np.ones((6, 1), np.float32)
        assert np.array_equal(eval_reference(m, g, x), x)           # constant fixed point
        x = np.zeros((6, 1), np.float32)
        x[2], x[3] = 2.0, 4.0
        out = eval_reference(m, g, x)
        assert out[0, 0] == np.float32((2 + 4 + 0) / 3)             # A = mean{C, D, A}
    finally:
        kernels.PRECISION = prev
    lm = build_linear(3, 2, seed=4)
    x = np.random.default_rng(0).normal(size=(6, 3)).astype(np.float32)
    w, b = lm.operators["lin"].params["weight"], lm.operators["lin"].params["bias"]
    assert rel_l2(eval_reference(lm, g, x), np.einsum("ij,kj->ik", x, w) + b) <= 1e-6


def test_eval_conv_and_normal_match_golden_kernels(golden, cuda):
    """eval_conv / eval_normal (model_ir.py:334-351) on the reference's kernel
    cases: ConvMean with W = I and the fp32 GEMM is exactly agg_mean's bytes;
    ConvAttn within 1e-5; Linear within 1e-5; elementwise / Concat bytes equal
    (Norm within 1e-6)."""
    from paper_2211_15082_b200 import kernels
    from paper_2211_15082_b200.model_ir import Operator, eval_conv, eval_normal

    def host(t):
        return t.cpu().numpy() if hasattr(t, "cpu") else np.asarray(t)

    arrs, meta = golden
    counts = {"mean": 0, "attn": 0, "normal": 0}
    prev = kernels.PRECISION
    for case in meta["kernels"]:
        g = golden_graph(arrs, case["graph"])
        x = arrs[case["x"]]
        d = x.shape[1]
        targets = arrs[case["targets"]]
        bc = kernels.build_batch_csc(g, targets)
        h = x[bc.input_ids.cpu().numpy() if hasattr(bc.input_ids, "cpu") else bc.input_ids]
        kernels.PRECISION = 0
        try:
            out = host(eval_conv(_identity_conv("c", ("x",), d), bc, h))
        finally:
            kernels.PRECISION = prev
        assert out.tobytes() == arrs[case["agg_mean"]].tobytes(), case["agg_mean"]
        counts["mean"] += 1
        if "agg_attn" in case:
            op = Operator("a", "ConvAttn", ("x",), {"weight": arrs[case["attn_w"]],
                                                   "attn": arrs[case["attn_a"]]})
            assert rel_l2(host(eval_conv(op, bc, h)), arrs[case["agg_attn"]]) <= 1e-5
            counts["attn"] += 1
        if "linear" in case:
            op = Operator("l", "Linear", ("x",), {"weight": arrs[case["lin_w"]],
                                                 "bias": arrs[case["lin_b"]]})
            assert rel_l2(host(eval_normal(op, [x])), arrs[case["linear"]]) <= 1e-5
            for kind in ("ReLU", "LeakyReLU", "DropoutIdentity", "Norm"):
                got = host(eval_normal(Operator("e", kind, ("x",)), [x]))
                want = arrs[case["ew_" + kind]]
                if kind == "Norm":
                    assert rel_l2(got, want) <= 1e-6
                else:
                    assert got.tobytes() == want.tobytes(), (kind, case["x"])
            got = host(eval_normal(Operator("s", "Add", ("x", "y", "z")), [x, x * 0.5, -x]))
            assert got.tobytes() == arrs[case["ew_Add"]].tobytes()
            got = host(eval_normal(Operator("c", "Concat", ("x", "y", "z")), [x, x[:, :1], 2 * x]))
            assert got.tobytes() == arrs[case["concat"]].tobytes()
            counts["normal"] += 1
    assert counts["mean"] >= 60 and counts["attn"] >= 8 and counts["normal"] >= 20, counts


def test_eval_reference_equals_layerwise_and_golden(golden, cuda):
    """C1's oracle side: whole-graph eval_reference == layer-wise bytes (same
    kernels, default settings), and within 1e-4 of the reference's output."""
    from test_host_logic import golden_models

    from paper_2211_15082_b200.executor import run_inference
    from paper_2211_15082_b200.model_ir import eval_reference

    arrs, meta = golden
    models = golden_models()
    done = 0
    for case in meta["e2e"]:
        if case["mode"] != "full" or case["order"] != "none" or case["budget"] != BIG \
                or "output" not in case:
            continue
        g = golden_graph(arrs, case["graph"])
        x = arrs[f"e/{case['graph']}/x"]
        m = models[case["model"]]
        ev = eval_reference(m, g, x)
        lw = run_inference(m, g, x, budget=_budget()).output
        assert ev.tobytes() == lw.tobytes(), case["name"]
        assert rel_l2(ev, arrs[case["output"]]) <= 1e-4, case["name"]
        done += 1
    assert done >= 8


def test_annotate_matches_reference_sets(golden, cuda):
    """Device frontier expansion == the reference's annotate() sets (golden)."""
    from paper_2211_15082_b200 import kernels
    from paper_2211_15082_b200.executor import annotate

    arrs, meta = golden
    assert meta["annotate"]
    for case in meta["annotate"]:
        g = golden_graph(arrs, case["graph"])
        for gg in (g, kernels.device_graph(g)):
            ts = annotate(gg, np.asarray(case["targets"]), case["depth"], "partial")
            assert ts.skip_from == case["skip_from"], case
            assert {str(k): np.asarray(v).tolist() for k, v in ts.v_sets.items()} == case["v"], case
