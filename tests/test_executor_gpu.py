"""End-to-end parity of run_inference on the GPU against the reference's own runs.

For every golden case (graphs x models x modes x orders x budgets, produced by
running the reference): the stats document -- batch membership, OOM retries,
threshold trajectory, footprints, transfer/input bytes, aggregation counts --
must be byte-identical, and the output embeddings within rel-L2 <= 1e-4.
"""

import numpy as np
import pytest

from conftest import golden_graph, rel_l2
from oracle import glint_oracle as orc

pytestmark = pytest.mark.gpu


def _run(case, arrs, models, **over):
    from paper_2211_15082_b200.batching import Thresholds
    from paper_2211_15082_b200.device import DeviceBudget
    from paper_2211_15082_b200.executor import run_inference

    g = golden_graph(arrs, case["graph"])
    x = arrs[f"e/{case['graph']}/x"]
    kw = dict(mode=case["mode"], order=case["order"], seed=case.get("seed", 13),
              budget=DeviceBudget(case["budget"]),
              thresholds=Thresholds(*case.get("thresholds", [64, 512])))
    if case["mode"] != "full":
        kw["targets"] = (arrs[f"e/{case['graph']}/partial"] if case["graph"] != "toy"
                         else np.array([3, 0]))
    if case["mode"] == "sampling":
        kw["fanout"] = case["fanout"]
    kw.update(over)
    return run_inference(models[case["model"]], g, x, **kw)


def test_all_golden_cases(golden, cuda):
    from test_host_logic import golden_models

    arrs, meta = golden
    models = golden_models()
    worst = 0.0
    for case in meta["e2e"]:
        res = _run(case, arrs, models)
        assert res.stats.document() == case["stats"], case["name"]
        err = rel_l2(res.output, arrs[case["output"]])
        worst = max(worst, err)
        assert err <= 1e-4, (case["name"], err)
    print(f"worst rel-L2 over {len(meta['e2e'])} cases: {worst:.2e}")


def test_nodewise_equals_layerwise_bytes(golden, cuda):
    """Both engines share kernels; batch invariance makes them bit-identical
    (reference test_executor.py:109-180), with the drop-in API's default
    settings (reassociation is opt-in: it is a different, equally
    row-invariant, fp32 evaluation order)."""
    from test_host_logic import golden_models

    arrs, meta = golden
    models = golden_models()
    done = 0
    for case in meta["e2e"]:
        if case["graph"] not in ("toy", "reg200") or case["budget"] != 1 << 30:
            continue
        lw = _run(case, arrs, models)
        nw = _run(case, arrs, models, executor="nodewise", batch_size=7)
        assert lw.output.tobytes() == nw.output.tobytes(), case["name"]
        done += 1
    assert done >= 8


def test_outputs_invariant_to_batching_and_order(golden, cuda):
    from paper_2211_15082_b200.batching import Thresholds
    from paper_2211_15082_b200.device import DeviceBudget
    from paper_2211_15082_b200.executor import run_inference
    from paper_2211_15082_b200.synth import build_gcn, build_jknet

    arrs, _ = golden
    g = golden_graph(arrs, "pow300")
    x = arrs["e/pow300/x"]
    for m in (build_gcn(8, 16, 4, 3, seed=1), build_jknet(8, 6, 4, 3, seed=2)):
        base = run_inference(m, g, x, budget=DeviceBudget(1 << 30)).output
        for th in (Thresholds(1, 10 ** 6), Thresholds(7, 40), Thresholds(1000, 10 ** 6)):
            for order in ("none", "rcmk", "degree", "random"):
                out = run_inference(m, g, x, budget=DeviceBudget(1 << 30), thresholds=th,
                                    order=order, seed=3).output
                assert out.tobytes() == base.tobytes(), (th, order)


def test_whole_layer_runs_equal_controller_batches(cuda, monkeypatch):
    """A full-mode conv layer the budget admits as one batch runs as one launch;
    the bytes and the stats document (the controller's bootstrap batches) must
    equal the batch-by-batch execution, for every conv kind, with hub rows."""
    import torch

    from paper_2211_15082_b200 import synth
    from paper_2211_15082_b200.batching import Thresholds
    from paper_2211_15082_b200.device import DeviceBudget
    from paper_2211_15082_b200.executor import run_inference

    n = 40_000
    g = synth.gen_products_like(n, n * 25, seed=5, device="cuda")
    assert int(g.in_degrees.max()) + 1 >= 512          # hub rows present
    x = synth.gen_features_device(n, 24, seed=5, device="cuda")
    models = [synth.build_gcn(24, 64, 7, 3, seed=1),
              synth.build_gat(24, 16, 7, 2, heads=4, seed=2),
              synth.build_jknet(24, 32, 7, 3, seed=3),
              synth.build_appnp(24, 32, 7, k=3, alpha=0.1, seed=4)]
    for m in models:
        outs, docs = [], []
        for whole in ("1", "0"):
            monkeypatch.setenv("GLINT_WHOLE_LAYER", whole)
            res = run_inference(m, g, x, budget=DeviceBudget(8 << 30),
                                thresholds=Thresholds(512, 4096), output="device")
            outs.append(res.output.clone())
            docs.append(res.stats.document())
            assert res.stats.batches > m.depth           # the controller did bootstrap
        assert torch.equal(outs[0], outs[1]), m
        assert docs[0] == docs[1]


def test_planning_counts_memoized_per_graph(cuda, monkeypatch):
    """Full-mode batch counts are a pure function of the graph and the range:
    a second run on the same DeviceGraph plans the same batches (identical
    stats document and bytes) without any counting kernel."""
    import torch

    from paper_2211_15082_b200 import kernels, synth
    from paper_2211_15082_b200.batching import Thresholds
    from paper_2211_15082_b200.device import DeviceBudget
    from paper_2211_15082_b200.executor import run_inference

    n = 40_000
    g = synth.gen_products_like(n, n * 25, seed=6, device="cuda")
    x = synth.gen_features_device(n, 24, seed=6, device="cuda")
    m = synth.build_gcn(24, 64, 7, 3, seed=1)
    calls = [0]
    orig = kernels.IdSet.finalize

    def counting(self, *a, **k):
        calls[0] += 1
        return orig(self, *a, **k)

    monkeypatch.setattr(kernels.IdSet, "finalize", counting)
    runs = []
    for _ in range(2):
        before = calls[0]
        res = run_inference(m, g, x, budget=DeviceBudget(8 << 30),
                            thresholds=Thresholds(512, 4096), output="device")
        runs.append((res.output.clone(), res.stats.document(), calls[0] - before))
    assert runs[0][2] > 0 and runs[1][2] == 0, [r[2] for r in runs]
    assert torch.equal(runs[0][0], runs[1][0]) and runs[0][1] == runs[1][1]
    # another graph object with the same content counts again and agrees
    g2 = synth.gen_products_like(n, n * 25, seed=6, device="cuda")
    before = calls[0]
    res = run_inference(m, g2, x, budget=DeviceBudget(8 << 30),
                        thresholds=Thresholds(512, 4096), output="device")
    assert calls[0] > before and res.stats.document() == runs[0][1]


def test_real_allocations_stay_within_the_budget(cuda):
    """The batch controller's capacity bounds the real per-batch allocations:
    peak device memory during a run, minus the resident bytes the budget does
    not cover (stores and a transform-first conv's transformed rows,
    executor._resident_bytes), stays under the capacity (the reference's
    footprint model is an upper bound of what the engine allocates per batch)."""
    import torch

    from paper_2211_15082_b200 import synth
    from paper_2211_15082_b200.batching import Thresholds
    from paper_2211_15082_b200.device import DeviceBudget
    from paper_2211_15082_b200.executor import _resident_bytes, annotate, run_inference
    from paper_2211_15082_b200.splitter import split

    n = 40_000
    g = synth.gen_products_like(n, n * 25, seed=7, device="cuda")
    x = synth.gen_features_device(n, 24, seed=7, device="cuda")
    for m in (synth.build_gcn(24, 64, 7, 3, seed=1), synth.build_gat(24, 16, 7, 2, heads=4, seed=2)):
        cap = 6 << 20
        resident = _resident_bytes(m, split(m), annotate(g, np.arange(0), m.depth, "full"), g)
        run_inference(m, g, x, budget=DeviceBudget(cap), thresholds=Thresholds(512, 4096),
                      output="device")                       # warm caches (schedules, id sets)
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
        base = torch.cuda.memory_allocated()
        torch.cuda.reset_peak_memory_stats()
        res = run_inference(m, g, x, budget=DeviceBudget(cap), thresholds=Thresholds(512, 4096),
                            output="device")
        torch.cuda.synchronize()
        peak = torch.cuda.max_memory_allocated() - base
        assert res.stats.batches > m.depth                    # really batched
        assert peak - resident <= cap, (m.depth, peak, resident, cap)


def test_reassociation_and_precision_agree(golden, cuda):
    """Transform-then-aggregate (narrowing ConvMean) and both GEMM precisions
    agree with the aggregate-first fp32 path within 1e-5 (bar 1e-4)."""
    from paper_2211_15082_b200 import _lib
    from paper_2211_15082_b200.device import DeviceBudget
    from paper_2211_15082_b200.executor import run_inference
    from paper_2211_15082_b200.synth import build_gcn, build_jknet

    arrs, _ = golden
    g = golden_graph(arrs, "pow300")
    x = arrs["e/pow300/x"]
    for m in (build_gcn(8, 16, 4, 3, seed=11), build_jknet(8, 6, 4, 3, seed=12)):
        want = orc.eval_model(orc.model_spec(m), g.indptr, g.indices, x)
        base = run_inference(m, g, x, budget=DeviceBudget(1 << 30), reassociate=False,
                             precision=_lib.PREC_FP32).output
        for reassoc in (False, True):
            for prec in (_lib.PREC_FP32, _lib.PREC_3XTF32):
                out = run_inference(m, g, x, budget=DeviceBudget(1 << 30), reassociate=reassoc,
                                    precision=prec).output
                assert rel_l2(out, base) <= 1e-5, (reassoc, prec)
                assert rel_l2(out, want) <= 1e-5, (reassoc, prec)


def test_device_budget_and_device_output(golden, cuda):
    import torch

    from paper_2211_15082_b200.executor import run_inference
    from paper_2211_15082_b200.synth import build_gcn

    arrs, _ = golden
    g = golden_graph(arrs, "reg200")
    x = arrs["e/reg200/x"]
    m = build_gcn(8, 16, 4, 2, seed=5)
    res = run_inference(m, g, torch.from_numpy(x).cuda(), budget="device")
    assert isinstance(res.output, torch.Tensor) and res.output.is_cuda
    want = orc.eval_model(orc.model_spec(m), g.indptr, g.indices, x)
    assert rel_l2(res.output.cpu().numpy(), want) <= 1e-5
    assert res.budget.capacity > 1 << 30


def test_partial_outputs_in_listed_order(golden, cuda):
    """Reference test_executor.py:120-128."""
    from paper_2211_15082_b200.device import DeviceBudget
    from paper_2211_15082_b200.executor import run_inference
    from paper_2211_15082_b200.synth import build_gcn, gen_features

    arrs, _ = golden
    toy = golden_graph(arrs, "toy")
    m = build_gcn(3, 4, 2, layers=2, seed=2)
    x = gen_features(6, 3, seed=0)
    big = DeviceBudget(1 << 30)
    full = run_inference(m, toy, x, budget=big)
    part = run_inference(m, toy, x, mode="partial", targets=[3, 0], budget=big)
    assert part.output.shape == (2, 2)
    assert part.output[0].tobytes() == full.output[3].tobytes()
    assert part.output[1].tobytes() == full.output[0].tobytes()


def test_repetition_elimination_counts(golden, cuda):
    """Reference test_executor.py:183-196: node-wise 6 vs layer-wise 4 aggregations."""
    from paper_2211_15082_b200.device import DeviceBudget
    from paper_2211_15082_b200.executor import run_inference
    from paper_2211_15082_b200.synth import build_gcn, gen_features

    arrs, _ = golden
    toy = golden_graph(arrs, "toy")
    m = build_gcn(1, 2, 2, layers=2, seed=0)
    x = gen_features(6, 1, seed=0)
    big = DeviceBudget(1 << 30)
    nw = run_inference(m, toy, x, mode="partial", targets=[0, 1], executor="nodewise",
                       budget=big, batch_size=1)
    lw = run_inference(m, toy, x, mode="partial", targets=[0, 1], budget=big)
    assert nw.stats.layer_aggregations[1] == 6
    assert lw.stats.layer_aggregations[1] == 4


def test_nodewise_hard_oom(golden, cuda):
    from paper_2211_15082_b200.device import DeviceBudget
    from paper_2211_15082_b200.errors import DeviceCapacityError
    from paper_2211_15082_b200.executor import run_inference
    from paper_2211_15082_b200.synth import build_gcn, gen_features

    arrs, _ = golden
    toy = golden_graph(arrs, "toy")
    with pytest.raises(DeviceCapacityError):
        run_inference(build_gcn(3, 4, 2, 2, seed=2), toy, gen_features(6, 3, 0),
                      executor="nodewise", budget=DeviceBudget(64), batch_size=6)


@pytest.mark.gpu
def test_two_ranks_on_one_gpu_bit_identical(tmp_path):
    """The torchrun path (edge-balanced row ranges + per-layer exchange) gives the
    single-rank bytes for GCN (aggregate-first and reassociated) and GAT, one
    batch and many batches per layer, and on a star graph whose edge-balanced
    ranges leave ranks empty.  2 and 4 ranks share cuda:0 over gloo (NCCL
    refuses duplicate devices)."""
    import json
    import os
    import pathlib
    import subprocess
    import sys

    root = pathlib.Path(__file__).resolve().parents[1]
    env = dict(os.environ, GLINT_DIST_BACKEND="gloo")
    for world in (2, 4):
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node",
               str(world), "--master-addr", "127.0.0.1", "--master-port", str(29533 + world),
               str(root / "tools" / "dist_check.py"), "20000"]
        out = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600, cwd=root)
        assert out.returncode == 0, out.stderr[-2000:]
        lines = [json.loads(x) for x in out.stdout.splitlines() if x.startswith("{")]
        runs = [x for x in lines if "model" in x]
        assert len(runs) == 2 * (6 + 3), lines        # replicate and halo exchange
        assert {x["exchange"] for x in runs} == {"replicate", "halo"}
        assert all(x["bit_identical_all_ranks"] for x in runs), runs
        star = next(x for x in lines if "star_cuts" in x)
        assert star["empty_ranks"] >= (world > 2)      # a rank without rows took part


@pytest.mark.gpu
def test_exchange_nccl_calls_on_one_gpu():
    """The NCCL calls of the row exchange (grouped broadcasts through the
    coalescing manager, the halo all-to-all, direct tensor exchanges) run in a
    1-rank NCCL group inside the engine; outputs bit-identical to no exchange."""
    import json
    import os
    import pathlib
    import subprocess
    import sys

    root = pathlib.Path(__file__).resolve().parents[1]
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT="29571")
    out = subprocess.run([sys.executable, str(root / "tools" / "nccl_single_check.py"), "20000"],
                         env=env, capture_output=True, text=True, timeout=600, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(x) for x in out.stdout.splitlines() if x.startswith("{")]
    runs = [x for x in lines if "model" in x]
    assert len(runs) == 4 and all(x["bit_identical"] and x["backend"] == "nccl" for x in runs)
    assert any("direct_exchanges" in x for x in lines)


@pytest.mark.gpu
def test_bench_json_contract():
    """bench.py (small graph) prints one JSON line carrying every key the driver
    reads, for both arms."""
    import json
    import pathlib
    import subprocess
    import sys

    root = pathlib.Path(__file__).resolve().parents[1]
    configs = []
    for extra in ([], ["--impl", "reference"]):
        out = subprocess.run([sys.executable, str(root / "bench.py"), "--nodes", "20000",
                              "--steps", "2", "--warmup", "3", "--cpu-sample", "256"] + extra,
                             capture_output=True, text=True, timeout=600, cwd=root)
        assert out.returncode == 0, out.stderr[-2000:]
        lines = [x for x in out.stdout.splitlines() if x.startswith("{")]
        assert len(lines) == 1
        d = json.loads(lines[0])
        for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                  "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
                  "cpu_baseline", "e2e"):
            assert k in d, k
        assert d["value"] > 0 and "workload" in d["config"]
        configs.append((d["config"], d["metric"], d["unit"], d["data"]))
        if extra:
            assert d["impl"] == "reference" and d["e2e"]["h2d_bytes_per_step"] == 0
        else:
            for k in ("roofline", "gpu_launches", "clocks"):
                assert k in d, k
            r = d["roofline"]
            for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
                assert k in r, k
            assert d["gpu_launches"] > 0
            for k in ("value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"):
                assert k in d["e2e"], k
            for k in ("value", "unit", "cores", "kind", "sample"):
                assert k in d["cpu_baseline"], k
            p = d["parity"]
            assert p["pass"] and p["k1_bytes_equal"] and p["records_equal"], p
            assert d["secondary"]["cfg3"]["parity"]["pass"]
    assert configs[0] == configs[1]         # the driver's same_config
