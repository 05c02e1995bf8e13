"""BASELINE.json configs[0] ("cfg1") run exactly, against the reference.

cfg1 = gen_regular(100_000, 20, seed=0), 128-d gen_features(seed=0),
build_gcn(128, 128, 128, 2, seed=0), full inference, layer-wise, default
thresholds (1024, 32768).  tests/golden/make_cfg1.py ran the REFERENCE on it
(order none and rcmk at 16 GiB, none at 256 MiB) and recorded the stats
documents, the RCMK permutation hash and sampled output rows.

Pass bars:
* stats document byte-identical (batch membership: layer 1 = 1024, 4096,
  16384, 65536, 12960 targets; footprints; transfer bytes; thresholds);
* the RCMK permutation identical (sha256);
* every output row within rel-L2 1e-4 of the oracle's whole-graph evaluation
  (3xTF32 GEMM) and the reference's sampled rows;
* the layer-1 and layer-2 aggregates byte-identical to agg_mean: a model
  whose convs are W = I with the fp32 GEMM outputs exactly the aggregate.
"""

import hashlib
import json

import numpy as np
import pytest

from conftest import GOLDEN, rel_l2

pytestmark = pytest.mark.gpu

N, DEG, DIM = 100_000, 20, 128


@pytest.fixture(scope="module")
def cfg1():
    from paper_2211_15082_b200.synth import build_gcn, gen_features, gen_regular

    gold = json.loads((GOLDEN / "cfg1.json").read_text())
    g = gen_regular(N, DEG, seed=0)
    assert hashlib.sha256(np.ascontiguousarray(g.indices, "<i8").tobytes()).hexdigest() \
        == gold["graph"]["indices_sha256"]
    x = gen_features(N, DIM, seed=0)
    m = build_gcn(DIM, DIM, DIM, 2, seed=0)
    return gold, g, x, m


@pytest.fixture(scope="module")
def oracle_out(cfg1):
    from oracle import glint_oracle as orc

    _, g, x, m = cfg1
    return orc.eval_model(orc.model_spec(m), g.indptr, g.indices, x)


@pytest.mark.parametrize("run", [0, 1, 2], ids=["none-16GiB", "rcmk-16GiB", "none-256MiB"])
def test_cfg1_matches_reference(cuda, cfg1, oracle_out, run):
    from paper_2211_15082_b200.batching import Thresholds
    from paper_2211_15082_b200.device import DeviceBudget
    from paper_2211_15082_b200.executor import run_inference

    gold, g, x, m = cfg1
    want = gold["runs"][run]
    res = run_inference(m, g, x, mode="full", order=want["order"],
                        budget=DeviceBudget(want["capacity"]), thresholds=Thresholds(1024, 32768))
    assert res.stats.document() == want["stats"]
    if want["capacity"] == 16 << 30:        # SURVEY P2's batch sequence
        assert res.stats.batch_sizes == [1024, 4096, 16384, 65536, 12960, 100000]
    if want["order"] == "rcmk":
        assert hashlib.sha256(np.ascontiguousarray(res.order.perm, "<i8").tobytes()).hexdigest() \
            == want["perm_sha256"]
    out = np.asarray(res.output)
    assert out.shape == (N, DIM)
    assert rel_l2(out, oracle_out) <= 1e-4
    rows = np.asarray(gold["rows"])
    ref_rows = np.frombuffer(bytes.fromhex(want["out_rows_hex"]), "<f4").reshape(len(rows), DIM)
    assert rel_l2(out[rows], ref_rows) <= 1e-4


@pytest.mark.parametrize("whole_layer", ["1", "0"])
def test_cfg1_aggregates_byte_exact(cuda, cfg1, monkeypatch, whole_layer):
    """Identity convs + fp32 GEMM: the output IS agg_mean(agg_mean(x)), byte for byte,
    through run_inference (whole-layer launch, or batch by batch)."""
    from oracle import glint_oracle as orc
    from paper_2211_15082_b200 import _lib
    from paper_2211_15082_b200.batching import Thresholds
    from paper_2211_15082_b200.device import DeviceBudget
    from paper_2211_15082_b200.executor import run_inference
    from paper_2211_15082_b200.model_ir import Operator, build_model

    monkeypatch.setenv("GLINT_WHOLE_LAYER", whole_layer)
    gold, g, x, _ = cfg1
    eye = np.eye(DIM, dtype=np.float32)
    ops = {"x": Operator("x", "Input", ()),
           "c1": Operator("c1", "ConvMean", ("x",), {"weight": eye, "bias": np.zeros(DIM, np.float32)}),
           "c2": Operator("c2", "ConvMean", ("c1",), {"weight": eye, "bias": np.zeros(DIM, np.float32)}),
           "out": Operator("out", "Output", ("c2",))}
    m = build_model(ops, DIM, "out")
    res = run_inference(m, g, x, budget=DeviceBudget(16 << 30), thresholds=Thresholds(1024, 32768),
                        precision=_lib.PREC_FP32)
    bc = orc.build_batch_csc(g.indptr, g.indices, np.arange(N))
    a1 = orc.agg_mean(bc, x)
    a2 = orc.agg_mean(bc, a1)
    assert np.asarray(res.output).tobytes() == a2.tobytes()
    assert res.stats.layer_batches[1] > 1       # bootstrap batches were planned
