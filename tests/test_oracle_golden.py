"""Pin the CPU oracle against golden vectors produced by the reference itself.

The oracle (oracle/glint_oracle.py) is the checker for every GPU parity test,
so it must reproduce the reference's bytes on the reference's own outputs.
"""

import numpy as np
import pytest

from conftest import golden_graph
from oracle import glint_oracle as orc


def _kcases(golden):
    arrs, meta = golden
    return [(arrs, c) for c in meta["kernels"]]


def test_build_batch_csc_and_agg_mean_bytes(golden):
    arrs, meta = golden
    for c in meta["kernels"]:
        g = golden_graph(arrs, c["graph"])
        bc = orc.build_batch_csc(g.indptr, g.indices, arrs[c["targets"]])
        for f in ("input_ids", "indptr", "local_srcs", "target_pos"):
            assert np.array_equal(getattr(bc, f), arrs[c[f]]), (c["targets"], f)
        x = arrs[c["x"]]
        out = orc.agg_mean(bc, x[bc.input_ids])
        assert out.tobytes() == arrs[c["agg_mean"]].tobytes(), c["targets"]


def test_agg_attn_bytes(golden):
    arrs, meta = golden
    n = 0
    for c in meta["kernels"]:
        if "agg_attn" not in c:
            continue
        g = golden_graph(arrs, c["graph"])
        bc = orc.build_batch_csc(g.indptr, g.indices, arrs[c["targets"]])
        out = orc.agg_attn(bc, arrs[c["x"]][bc.input_ids], arrs[c["attn_w"]], arrs[c["attn_a"]])
        assert out.tobytes() == arrs[c["agg_attn"]].tobytes()
        n += 1
    assert n > 0


def test_dense_and_elementwise_bytes(golden):
    arrs, meta = golden
    for c in meta["kernels"]:
        if "linear" not in c:
            continue
        x = arrs[c["x"]]
        assert orc.linear(x, arrs[c["lin_w"]], arrs[c["lin_b"]]).tobytes() == arrs[c["linear"]].tobytes()
        for kind in ("ReLU", "LeakyReLU", "Norm", "DropoutIdentity"):
            assert orc.elementwise(kind, [x]).tobytes() == arrs[c["ew_" + kind]].tobytes(), kind
        assert orc.elementwise("Add", [x, x * 0.5, -x]).tobytes() == arrs[c["ew_Add"]].tobytes()
        assert orc.concat([x, x[:, :1], 2 * x]).tobytes() == arrs[c["concat"]].tobytes()


def test_whole_graph_model_matches_reference_layerwise(golden):
    """eval_reference == layer-wise bytes in the reference (test_executor.py:109-118),
    so the oracle's whole-graph pass must equal every full/none golden output."""
    from paper_2211_15082_b200.model_ir import model_document, model_tensors  # noqa: F401
    from test_host_logic import golden_models

    arrs, meta = golden
    models = golden_models()
    n = 0
    for c in meta["e2e"]:
        if c["mode"] != "full" or c["order"] != "none":
            continue
        g = golden_graph(arrs, c["graph"])
        x = arrs[f"e/{c['graph']}/x"]
        out = orc.eval_model(orc.model_spec(models[c["model"]]), g.indptr, g.indices, x)
        assert out.tobytes() == arrs[c["output"]].tobytes(), c["name"]
        n += 1
    assert n >= 8


def test_rcmk_oracle_matches_reference(golden):
    arrs, meta = golden
    for c in meta["orders"]:
        if c["kind"] != "rcmk":
            continue
        g = golden_graph(arrs, c["graph"])
        assert np.array_equal(orc.rcmk(g.indptr, g.indices), arrs[c["perm"]]), c["graph"]


@pytest.mark.parametrize("case", range(6))
def test_batch_replay_matches_reference(golden, case):
    _, meta = golden
    c = meta["batching"][case]
    degs = np.asarray(c["degs"], dtype=np.int64)
    prefix = np.zeros(len(degs) + 1, dtype=np.int64)
    np.cumsum(degs, out=prefix[1:])

    def peak(s, e):
        edges = int(prefix[e] - prefix[s])
        return (e - s) * 13 + edges * 5 + (edges * edges) % 97

    nt, ni = c["init"]
    got = []
    for layer in (1, 2):
        recs, (nt, ni) = orc.replay_batches(prefix, c["cap"], nt, ni, peak)
        got += [[layer, s, e, r, a, b, p] for s, e, r, a, b, p in recs]
    assert got == c["records"]
