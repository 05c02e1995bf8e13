"""Golden fixture for BASELINE.json configs[0] ("cfg1"), made by running the REFERENCE.

    python tests/golden/make_cfg1.py          (needs /root/reference; ~1 min)

cfg1: gen_regular(100_000, 20, seed=0), gen_features(100_000, 128, seed=0),
build_gcn(128, 128, 128, 2, seed=0) (GraphSAGE-mean / GCN stand-in), full
inference, layer-wise executor, default thresholds (1024, 32768).  Runs:
order none and rcmk at a 16 GiB capacity, and order none at 256 MiB.

Writes tests/golden/cfg1.json: each run's stats document (glint-stats-v1), the
sha256 of the RCMK permutation, and 96 sampled output rows per run (the
reference's own output, float32 hex) with their row ids.  The GPU test
(tests/test_cfg1_gpu.py) compares the B200 run with these and with the oracle
over every row.  /root/reference is read here only, never on the GPU box.
"""

from __future__ import annotations

import hashlib
import json
import pathlib
import sys
import time

import numpy as np

HERE = pathlib.Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(ROOT))

from glint import batching as r_batching  # noqa: E402
from glint import executor as r_exec  # noqa: E402
from glint import model_ir as r_ir  # noqa: E402
from glint import reorder as r_reorder  # noqa: E402
from glint import storage as r_storage  # noqa: E402
from glint import synth as r_synth  # noqa: E402
from glint.device import DeviceBudget as RBudget  # noqa: E402

from paper_2211_15082_b200 import model_ir as my_ir  # noqa: E402
from paper_2211_15082_b200 import synth as my_synth  # noqa: E402

N, DEG, DIM = 100_000, 20, 128
RUNS = [("none", 16 << 30), ("rcmk", 16 << 30), ("none", 256 << 20)]


def main():
    g = r_synth.gen_regular(N, DEG, seed=0)
    x = r_synth.gen_features(N, DIM, seed=0)
    xs = r_storage.open_store(N, DIM)
    xs.scatter(np.arange(N), x)
    m = my_synth.build_gcn(DIM, DIM, DIM, 2, seed=0)
    rm = r_ir.model_from_document(my_ir.model_document(m), my_ir.model_tensors(m))
    rows = np.sort(np.random.default_rng(5).choice(N, size=96, replace=False))
    out = {"graph": {"kind": "regular", "n": N, "d": DEG, "seed": 0,
                     "indices_sha256": hashlib.sha256(
                         np.ascontiguousarray(g.indices, "<i8").tobytes()).hexdigest()},
           "features": {"dim": DIM, "seed": 0}, "model": "build_gcn(128,128,128,2,seed=0)",
           "thresholds": [1024, 32768], "rows": rows.tolist(), "runs": []}
    for order, cap in RUNS:
        t0 = time.perf_counter()
        res = r_exec.run_inference(rm, g, xs, mode="full", order=order, budget=RBudget(cap),
                                   executor="layerwise",
                                   thresholds=r_batching.Thresholds(1024, 32768))
        secs = time.perf_counter() - t0
        rec = {"order": order, "capacity": cap, "stats": res.stats.document(),
               "seconds": round(secs, 2),
               "out_rows_hex": np.ascontiguousarray(res.output[rows], "<f4").tobytes().hex()}
        if order == "rcmk":
            perm = r_reorder.rcmk(g).perm
            rec["perm_sha256"] = hashlib.sha256(np.ascontiguousarray(perm, "<i8").tobytes()).hexdigest()
        out["runs"].append(rec)
        print(order, cap, f"{secs:.1f}s", res.stats.document().count("\n"), "stats lines",
              flush=True)
    (HERE / "cfg1.json").write_text(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    main()
