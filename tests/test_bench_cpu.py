"""CPU checks of the bench plumbing: the shared workload, the reference arm's
isolation from the product, and the oracle's plan-only replay helpers."""

import json
import pathlib
import subprocess
import sys

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parents[1]


def test_workload_graph_equals_synth_generator():
    """workload.products_like_csc (bench, both arms) == synth.gen_products_like."""
    import workload
    from paper_2211_15082_b200 import synth

    ip, ix = workload.products_like_csc(3000, 40000, seed=0, device="cpu")
    g = synth.gen_products_like(3000, 40000, seed=0, device="cpu")
    assert np.array_equal(ip.numpy(), g.indptr.numpy())
    assert np.array_equal(ix.numpy(), g.indices.numpy().astype(np.int64))
    assert int(ip[-1]) == 80000
    # symmetric, ascending slices, no self loops
    dst = np.repeat(np.arange(3000), np.diff(ip.numpy()))
    src = ix.numpy()
    assert not np.any(src == dst)
    fwd = set(zip(dst.tolist(), src.tolist()))
    assert all((s, d) in fwd for d, s in list(fwd)[:2000])
    x = workload.features(50, 7, seed=0, device="cpu")
    assert np.array_equal(x.numpy(), synth.gen_features_device(50, 7, 0, device="cpu").numpy())


def test_workload_weights_equal_model_builders():
    import workload
    from paper_2211_15082_b200 import synth

    m = synth.build_gcn(100, 256, 47, 3, seed=0)
    for i, (w, b) in enumerate(workload.gcn_params(100, 256, 47, 3, seed=0), start=1):
        assert np.array_equal(w, m.operators[f"conv{i}"].params["weight"])
        assert np.array_equal(b, m.operators[f"conv{i}"].params["bias"])
    m = synth.build_gat(100, 64, 47, 3, heads=4, seed=0)
    for i, (w, a) in enumerate(workload.gat_params(100, 64, 47, 3, heads=4, seed=0), start=1):
        assert np.array_equal(w, m.operators[f"attn{i}"].params["weight"])
        assert np.array_equal(a, m.operators[f"attn{i}"].params["attn"])


def test_reference_arm_never_imports_the_product(tmp_path):
    code = (
        "import runpy, sys\n"
        f"sys.argv = ['bench.py', '--impl', 'reference', '--nodes', '3000', '--steps', '1',"
        " '--warmup', '1', '--cpu-sample', '64']\n"
        f"runpy.run_path({str(ROOT / 'bench.py')!r}, run_name='__main__')\n"
        "bad = [k for k in sys.modules if k.startswith('paper_2211_15082_b200')]\n"
        "assert not bad, bad\n"
        "import os\n"
        "maps = open('/proc/self/maps').read()\n"
        "assert 'libglint_b200' not in maps\n")
    r = subprocess.run([sys.executable, "-c", code], cwd=tmp_path, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["cpu_model"]
    assert line["e2e"]["h2d_bytes_per_step"] == 0


def test_replay_matches_package_controller():
    """oracle.parity.replay_layers == the package's BatchController on a
    full-mode GCN at a capacity that forces bootstrap batches and retries."""
    from oracle import parity
    from paper_2211_15082_b200 import device as devmodel
    from paper_2211_15082_b200.batching import BatchController, Thresholds
    from paper_2211_15082_b200.device import DeviceBudget
    from paper_2211_15082_b200.executor import _dims_table
    from paper_2211_15082_b200.splitter import split
    from paper_2211_15082_b200.synth import build_gcn, gen_powerlaw

    g = gen_powerlaw(3000, seed=3)
    m = build_gcn(16, 32, 8, 3, seed=0)
    sch = split(m)
    dims = _dims_table(m, sch)
    cap = 400_000
    blocks = [{"layer": b.layer, "has_conv": b.has_conv,
               "input_widths": [dims[k] for k in b.input_keys()],
               "ops": [(dom, dims[o]) for o, kind, dom in b.iter_ops()
                       if kind not in ("Input", "Output")],
               "output_widths": [dims[o] for o in b.output_ids()]} for b in sch.blocks]
    want = parity.replay_layers(g.indptr, g.indices, cap, 64, 512, blocks)
    ctl = BatchController(Thresholds(64, 512), DeviceBudget(cap))
    count = parity.InputCounter(g.indptr, g.indices)
    got = []
    for b in sch.blocks:
        def plan(a, e, b=b):
            n_e = int(g.indptr[e] - g.indptr[a])
            return None, devmodel.footprint_counts(b, e - a, count(a, e), n_e, dims)
        recs = ctl.run_layer(b.layer, np.arange(g.num_nodes), g.indptr, plan, lambda p: None)
        got += [(b.layer, r.n_targets, r.footprint.peak, r.n_t, r.n_i, r.oom_retries)
                for r in recs]
    assert got == want
    assert len(want) > 6 and any(w[5] for w in want)


def test_spot_targets_include_hubs():
    from oracle import parity
    from paper_2211_15082_b200.synth import gen_powerlaw

    g = gen_powerlaw(2000, seed=1)
    t = parity.spot_targets(g.indptr, 100, 10)
    deg = np.diff(g.indptr)
    assert np.all(np.diff(t) > 0) and t[0] == 0 and t[-1] == 1999
    assert set(np.argsort(deg)[-10:]).issubset(set(t.tolist())) or \
        deg[t].max() == deg.max()
