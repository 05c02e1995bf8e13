"""K7, the fused aggregate -> transform ConvMean (glint_conv_mean_f32), against
K1 + K2 (the unfused path) and the CPU oracle.

Reference: model_ir.py:336-338 (ConvMean = agg_mean, kernels.py:122-135, then
linear, kernels.py:95-107).  K7 computes each row's mean with K1's add chain
and division and feeds it to the tensor core in K2's 3xTF32 product order, so
the bar against K1 + K2 is BYTE equality; against the oracle (numpy einsum
order) rel-L2 <= 1e-5.
"""

import numpy as np
import pytest

from conftest import rel_l2
from oracle import glint_oracle as orc

pytestmark = pytest.mark.gpu


def _graph(rng, n, hubs=True):
    degs = rng.integers(0, 40, size=n)
    degs[rng.integers(0, n, size=20)] = 0                     # isolated rows
    if hubs:
        degs[[1, n // 2, n - 1]] = [3000, 700, 1200]           # hub rows, longest first
    indptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(degs, out=indptr[1:])
    indices = rng.integers(0, n, size=int(indptr[-1]))
    if len(indices) > 8:
        indices[:6] = indices[0]                               # duplicate edges
        indices[int(indptr[5])] = 5                            # a self loop
    return indptr, indices


def _dev(torch, a, dtype):
    return torch.as_tensor(a, dtype=dtype).cuda()


def _padded(torch, x, pitch):
    t = torch.zeros((x.shape[0], pitch), dtype=torch.float32, device="cuda")
    t[:, : x.shape[1]] = torch.from_numpy(x).cuda()
    return t[:, : x.shape[1]]


def _unfused(kernels, _lib, torch, h, W, b, act, ip, ix, n, sched, n_hub, d_out, **kw):
    d_in = int(h.shape[1])
    agg = torch.empty((n, (d_in + 3) // 4 * 4), dtype=torch.float32, device="cuda")[:, :d_in]
    kernels.spmm_mean(agg, h, ip, ix, n, schedule=sched, n_hub=n_hub, **kw)
    out = torch.empty((n, (d_out + 3) // 4 * 4), dtype=torch.float32, device="cuda")[:, :d_out]
    kernels.linear_into(out, agg, W, b, act, precision=_lib.PREC_3XTF32)
    return out


@pytest.mark.parametrize("d_in,d_out,act,bias", [
    (100, 256, 1, True), (128, 128, 0, True), (64, 47, 1, False), (4, 16, 0, True),
    (128, 200, 2, True), (32, 256, 1, True), (100, 47, 0, False), (96, 64, 1, True)])
def test_conv_mean_equals_k1_k2_bytes(cuda, d_in, d_out, act, bias):
    import torch

    from paper_2211_15082_b200 import _lib, kernels

    rng = np.random.default_rng(d_in * 1000 + d_out)
    n = 5000
    indptr, indices = _graph(rng, n)
    x = rng.normal(size=(n, d_in)).astype(np.float32)
    W = (rng.normal(size=(d_out, d_in)) / np.sqrt(d_in)).astype(np.float32)
    bv = rng.normal(size=d_out).astype(np.float32) if bias else None
    ip, ix = _dev(torch, indptr, torch.int64), _dev(torch, indices, torch.int32)
    h = _padded(torch, x, (d_in + 3) // 4 * 4)
    Wt = torch.from_numpy(W).cuda()
    bt = torch.from_numpy(bv).cuda() if bias else None
    sched, n_hub = kernels.degree_schedule(ip, None, 0, n)
    n_hub = int(n_hub.item())
    assert kernels.conv_mean_supported(h, d_out)
    want = _unfused(kernels, _lib, torch, h, Wt, bt, act, ip, ix, n, sched, n_hub, d_out)
    got = torch.empty((n, (d_out + 3) // 4 * 4), dtype=torch.float32, device="cuda")[:, :d_out]
    got.fill_(float("nan"))
    kernels.conv_mean(got, h, Wt, bt, act, ip, ix, n, schedule=sched)
    g, w = got.cpu().numpy(), want.cpu().numpy()
    assert np.isfinite(g).all()
    assert g.tobytes() == w.tobytes(), rel_l2(g, w)
    # the gather warps one row at a time (GLINT_TUNE_FUSED_PIPE = 1): same bytes
    _lib.call("glint_set_tuning", 19, 1)
    try:
        kernels.conv_mean(got, h, Wt, bt, act, ip, ix, n, schedule=sched)
        assert got.cpu().numpy().tobytes() == w.tobytes()
    finally:
        _lib.call("glint_set_tuning", 19, 0)
    # and against the oracle (numpy add.at mean + float64 transform)
    bc = orc.build_batch_csc(indptr, indices, np.arange(n))
    agg = orc.agg_mean(bc, x).astype(np.float64)
    ref = agg @ W.astype(np.float64).T + (bv if bias else 0.0)
    if act == 1:
        ref = np.maximum(ref, 0.0)
    elif act == 2:
        ref = np.where(ref >= 0, ref, 0.2 * ref)
    assert rel_l2(g, ref) <= 1e-5


def test_conv_mean_natural_order_row_ids_and_col_map(cuda):
    """No schedule (natural order), a target subset through row_ids, and source
    rows through a col_map into a permuted compact matrix: equal bytes to K1 + K2
    with the same addressing, and a tail tile of fewer than 128 rows."""
    import torch

    from paper_2211_15082_b200 import _lib, kernels

    rng = np.random.default_rng(7)
    n, d_in, d_out = 3000, 100, 256
    indptr, indices = _graph(rng, n)
    x = rng.normal(size=(n, d_in)).astype(np.float32)
    perm = rng.permutation(n)
    xc = np.empty_like(x)
    xc[perm] = x                                            # row perm[u] holds node u
    W = (rng.normal(size=(d_out, d_in)) / 10).astype(np.float32)
    bv = rng.normal(size=d_out).astype(np.float32)
    ip, ix = _dev(torch, indptr, torch.int64), _dev(torch, indices, torch.int32)
    cmap = _dev(torch, perm, torch.int32)
    targets = np.sort(rng.choice(n, size=1001, replace=False))
    rid = _dev(torch, targets, torch.int64)
    h = _padded(torch, xc, 100)
    Wt, bt = torch.from_numpy(W).cuda(), torch.from_numpy(bv).cuda()
    B = len(targets)
    want = _unfused(kernels, _lib, torch, h, Wt, bt, 1, ip, ix, B, None, 0, d_out,
                    row_ids=rid, col_map=cmap)
    got = torch.empty((B, d_out), dtype=torch.float32, device="cuda")
    kernels.conv_mean(got, h, Wt, bt, 1, ip, ix, B, row_ids=rid, col_map=cmap)
    assert got.cpu().numpy().tobytes() == want.cpu().numpy().tobytes()
    _lib.call("glint_set_tuning", 19, 1)
    try:
        kernels.conv_mean(got, h, Wt, bt, 1, ip, ix, B, row_ids=rid, col_map=cmap)
        assert got.cpu().numpy().tobytes() == want.cpu().numpy().tobytes()
    finally:
        _lib.call("glint_set_tuning", 19, 0)
    bc = orc.build_batch_csc(indptr, indices, targets)
    ref = np.maximum(orc.agg_mean(bc, x[bc.input_ids]).astype(np.float64) @ W.T.astype(np.float64)
                     + bv, 0.0)
    assert rel_l2(got.cpu().numpy(), ref) <= 1e-5


def test_conv_mean_tiny_and_unsupported(cuda):
    import torch

    from paper_2211_15082_b200 import _lib, kernels

    rng = np.random.default_rng(3)
    indptr, indices = _graph(rng, 3, hubs=False)
    ip, ix = _dev(torch, indptr, torch.int64), _dev(torch, indices, torch.int32)
    x = rng.normal(size=(3, 8)).astype(np.float32)
    h = torch.from_numpy(x).cuda()
    W = torch.from_numpy(rng.normal(size=(5, 8)).astype(np.float32)).cuda()
    out = torch.empty((3, 8), dtype=torch.float32, device="cuda")[:, :5]
    kernels.conv_mean(out, h, W, None, 0, ip, ix, 3, max_ctas=1)
    want = _unfused(kernels, _lib, torch, h, W, None, 0, ip, ix, 3, None, 0, 5)
    assert out.cpu().numpy().tobytes() == want.cpu().numpy().tobytes()
    assert not kernels.conv_mean_supported(torch.empty((4, 256), device="cuda"), 256)
    assert not kernels.conv_mean_supported(h, 300)
    assert not kernels.conv_mean_supported(torch.empty((4, 6), device="cuda"), 8)


def test_engine_fused_equals_unfused(cuda):
    """run_inference with K7 (default) and with K1 + K2 (FUSE_CONV off): the same
    bytes for GCN and JKNet-style models, one batch and many batches per layer."""
    from paper_2211_15082_b200 import kernels
    from paper_2211_15082_b200.device import DeviceBudget
    from paper_2211_15082_b200.executor import run_inference
    from paper_2211_15082_b200.synth import build_gcn, build_jknet, gen_features, gen_powerlaw

    from paper_2211_15082_b200 import executor

    g = gen_powerlaw(4000, 4, exponent=1.8, max_deg=3000)
    assert (np.diff(g.indptr) + 1 >= kernels.HUB_MIN_DEGREE).sum() >= 2   # hub rows
    x = gen_features(4000, 100, seed=4)
    modes = {"whole": 0, "split": 0}
    orig = executor.LayerwiseEngine.run

    def counting_run(self, *a, **k):
        try:
            return orig(self, *a, **k)
        finally:
            for key in modes:
                modes[key] += self.k7_launches[key]

    executor.LayerwiseEngine.run = counting_run
    try:
        for m in (build_gcn(100, 128, 47, layers=3, seed=1),
                  build_jknet(100, 64, 16, layers=2, seed=2)):
            for cap in (1 << 32, 2 << 20):
                outs = []
                for fuse in (True, False):
                    kernels.FUSE_CONV = fuse
                    try:
                        res = run_inference(m, g, x, budget=DeviceBudget(cap))
                    finally:
                        kernels.FUSE_CONV = True
                    outs.append(res.output)
                assert outs[0].tobytes() == outs[1].tobytes()
                want = orc.eval_model(orc.model_spec(m), g.indptr, g.indices, x)
                assert rel_l2(outs[0], want) <= 1e-4
    finally:
        executor.LayerwiseEngine.run = orig
    # whole-layer launches (hub rows inside K7) and batches whose hub rows ran
    # beside K7 on the side stream
    assert modes["whole"] > 0 and modes["split"] > 0, modes
