"""GPU parity of every kernel against the golden vectors and the CPU oracle.

Bars: integer / index work and the mean aggregation are BIT-EXACT; attention
and dense transforms (fp32 accumulation in a different order than numpy's
einsum) are held to rel-L2 <= 1e-5 per kernel.
"""

import numpy as np
import pytest

from conftest import golden_graph, rel_l2
from oracle import glint_oracle as orc

pytestmark = pytest.mark.gpu


def test_build_batch_csc_bit_exact(golden, cuda):
    from paper_2211_15082_b200 import kernels

    arrs, meta = golden
    for c in meta["kernels"]:
        g = golden_graph(arrs, c["graph"])
        bc = kernels.build_batch_csc(g, arrs[c["targets"]])
        assert np.array_equal(bc.input_ids.cpu().numpy(), arrs[c["input_ids"]])
        assert np.array_equal(bc.indptr.cpu().numpy(), arrs[c["indptr"]])
        assert np.array_equal(bc.local_srcs.cpu().numpy(), arrs[c["local_srcs"]])
        assert np.array_equal(bc.target_pos.cpu().numpy(), arrs[c["target_pos"]])


def test_gather_slices_and_trivial(golden, cuda):
    from paper_2211_15082_b200 import kernels

    arrs, _ = golden
    g = golden_graph(arrs, "pow300")
    t = np.array([5, 0, 299, 17, 17])
    srcs, ip = kernels.gather_slices(g, t)
    s2, ip2 = orc.gather_slices(g.indptr, g.indices, t)
    assert np.array_equal(srcs, s2) and np.array_equal(ip, ip2)
    tb = kernels.trivial_batch_csc(np.array([4, 7, 2]))
    assert tb.input_ids.cpu().tolist() == [2, 4, 7] and tb.target_pos.cpu().tolist() == [1, 2, 0]


def test_agg_mean_bit_exact_vs_reference(golden, cuda):
    from paper_2211_15082_b200 import kernels

    arrs, meta = golden
    for c in meta["kernels"]:
        g = golden_graph(arrs, c["graph"])
        bc = kernels.build_batch_csc(g, arrs[c["targets"]])
        x = arrs[c["x"]]
        out = kernels.agg_mean(bc, x[bc.input_ids.cpu().numpy()])
        assert out.tobytes() == arrs[c["agg_mean"]].tobytes(), (c["graph"], c["dim"])


@pytest.mark.parametrize("dim", [1, 5, 47, 64, 100, 128, 188, 256, 300, 768, 1100])
def test_agg_mean_widths_and_hubs_bit_exact(cuda, dim):
    """Regular, sub-warp and hub (CTA) paths, aligned and unaligned pitches,
    duplicate edges and self loops, tile loop beyond 1024 columns."""
    import torch

    from paper_2211_15082_b200 import kernels

    rng = np.random.default_rng(dim)
    n = 3000
    degs = rng.integers(0, 12, size=n)
    degs[[3, 100, 2999]] = [2500, 700, 5000]          # hubs (deg+1 >= 512)
    indptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(degs, out=indptr[1:])
    indices = rng.integers(0, n, size=int(indptr[-1]))
    indices[:5] = 0                                     # duplicates
    from paper_2211_15082_b200.storage import CscGraph

    g = CscGraph(n, int(indptr[-1]), indptr, indices)
    x = rng.normal(size=(n, dim)).astype(np.float32)
    bc_ref = orc.build_batch_csc(indptr, indices, np.arange(n))
    want = orc.agg_mean(bc_ref, x)
    bc = kernels.build_batch_csc(g, np.arange(n))
    got = kernels.agg_mean(bc, torch.from_numpy(x).cuda()).cpu().numpy()
    assert got.tobytes() == want.tobytes()
    # same rows through the resident (global-id) form with a padded pitch
    dg = kernels.device_graph(g)
    pitch = (dim + 3) // 4 * 4
    hp = torch.zeros((n, pitch), dtype=torch.float32, device="cuda")
    hp[:, :dim] = torch.from_numpy(x).cuda()
    out = torch.zeros((n, pitch), dtype=torch.float32, device="cuda")
    sched, nh = kernels.degree_schedule(dg.indptr, None, 0, n)
    kernels.spmm_mean(out[:, :dim], hp[:, :dim], dg.indptr, dg.indices, n, schedule=sched,
                      n_hub=int(nh.item()))
    assert out[:, :dim].cpu().numpy().tobytes() == want.tobytes()
    assert not out[:, dim:].any()


@pytest.mark.parametrize("dim", [5, 48, 100, 256])
def test_agg_mean_every_variant_bit_exact(cuda, dim):
    """Every K1 launch variant (register-staged and cp.async ring) and both hub
    paths give the oracle's bytes (tuning knobs are performance-only)."""
    import torch

    from paper_2211_15082_b200 import _lib, kernels

    rng = np.random.default_rng(7 + dim)
    n = 4000
    degs = rng.integers(0, 70, size=n)
    degs[[11, 2500]] = [3000, 600]
    indptr = np.concatenate([[0], np.cumsum(degs)]).astype(np.int64)
    indices = rng.integers(0, n, size=int(indptr[-1]))
    x = rng.normal(size=(n, dim)).astype(np.float32)
    want = orc.agg_mean(orc.build_batch_csc(indptr, indices, np.arange(n)), x)
    pitch = (dim + 3) // 4 * 4
    hp = torch.zeros((n, pitch), dtype=torch.float32, device="cuda")
    hp[:, :dim] = torch.from_numpy(x).cuda()
    ip = torch.from_numpy(indptr).cuda()
    ix = torch.from_numpy(indices.astype(np.int32)).cuda()
    sched, nh = kernels.degree_schedule(ip, None, 0, n)
    try:
        for variant in range(16):
            for hub in (0, 1, 2, 3, 4, 5):
                _lib.call("glint_set_tuning", 0, variant)
                _lib.call("glint_set_tuning", 2, hub)
                out = torch.full((n, pitch), 7.0, dtype=torch.float32, device="cuda")
                kernels.spmm_mean(out[:, :dim], hp[:, :dim], ip, ix, n, schedule=sched,
                                  n_hub=int(nh.item()))
                assert out[:, :dim].cpu().numpy().tobytes() == want.tobytes(), (variant, hub)
    finally:
        _lib.call("glint_set_tuning", 0, 0)
        _lib.call("glint_set_tuning", 2, 0)


@pytest.mark.parametrize("act", [0, 1, 2])
def test_agg_mean_bias_act_epilogue_bit_exact(cuda, act):
    """K1 epilogue act(mean + b) == numpy (agg_mean + b) then ReLU/LeakyReLU, bytes."""
    import torch

    from paper_2211_15082_b200 import kernels
    from paper_2211_15082_b200.synth import gen_powerlaw

    g = gen_powerlaw(700, seed=5)
    rng = np.random.default_rng(act)
    x = rng.normal(size=(700, 48)).astype(np.float32)
    b = rng.normal(size=48).astype(np.float32)
    want = orc.agg_mean(orc.build_batch_csc(g.indptr, g.indices, np.arange(700)), x) + b
    want = [want, orc.elementwise("ReLU", [want]), orc.leaky_relu(want)][act]
    dg = kernels.device_graph(g)
    out = torch.empty((700, 48), device="cuda")
    sched, nh = kernels.degree_schedule(dg.indptr, None, 0, 700)
    kernels.spmm_mean(out, torch.from_numpy(x).cuda(), dg.indptr, dg.indices, 700,
                      schedule=sched, n_hub=int(nh.item()), bias=torch.from_numpy(b).cuda(), act=act)
    assert out.cpu().numpy().tobytes() == want.tobytes()


def test_agg_mean_reference_kats(cuda):
    """Reference test_kernels.py:50-67 known answers."""
    from paper_2211_15082_b200 import kernels
    from paper_2211_15082_b200.storage import make_graph

    toy = make_graph(6, {0: [2, 3], 1: [2, 3], 2: [4, 5]})
    bc = kernels.build_batch_csc(toy, np.array([0]))
    h = np.zeros((3, 1), np.float32)
    ids = bc.input_ids.cpu().tolist()
    h[ids.index(2)] = 2.0
    h[ids.index(3)] = 4.0
    assert kernels.agg_mean(bc, h).tolist() == [[2.0]]
    assert kernels.agg_mean(kernels.build_batch_csc(toy, np.array([3])),
                            np.array([[7.0]], np.float32)).tolist() == [[7.0]]
    full = kernels.build_batch_csc(toy, np.arange(6))
    assert np.array_equal(kernels.agg_mean(full, np.full((6, 2), 3.25, np.float32)),
                          np.full((6, 2), 3.25, np.float32))


def test_batch_invariance_on_device(cuda):
    from paper_2211_15082_b200 import kernels
    from paper_2211_15082_b200.synth import gen_powerlaw

    g = gen_powerlaw(500, seed=3)
    rng = np.random.default_rng(1)
    x = rng.normal(size=(500, 33)).astype(np.float32)
    full_bc = kernels.build_batch_csc(g, np.arange(500))
    full = kernels.agg_mean(full_bc, x)
    for _ in range(5):
        sub = np.sort(rng.choice(500, size=int(rng.integers(1, 500)), replace=False))
        bc = kernels.build_batch_csc(g, sub)
        out = kernels.agg_mean(bc, x[bc.input_ids.cpu().numpy()])
        assert out.tobytes() == full[sub].tobytes()


def test_agg_attn_vs_reference(golden, cuda):
    from paper_2211_15082_b200 import kernels

    arrs, meta = golden
    n = 0
    for c in meta["kernels"]:
        if "agg_attn" not in c:
            continue
        g = golden_graph(arrs, c["graph"])
        bc = kernels.build_batch_csc(g, arrs[c["targets"]])
        out = kernels.agg_attn(bc, arrs[c["x"]][bc.input_ids.cpu().numpy()],
                               kernels.AttnParams(arrs[c["attn_w"]], arrs[c["attn_a"]]))
        assert rel_l2(out, arrs[c["agg_attn"]]) <= 1e-5, c["targets"]
        n += 1
    assert n > 0


@pytest.mark.parametrize("heads,dh", [(1, 2), (4, 64), (4, 47), (8, 16)])
def test_agg_attn_hubs_and_widths(cuda, heads, dh):
    from paper_2211_15082_b200 import kernels
    from paper_2211_15082_b200.storage import CscGraph

    rng = np.random.default_rng(heads * 100 + dh)
    n = 1500
    degs = rng.integers(0, 9, size=n)
    degs[[7, 800]] = [3000, 600]
    indptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(degs, out=indptr[1:])
    indices = rng.integers(0, n, size=int(indptr[-1]))
    g = CscGraph(n, int(indptr[-1]), indptr, indices)
    din = 24
    x = (rng.normal(size=(n, din)) * 3).astype(np.float32)
    w = (rng.normal(size=(heads, dh, din)) / np.sqrt(din)).astype(np.float32)
    a = rng.normal(size=(heads, 2 * dh)).astype(np.float32)
    want = orc.agg_attn(orc.build_batch_csc(indptr, indices, np.arange(n)), x, w, a)
    got = kernels.agg_attn(kernels.build_batch_csc(g, np.arange(n)), x, kernels.AttnParams(w, a))
    assert np.all(np.isfinite(got))
    assert rel_l2(got, want) <= 1e-5


@pytest.mark.parametrize("heads,dh", [(4, 64), (4, 47), (3, 5)])
def test_gat_hub_paths_and_act_bit_identical(cuda, heads, dh):
    """Hub rows: bulk-copy ring kernel == one-CTA register path, byte for byte
    (same per-column order); the fused ReLU epilogue == ReLU of the output."""
    import torch

    from paper_2211_15082_b200 import _lib, kernels

    rng = np.random.default_rng(dh)
    n = 3000
    degs = rng.integers(0, 40, size=n)
    degs[[5, 1200, 2999]] = [4500, 700, 2048]
    indptr = torch.from_numpy(np.concatenate([[0], np.cumsum(degs)]).astype(np.int64)).cuda()
    indices = torch.from_numpy(rng.integers(0, n, size=int(degs.sum())).astype(np.int32)).cuda()
    hp = kernels.head_pitch(dh)
    Z = torch.randn((n, heads * hp), device="cuda")
    Z.view(n, heads, hp)[:, :, dh:] = 0
    s_src = torch.randn((n, heads), device="cuda")
    s_dst = torch.randn((n, heads), device="cuda")
    sched, nh = kernels.degree_schedule(indptr, None, 0, n)
    outs = []
    for inline, act in ((0, 0), (1, 0), (0, 1), (3, 0), (2, 0), (4, 0)):
        _lib.call("glint_set_tuning", 2, inline)
        out = torch.empty((n, heads * dh), device="cuda")
        kernels.gat_aggregate(out, Z, s_src, s_dst, heads, dh, indptr, indices, n,
                              schedule=sched, n_hub=int(nh.item()), act=act)
        outs.append(out)
    _lib.call("glint_set_tuning", 2, 0)
    assert int(nh.item()) == 3
    assert torch.equal(outs[0], outs[1])
    assert torch.equal(torch.relu(outs[0]), outs[2])
    assert torch.equal(outs[0], outs[3])
    assert torch.equal(outs[0], outs[4]) and torch.equal(outs[0], outs[5])
    # the K4 ring's L2 policy (scores evict_last, Z evict_first) off: same bytes
    _lib.call("glint_set_tuning", 14, 1)
    try:
        nopol = torch.empty_like(outs[0])
        kernels.gat_aggregate(nopol, Z, s_src, s_dst, heads, dh, indptr, indices, n,
                              schedule=sched, n_hub=int(nh.item()))
        assert torch.equal(nopol, outs[0])
    finally:
        _lib.call("glint_set_tuning", 14, 0)
    # the peak pass before the ring prologue (the pre-round-2 order): same bytes
    _lib.call("glint_set_tuning", 18, 1)
    try:
        first = torch.empty_like(outs[0])
        kernels.gat_aggregate(first, Z, s_src, s_dst, heads, dh, indptr, indices, n,
                              schedule=sched, n_hub=int(nh.item()))
        assert torch.equal(first, outs[0])
    finally:
        _lib.call("glint_set_tuning", 18, 0)
    # and the same bytes without any hub path (every row in the regular kernel),
    # for every launch variant (register-staged and cp.async ring)
    try:
        for v in range(10):
            _lib.call("glint_set_tuning", 3, v)
            plain = torch.empty_like(outs[0])
            kernels.gat_aggregate(plain, Z, s_src, s_dst, heads, dh, indptr, indices, n)
            assert torch.equal(plain, outs[0]), v
            kernels.gat_aggregate(plain, Z, s_src, s_dst, heads, dh, indptr, indices, n,
                                  schedule=sched, n_hub=int(nh.item()))
            assert torch.equal(plain, outs[0]), v
            # two-phase (edge softmax + weighted SpMM) path, whole and offset edge ranges
            for rng_ in ((0, int(degs.sum())), (-5, int(degs.sum()) + 9)):
                if rng_[0] < 0:
                    continue
                kernels.gat_aggregate(plain, Z, s_src, s_dst, heads, dh, indptr, indices, n,
                                      schedule=sched, n_hub=int(nh.item()), edge_range=rng_)
                assert torch.equal(plain, outs[0]), (v, rng_)
            half = n // 2
            e0 = int(degs[:half].sum())
            part = torch.empty((n - half, heads * dh), device="cuda")
            s2, nh2 = kernels.degree_schedule(indptr, None, half, n - half)
            kernels.gat_aggregate(part, Z, s_src, s_dst, heads, dh, indptr, indices, n - half,
                                  row_base=half, schedule=s2, n_hub=int(nh2.item()),
                                  edge_range=(e0, int(degs.sum()) - e0))
            assert torch.equal(part, outs[0][half:]), v
    finally:
        _lib.call("glint_set_tuning", 3, 0)


def test_attn_zero_logits_equal_mean_after_transform(cuda):
    """Reference test_kernels.py:101-109 (tolerance: the transform is a GEMM)."""
    from paper_2211_15082_b200 import kernels
    from paper_2211_15082_b200.storage import make_graph

    toy = make_graph(6, {0: [2, 3], 1: [2, 3], 2: [4, 5]})
    bc = kernels.build_batch_csc(toy, np.arange(6))
    rng = np.random.default_rng(3)
    w = rng.normal(size=(1, 2, 3)).astype(np.float32)
    h = rng.normal(size=(6, 3)).astype(np.float32)
    att = kernels.agg_attn(bc, h, kernels.AttnParams(w, np.zeros((1, 4), np.float32)))
    mean = kernels.agg_mean(bc, kernels.linear(h, w[0]))
    assert rel_l2(att, mean) <= 1e-6


def test_linear_elementwise_concat(golden, cuda):
    from paper_2211_15082_b200 import kernels

    arrs, meta = golden
    for c in meta["kernels"]:
        if "linear" not in c:
            continue
        x = arrs[c["x"]]
        assert rel_l2(kernels.linear(x, arrs[c["lin_w"]], arrs[c["lin_b"]]), arrs[c["linear"]]) <= 1e-5
        for kind in ("ReLU", "LeakyReLU", "DropoutIdentity"):
            assert kernels.elementwise(kind, [x]).tobytes() == arrs[c["ew_" + kind]].tobytes(), kind
        assert rel_l2(kernels.elementwise("Norm", [x]), arrs[c["ew_Norm"]]) <= 1e-6
        assert kernels.elementwise("Add", [x, x * 0.5, -x]).tobytes() == arrs[c["ew_Add"]].tobytes()
        assert kernels.concat([x, x[:, :1], 2 * x]).tobytes() == arrs[c["concat"]].tobytes()


def test_linear_row_invariance(cuda):
    """Rows computed alone equal the all-at-once bytes (test_kernels.py:31-44)."""
    from paper_2211_15082_b200 import kernels

    rng = np.random.default_rng(0)
    x = rng.normal(size=(300, 100)).astype(np.float32)
    w = rng.normal(size=(47, 100)).astype(np.float32)
    b = rng.normal(size=47).astype(np.float32)
    full = kernels.linear(x, w, b)
    for i in (0, 1, 150, 299):
        assert kernels.linear(x[i:i + 1], w, b).tobytes() == full[i:i + 1].tobytes()
    assert rel_l2(full, orc.linear(x, w, b)) <= 5e-6


@pytest.mark.parametrize("M,N,K", [(1, 47, 100), (300, 47, 100), (1000, 256, 256),
                                   (129, 300, 64), (257, 16, 3), (4096, 128, 128),
                                   (77, 48, 188), (5000, 256, 100)])
@pytest.mark.parametrize("act", [0, 1, 2])
def test_tcgen05_3xtf32_linear(cuda, M, N, K, act):
    """Tensor-core split-TF32 GEMM vs fp64: rel-L2 <= 5e-6 (plain TF32 would be ~3e-4),
    bias + activation epilogue, row gather, M/N/K tails, N > 256 (two column tiles)."""
    import torch

    from paper_2211_15082_b200 import _lib, kernels

    rng = np.random.default_rng(M * 7 + N + K + act)
    x = rng.normal(size=(M + 5, K)).astype(np.float32)
    w = (rng.normal(size=(N, K)) / np.sqrt(K)).astype(np.float32)
    b = rng.normal(size=N).astype(np.float32)
    rows = rng.permutation(M + 5)[:M].astype(np.int64)
    want = x[rows].astype(np.float64) @ w.T.astype(np.float64) + b
    if act == 1:
        want = np.maximum(want, 0)
    elif act == 2:
        want = np.where(want >= 0, want, 0.2 * want)
    xd, wd, bd = (torch.from_numpy(a).cuda() for a in (x, w, b))
    rd = torch.from_numpy(rows).cuda()
    base = torch.full((M, N + 3), 7.0, device="cuda")
    out = base[:, :N]
    kernels.linear_into(out, xd, wd, bd, act, a_rows=rd, precision=_lib.PREC_3XTF32)
    got = out.cpu().numpy()
    assert rel_l2(got, want) <= 5e-6, rel_l2(got, want)
    assert torch.all(base[:, N:] == 7.0)             # no writes past N
    # row invariance on the tensor cores
    one = torch.empty((1, N), device="cuda")
    kernels.linear_into(one, xd, wd, bd, act, a_rows=rd[M // 2:M // 2 + 1], precision=_lib.PREC_3XTF32)
    assert one.cpu().numpy().tobytes() == got[M // 2:M // 2 + 1].tobytes()


@pytest.mark.parametrize("M,N,K", [(1, 47, 100), (300, 47, 256), (1000, 256, 256), (1000, 256, 100),
                                   (129, 300, 64), (257, 16, 3), (4096, 128, 128), (77, 48, 188),
                                   (5000, 256, 100), (513, 172, 128), (700, 65, 40), (300, 64, 600),
                                   (2000, 600, 36), (33, 1, 9), (600, 64, 512), (400, 48, 480)])
@pytest.mark.parametrize("act", [0, 1])
def test_tcgen05_v3_linear(cuda, M, N, K, act):
    """The v3 GEMM (tensor-map TMA, CTA pairs for N > 64, resident W for N <= 64)
    vs fp64: rel-L2 <= 5e-6; M/N/K tails (partial 256-row pair tiles, K not a
    multiple of the 32-wide chunk), N > 256 (column tiles), no writes past N,
    rows computed alone equal the batch bytes, and agreement with v2."""
    import torch

    from paper_2211_15082_b200 import _lib, kernels

    rng = np.random.default_rng(M * 11 + N * 3 + K + act)
    x = rng.normal(size=(M, K)).astype(np.float32)
    w = (rng.normal(size=(N, K)) / np.sqrt(K)).astype(np.float32)
    b = rng.normal(size=N).astype(np.float32)
    want = x.astype(np.float64) @ w.T.astype(np.float64) + b
    if act == 1:
        want = np.maximum(want, 0)
    xd, wd, bd = (torch.from_numpy(a).cuda() for a in (x, w, b))
    base = torch.full((M, N + 3), 7.0, device="cuda")
    out = base[:, :N]
    kernels.linear_into(out, xd, wd, bd, act, precision=_lib.PREC_3XTF32)
    got = out.cpu().numpy()
    assert rel_l2(got, want) <= 5e-6, rel_l2(got, want)
    assert torch.all(base[:, N:] == 7.0)
    i = M // 2
    one = torch.empty((1, N), device="cuda")
    kernels.linear_into(one, xd[i:i + 1], wd, bd, act, precision=_lib.PREC_3XTF32)
    assert one.cpu().numpy().tobytes() == got[i:i + 1].tobytes()
    _lib.call("glint_set_tuning", 9, 1)          # the v2 kernel
    try:
        ref = torch.empty((M, N), device="cuda")
        kernels.linear_into(ref, xd, wd, bd, act, precision=_lib.PREC_3XTF32)
    finally:
        _lib.call("glint_set_tuning", 9, 0)
    assert rel_l2(got, ref.cpu().numpy()) <= 2e-6


@pytest.mark.parametrize("M,heads,dh,K", [(1000, 4, 64, 100), (777, 4, 47, 256), (300, 2, 32, 64),
                                          (5, 8, 8, 16)])
def test_tcgen05_v3_gat_project(cuda, M, heads, dh, K):
    """Fused projection + score epilogue on the v3 kernel vs fp64 (Z and s_src/s_dst)."""
    import torch

    from paper_2211_15082_b200 import _lib, kernels

    rng = np.random.default_rng(M + heads * dh + K)
    x = rng.normal(size=(M, K)).astype(np.float32)
    w = (rng.normal(size=(heads, dh, K)) / np.sqrt(K)).astype(np.float32)
    att = rng.normal(size=(heads, 2 * dh)).astype(np.float32)
    xd = torch.from_numpy(x).cuda()
    w_pad = kernels.padded_head_weight(torch.from_numpy(w).cuda())
    Z, ss, sd = kernels.attn_project(xd, w_pad, torch.from_numpy(att).cuda(), heads, dh,
                                     precision=_lib.PREC_3XTF32)
    hp = kernels.head_pitch(dh)
    z = Z.cpu().numpy().reshape(M, heads, hp)[:, :, :dh]
    want = np.einsum("mk,hdk->mhd", x.astype(np.float64), w.astype(np.float64))
    assert rel_l2(z, want) <= 5e-6
    ws = np.einsum("mhd,hd->mh", want, att[:, :dh].astype(np.float64))
    wdst = np.einsum("mhd,hd->mh", want, att[:, dh:].astype(np.float64))
    assert rel_l2(ss.cpu().numpy(), ws) <= 1e-5
    assert rel_l2(sd.cpu().numpy(), wdst) <= 1e-5


@pytest.mark.parametrize("M,heads,dh,K", [(1000, 4, 64, 100), (777, 4, 47, 256), (513, 4, 64, 256),
                                          (300, 4, 10, 200), (65, 8, 32, 192)])
def test_gat_score_epilogue_modes_same_bytes(cuda, M, heads, dh, K):
    """The one-head half-chunk score path (GLINT_TUNE_GAT_EPI 0: 32-column
    chunks, v3 for every K; 3: 16-column chunks) and the per-column head walk
    (1: v2 for K < 192) give the same Z, s_src and s_dst bytes, on v3 and on v2
    (GLINT_TUNE_GEMM_V3 1); head pitch 12 (dh 10) takes the per-column walk."""
    import torch

    from paper_2211_15082_b200 import _lib, kernels

    rng = np.random.default_rng(7 * M + K)
    xd = torch.from_numpy(rng.normal(size=(M, K)).astype(np.float32)).cuda()
    w = (rng.normal(size=(heads, dh, K)) / np.sqrt(K)).astype(np.float32)
    w_pad = kernels.padded_head_weight(torch.from_numpy(w).cuda())
    att = torch.from_numpy(rng.normal(size=(heads, 2 * dh)).astype(np.float32)).cuda()
    outs = {}
    try:
        for v3off in (0, 1):
            for mode in (0, 1, 3):
                _lib.call("glint_set_tuning", 9, v3off)
                _lib.call("glint_set_tuning", 20, mode)
                res = kernels.attn_project(xd, w_pad, att, heads, dh, precision=_lib.PREC_3XTF32)
                torch.cuda.synchronize()
                outs[(v3off, mode)] = [t.cpu().numpy().tobytes() for t in res]
    finally:
        _lib.call("glint_set_tuning", 9, 0)
        _lib.call("glint_set_tuning", 20, 0)
    base = outs[(0, 1)]
    for key, got in outs.items():
        assert got == base, key


def test_shape_errors_are_value_errors(cuda):
    from paper_2211_15082_b200 import kernels

    with pytest.raises(ValueError):
        kernels.linear(np.zeros((1, 3), np.float32), np.zeros((2, 2), np.float32))
    with pytest.raises(ValueError):
        kernels.elementwise("Add", [np.zeros((1, 2), np.float32), np.zeros((2, 2), np.float32)])
    with pytest.raises(ValueError):
        kernels.concat([np.zeros((1, 2), np.float32), np.zeros((2, 2), np.float32)])


def test_device_rcmk_matches_reference_and_host_path(golden, cuda):
    """RCMK from the device-built (degree, id)-sorted adjacency == the reference's
    golden orders and == the all-host native path on random directed graphs with
    duplicates, self loops and several components."""
    from paper_2211_15082_b200 import kernels, reorder
    from paper_2211_15082_b200.storage import CscGraph

    arrs, meta = golden
    n_checked = 0
    for c in meta["orders"]:
        if c["kind"] != "rcmk":
            continue
        g = golden_graph(arrs, c["graph"])
        got = reorder.rcmk(kernels.device_graph(g)).perm
        assert np.array_equal(got, arrs[c["perm"]]), c["graph"]
        n_checked += 1
    assert n_checked > 0
    rng = np.random.default_rng(11)
    for n, e in ((1, 0), (50, 0), (300, 900), (5000, 40000)):
        dst = np.sort(rng.integers(0, n, size=e))
        src = rng.integers(0, max(n // 2, 1), size=e)      # ids >= n/2 only as targets
        indptr = np.concatenate([[0], np.cumsum(np.bincount(dst, minlength=n))]).astype(np.int64)
        g = CscGraph(n, e, indptr, src.astype(np.int64))
        host = reorder.rcmk(g).perm
        dev = reorder.rcmk(kernels.device_graph(g)).perm
        assert np.array_equal(host, dev), (n, e)


def test_device_rcmk_bfs_levels_and_fallback(cuda, monkeypatch):
    """The level-synchronous device BFS (union-find components, first-parent
    ordering) equals the sequential native RCMK on a heavy-tailed graph with
    isolated nodes and many components, on a path (one node per level), and
    through the host fallback once the level cap is hit."""
    import torch

    from paper_2211_15082_b200 import kernels, reorder, synth
    from paper_2211_15082_b200.storage import CscGraph

    dg = synth.gen_products_like(60_000, 60_000 * 12, seed=9, device="cuda")
    hg = CscGraph(dg.num_nodes, dg.num_edges, dg.indptr_host,
                  dg.indices.to(torch.int64).cpu().numpy())
    want = reorder.rcmk(hg).perm
    assert np.array_equal(reorder.rcmk(dg).perm, want)
    # a path 0-1-...-999 plus isolated nodes and a triangle: 1000 BFS levels
    n = 1010
    edges = [(i + 1, i) for i in range(999)] + [(1001, 1000), (1002, 1001), (1000, 1002)]
    dst = np.array([d for d, _ in edges])
    srcs = np.array([s_ for _, s_ in edges])
    order = np.argsort(dst, kind="stable")
    indptr = np.concatenate([[0], np.cumsum(np.bincount(dst, minlength=n))]).astype(np.int64)
    g = CscGraph(n, len(edges), indptr, srcs[order].astype(np.int64))
    want = reorder.rcmk(g).perm
    assert np.array_equal(reorder.rcmk(kernels.device_graph(g)).perm, want)
    monkeypatch.setattr(reorder, "RCMK_MAX_DEVICE_LEVELS", 10)
    assert reorder._rcmk_device(kernels.device_graph(g)) is None
    assert np.array_equal(reorder.rcmk(kernels.device_graph(g)).perm, want)


def test_device_sampling_matches_reference(golden, cuda):
    """glint_sample_neighbors == the reference's draws (golden) and == the host
    restatement on random graphs with duplicates, for all-node and subset draws."""
    from paper_2211_15082_b200 import kernels
    from paper_2211_15082_b200.executor import sample_neighbors
    from paper_2211_15082_b200.storage import CscGraph

    arrs, meta = golden
    n_checked = 0
    for c in meta["sampling"]:
        g = golden_graph(arrs, c["graph"])
        s = sample_neighbors(kernels.device_graph(g), np.arange(g.num_nodes), c["fanout"],
                             c["seed"], c["layer"])
        assert np.array_equal(np.asarray(s.indptr_host), arrs[c["indptr"]])
        assert np.array_equal(s.indices.cpu().numpy().astype(np.int64), arrs[c["indices"]])
        n_checked += 1
    assert n_checked > 0
    rng = np.random.default_rng(5)
    for n, e, fanout in ((200, 3000, 5), (3000, 60000, 10), (1000, 20000, 1)):
        dst = np.sort(rng.integers(0, n, size=e))
        dst[:600] = 7                                       # one heavy row
        dst = np.sort(dst)
        src = rng.integers(0, n, size=e)
        indptr = np.concatenate([[0], np.cumsum(np.bincount(dst, minlength=n))]).astype(np.int64)
        g = CscGraph(n, e, indptr, src.astype(np.int64))
        dg = kernels.device_graph(g)
        for nodes in (np.arange(n), np.sort(rng.choice(n, n // 3, replace=False))):
            for seed, layer in ((0, 1), (-3, 2)):
                h = sample_neighbors(g, nodes, fanout, seed, layer)
                d = sample_neighbors(dg, nodes, fanout, seed, layer)
                assert np.array_equal(h.indptr, np.asarray(d.indptr_host))
                assert np.array_equal(h.indices, d.indices.cpu().numpy().astype(np.int64))


def test_streaming_graph_loader(tmp_path, cuda):
    """load_graph_device (mmap + chunked pinned upload + device narrowing) gives
    load_graph's arrays, and rejects the reference's malformed-file cases."""
    import struct

    from paper_2211_15082_b200.errors import FormatError
    from paper_2211_15082_b200.storage import (CscGraph, load_graph, load_graph_device,
                                               save_graph)

    rng = np.random.default_rng(2)
    n, e = 5000, 80000
    dst = np.sort(rng.integers(0, n, size=e))
    indptr = np.concatenate([[0], np.cumsum(np.bincount(dst, minlength=n))]).astype(np.int64)
    g = CscGraph(n, e, indptr, rng.integers(0, n, size=e).astype(np.int64))
    p = tmp_path / "g.dgig"
    save_graph(g, p)
    ref = load_graph(p)
    for chunk in (1 << 25, 7777):
        dg = load_graph_device(p, chunk_edges=chunk)
        assert np.array_equal(np.asarray(dg.indptr_host), ref.indptr)
        assert np.array_equal(dg.indptr.cpu().numpy(), ref.indptr)
        assert np.array_equal(dg.indices.cpu().numpy().astype(np.int64), ref.indices)
    empty = tmp_path / "e.dgig"
    save_graph(CscGraph(3, 0, np.zeros(4, np.int64), np.zeros(0, np.int64)), empty)
    assert load_graph_device(empty).num_edges == 0
    raw = p.read_bytes()
    cases = {
        "magic": b"XXXX" + raw[4:],
        "trunc": raw[:-8],
        "trail": raw + b"\0",
        "range": raw[:-8] + struct.pack("<Q", n),
        "mono": raw[:struct.calcsize("<4sIQQ") + 8] + struct.pack("<Q", 10 ** 9)
        + raw[struct.calcsize("<4sIQQ") + 16:],
    }
    for name, data in cases.items():
        q = tmp_path / f"{name}.dgig"
        q.write_bytes(data)
        with pytest.raises(FormatError):
            load_graph_device(q, chunk_edges=10000)


@pytest.mark.parametrize("pack24", ["1", "0"])
def test_async_csr_upload_equals_host_graph(cuda, monkeypatch, pack24):
    """DeviceGraph.upload_async (native thread: host narrowing or 24-bit packing,
    chunked H2D, per-chunk events) lands the same CSR as the host graph, for
    uniform and geometric chunks and ragged chunk sizes."""
    import torch

    from paper_2211_15082_b200 import storage

    monkeypatch.setattr(storage, "PACK24", pack24 == "1")
    if True:
        rng = np.random.default_rng(7)
        n = 70_000
        degs = rng.integers(0, 40, n)
        degs[:3] = [0, 5000, 1]
        ptr = np.concatenate([[0], np.cumsum(degs)]).astype(np.int64)
        idx = rng.integers(0, n, int(ptr[-1])).astype(np.int64)
        idx[:5] = [n - 1, 0, 65535, 65536, n - 2]
        g = storage.CscGraph(n, int(ptr[-1]), ptr, idx)
        copy = torch.cuda.Stream()
        for chunks, geometric in ((1, False), (5, True), (7, False)):
            dg = storage.DeviceGraph.upload_async(g, torch.device("cuda"), copy, chunks=chunks,
                                                  geometric=geometric)
            dg.wait_rows()
            torch.cuda.synchronize()
            assert np.array_equal(dg.indices.cpu().numpy(), idx.astype(np.int32))
            assert np.array_equal(dg.indptr.cpu().numpy(), ptr)
            assert not dg.upload_in_flight()


def test_packed_upload_rejects_wide_ids(cuda):
    """glint_upload_start_packed: an id >= 2^24 fails its chunk with EINVAL
    (the caller only packs when N <= 2^24), ids up to 2^24 - 1 round-trip."""
    import ctypes

    import torch

    from paper_2211_15082_b200 import _lib

    lib = _lib.load()
    for ids, ok in (([0, 1, (1 << 24) - 1, 12345, 7], True), ([3, 1 << 24, 5], False)):
        src = np.asarray(ids, dtype=np.int64)
        m = len(src)
        dst = torch.full((m,), -1, dtype=torch.int32, device="cuda")
        stage = torch.empty(3 * m, dtype=torch.uint8, pin_memory=True)
        dstage = torch.empty(3 * m, dtype=torch.uint8, device="cuda")
        edges = np.asarray([0, m], dtype=np.int64)
        h = ctypes.c_void_p()
        s = torch.cuda.current_stream()
        assert lib.glint_upload_start_packed(src.ctypes.data, dst.data_ptr(), stage.data_ptr(),
                                             dstage.data_ptr(), 3, edges.ctypes.data, 1, 2,
                                             ctypes.c_void_p(s.cuda_stream), ctypes.byref(h)) == 0
        rc = lib.glint_upload_wait(h, 0, ctypes.c_void_p(s.cuda_stream))
        lib.glint_upload_finish(h)
        torch.cuda.synchronize()
        if ok:
            assert rc == 0 and dst.cpu().tolist() == ids
        else:
            assert rc != 0 and "24 bits" in _lib.last_error()


def test_async_upload_wide_ids_use_int32(cuda):
    """N > 2^24: ids no longer fit 24 bits, so the upload narrows to int32 (the
    packed path is only taken when every id fits); ids near 2^24 and N-1 land
    intact."""
    import torch

    from paper_2211_15082_b200 import storage

    n = (1 << 24) + 5
    ptr = np.zeros(n + 1, dtype=np.int64)
    ids = np.array([0, (1 << 24) - 1, 1 << 24, (1 << 24) + 1, n - 1, 12345], dtype=np.int64)
    ptr[3:] = 2                     # node 2 gets ids[0:2]
    ptr[n - 1:] = 6                 # node n-2 gets ids[2:6]
    ptr[-1] = 6
    g = storage.CscGraph(n, 6, ptr, ids)
    copy = torch.cuda.Stream()
    dg = storage.DeviceGraph.upload_async(g, torch.device("cuda"), copy, chunks=2)
    dg.wait_rows()
    torch.cuda.synchronize()
    assert dg.indices.cpu().numpy().tolist() == ids.tolist()


def test_k1_hot_row_l2_steering_same_bytes(cuda, monkeypatch):
    """K1 on the hot-annotated index copy (bit 31 on the most-read source ids,
    evict_last for them and evict_first for the rest) gives the same bytes;
    the annotated ids mask back to the graph's ids."""
    import torch

    from paper_2211_15082_b200 import kernels, synth

    g = synth.gen_products_like(30_000, 30_000 * 20, seed=3, device="cuda")
    monkeypatch.setattr(kernels, "HOT_MB", 4)           # a few thousand hot rows
    h = torch.randn((g.num_nodes, 256), device="cuda")
    sched, nh = kernels.degree_schedule(g.indptr, None, 0, g.num_nodes)
    assert kernels.hot_indices(g, 256 * 4) is None        # first request: not built yet
    ann = kernels.hot_indices(g, 256 * 4)
    assert ann is not None and int((ann < 0).sum()) > 0
    assert torch.equal(ann & 0x7FFFFFFF, g.indices)
    want = torch.empty_like(h)
    kernels.spmm_mean(want, h, g.indptr, g.indices, g.num_nodes, schedule=sched,
                      n_hub=int(nh.item()))
    got = torch.empty_like(h)
    kernels.spmm_mean_hot(got, h, g, g.num_nodes, schedule=sched, n_hub=int(nh.item()))
    assert torch.equal(got, want)
    assert kernels.hot_indices(g, 48 * 4) is None        # narrow rows: no steering


def test_sampling_select_path_equals_sort_path(cuda):
    """fanout <= 32 selects each node's draws with warp bitonic merges; the
    segmented-sort pipeline (GLINT_TUNE_SAMPLE_SORT = 1, and every fanout > 32)
    gives the same sampled graph, for every node and for a node subset, on a
    graph with hub rows and duplicate edges."""
    import torch

    from paper_2211_15082_b200 import _lib, kernels, synth

    g = synth.gen_products_like(30_000, 30_000 * 15, seed=4, device="cuda")
    sub = np.sort(np.random.default_rng(1).choice(g.num_nodes, 5000, replace=False))
    for nodes in (None, sub):
        for fanout in (1, 10, 32):
            a = kernels.sample_neighbors_dev(g, nodes, fanout, 7, 2)
            _lib.call("glint_set_tuning", 15, 1)
            try:
                b = kernels.sample_neighbors_dev(g, nodes, fanout, 7, 2)
            finally:
                _lib.call("glint_set_tuning", 15, 0)
            assert np.array_equal(a.indptr_host, b.indptr_host)
            assert torch.equal(a.indices, b.indices), (fanout, nodes is None)


@pytest.mark.parametrize("dim", [1, 3, 4, 5, 47, 48, 100, 130, 256])
def test_elementwise_row_chunks_pitched_and_gathered(cuda, dim):
    """K5 pointwise kinds on pitched stores (the 16-byte row-chunk kernel, whose
    last chunk reads pad columns it never stores) and on unaligned views (the
    per-element kernel), with row-gathered operands: bytes equal to numpy's
    float32 arithmetic (reference kernels.py:206-231), pads untouched."""
    import torch

    from paper_2211_15082_b200 import kernels
    from paper_2211_15082_b200.storage import pitch_of

    rng = np.random.default_rng(dim)
    n = 777
    p = pitch_of(dim)

    def padded(x, fill):
        t = torch.full((x.shape[0], p + 4), fill, dtype=torch.float32, device="cuda")
        t[:, :dim] = torch.from_numpy(x).cuda()
        return t

    xs = [rng.normal(size=(n, dim)).astype(np.float32) for _ in range(3)]
    xs[0][::7, 0] = np.nan
    xs[0][1::5, -1] = -0.0
    sel = rng.integers(0, n, size=n)
    for aligned in (True, False):
        c0 = 0 if aligned else 1               # a 4-byte offset view: the per-element kernel
        bufs = [padded(x, float("nan")) for x in xs]
        ops = [b[:, c0:c0 + dim] if aligned else torch.roll(b, 1, 1)[:, c0:c0 + dim]
               for b in bufs]
        host = [o.cpu().numpy() for o in ops]
        sel_t = torch.from_numpy(sel).cuda()
        for kind in ("ReLU", "LeakyReLU", "DropoutIdentity", "Add"):
            out_buf = torch.full((n, p + 4), 7.0, device="cuda")
            out = out_buf[:, c0:c0 + dim]
            if kind == "Add":
                kernels.elementwise_into(out, kind, ops, [None, sel_t, None])
                want = (host[0] + host[1][sel]) + host[2]
            else:
                kernels.elementwise_into(out, kind, ops[:1], None)
                x = host[0]
                want = {"ReLU": np.maximum(x, np.float32(0)),
                        "LeakyReLU": np.where(x >= 0, x, np.float32(0.2) * x),
                        "DropoutIdentity": x}[kind]
            got = out_buf.cpu().numpy()
            g, w = got[:, c0:c0 + dim], want.astype(np.float32)
            # NaN kept where numpy keeps it (its payload is not part of the contract);
            # every other element bit-equal (so -0.0 vs +0.0 counts)
            assert (np.isnan(g) == np.isnan(w)).all(), (kind, aligned)
            fin = ~np.isnan(w)
            assert g[fin].tobytes() == w[fin].tobytes(), (kind, aligned)
            # nothing outside the view was written
            assert (got[:, :c0] == 7.0).all() and (got[:, c0 + dim:] == 7.0).all(), (kind, aligned)


@pytest.mark.parametrize("K,N", [(47, 47), (5, 16), (50, 100), (130, 47), (47, 256)])
def test_linear_unaligned_k_pitched_rows(cuda, K, N):
    """K2 with K % 4 != 0 on 16-byte pitched rows (v3's tensor maps zero-fill
    the box beyond K): the same bytes as the v1 kernel and as the row-gathered
    (a_rows) path, and within the 3xTF32 bar of fp64 (reference kernels.py:95-107)."""
    import torch

    from paper_2211_15082_b200 import _lib, kernels
    from paper_2211_15082_b200.storage import pitch_of

    rng = np.random.default_rng(K * 1000 + N)
    M = 3001
    x = rng.normal(size=(M, K)).astype(np.float32)
    w = (rng.normal(size=(N, K)) / np.sqrt(K)).astype(np.float32)
    b = rng.normal(size=N).astype(np.float32)

    def pitched(a, fill=float("nan")):
        t = torch.full((a.shape[0], pitch_of(a.shape[1])), fill, dtype=torch.float32, device="cuda")
        t[:, : a.shape[1]] = torch.from_numpy(a).cuda()
        return t[:, : a.shape[1]]

    xd, wd = pitched(x), pitched(w, 0.0)
    bd = torch.from_numpy(b).cuda()

    def run(**kw):
        o = torch.empty((M, pitch_of(N)), device="cuda")[:, :N]
        kernels.linear_into(o, xd, wd, bd, _lib.ACT_RELU, precision=_lib.PREC_3XTF32, **kw)
        return o.cpu().numpy()

    got = run()
    _lib.call("glint_set_tuning", 4, 1)          # the v1 kernel
    try:
        v1 = run()
    finally:
        _lib.call("glint_set_tuning", 4, 0)
    assert got.tobytes() == v1.tobytes()
    rows = torch.arange(M, device="cuda", dtype=torch.int64)
    assert run(a_rows=rows).tobytes() == got.tobytes()
    ref = np.maximum(x.astype(np.float64) @ w.T.astype(np.float64) + b, 0.0)
    assert rel_l2(got, ref) <= 5e-6


@pytest.mark.parametrize("n_floats", [1, 1 << 20, (2 << 20) + 3, (13 << 20) + 1, 25_000_001])
def test_h2d_pageable_bytes(cuda, n_floats):
    """glint_h2d_pageable (pinned staging on host threads) lands the exact bytes
    of a pageable numpy array, for sizes below, at and across its chunking."""
    import torch

    from paper_2211_15082_b200 import _lib, kernels

    rng = np.random.default_rng(n_floats % 1000)
    a = rng.normal(size=n_floats).astype(np.float32)
    out = torch.empty(n_floats, dtype=torch.float32, device="cuda")
    for threads in (1, 3, 8):
        out.fill_(float("nan"))
        _lib.call("glint_h2d_pageable", out.data_ptr(), a.ctypes.data, a.nbytes, threads,
                  kernels.stream_handle())
        assert out.cpu().numpy().tobytes() == a.tobytes(), threads
    # and through to_device (the path run_inference takes for numpy features)
    t = kernels.to_device(a.reshape(-1, 1) if n_floats % 4 else a.reshape(-1, 4))
    assert t.cpu().numpy().tobytes() == a.tobytes()
