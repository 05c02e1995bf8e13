#!/usr/bin/env python
"""Kernel-level sweep on the headline graph (run on the B200 box).

Times K1 (mean aggregation) for every launch variant at the widths of the
3-layer GCN workload, and K2 (GEMM) in fp32 SIMT vs tcgen05 3xTF32, with CUDA
events on the launching stream, inputs larger than L2.  Prints one JSON line
per measurement.  Also checks every variant's output bytes against variant 0.
"""

from __future__ import annotations

import json
import pathlib
import sys

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def timed(fn, reps=5):
    import torch

    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def main():
    import torch

    from paper_2211_15082_b200 import _lib, kernels, synth
    from paper_2211_15082_b200.executor import agg_bytes

    import argparse

    ap = argparse.ArgumentParser()
    ap.add_argument("--nodes", type=int, default=synth.PRODUCTS_NODES)
    ap.add_argument("--what", default="spmm,gemm")
    ap.add_argument("--dims", default="100,256,48")
    ap.add_argument("--variants", type=int, default=5)
    ap.add_argument("--gemm", default="100x256,256x256,256x47,256x192,100x192")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--tune", action="append", default=[],
                    help="glint_set_tuning KEY=VALUE applied before the sweep")
    args = ap.parse_args()
    args.what = set(args.what.split(","))
    for kv in args.tune:
        k, v = kv.split("=")
        _lib.call("glint_set_tuning", int(k), int(v))
        print(json.dumps({"tuning": {int(k): int(v)}}), flush=True)
    n = args.nodes
    und = int(round(n * synth.PRODUCTS_UNDIRECTED / synth.PRODUCTS_NODES))
    g = synth.gen_products_like(n, und, seed=0, device="cuda") \
        if ("spmm" in args.what or "gat" in args.what) else None
    if g is None:
        if "gatproj" in args.what:
            sweep_gat_project(args, n)
        if "gemm" in args.what:
            gemm_only(args, n)
        return
    deg = g.in_degrees
    hub_pre = int(((deg + 1) >= kernels.HUB_MIN_DEGREE).sum())
    sched, nh = kernels.degree_schedule(g.indptr, None, 0, n)
    assert int(nh.item()) == hub_pre
    print(json.dumps({"graph": {"nodes": n, "edges": g.num_edges, "max_deg": int(deg.max()),
                                "hubs": hub_pre}}), flush=True)
    if "gat" in args.what:
        sweep_gat(args, g, n)
    dims = [int(x) for x in args.dims.split(",")] if "spmm" in args.what else []
    for d in dims:
        h = torch.randn((n, d), device="cuda")
        out = torch.empty_like(h)
        ref = None
        for variant in range(args.variants):
            _lib.call("glint_set_tuning", 0, variant)

            def run():
                kernels.spmm_mean(out, h, g.indptr, g.indices, n, schedule=sched, n_hub=hub_pre)

            ms = timed(run, args.reps)
            nb = agg_bytes(d, g.num_edges, n)
            same = None
            if ref is None:
                ref = out.clone()
            else:
                same = bool(torch.equal(ref, out))
            print(json.dumps({"kernel": "spmm_mean", "dim": d, "variant": variant, "ms": ms,
                              "GBps": nb / ms / 1e6, "identical_to_v0": same}), flush=True)
        # row pitch rounded to 32 B / 128 B (sector / line aligned source rows)
        _lib.call("glint_set_tuning", 0, 0)
        for pad in (4, 8, 32):
            pitch = (d + pad - 1) // pad * pad
            if pitch == d:
                continue
            hp = torch.zeros((n, pitch), device="cuda")
            hp[:, :d] = h
            hv = hp[:, :d]
            op = torch.zeros((n, pitch), device="cuda")
            ov = op[:, :d]
            ms = timed(lambda: kernels.spmm_mean(ov, hv, g.indptr, g.indices, n, schedule=sched,
                                                 n_hub=hub_pre), args.reps)
            out.copy_(ov)
            print(json.dumps({"kernel": "spmm_mean_pitch", "dim": d, "pitch": pitch, "ms": ms,
                              "GBps": agg_bytes(d, g.num_edges, n) / ms / 1e6,
                              "identical_to_v0": bool(torch.equal(ref, out))}), flush=True)
            del hp, hv, op, ov
        # hub rows in the register path of the main kernel (vs bulk-copy hub kernel)
        _lib.call("glint_set_tuning", 0, 0)
        _lib.call("glint_set_tuning", 2, 1)
        ms = timed(lambda: kernels.spmm_mean(out, h, g.indptr, g.indices, n, schedule=sched,
                                             n_hub=hub_pre), args.reps)
        _lib.call("glint_set_tuning", 2, 0)
        print(json.dumps({"kernel": "spmm_mean_hub_inline", "dim": d, "ms": ms,
                          "GBps": agg_bytes(d, g.num_edges, n) / ms / 1e6,
                          "identical_to_v0": bool(torch.equal(ref, out))}), flush=True)
        # the bootstrap batch sizes of layer 1 (contiguous row ranges)
        pos = 0
        for size in (1024, 4096, 16384, 65536, 262144, 1048576):
            if pos + size > n:
                break
            hp = kernels.hub_prefix_dev(g, None, pos, size)
            nh_r = int(hp[-1].item())
            sch, _ = kernels.degree_schedule(g.indptr, None, pos, size)
            o2 = out[pos:pos + size]
            for inline in (2, 3, 4, 1):  # ring: 2 LDGSTS 32-col, 3 TMA 32-col, 4 LDGSTS 64-col; 1 register
                _lib.call("glint_set_tuning", 2, inline)
                ms = timed(lambda: kernels.spmm_mean(o2, h, g.indptr, g.indices, size,
                                                     row_base=pos, schedule=sch, n_hub=nh_r),
                           args.reps)
                e_r = int(g.indptr_host[pos + size] - g.indptr_host[pos])
                print(json.dumps({"kernel": "spmm_mean_batch", "dim": d, "rows": size,
                                  "hubs": nh_r, "hub_inline": inline, "ms": ms,
                                  "GBps": agg_bytes(d, e_r, size) / ms / 1e6}), flush=True)
            _lib.call("glint_set_tuning", 2, 0)
            pos += size
        _lib.call("glint_set_tuning", 8, 1)   # hub rows after the regular rows
        ms = timed(lambda: kernels.spmm_mean(out, h, g.indptr, g.indices, n, schedule=sched,
                                             n_hub=hub_pre), args.reps)
        _lib.call("glint_set_tuning", 8, 0)
        print(json.dumps({"kernel": "spmm_mean_hubs_after", "dim": d, "ms": ms,
                          "GBps": agg_bytes(d, g.num_edges, n) / ms / 1e6,
                          "identical_to_v0": bool(torch.equal(ref, out))}), flush=True)
        # register hub kernel: k CTAs per SM, persistent (0 = one CTA per hub unit)
        for per_sm in (1, 2, 4, 0):
            _lib.call("glint_set_tuning", 6, per_sm)
            ms = timed(lambda: kernels.spmm_mean(out, h, g.indptr, g.indices, n, schedule=sched,
                                                 n_hub=hub_pre), args.reps)
            print(json.dumps({"kernel": "spmm_mean_hub_per_sm", "dim": d, "per_sm": per_sm,
                              "ms": ms, "GBps": agg_bytes(d, g.num_edges, n) / ms / 1e6,
                              "identical_to_v0": bool(torch.equal(ref, out))}), flush=True)
        _lib.call("glint_set_tuning", 6, 0)
        # natural order, no hub path (effect of the LPT schedule)
        _lib.call("glint_set_tuning", 0, 0)
        ms = timed(lambda: kernels.spmm_mean(out, h, g.indptr, g.indices, n))
        print(json.dumps({"kernel": "spmm_mean_nosched", "dim": d, "ms": ms,
                          "GBps": agg_bytes(d, g.num_edges, n) / ms / 1e6,
                          "identical_to_v0": bool(torch.equal(ref, out))}), flush=True)
        del h, out, ref
    shapes = [tuple(int(v) for v in x.split("x")) for x in args.gemm.split(",")] \
        if "gemm" in args.what else []
    for (K, N) in shapes:
        a = torch.randn((n, K), device="cuda")
        w = torch.randn((N, K), device="cuda") / K ** 0.5
        b = torch.randn((N,), device="cuda")
        c = torch.empty((n, (N + 3) // 4 * 4), device="cuda")[:, :N]
        res = {}
        for prec in (0, 1):
            ms = timed(lambda: kernels.linear_into(c, a, w, b, 1, precision=prec), args.reps)
            res[prec] = c.clone()
            print(json.dumps({"kernel": "linear", "K": K, "N": N, "precision": prec, "ms": ms,
                              "TFLOPs": 2 * n * K * N / ms / 1e9,
                              "GBps": (n * K * 4 + n * N * 4) / ms / 1e6}), flush=True)
        err = float((res[0] - res[1]).norm() / res[0].norm())
        print(json.dumps({"kernel": "linear_agree", "K": K, "N": N, "rel_l2_fp32_vs_3xtf32": err}))
        del a, c


def sweep_gat(args, g, n):
    """K4 (GAT edge-softmax aggregation) variants at the cfg3 widths (4 heads x 64 / 47)."""
    import torch

    from paper_2211_15082_b200 import _lib, kernels
    from paper_2211_15082_b200.executor import agg_bytes

    heads = 4
    sched, nh = kernels.degree_schedule(g.indptr, None, 0, n)
    n_hub = int(nh.item())
    for dh in (64, 47):
        hp = kernels.head_pitch(dh)
        Z = torch.randn((n, heads * hp), device="cuda")
        s_src = torch.randn((n, heads), device="cuda")
        s_dst = torch.randn((n, heads), device="cuda")
        out = torch.empty((n, heads * dh), device="cuda")
        ref = None
        for variant in range(args.variants):
            _lib.call("glint_set_tuning", 3, variant)

            def run():
                kernels.gat_aggregate(out, Z, s_src, s_dst, heads, dh, g.indptr, g.indices, n,
                                      schedule=sched, n_hub=n_hub)

            ms = timed(run, args.reps)
            nb = agg_bytes(heads * hp, g.num_edges, n, heads=heads)
            same = None
            if ref is None:
                ref = out.clone()
            else:
                same = bool(torch.equal(ref, out))
            print(json.dumps({"kernel": "gat_aggregate", "heads": heads, "head_dim": dh,
                              "variant": variant, "ms": ms, "GBps": nb / ms / 1e6,
                              "identical_to_v0": same}), flush=True)
        _lib.call("glint_set_tuning", 8, 1)   # hub rows after the regular rows
        for hub_knob in (0, 4, 1):
            _lib.call("glint_set_tuning", 2, hub_knob)
            ms = timed(run, args.reps)
            print(json.dumps({"kernel": "gat_aggregate_hubs_after", "heads": heads,
                              "head_dim": dh, "hub_knob": hub_knob, "ms": ms,
                              "GBps": agg_bytes(heads * hp, g.num_edges, n, heads=heads) / ms / 1e6,
                              "identical_to_v0": bool(torch.equal(ref, out))}), flush=True)
        _lib.call("glint_set_tuning", 2, 0)
        _lib.call("glint_set_tuning", 8, 0)
        for hub_knob in (1, 3):         # hub rows: register CTAs / TMA ring (default: LDGSTS ring)
            _lib.call("glint_set_tuning", 3, 0)
            _lib.call("glint_set_tuning", 2, hub_knob)
            ms = timed(run, args.reps)
            _lib.call("glint_set_tuning", 2, 0)
            print(json.dumps({"kernel": "gat_aggregate_hub_path", "heads": heads, "head_dim": dh,
                              "hub_knob": hub_knob, "ms": ms,
                              "GBps": agg_bytes(heads * hp, g.num_edges, n, heads=heads) / ms / 1e6,
                              "identical_to_v0": bool(torch.equal(ref, out))}), flush=True)
        _lib.call("glint_set_tuning", 3, 0)
        ms = timed(lambda: kernels.gat_aggregate(out, Z, s_src, s_dst, heads, dh, g.indptr,
                                                 g.indices, n), args.reps)
        print(json.dumps({"kernel": "gat_aggregate_no_hub_split", "heads": heads, "head_dim": dh,
                          "ms": ms, "GBps": agg_bytes(heads * hp, g.num_edges, n, heads=heads) / ms / 1e6,
                          "identical_to_v0": bool(torch.equal(ref, out))}), flush=True)
        for variant in range(4):        # two-phase path (edge softmax + weighted SpMM)
            _lib.call("glint_set_tuning", 3, variant)

            def run2():
                kernels.gat_aggregate(out, Z, s_src, s_dst, heads, dh, g.indptr, g.indices, n,
                                      schedule=sched, n_hub=n_hub, edge_range=(0, g.num_edges))

            ms = timed(run2, args.reps)
            print(json.dumps({"kernel": "gat_aggregate_two_phase", "heads": heads, "head_dim": dh,
                              "variant": variant, "ms": ms,
                              "GBps": agg_bytes(heads * hp, g.num_edges, n, heads=heads) / ms / 1e6,
                              "identical_to_v0": bool(torch.equal(ref, out))}), flush=True)
        _lib.call("glint_set_tuning", 3, 0)
        del Z, out, ref


def sweep_gat_project(args, n):
    """GAT projection with the fused score epilogue vs the plain GEMM + scores kernel."""
    import torch

    from paper_2211_15082_b200 import kernels

    for K, H, dh in ((100, 4, 64), (256, 4, 64), (256, 4, 47)):
        h = torch.randn((n, K), device="cuda")
        w = torch.randn((H, dh, K), device="cuda") / K ** 0.5
        att = torch.randn((H, 2 * dh), device="cuda")
        wp = kernels.padded_head_weight(w)
        fused = timed(lambda: kernels.attn_project(h, wp, att, H, dh, precision=1), args.reps)
        Z, s1, s2 = kernels.attn_project(h, wp, att, H, dh, precision=1)
        hp = kernels.head_pitch(dh)
        Zp = torch.empty((n, H * hp), device="cuda")
        plain = timed(lambda: kernels.linear_into(Zp, h, wp, None, 0, precision=1), args.reps)
        print(json.dumps({"kernel": "gat_project", "K": K, "heads": H, "head_dim": dh,
                          "ms_fused_scores": fused, "ms_gemm_only": plain,
                          "Z_identical": bool(torch.equal(Z, Zp))}), flush=True)
        del h, Z, Zp


def gemm_only(args, n):
    import torch

    from paper_2211_15082_b200 import _lib, kernels

    for x in args.gemm.split(","):
        K, N = (int(v) for v in x.split("x"))
        a = torch.randn((n, K), device="cuda")
        w = torch.randn((N, K), device="cuda") / K ** 0.5
        b = torch.randn((N,), device="cuda")
        c = torch.empty((n, (N + 3) // 4 * 4), device="cuda")[:, :N]
        outs = []
        for v1 in (0, 1):
            _lib.call("glint_set_tuning", 4, v1)
            ms = timed(lambda: kernels.linear_into(c, a, w, b, 1, precision=1), args.reps)
            outs.append(c.clone())
            print(json.dumps({"kernel": "linear", "K": K, "N": N, "precision": 1,
                              "impl": "v1" if v1 else "v2", "ms": ms,
                              "TFLOPs": 2 * n * K * N / ms / 1e9,
                              "GBps": (n * K * 4 + n * N * 4) / ms / 1e6}), flush=True)
        _lib.call("glint_set_tuning", 4, 0)
        if N <= 128:                    # 128-row tiles (experiment knob 7 = 3)
            _lib.call("glint_set_tuning", 7, 3)
            ms = timed(lambda: kernels.linear_into(c, a, w, b, 1, precision=1), args.reps)
            _lib.call("glint_set_tuning", 7, 0)
            print(json.dumps({"kernel": "linear_128row_tiles", "K": K, "N": N, "ms": ms,
                              "TFLOPs": 2 * n * K * N / ms / 1e9,
                              "identical": bool(torch.equal(c, outs[0]))}), flush=True)
        if 128 < N <= 256:              # 256-row x N/2 tiles instead of 128-row x N
            _lib.call("glint_set_tuning", 7, 2)
            ms = timed(lambda: kernels.linear_into(c, a, w, b, 1, precision=1), args.reps)
            _lib.call("glint_set_tuning", 7, 0)
            print(json.dumps({"kernel": "linear_256row_tiles", "K": K, "N": N, "ms": ms,
                              "TFLOPs": 2 * n * K * N / ms / 1e9,
                              "identical": bool(torch.equal(c, outs[0]))}), flush=True)
        for diag, name in ((2, "linear_mma_only"), (3, "linear_no_lo_pass")):
            _lib.call("glint_set_tuning", 1, diag)   # diagnostics (wrong results)
            ms = timed(lambda: kernels.linear_into(c, a, w, b, 1, precision=1), args.reps)
            _lib.call("glint_set_tuning", 1, 0)
            print(json.dumps({"kernel": name, "K": K, "N": N, "ms": ms,
                              "TFLOPs": 2 * n * K * N / ms / 1e9}), flush=True)
        print(json.dumps({"kernel": "linear_v1_v2_identical", "K": K, "N": N,
                          "identical": bool(torch.equal(outs[0], outs[1]))}), flush=True)


if __name__ == "__main__":
    main()
