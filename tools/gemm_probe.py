#!/usr/bin/env python
"""K2/K3 GEMM probe (run on the B200 box): v3 (tensor-map TMA, CTA pairs,
resident W) against v2 on the workload's shapes.

For each shape: CUDA-event time per call (inputs larger than L2, 5 reps after
a warm-up), rel-L2 of a 4096-row sample against an fp64 host product, and
whether v3's bytes equal v2's.  One JSON line per (shape, kernel).

  python tools/gemm_probe.py [--m 2449029] [--shapes 100x256r,256x256r,256x47,...]
Shape tokens: KxN, suffix r = ReLU epilogue with bias, s = GAT score
epilogue (N = heads x head_dim, 4 heads).
"""

from __future__ import annotations

import argparse
import json
import pathlib
import sys

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import numpy as np
    import torch

    from paper_2211_15082_b200 import _lib, kernels

    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=2_449_029)
    ap.add_argument("--shapes", default="100x256r,256x256r,256x47,128x128r,128x172,100x256s,256x256s,256x188s")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--kernels", default="3,2")
    ap.add_argument("--tune", action="append", default=[], help="glint_set_tuning KEY=VALUE")
    args = ap.parse_args()
    tune = {}
    for kv in args.tune:
        k, v = kv.split("=")
        _lib.call("glint_set_tuning", int(k), int(v))
        tune[int(k)] = int(v)
    M = args.m
    torch.manual_seed(0)
    for tok in args.shapes.split(","):
        kind = tok[-1] if tok[-1] in "rs" else ""
        K, N = (int(v) for v in tok.rstrip("rs").split("x"))
        x = torch.randn((M, K), device="cuda")
        w = torch.randn((N, K), device="cuda") / K ** 0.5
        b = torch.randn(N, device="cuda") if kind == "r" else None
        act = _lib.ACT_RELU if kind == "r" else _lib.ACT_NONE
        sample = torch.randint(0, M, (4096,), device="cuda")
        sample[:2] = torch.tensor([0, M - 1])
        xs = x[sample].double().cpu()
        want = xs @ w.double().cpu().T
        if b is not None:
            want = want + b.double().cpu()
        if act == _lib.ACT_RELU:
            want = want.clamp_min(0)
        heads = 4
        if kind == "s":
            hd = N // heads
            attn = torch.randn((heads, 2 * hd), device="cuda") / hd ** 0.5
            w_pad = kernels.padded_head_weight(w.reshape(heads, hd, K))
            pitch = kernels.head_pitch(hd)
            wp = w_pad.reshape(heads, pitch, K)[:, :hd, :].reshape(N, K).double().cpu()
            want = xs @ wp.T
        outs = {}
        for kv in (int(v) for v in args.kernels.split(",")):
            _lib.call("glint_set_tuning", 9, 1 if kv == 2 else tune.get(9, 0))
            if kind == "s":
                # outputs allocated once: a fresh 2.5 GB Z per call put cudaMalloc
                # inside the timed reps (noisy, up to 10x)
                pitch = kernels.head_pitch(hd)
                out = (torch.empty((M, heads * pitch), device="cuda"),
                       torch.empty((M, heads), device="cuda"), torch.empty((M, heads), device="cuda"))

                def run():
                    kernels.attn_project(x, w_pad, attn, heads, hd, precision=_lib.PREC_3XTF32,
                                         out=out)
            else:
                out = torch.empty((M, N), device="cuda")

                def run():
                    kernels.linear_into(out, x, w, b, act, precision=_lib.PREC_3XTF32)
            run()
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            for _ in range(args.reps):
                run()
            e.record()
            torch.cuda.synchronize()
            ms = s.elapsed_time(e) / args.reps
            z = out[0] if isinstance(out, tuple) else out
            if kind == "s":
                pitch = kernels.head_pitch(N // heads)
                z = z.reshape(M, heads, pitch)[:, :, :N // heads].reshape(M, N)
            got = z[sample].double().cpu()
            err = float((got - want).norm() / want.norm())
            sc_err = None
            if kind == "s":
                hd = N // heads
                wz = want.reshape(-1, heads, hd)
                a64 = attn.double().cpu()
                ws = (wz * a64[None, :, :hd]).sum(-1)
                wd = (wz * a64[None, :, hd:]).sum(-1)
                gs, gd = out[1][sample].double().cpu(), out[2][sample].double().cpu()
                sc_err = max(float((gs - ws).norm() / ws.norm()), float((gd - wd).norm() / wd.norm()))
            flops = 3 * 2 * M * N * K
            hbm = 4 * M * (K + N)
            outs[kv] = z
            rec = {"tune": tune, "shape": tok, "M": M, "K": K, "N": N, "kernel": f"v{kv}", "ms": round(ms, 4),
                   "rel_l2_vs_fp64": err, "tflops_3x": round(flops / ms / 1e9, 1),
                   "hbm_gbs": round(hbm / ms / 1e6, 1)}
            if sc_err is not None:
                rec["scores_rel_l2_vs_fp64"] = sc_err
            if kv != 3 and 3 in outs:
                rec["bytes_equal_v3"] = bool(torch.equal(outs[3], z))
            print(json.dumps(rec), flush=True)
        _lib.call("glint_set_tuning", 9, tune.get(9, 0))
        del x, w, outs


if __name__ == "__main__":
    main()
