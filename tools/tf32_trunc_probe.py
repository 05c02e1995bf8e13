#!/usr/bin/env python
"""Does tcgen05.mma kind::tf32 ignore the low 13 mantissa bits of an fp32
operand (truncation)?  Runs the split-TF32 GEMM once with the masked "hi"
operand and once with the raw fp32 word in its place; identical bytes over
random data mean the tensor core truncates."""
import json
import pathlib
import sys

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import torch

    from paper_2211_15082_b200 import _lib, kernels

    torch.manual_seed(0)
    for (M, K, N) in ((4096, 256, 256), (3000, 100, 48), (512, 64, 128)):
        a = torch.randn((M, K), device="cuda") * 3
        w = torch.randn((N, K), device="cuda") / K ** 0.5
        c0 = torch.empty((M, N), device="cuda")
        c1 = torch.empty((M, N), device="cuda")
        _lib.call("glint_set_tuning", 4, 1)      # v1 kernel: explicit hi/lo split
        kernels.linear_into(c0, a, w, None, 0, precision=1)
        _lib.call("glint_set_tuning", 5, 1)      # ... with the raw fp32 word as "hi"
        kernels.linear_into(c1, a, w, None, 0, precision=1)
        _lib.call("glint_set_tuning", 5, 0)
        _lib.call("glint_set_tuning", 4, 0)
        ref = (a.double() @ w.double().T)
        e0 = float((c0.double() - ref).norm() / ref.norm())
        e1 = float((c1.double() - ref).norm() / ref.norm())
        print(json.dumps({"M": M, "K": K, "N": N, "identical": bool(torch.equal(c0, c1)),
                          "max_abs_diff": float((c0 - c1).abs().max()),
                          "rel_l2_masked": e0, "rel_l2_raw": e1}), flush=True)


if __name__ == "__main__":
    main()
