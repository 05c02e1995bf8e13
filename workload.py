"""The bench workload (BASELINE.json configs[1]/[2]) shared by BOTH bench arms.

Torch + numpy only: this module never imports ``paper_2211_15082_b200`` or
loads its library, so ``bench.py --impl reference`` can build exactly the
same inputs as the B200 arm without touching the product.

* ``products_like_csc`` -- the OGBN-Products-shaped symmetric graph
  (2,449,029 nodes, 61,859,140 undirected edges stored both ways =
  123,718,280 in-edges, Chung-Lu degrees, slices ascending), drawn with a
  seeded torch generator on ``device``.  The same draw sequence as
  ``paper_2211_15082_b200.synth.gen_products_like`` (tests assert the bytes
  are equal), returned as plain int64 (indptr, indices) tensors.
* ``features`` -- N(0,1) fp32 node features (same stream as
  ``synth.gen_features_device``).
* ``gcn_params`` / ``gat_params`` -- the random-init weights of
  ``synth.build_gcn`` / ``synth.build_gat`` (the reference's numpy draw
  sequence, glint/synth.py), as plain arrays.
"""

from __future__ import annotations

import numpy as np

PRODUCTS_NODES = 2_449_029
PRODUCTS_UNDIRECTED = 61_859_140


def products_like_csc(n=PRODUCTS_NODES, n_undirected=PRODUCTS_UNDIRECTED, seed=0, alpha=0.45,
                      device="cuda"):
    """(indptr int64 [n+1], indices int64 [2*n_undirected]) on `device`."""
    import torch

    dev = torch.device(device)
    gen = torch.Generator(device=dev)
    gen.manual_seed(int(seed) * 1_000_003 + 20)
    w = torch.arange(1, n + 1, device=dev, dtype=torch.float64).pow_(-alpha)
    label = torch.randperm(n, generator=gen, device=dev)
    wn = torch.empty_like(w)
    wn[label] = w
    cdf = torch.cumsum(wn, 0)
    cdf /= cdf[-1].clone()
    keys = torch.zeros(0, dtype=torch.int64, device=dev)
    while keys.numel() < n_undirected:
        m = int((n_undirected - keys.numel()) * 1.08) + 4096
        a = torch.searchsorted(cdf, torch.rand(m, generator=gen, device=dev, dtype=torch.float64),
                               right=True).clamp_(max=n - 1)
        b = torch.searchsorted(cdf, torch.rand(m, generator=gen, device=dev, dtype=torch.float64),
                               right=True).clamp_(max=n - 1)
        lo, hi = torch.minimum(a, b), torch.maximum(a, b)
        keep = lo != hi
        keys = torch.unique(torch.cat([keys, lo[keep] * n + hi[keep]]))
        del a, b, lo, hi, keep
    if keys.numel() > n_undirected:
        pick = torch.randperm(keys.numel(), generator=gen, device=dev)[:n_undirected]
        keys = torch.sort(keys[pick]).values
    lo, hi = keys // n, keys % n
    del keys
    dst = torch.cat([lo, hi])
    src = torch.cat([hi, lo])
    del lo, hi
    order = torch.sort(dst * n + src).values
    dst = order // n
    src = order - dst * n
    del order
    counts = torch.bincount(dst, minlength=n)
    indptr = torch.zeros(n + 1, dtype=torch.int64, device=dev)
    torch.cumsum(counts, 0, out=indptr[1:])
    return indptr, src


def features(n, dim, seed=0, device="cuda"):
    """N(0,1) fp32 [n, dim]."""
    import torch

    gen = torch.Generator(device=torch.device(device))
    gen.manual_seed(int(seed) * 1_000_003 + 3)
    return torch.randn((n, dim), generator=gen, device=device, dtype=torch.float32)


def _w(rng, shape):
    return rng.normal(0.0, 1.0 / np.sqrt(shape[-1]), size=shape).astype(np.float32)


def gcn_params(input_dim, hidden, out_dim, layers, seed=0):
    """[(weight [d_out, d_in], bias [d_out])] per ConvMean layer; ReLU between layers."""
    rng = np.random.default_rng([seed, 10, layers])
    out, width = [], input_dim
    for i in range(1, layers + 1):
        d = out_dim if i == layers else hidden
        out.append((_w(rng, (d, width)), np.zeros(d, np.float32)))
        width = d
    return out


def gat_params(input_dim, head_dim, out_dim, layers, heads=2, seed=0):
    """[(weight [H, dh, d_in], attn [H, 2*dh])] per ConvAttn layer; ReLU between layers."""
    rng = np.random.default_rng([seed, 11, layers])
    out, width = [], input_dim
    for i in range(1, layers + 1):
        dh = out_dim if i == layers else head_dim
        out.append((_w(rng, (heads, dh, width)), _w(rng, (heads, 2 * dh))))
        width = heads * dh
    return out


def cpu_model_name() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform

    return platform.processor() or "unknown"
