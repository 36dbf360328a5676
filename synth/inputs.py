"""Seeded synthetic inputs for the K-FAC hot path (CPU, torch generators).

This module is shared by the oracle side (tests) and the CUDA side (tests,
bench.py).  It holds none of the method's arithmetic: it only draws tensors
with the structure of the paper's workload:

  x   layer input, NHWC  [N, H_in, W_in, C_in] (FC: [N, C_in]),
      ReLU(N(0,1)) (post-BN-ReLU activations; the network stem input is N(0,1))
  gy  gradient w.r.t. the layer output, NHWC [N, H_out, W_out, C_out]
      (FC: [N, C_out]), N(0,1)
  dW  the rank-local weight gradient [C_out, dA] fp32 N(0,1) (bias column last)

Every per-sample tensor is drawn from its own generator, seeded by
(seed, layer index, tensor id, GLOBAL sample index), so the global batch is
identical for every world size P: rank r holds global samples
[r*n_local, (r+1)*n_local).  dW is seeded by the rank (a rank-local gradient).
Half-precision tensors are produced by round-to-nearest-even from fp32.
"""

from __future__ import annotations

import numpy as np
import torch

from . import shapes

_M64 = (1 << 64) - 1


def _mix(*vals: int) -> int:
    """splitmix64 over a tuple of integers -> 63-bit seed (stable, platform-free)."""
    h = 0x9E3779B97F4A7C15
    for v in vals:
        z = (h + (v & _M64) * 0xBF58476D1CE4E5B9 + 0x94D049BB133111EB) & _M64
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
        h = z ^ (z >> 31)
    return h & ((1 << 63) - 1)


TID_X, TID_GY, TID_DW = 0, 1, 2

_HALF = {"bf16": torch.bfloat16, "fp16": torch.float16}


def _sample(seed, li, tid, ng, shape, relu):
    g = torch.Generator().manual_seed(_mix(seed, li, tid, ng))
    t = torch.randn(shape, generator=g, dtype=torch.float32)
    if relu:
        t.clamp_(min=0.0)
    return t


def layer_x(layer, li, n_local, rank=0, seed=1811, dtype="bf16", stem=None):
    """x for layer `li` on `rank`: [n_local, H, W, C] (conv) or [n_local, C] (FC)."""
    if stem is None:
        stem = li == 0
    if layer["kind"] == 1:
        shp = (layer["c_in"],)
    else:
        shp = (layer["h_in"], layer["w_in"], layer["c_in"])
    out = torch.empty((n_local,) + shp, dtype=_HALF[dtype])
    for n in range(n_local):
        out[n] = _sample(seed, li, TID_X, rank * n_local + n, shp, relu=not stem).to(_HALF[dtype])
    return out


def layer_gy(layer, li, n_local, rank=0, seed=1811, dtype="bf16"):
    """gy for layer `li` on `rank`: [n_local, Ho, Wo, C_out] (conv) or [n_local, C_out] (FC)."""
    if layer["kind"] == 1:
        shp = (layer["c_out"],)
    else:
        ho, wo = shapes.out_hw(layer)
        shp = (ho, wo, layer["c_out"])
    out = torch.empty((n_local,) + shp, dtype=_HALF[dtype])
    for n in range(n_local):
        out[n] = _sample(seed, li, TID_GY, rank * n_local + n, shp, relu=False).to(_HALF[dtype])
    return out


def layer_dw(layer, li, rank=0, seed=1811):
    """Rank-local gradient dW [C_out, dA] fp32 (bias column last)."""
    d_a, d_g = shapes.dims(layer)
    g = torch.Generator().manual_seed(_mix(seed, li, TID_DW, rank))
    return torch.randn((d_g, d_a), generator=g, dtype=torch.float32)


def half_bits(t: torch.Tensor) -> np.ndarray:
    """The raw 16-bit patterns of a bf16/fp16 tensor as a contiguous uint16 array."""
    return t.contiguous().view(torch.int16).numpy().view(np.uint16)


def rank_inputs(layers, n_local, rank=0, seed=1811, dtype="bf16"):
    """All inputs of one rank: lists xs, gys (half, CPU) and dWs (fp32, CPU)."""
    xs = [layer_x(L, i, n_local, rank, seed, dtype) for i, L in enumerate(layers)]
    gys = [layer_gy(L, i, n_local, rank, seed, dtype) for i, L in enumerate(layers)]
    dws = [layer_dw(L, i, rank, seed) for i, L in enumerate(layers)]
    return xs, gys, dws
