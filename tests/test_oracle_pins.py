"""Pins for the fp64 oracle against what the paper and the mathematics fix.

Each test pins an oracle function to something other than itself: values
printed in SPEC.md / PAPER.md (tests/golden/*.json, cited), closed forms,
library routines on special cases (LAPACK inverse, torch unfold/conv2d,
numpy kron/solve), invariants (symmetry, PSD, residuals, P-invariance).
"""
import json
import math
import os

import numpy as np
import pytest
import torch

from synth import shapes, inputs

GOLD = os.path.join(os.path.dirname(__file__), "golden")
SPEC = json.load(open(os.path.join(GOLD, "spec_examples.json")))


def _fc(c_in, c_out=1, bias=0):
    return shapes.linear("fc", c_in, c_out, bias)


def _bits(a):
    """Exact bf16 bit patterns of small float arrays (test values are bf16-exact)."""
    t = torch.as_tensor(np.asarray(a, dtype=np.float32)).to(torch.bfloat16)
    assert torch.equal(t.float(), torch.as_tensor(np.asarray(a, dtype=np.float32)))
    return inputs.half_bits(t)


def relerr(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(np.asarray(b)), 1e-300))


# ---------------------------------------------------------------- packing
def test_pack_spec_examples(orc):
    e = SPEC["pack_identity3"]
    assert orc.pack(np.array(e["input"], float)).tolist() == e["expected"]
    e = SPEC["unpack_213"]
    assert orc.unpack(np.array(e["input"], float)).tolist() == e["expected"]
    for k in ("packed_count_2304", "packed_count_100"):
        assert orc.packed_len(SPEC[k]["dim"]) == SPEC[k]["expected"]
    rng = np.random.default_rng(0)
    B = rng.standard_normal((100, 100))
    assert len(orc.pack(B + B.T)) == SPEC["packed_count_100"]["expected"]


def test_pack_roundtrip_bitwise(orc):
    rng = np.random.default_rng(1)
    for n in (1, 2, 5, 17, 64):
        B = rng.standard_normal((n, n))
        S = B + B.T
        assert np.array_equal(orc.unpack(orc.pack(S)), S)
        # row-major upper order: element (i, j) at i*n - i(i-1)/2 + (j - i)
        p = orc.pack(S)
        for i in range(n):
            for j in range(i, n):
                assert p[i * n - i * (i - 1) // 2 + (j - i)] == S[i, j]
    with pytest.raises(ValueError):
        orc.pack(rng.standard_normal((4, 4)))
    with pytest.raises(ValueError):
        orc.unpack(np.zeros(5))


# ---------------------------------------------------------------- inverse
def test_inverse_spec_examples(orc):
    e = SPEC["invert_scalar"]
    X, st = orc.inverse(e["c"] * np.eye(4))
    assert st == 0 and np.allclose(X, e["expected_diag"] * np.eye(4), rtol=1e-15, atol=0)
    e = SPEC["invert_2x2"]
    X, st = orc.inverse(np.array(e["input"], float))
    assert st == 0 and np.allclose(X, np.array(e["expected"]), rtol=1e-15, atol=1e-16)


@pytest.mark.parametrize("n", [1, 3, 8, 33, 64, 130])
def test_inverse_vs_lapack_and_residual(orc, n):
    rng = np.random.default_rng(n)
    B = rng.standard_normal((n, n))
    M = B.T @ B + np.eye(n)
    X, st = orc.inverse(M)
    assert st == 0
    assert np.linalg.norm(M @ X - np.eye(n)) <= 1e-8 * n
    assert relerr(X, np.linalg.inv(M)) < 1e-12  # LAPACK getrf/getri
    L, st = orc.cholesky(M)
    assert st == 0 and np.allclose(L, np.linalg.cholesky(M), rtol=1e-12, atol=1e-12)


def test_inverse_reports_pivot(orc):
    M = np.diag([1.0, 2.0, -1.0, 3.0])
    _, st = orc.inverse(M)
    assert st == 3  # failing pivot index 2, reported +1
    _, st = orc.inverse(np.zeros((2, 2)))
    assert st == 1


# ---------------------------------------------------------------- factors
def test_factor_spec_examples(orc):
    for k in ("a_factor_single_row", "a_factor_orthonormal", "a_factor_zero_bias"):
        e = SPEC[k]
        rows = np.array(e["rows"], float)
        layer = _fc(rows.shape[1], bias=e["bias"])
        A = orc.factor_A(layer, _bits(rows), rows.shape[0])
        assert A.tolist() == e["expected"], k
    for k in ("g_factor_single", "g_factor_orthonormal"):
        e = SPEC[k]
        rows = np.array(e["rows"], float)
        G = orc.factor_G(_bits(rows), rows.shape[0], rows.shape[1])
        assert G.tolist() == e["expected"], k


GEOMS = [  # (C_in, k, stride, pad, H, W, bias, N)
    (16, 3, 1, 1, 8, 8, 1, 2),      # config-1 geometry
    (3, 7, 2, 3, 13, 11, 0, 2),     # stem-like, ragged spatial size
    (8, 1, 2, 0, 9, 9, 0, 3),       # strided 1x1 downsample
    (5, 3, 2, 1, 7, 6, 1, 1),       # odd channels, stride 2
    (4, 1, 1, 0, 5, 5, 0, 2),       # plain 1x1
]


def _rand_x(rng, N, H, W, C, relu=True):
    x = rng.standard_normal((N, H, W, C)).astype(np.float32)
    if relu:
        x = np.maximum(x, 0)
    t = torch.as_tensor(x).to(torch.bfloat16)
    return t, inputs.half_bits(t)


@pytest.mark.parametrize("geom", GEOMS)
def test_factor_A_vs_torch_unfold(orc, geom):
    """Library im2col (torch.nn.functional.unfold) + matmul reproduces A (R-5..R-7)."""
    C, k, s, p, H, W, bias, N = geom
    layer = dict(kind=0, c_in=C, c_out=1, kh=k, kw=k, stride_h=s, stride_w=s, pad_h=p, pad_w=p,
                 h_in=H, w_in=W, has_bias=bias)
    rng = np.random.default_rng(sum(geom))
    t, bits = _rand_x(rng, N, H, W, C, relu=False)
    A = orc.factor_A(layer, bits, N)
    xn = t.double().permute(0, 3, 1, 2)  # NCHW
    cols = torch.nn.functional.unfold(xn, k, padding=p, stride=s)  # [N, C*k*k, L], (c, kh, kw)
    Lp = cols.shape[-1]
    cols = cols.reshape(N, C, k, k, Lp).permute(0, 4, 2, 3, 1).reshape(N * Lp, k * k * C)  # (kh, kw, c)
    if bias:
        cols = torch.cat([cols, torch.ones(N * Lp, 1, dtype=torch.float64)], 1)
    Aref = (cols.T @ cols / cols.shape[0]).numpy()
    assert A.shape == Aref.shape
    assert relerr(A, Aref) < 1e-13
    assert np.array_equal(A, A.T)


@pytest.mark.parametrize("geom", GEOMS[:4])
def test_factor_A_quadratic_form_vs_conv2d(orc, geom):
    """vᵀAv = α‖conv2d(x, v)‖² for any filter v (independent of im2col)."""
    C, k, s, p, H, W, bias, N = geom
    layer = dict(kind=0, c_in=C, c_out=1, kh=k, kw=k, stride_h=s, stride_w=s, pad_h=p, pad_w=p,
                 h_in=H, w_in=W, has_bias=bias)
    rng = np.random.default_rng(7 + sum(geom))
    t, bits = _rand_x(rng, N, H, W, C)
    A = orc.factor_A(layer, bits, N)
    for trial in range(3):
        v = rng.standard_normal(A.shape[0])
        filt = torch.as_tensor(v[:k * k * C].reshape(k, k, C)).permute(2, 0, 1)[None]  # [1,C,k,k]
        b = torch.tensor([v[-1]], dtype=torch.float64) if bias else None
        y = torch.nn.functional.conv2d(t.double().permute(0, 3, 1, 2), filt, b, stride=s, padding=p)
        q = float((y ** 2).sum()) / y.numel()
        assert abs(v @ A @ v - q) <= 1e-12 * abs(q)


def test_factor_A_1x1_is_gram(orc):
    rng = np.random.default_rng(3)
    t, bits = _rand_x(rng, 3, 4, 5, 6)
    layer = dict(kind=0, c_in=6, c_out=1, kh=1, kw=1, stride_h=1, stride_w=1, pad_h=0, pad_w=0,
                 h_in=4, w_in=5, has_bias=0)
    X = t.double().reshape(-1, 6).numpy()
    assert relerr(orc.factor_A(layer, bits, 3), X.T @ X / X.shape[0]) < 1e-14


def test_factor_entries_match_full(orc):
    rng = np.random.default_rng(4)
    C, k, s, p, H, W, bias, N = GEOMS[0]
    layer = dict(kind=0, c_in=C, c_out=1, kh=k, kw=k, stride_h=s, stride_w=s, pad_h=p, pad_w=p,
                 h_in=H, w_in=W, has_bias=bias)
    t, bits = _rand_x(rng, N, H, W, C)
    A = orc.factor_A(layer, bits, N)
    ij = rng.integers(0, A.shape[0], size=(50, 2))
    assert np.allclose(orc.factor_A_entries(layer, bits, N, ij), A[ij[:, 0], ij[:, 1]], rtol=1e-13, atol=1e-15)
    g = rng.standard_normal((40, 9)).astype(np.float32)
    gb = _bits(torch.as_tensor(g).to(torch.bfloat16).float().numpy())
    G = orc.factor_G(gb, 40, 9)
    ij = rng.integers(0, 9, size=(20, 2))
    assert np.allclose(orc.factor_G_entries(gb, 40, 9, ij), G[ij[:, 0], ij[:, 1]], rtol=1e-13, atol=1e-15)


def test_factors_symmetric_psd(orc):
    layer = shapes.single_conv()[0]
    x = inputs.layer_x(layer, 0, 4, stem=False)
    gy = inputs.layer_gy(layer, 0, 4)
    A = orc.factor_A(layer, inputs.half_bits(x), 4)
    G = orc.factor_G(inputs.half_bits(gy), shapes.rows(layer, 4), 32)
    for M in (A, G):
        assert np.array_equal(M, M.T)
        assert np.linalg.eigvalsh(M).min() >= -1e-10 * np.linalg.norm(M)


def test_exact_fim_special_case(orc):
    """One example, FC layer: G ⊗ A equals the exact empirical FIM block.

    The per-example gradient of W (dG x dA, row-major vec) is g ãᵀ, so
    vec(∇)vec(∇)ᵀ = (g⊗ã)(g⊗ã)ᵀ = (g gᵀ)⊗(ã ãᵀ) = G ⊗ A.
    """
    rng = np.random.default_rng(5)
    a = rng.standard_normal(3).astype(np.float32)
    g = rng.standard_normal(2).astype(np.float32)
    ab = torch.as_tensor(a).to(torch.bfloat16)
    gb = torch.as_tensor(g).to(torch.bfloat16)
    A = orc.factor_A(_fc(3, bias=1), inputs.half_bits(ab), 1)
    G = orc.factor_G(inputs.half_bits(gb), 1, 2)
    at = np.concatenate([ab.double().numpy(), [1.0]])
    grad = np.outer(gb.double().numpy(), at).reshape(-1)
    assert np.allclose(np.kron(G, A), np.outer(grad, grad), rtol=1e-15, atol=1e-15)


def test_factor_P_invariance(orc):
    """Mean over P equal shards of per-shard factors = factor of the global batch."""
    layer = shapes.single_conv()[0]
    n_glob = 8
    xg = inputs.layer_x(layer, 0, n_glob, rank=0, stem=False)
    A1 = orc.factor_A(layer, inputs.half_bits(xg), n_glob)
    for P in (2, 4):
        nl = n_glob // P
        acc = 0
        for r in range(P):
            xr = inputs.layer_x(layer, 0, nl, rank=r, stem=False)
            assert torch.equal(xr, xg[r * nl:(r + 1) * nl])  # generator is global-index seeded
            acc = acc + orc.factor_A(layer, inputs.half_bits(xr), nl)
        assert relerr(acc / P, A1) < 1e-13


# ---------------------------------------------------------------- damping
def test_damping_spec_examples(orc):
    for k in ("damp_identity", "damp_ratio"):
        e = SPEC[k]
        A = e["trA_per_dim"] * np.eye(e["dA"])
        G = e["trG_per_dim"] * np.eye(e["dG"])
        Ad, Gd, pi = orc.damp(A, G, e["gamma"])
        assert abs(pi - e["pi"]) < 1e-15
        assert np.allclose(Ad - A, e["a_add"] * np.eye(e["dA"]), rtol=1e-14, atol=0)
        assert np.allclose(Gd - G, e["g_add"] * np.eye(e["dG"]), rtol=1e-14, atol=0)
    Ad, Gd, pi = orc.damp(np.zeros((2, 2)), np.eye(2), 0.04)
    assert pi == 1.0  # a zero trace falls back to pi = 1
    with pytest.raises(ValueError):
        orc.damp(np.eye(2), np.eye(2), 0.0)


def test_damped_kronecker_dominates_tikhonov(orc):
    """(G+cI)⊗(A+dI) ⪰ G⊗A + γI with c·d = γ (the factored form damps at least γ; R-1)."""
    rng = np.random.default_rng(6)
    for _ in range(5):
        Ba, Bg = rng.standard_normal((3, 3)), rng.standard_normal((2, 2))
        A, G = Ba @ Ba.T, Bg @ Bg.T
        Ad, Gd, pi = orc.damp(A, G, 0.3)
        D = np.kron(Gd, Ad) - np.kron(G, A) - 0.3 * np.eye(6)
        assert np.linalg.eigvalsh(D).min() >= -1e-12


def test_warmup_damping_schedule(orc):
    e = SPEC["warmup_damping_bs4096"]
    a = orc.damping_alpha(e["gamma0"], e["gamma_target"], e["t_warmup"])
    assert abs(a - e["alpha"]) < 1e-15 and abs(a - 4 / 313) < 1e-15
    g = orc.damping_schedule(e["gamma0"], e["gamma_target"], e["t_warmup"], 400)
    assert abs(g[1] - e["gamma1"]) <= 5e-8  # printed to 6 significant digits
    d = [abs(v - e["gamma_target"]) for v in g]
    assert all(d[i + 1] < d[i] for i in range(len(d) - 1))  # monotone contraction
    assert orc.damping_schedule(1e-3, 1e-3 / 10, 10, 1)[0] == 1e-3
    fixed = orc.damping_schedule(2.5e-4, 2.5e-4 / 100, 50, 0)
    assert fixed == [2.5e-4]


# ---------------------------------------------------------------- precondition
def test_precondition_identity(orc):
    e = SPEC["precondition_identity"]
    rng = np.random.default_rng(8)
    dW = rng.standard_normal((3, 4))
    Ad, Gd, _ = orc.damp(np.eye(4), np.eye(3), e["gamma"])
    Ai, _ = orc.inverse(Ad)
    Gi, _ = orc.inverse(Gd)
    assert np.allclose(orc.precondition(Gi, Ai, dW), dW / e["scale"], rtol=1e-14, atol=0)
    assert np.allclose(orc.precondition(2 * np.eye(3), 3 * np.eye(4), dW), 6 * dW, rtol=1e-15, atol=0)


@pytest.mark.parametrize("da,dg", [(1, 1), (3, 2), (5, 4), (8, 8), (7, 3)])
def test_kronecker_identity_explicit(orc, da, dg):
    """(G_d⊗A_d)⁻¹ vec_row(∇W) = vec_row(G_d⁻¹ ∇W A_d⁻¹) with explicit Kronecker products
    (P:247-273 Eqs. inv_fim, K-FAC update; R-14: also (A_d⊗G_d)⁻¹ vec_col)."""
    rng = np.random.default_rng(100 * da + dg)
    Ba, Bg = rng.standard_normal((da, 2 * da)), rng.standard_normal((dg, 2 * dg))
    Ad, Gd, _ = orc.damp(Ba @ Ba.T / 2, Bg @ Bg.T / 2, 2.5e-2)
    dW = rng.standard_normal((dg, da))
    Ai, _ = orc.inverse(Ad)
    Gi, _ = orc.inverse(Gd)
    pre = orc.precondition(Gi, Ai, dW)
    ref_row = np.linalg.solve(np.kron(Gd, Ad), dW.reshape(-1))
    assert relerr(pre.reshape(-1), ref_row) < 1e-10
    ref_col = np.linalg.solve(np.kron(Ad, Gd), dW.reshape(-1, order="F"))
    assert relerr(pre.reshape(-1, order="F"), ref_col) < 1e-10
    ij = np.array([[i, j] for i in range(dg) for j in range(da)])
    assert np.allclose(orc.precondition_entries(Gi, Ai, dW, ij), pre.reshape(-1), rtol=1e-12, atol=1e-14)


def test_large_gamma_limit(orc):
    """γ→∞: ‖γ𝒢 − ∇W‖/‖∇W‖ ≤ 0.01 at γ = 1e6 on unit-scale factors."""
    rng = np.random.default_rng(9)
    Ba, Bg = rng.standard_normal((6, 12)), rng.standard_normal((4, 8))
    A, G = Ba @ Ba.T / 12, Bg @ Bg.T / 8
    dW = rng.standard_normal((4, 6))
    Ad, Gd, _ = orc.damp(A, G, 1e6)
    pre = orc.precondition(orc.inverse(Gd)[0], orc.inverse(Ad)[0], dW)
    assert relerr(1e6 * pre, dW) <= 0.01


# ---------------------------------------------------------------- shapes pinned by Fig. 4
def test_resnet50_shapes_reproduce_fig4(orc):
    g = json.load(open(os.path.join(GOLD, "paper_fig4.json")))
    L = shapes.resnet50()
    n_conv = sum(1 for l in L if l["kind"] == 0)
    n_fc = sum(1 for l in L if l["kind"] == 1)
    assert (n_conv, n_fc) == (g["n_conv"], g["n_fc"])
    kf = sum(orc.dims(l)[0] ** 2 + orc.dims(l)[1] ** 2 for l in L)
    bn_c = [l["c_out"] for l in L if l["kind"] == 0]  # one BN per conv output
    assert len(bn_c) == g["n_bn"]
    mib = 4 / 2 ** 20
    diag = (kf + sum(2 * c for c in bn_c)) * mib
    full = (kf + sum((2 * c) ** 2 for c in bn_c)) * mib
    assert round(diag) == g["diag_bn_mib"] and round(full) == g["full_bn_mib"]
    # the survey's derived totals (App. A.1)
    assert abs(kf * mib - 586.90) < 0.01 and abs(full - 1017.33) < 0.01
    assert sum(orc.packed_len(orc.dims(l)[0]) + orc.packed_len(orc.dims(l)[1]) for l in L) == 76967027
    assert sum(orc.dims(l)[0] * orc.dims(l)[1] for l in L) == 25503912
