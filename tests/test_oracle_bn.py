"""Pins for the oracle's Batch Normalization Fisher (NEXT-2; P:493-494, P:665-668, P:740-763;
S:231-246).

SPEC's hand-averaged example and elementwise example, the trivial cases (zero
gradients, F = 0, a truly diagonal F), the per-sample gradients against torch autograd of the BN
affine map y = γ·x̂ + β (a library routine on the definition), and (F + γ_BN I)·x = grad.
"""
import numpy as np
import pytest
import torch

from synth import inputs


def test_bn_fisher_spec_examples(orc):
    S = np.array([[1.0, 2.0], [3.0, 4.0]])  # C = 1: per-sample [dγ, dβ]
    assert orc.bn_fisher(S, "full").tolist() == [[5.0, 7.0], [7.0, 10.0]]
    assert orc.bn_fisher(S, "diag").tolist() == [5.0, 10.0]
    assert np.array_equal(orc.bn_fisher(np.zeros((3, 4)), "full"), np.zeros((4, 4)))
    rng = np.random.default_rng(0)
    R = rng.standard_normal((7, 6))
    assert np.array_equal(np.diag(orc.bn_fisher(R, "full")), orc.bn_fisher(R, "diag")) or \
        np.allclose(np.diag(orc.bn_fisher(R, "full")), orc.bn_fisher(R, "diag"), rtol=1e-15)
    with pytest.raises(ValueError):
        orc.bn_fisher(R, "nope")


def test_bn_precondition_spec_examples(orc):
    assert orc.bn_precondition(np.array([5.0, 10.0]), np.array([6.0, 22.0]), 1.0).tolist() == [1.0, 2.0]
    g = np.array([1.0, -2.0, 3.0])
    assert np.allclose(orc.bn_precondition(np.zeros((3, 3)), g, 0.4), g / 0.4, rtol=1e-15)  # F = 0
    d = np.array([0.5, 2.0, 7.0])
    assert np.allclose(orc.bn_precondition(np.diag(d), g, 0.4), orc.bn_precondition(d, g, 0.4), rtol=1e-14)
    rng = np.random.default_rng(1)
    S = rng.standard_normal((5, 8))
    F = orc.bn_fisher(S, "full")
    v = rng.standard_normal(8)
    x = orc.bn_precondition(F, v, 0.4)
    assert np.allclose(F @ x + 0.4 * x, v, rtol=0, atol=1e-12)  # the defining equation
    with pytest.raises(ValueError):
        orc.bn_precondition(F, v, 0.0)
    with pytest.raises(ValueError):
        orc.bn_precondition(F, v[:3], 0.4)


@pytest.mark.parametrize("fmt", ["bf16", "fp16"])
def test_bn_sample_grads_vs_autograd(orc, fmt):
    n, h, w, c = 3, 5, 4, 6
    dt = torch.bfloat16 if fmt == "bf16" else torch.float16
    g = torch.Generator().manual_seed(11)
    xh = torch.randn(n, h, w, c, generator=g).to(dt)
    gy = torch.randn(n, h, w, c, generator=g).to(dt)
    S = orc.bn_sample_grads(inputs.half_bits(xh), inputs.half_bits(gy), n, h * w, c, fmt)
    for s in range(n):  # per sample: d/dγ, d/dβ of Σ gy·(γ x̂ + β) by autograd in fp64
        gam = torch.ones(c, dtype=torch.float64, requires_grad=True)
        bet = torch.zeros(c, dtype=torch.float64, requires_grad=True)
        y = gam * xh[s].double() + bet
        (y * gy[s].double()).sum().backward()
        want = torch.cat([gam.grad, bet.grad]).numpy()
        assert np.allclose(S[s], want, rtol=1e-12, atol=1e-12)


def test_bn_fisher_rank_mean(orc):
    """The ranks' mean of F (the paper's ReduceScatter mean) is F of the concatenated
    per-sample gradients (what kfac_bn_exchange + a replicated solve computes, R-22)."""
    rng = np.random.default_rng(2)
    parts = [rng.standard_normal((4, 10)) for _ in range(3)]
    mean_F = sum(orc.bn_fisher(p, "full") for p in parts) / 3
    assert np.allclose(orc.bn_fisher(np.concatenate(parts), "full"), mean_F, rtol=1e-13, atol=1e-13)
    mean_d = sum(orc.bn_fisher(p, "diag") for p in parts) / 3
    assert np.allclose(orc.bn_fisher(np.concatenate(parts), "diag"), mean_d, rtol=1e-13, atol=1e-13)
