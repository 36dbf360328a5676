"""GPU parity of the post-AllGather update (NEXT-3; R-21) through the C-ABI.

kfac_update against oracle.update_layer on the same seeded fp32 weights, previous weights
and preconditioned gradients (written into the AllGather buffer at the plan's ag_off):
small multi-layer nets (bias and no bias, vector and scalar access) and the full ResNet-50
parameter set.  Elementwise fp32 arithmetic against fp64: relative Frobenius error <= 1e-6
per layer; w_prev must receive the old weights bitwise.
"""
import numpy as np
import pytest
import torch

from synth import shapes

pytestmark = pytest.mark.gpu
TOL = 1e-6

NET = [shapes.conv("stem", 3, 16, 7, 2, 3, 20), shapes.conv("a", 16, 32, 3, 1, 1, 10, bias=1),
       shapes.conv("b", 32, 64, 1, 2, 0, 10), shapes.linear("fc", 64, 10), shapes.linear("odd", 37, 3, 1)]


@pytest.fixture(scope="module")
def K():
    if not torch.cuda.is_available():
        pytest.fail("GPU test run without a GPU")
    from conftest import build_lib
    build_lib()
    import paper_1811_12019_b200 as K
    return K


def relerr(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / max(np.linalg.norm(b), 1e-300))


def _case(K, orc, layers, lr, mom, rescale, misalign=False, seed=0):
    plan = K.Plan(layers, 1, 1)
    q = plan.query()
    g = torch.Generator().manual_seed(seed)
    ag = torch.zeros(q["ag_chunk"])
    ws, wps, want = [], [], []
    for l, L in enumerate(layers):
        da, dg = shapes.dims(L)
        w = torch.randn(dg, da, generator=g) * 0.05
        wp = w + 0.01 * torch.randn(dg, da, generator=g)
        pre = torch.randn(dg, da, generator=g)
        ag[q["ag_off"][l]:q["ag_off"][l] + dg * da] = pre.reshape(-1)
        want.append(orc.update_layer(w.double().numpy(), wp.double().numpy(), pre.double().numpy(), lr, mom,
                                     bool(L["has_bias"]), rescale))
        ws.append(w)
        wps.append(wp)
    dev_w, dev_p = [], []
    for w, wp in zip(ws, wps):
        if misalign:  # 4-byte offset: the scalar path
            bw = torch.zeros(w.numel() + 1, device="cuda")
            bp = torch.zeros(w.numel() + 1, device="cuda")
            bw[1:].copy_(w.reshape(-1))
            bp[1:].copy_(wp.reshape(-1))
            dev_w.append(bw[1:])
            dev_p.append(bp[1:])
        else:
            dev_w.append(w.cuda().reshape(-1))
            dev_p.append(wp.cuda().reshape(-1))
    wsb = torch.empty(q["ws_bytes"], dtype=torch.uint8, device="cuda")
    K.update(plan, ag.cuda(), dev_w, dev_p, lr, mom, wsb, rescale=rescale)
    torch.cuda.synchronize()
    worst = 0.0
    for l, L in enumerate(layers):
        da, dg = shapes.dims(L)
        got = dev_w[l].cpu().double().numpy().reshape(dg, da)
        e = relerr(got, want[l][0])
        worst = max(worst, e)
        assert e <= TOL, (l, e)
        assert torch.equal(dev_p[l].cpu().reshape(dg, da), ws[l])
        if rescale:
            nb = da - (1 if L["has_bias"] else 0)
            assert abs(np.linalg.norm(got[:, :nb]) - np.sqrt(2 * dg)) <= 1e-5 * np.sqrt(2 * dg)
    return worst


@pytest.mark.parametrize("rescale", [True, False])
@pytest.mark.parametrize("misalign", [False, True])
def test_update_small(K, orc, rescale, misalign):
    e = _case(K, orc, NET, 3.994e-3, 0.4868, rescale, misalign)
    print(f"update rescale={rescale} misalign={misalign}: max rel err {e:.2e}")


def test_update_special_cases(K, orc):
    _case(K, orc, NET, 0.1, 0.0, True, seed=1)  # m = 0
    _case(K, orc, NET, 0.0, 1.0, False, seed=2)  # eta = 0, m = 1


@pytest.mark.timeout(600)
def test_update_resnet50(K, orc):
    layers, _ = shapes.config("resnet50")
    e = _case(K, orc, layers, 8.18e-3, 0.997, True, seed=3)
    print(f"update resnet50 ({len(layers)} layers): max rel err {e:.2e}")
