"""GPU parity of the Batch Normalization Fisher (NEXT-2; R-22).

kfac_bn_grads against oracle.bn_sample_grads on the same seeded half inputs (factor tolerance
2e-3), kfac_bn_precondition (diagonal, and full through the Woodbury identity) against
oracle.bn_precondition of the dense (F + gamma_BN I): stage-wise on the GPU's own fp32 S (fp64
on both sides, 1e-8) and end to end from the half inputs (2e-3), at small shapes, every
ResNet-50 BN shape at batch 32, n = 128 (K in shared memory) and n = 256 (K in the workspace).
"""
import numpy as np
import pytest
import torch

from synth import inputs, shapes

pytestmark = pytest.mark.gpu
TOL = 2e-3
RHO_BN, GAMMA = 16.0, 2.5e-2  # Table 3: gamma_BN = rho_BN * gamma = 0.4
DENSE_MAX = 1024  # largest 2C checked against the dense oracle inverse


@pytest.fixture(scope="module")
def K():
    if not torch.cuda.is_available():
        pytest.fail("GPU test run without a GPU")
    from conftest import build_lib
    build_lib()
    import paper_1811_12019_b200 as K
    return K


def relerr(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def _layers_inputs(cs, hws, n, dt, seed):
    g = torch.Generator().manual_seed(seed)
    xs = [torch.randn(n, hw, c, generator=g).to(dt) for c, hw in zip(cs, hws)]
    gys = [(torch.randn(n, hw, c, generator=g) * 0.01).to(dt) for c, hw in zip(cs, hws)]
    grads = [torch.randn(2 * c, generator=g) for c in cs]
    return xs, gys, grads


def _run(K, orc, cs, hws, n, dt=torch.bfloat16, seed=0, check_e2e=True):
    fmt = "bf16" if dt == torch.bfloat16 else "fp16"
    xs, gys, grads = _layers_inputs(cs, hws, n, dt, seed)
    S = [torch.empty(n, 2 * c, device="cuda") for c in cs]
    K.bn_grads(cs, hws, [x.cuda() for x in xs], [g.cuda() for g in gys], n, S)
    lam = RHO_BN * GAMMA
    outs = {}
    ws = torch.empty(K.bn_ws_bytes(cs, n), dtype=torch.uint8, device="cuda")
    for full in (0, 1):
        o = [torch.empty(2 * c, device="cuda") for c in cs]
        K.bn_precondition(cs, n, S, [g.cuda() for g in grads], lam, full, o, ws if full else None)
        outs[full] = o
    torch.cuda.synchronize()
    worst = {"S": 0.0, "diag": 0.0, "full": 0.0, "stage": 0.0}
    for l, (c, hw) in enumerate(zip(cs, hws)):
        Sg = S[l].cpu().double().numpy()
        gr = grads[l].double().numpy()
        So = orc.bn_sample_grads(inputs.half_bits(xs[l]), inputs.half_bits(gys[l]), n, hw, c, fmt) if check_e2e else None
        if So is not None:
            worst["S"] = max(worst["S"], relerr(Sg, So))
        for full, key in ((0, "diag"), (1, "full")):
            got = outs[full][l].cpu().double().numpy()
            if full and 2 * c > DENSE_MAX:
                # past DENSE_MAX the dense oracle inverse is minutes of CPU: check the defining equation
                # (F + lambda I) x = grad instead, F x = S^T (S x) / n in fp64 (holds at any size)
                for Sx, k2, tol in ((Sg, "stage", 1e-6), (So, key, TOL)):
                    if Sx is None:
                        continue
                    Fx = Sx.T @ (Sx @ got) / n
                    r = np.linalg.norm(Fx + lam * got - gr) / (np.linalg.norm(Fx) + lam * np.linalg.norm(got) + np.linalg.norm(gr))
                    worst[k2] = max(worst[k2], r)
                continue
            F_same = orc.bn_fisher(Sg, "full" if full else "diag")
            worst["stage"] = max(worst["stage"], relerr(got, orc.bn_precondition(F_same, gr, lam)))
            if So is not None:
                want = orc.bn_precondition(orc.bn_fisher(So, "full" if full else "diag"), gr, lam)
                worst[key] = max(worst[key], relerr(got, want))
    print({k: f"{v:.2e}" for k, v in worst.items()})
    assert worst["stage"] <= 1e-6
    assert worst["S"] <= TOL and worst["diag"] <= TOL and worst["full"] <= TOL
    return worst


@pytest.mark.parametrize("dt", [torch.bfloat16, torch.float16])
def test_bn_small(K, orc, dt):
    _run(K, orc, [6, 64, 130, 256], [20, 49, 9, 196], 4, dt)


def test_bn_resnet50_shapes(K, orc):
    layers, n = shapes.config("resnet50")
    convs = [l for l in layers if l["kind"] == 0]  # one BN after every conv (53)
    cs = [l["c_out"] for l in convs]
    hws = [shapes.out_hw(l)[0] * shapes.out_hw(l)[1] for l in convs]
    _run(K, orc, cs, hws, n, seed=1)


def test_bn_sample_limit(K, orc):
    _run(K, orc, [64, 512], [4, 1], 128, seed=2)  # K in shared memory
    _run(K, orc, [64, 512, 6], [4, 1, 3], 256, seed=3)  # K in the workspace (8 ranks x 32 samples)
    S = [torch.zeros(257, 128, device="cuda")]
    g = [torch.zeros(128, device="cuda")]
    with pytest.raises(K.KfacError, match="ERR_UNSUPPORTED"):
        K.bn_precondition([64], 257, S, g, 0.4, 1, [torch.empty(128, device="cuda")])
    with pytest.raises(K.KfacError, match="ERR_ARG"):  # full mode without its workspace
        K.bn_precondition([64], 4, S, g, 0.4, 1, [torch.empty(128, device="cuda")])
    K.bn_precondition([64], 257, S, g, 0.4, 0, [torch.empty(128, device="cuda")])  # diag: any n
    with pytest.raises(K.KfacError, match="ERR_ARG"):
        K.bn_precondition([64], 4, S, g, 0.0, 0, [torch.empty(128, device="cuda")])
