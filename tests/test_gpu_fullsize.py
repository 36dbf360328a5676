"""Full-size parity of the whole step (BASELINE configs 2, 3 and 5) at world 1, in the launch
configuration bench.py times (kfac_factor_all over every layer, LPT plan, one persistent inverse
launch, grouped precondition), against the fp64 oracle on the same seeded bf16 inputs.

Every stage is compared densely, layer by layer (Algorithm 1):
  a1/a2 factors   rs_recv's packed A, G vs oracle.factor_A / factor_G           <= 2e-3
  a5 damping      pi vs oracle.damp on the same fp32 factors                    <= 1e-6 rel
  a6 inverse      A_d^-1, G_d^-1 vs oracle.inverse of the SAME fp32 damped matrices <= 1e-5
  a7 precondition 𝒢 vs oracle.precondition(GPU G_d^-1, GPU A_d^-1, ∇W)           <= 2e-3 (expect ~1e-6..3e-5)
  end to end      𝒢 vs oracle (factors -> damp -> inverse -> precondition, all fp64) <= 2e-3
(relative Frobenius errors over full matrices, BASELINE.json north_star tolerances).  The
oracle's work is large at these sizes (RN50: ~0.8 TFLOP of factors, 2 x 0.45 TFLOP of
inverses and 2 x 0.16 TFLOP of products per gamma), hence the long timeouts.
"""
import numpy as np
import pytest
import torch

from synth import inputs, shapes

pytestmark = pytest.mark.gpu

TOL_FACTOR, TOL_INV, TOL_PREC = 2e-3, 1e-5, 2e-3
LPT = 1

# config -> gammas (R-2: the benchmark's 2.5e-2 and the decayed 2.5e-4)
CASES = [("resnet50", 2.5e-2), ("resnet50", 2.5e-4), ("stress", 2.5e-4), ("resnet18_cifar", 2.5e-2)]


def relerr(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def unpack_f32(p, d):
    M = np.zeros((d, d))
    M[np.triu_indices(d)] = p
    return M + M.T - np.diag(np.diag(M))


@pytest.fixture(scope="module")
def K():
    if not torch.cuda.is_available():
        pytest.fail("GPU test run without a GPU")
    from conftest import build_lib
    build_lib()
    import paper_1811_12019_b200 as K
    return K


_INPUTS, _ORACLE_FACTORS = {}, {}


def cfg_inputs(cfg):
    if cfg not in _INPUTS:
        layers, n = shapes.config(cfg)
        xs = [inputs.layer_x(l, i, n) for i, l in enumerate(layers)]
        gys = [inputs.layer_gy(l, i, n) for i, l in enumerate(layers)]
        dws = [inputs.layer_dw(l, i) for i, l in enumerate(layers)]
        _INPUTS[cfg] = (layers, n, xs, gys, dws)
    return _INPUTS[cfg]


def oracle_factors(orc, cfg):
    """Stages a1/a2 of the oracle (fp64, explicit patch loops) from the GPU's own bf16 bits."""
    if cfg not in _ORACLE_FACTORS:
        layers, n, xs, gys, _ = cfg_inputs(cfg)
        out = []
        for l, layer in enumerate(layers):
            A = orc.factor_A(layer, inputs.half_bits(xs[l]), n)
            G = orc.factor_G(inputs.half_bits(gys[l]), shapes.rows(layer, n), layer["c_out"])
            out.append((A, G))
        _ORACLE_FACTORS[cfg] = out
    return _ORACLE_FACTORS[cfg]


@pytest.mark.timeout(1800)
@pytest.mark.parametrize("cfg,gamma", CASES)
def test_fullsize_step_parity(K, orc, cfg, gamma):
    layers, n, xs, gys, dws = cfg_inputs(cfg)
    st = K.KfacStep(layers, n, policy=LPT)
    st.set_dw([d.cuda() for d in dws])
    st.run([x.cuda() for x in xs], [g.cuda() for g in gys], gamma)
    torch.cuda.synchronize()
    status = st.dev_status.cpu().tolist()
    pis = st.pi.cpu().double().numpy()
    ref_f = oracle_factors(orc, cfg)
    worst = {k: (0.0, None) for k in ("factor", "pi", "inverse", "precond", "precond_vs_fp32", "e2e")}

    def note(kind, e, where):
        if e > worst[kind][0]:
            worst[kind] = (e, where)

    for k, l in enumerate(st.rl["layers"]):
        name = layers[l]["name"]
        d_a, d_g = shapes.dims(layers[l])
        dW, pa, pg = st.recv_views(k)
        dW = dW.cpu().double().numpy()
        A32 = unpack_f32(pa.cpu().double().numpy(), d_a)
        G32 = unpack_f32(pg.cpu().double().numpy(), d_g)
        A64, G64 = ref_f[l]
        # a1/a2 (world 1: the ReduceScatter mean is the send buffer itself)
        ea, eg = relerr(A32, A64), relerr(G32, G64)
        note("factor", max(ea, eg), name)
        assert ea <= TOL_FACTOR and eg <= TOL_FACTOR, (name, ea, eg)
        assert np.array_equal(dW, dws[l].double().numpy())
        # a5 on the same fp32 factors
        Ad, Gd, pi = orc.damp(A32, G32, gamma)
        ep = abs(pis[k] - pi) / pi
        note("pi", ep, name)
        assert ep <= 1e-6, (name, pis[k], pi)
        # a6 vs the fp64 inverse of the same fp32 damped matrices
        Ai, Gi = (v.cpu().double().numpy() for v in st.inv_views(k))
        for which, (Md, Mi) in enumerate(((Ad, Ai), (Gd, Gi))):
            ref, s = orc.inverse(Md)
            assert s == 0 and status[2 * k + which] == 0, (name, which, s, status[2 * k + which])
            e = relerr(Mi, ref)
            note("inverse", e, name + "AG"[which])
            assert e <= TOL_INV, (name, "AG"[which], e)
        # a7 on the GPU's own inverses
        got = st.result(l).cpu().double().numpy()
        want = orc.precondition(Gi, Ai, dW)
        e = relerr(got, want)
        note("precond", e, name)
        assert e <= TOL_PREC, (name, e)
        # R-13: 3xTF32 is fp32-class.  Cancellation in A_d^-1 (kappa ~ 2e3) lifts any fp32 product chain
        # above 1e-5 on some layers, so the yardstick is plain fp32 GEMMs of the same operands (CPU)
        f32 = (torch.from_numpy(Gi).float() @ torch.from_numpy(dW).float()) @ torch.from_numpy(Ai).float()
        e32 = relerr(f32.double().numpy(), want)
        note("precond_vs_fp32", e / max(e32, 1e-12), name)
        assert e <= max(1e-5, 4 * e32), (name, e, e32)
        # end to end: the all-fp64 oracle pipeline from the same half inputs
        Ad64, Gd64, _ = orc.damp(A64, G64, gamma)
        Ai64, sa = orc.inverse(Ad64)
        Gi64, sg = orc.inverse(Gd64)
        assert sa == 0 and sg == 0
        e = relerr(got, orc.precondition(Gi64, Ai64, dW))
        note("e2e", e, name)
        assert e <= TOL_PREC, (name, e)
    print(f"{cfg} gamma={gamma}: worst " + ", ".join(f"{k} {v[0]:.2e} ({v[1]})" for k, v in worst.items()))
