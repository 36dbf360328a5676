"""GPU parity of the stale-Fisher path (NEXT-1) through the C-ABI.

* kfac_factor_diff against oracle.fim_diff: stage-wise on the same fp32 factors
  (fp64 arithmetic on both sides, 1e-10), end to end against the all-fp64
  oracle factors (the factor tolerance 2e-3), the degenerate cases (equal
  factors -> 0 exactly, a zero previous factor -> NaN) and the full
  ResNet-50 layout.
* a stale step (dW-only ReduceScatter, cached inverses, R-20) against
  oracle.stale_results, world 1 (world 2/4 in tests/mp_parity.py).
"""
import numpy as np
import pytest
import torch

from synth import inputs, shapes

pytestmark = pytest.mark.gpu

TOL_PREC, TOL_FACTOR = 2e-3, 2e-3

NET = [shapes.conv("stem", 3, 16, 7, 2, 3, 20), shapes.conv("a", 16, 32, 3, 1, 1, 10, bias=1),
       shapes.conv("b", 32, 64, 1, 2, 0, 10), shapes.conv("c", 64, 64, 3, 1, 1, 5), shapes.linear("fc", 64, 10)]


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


def unpack(p, d):
    M = np.zeros((d, d))
    M[np.triu_indices(d)] = p
    return M + M.T - np.diag(np.diag(M))


def _inputs(layers, n, seed):
    xs = [inputs.layer_x(l, i, n, 0, seed) for i, l in enumerate(layers)]
    gys = [inputs.layer_gy(l, i, n, 0, seed) for i, l in enumerate(layers)]
    dws = [inputs.layer_dw(l, i, 0, seed) for i, l in enumerate(layers)]
    return xs, gys, dws


def _oracle_in(xs, gys, dws, n):
    return [([inputs.half_bits(x) for x in xs], [inputs.half_bits(g) for g in gys], [d.numpy() for d in dws], n)]


def test_factor_diff_two_refreshes(K, orc):
    n, gamma = 4, 2.5e-2
    st = K.KfacStep(NET, n, stale=True)
    ins = [_inputs(NET, n, s) for s in (1811, 1812)]
    for xs, gys, dws in ins:
        st.set_dw([d.cuda() for d in dws])
        st.run_refresh([x.cuda() for x in xs], [g.cuda() for g in gys], gamma)
    torch.cuda.synchronize()
    got = st.diff.cpu().numpy()
    cur, prev = st.rs_recv.cpu().double().numpy(), st.rs_recv_prev.cpu().double().numpy()
    refs = [orc.kfac_step(NET, _oracle_in(*i, n), 1, gamma)["results"][0] for i in ins]
    rl = st.plan.rank_layers(0)
    for k, l in enumerate(rl["layers"]):
        da, dg = shapes.dims(NET[l])
        o = rl["local_off"][k]
        for w, (off, d) in enumerate(((o[1], da), (o[2], dg))):
            seg = slice(off, off + d * (d + 1) // 2)
            same = orc.fim_diff(unpack(cur[seg], d), unpack(prev[seg], d))  # stage-wise: the same fp32 factors
            key = "A" if w == 0 else "G"
            e2e = orc.fim_diff(refs[1][l][key], refs[0][l][key])  # all-fp64 oracle factors
            print(f"layer {l} {key}: diff {got[2 * k + w]:.6e} (stage-wise ref {same:.6e}, oracle {e2e:.6e})")
            assert abs(got[2 * k + w] - same) <= 1e-10 * same
            assert abs(got[2 * k + w] - e2e) <= TOL_FACTOR * e2e


def test_factor_diff_degenerate(K):
    n = 4
    st = K.KfacStep(NET, n, stale=True)
    xs, gys, dws = _inputs(NET, n, 7)
    st.set_dw([d.cuda() for d in dws])
    for _ in range(2):  # the same inputs twice: the factor kernels are deterministic -> Diff = 0 exactly
        st.run_refresh([x.cuda() for x in xs], [g.cuda() for g in gys], 2.5e-2)
    torch.cuda.synchronize()
    assert (st.diff.cpu() == 0).all()
    zero = torch.zeros_like(st.rs_recv)
    K.factor_diff(st.plan, 0, st.rs_recv, zero, st.diff, st.ws)  # previous = 0: missing
    torch.cuda.synchronize()
    assert torch.isnan(st.diff.cpu()).all()
    K.factor_diff(st.plan, 0, st.rs_recv.mul(3.0), st.rs_recv, st.diff, st.ws)  # X = 3 X_prev -> 2
    torch.cuda.synchronize()
    assert torch.allclose(st.diff.cpu(), torch.full_like(st.diff.cpu(), 2.0), rtol=1e-6, atol=0)
    with pytest.raises(K.KfacError, match="ERR_STATE"):
        K.factor_diff(st.splan, 0, st.rs_recv, zero, st.diff, st.ws)


@pytest.mark.timeout(600)
def test_factor_diff_resnet50_layout(K, orc):
    """The full ResNet-50 recv layout (dims up to 4608, 108 matrices) with seeded packed values."""
    layers, n = shapes.config("resnet50")
    plan = K.Plan(layers, 1, n)
    q, rl = plan.query(), plan.rank_layers(0)
    g = torch.Generator(device="cuda").manual_seed(5)
    prev = torch.rand(q["rs_chunk"], generator=g, device="cuda")
    cur = prev + 0.05 * torch.randn(q["rs_chunk"], generator=g, device="cuda")
    ws = torch.empty(q["ws_bytes"], dtype=torch.uint8, device="cuda")
    diff = torch.empty(2 * len(rl["layers"]), dtype=torch.float64, device="cuda")
    K.factor_diff(plan, 0, cur, prev, diff, ws)
    torch.cuda.synchronize()
    got = diff.cpu().numpy()
    c, p = cur.cpu().double().numpy(), prev.cpu().double().numpy()
    worst = 0.0
    for k, l in enumerate(rl["layers"]):
        da, dg = shapes.dims(layers[l])
        o = rl["local_off"][k]
        for w, (off, d) in enumerate(((o[1], da), (o[2], dg))):
            seg = slice(off, off + d * (d + 1) // 2)
            want = orc.fim_diff(unpack(c[seg], d), unpack(p[seg], d))
            worst = max(worst, abs(got[2 * k + w] - want) / want)
    print(f"resnet50 layout: {len(got)} matrices, max rel err {worst:.2e}")
    assert worst <= 1e-10


@pytest.mark.parametrize("gamma", [2.5e-2, 2.5e-4])
def test_stale_step_end_to_end(K, orc, gamma):
    n = 4
    st = K.KfacStep(NET, n, stale=True)
    xs, gys, dws = _inputs(NET, n, 1811)
    st.set_dw([d.cuda() for d in dws])
    st.run([x.cuda() for x in xs], [g.cuda() for g in gys], gamma)
    dws2 = [inputs.layer_dw(l, i, 0, 99) for i, l in enumerate(NET)]
    st.set_stale_dw([d.cuda() for d in dws2])
    before = K.kfac.launch_count()
    st.run_stale()
    torch.cuda.synchronize()
    assert K.kfac.launch_count() > before
    assert st.dev_status.cpu().abs().sum().item() == 0
    full = orc.kfac_step(NET, _oracle_in(xs, gys, dws, n), 1, gamma)
    sp = orc.plan(NET, 1, 0, stale=True)
    recv = orc.reduce_scatter([orc.build_send(NET, sp, 0, None, [d.numpy() for d in dws2])], sp)[0]
    cached = {l: (v["Ainv"], v["Ginv"]) for l, v in full["results"][0].items()}
    ref = orc.stale_results(NET, sp, 0, recv, cached)
    rl = st.plan.rank_layers(0)
    for k, l in enumerate(rl["layers"]):
        Ai, Gi = st.inv_views(k)
        stage = orc.precondition(Gi.cpu().double().numpy(), Ai.cpu().double().numpy(), dws2[l].double().numpy())
        got = st.result(l).cpu().double().numpy()
        es, ee = relerr(got, stage), relerr(got, ref[l]["precond"])
        print(f"layer {l}: stale precond err {es:.2e} (same inverses), e2e {ee:.2e}")
        assert es <= 1e-5 and ee <= TOL_PREC
    with pytest.raises(K.KfacError, match="ERR_STATE"):
        K.damped_inverse(st.splan, 0, st.s_recv, gamma, st.inv_ws, st.dev_status, st.pi, st.ws)


@pytest.mark.parametrize("gamma", [2.5e-2, 2.5e-4])
def test_grefresh_step_end_to_end(K, orc, gamma):
    """Full step (seed 1811), then a G refresh with new gy and dW (seed 99): G factors, [dW, G]
    ReduceScatter, G_d^-1 with the cached pi, the cached A_d^-1 (R-20), against oracle.grefresh_results."""
    n = 4
    st = K.KfacStep(NET, n, stale=True)
    xs, gys, dws = _inputs(NET, n, 1811)
    st.set_dw([d.cuda() for d in dws])
    st.run([x.cuda() for x in xs], [g.cuda() for g in gys], gamma)
    _, gys2, dws2 = _inputs(NET, n, 99)
    st.set_grefresh_dw([d.cuda() for d in dws2])
    st.run_grefresh([g.cuda() for g in gys2], gamma)
    torch.cuda.synchronize()
    assert st.dev_status.cpu().abs().sum().item() == 0
    full = orc.kfac_step(NET, _oracle_in(xs, gys, dws, n), 1, gamma)
    gp = orc.plan(NET, 1, 0, g_only=True)
    facs = [(None, orc.factor_G(inputs.half_bits(gys2[l]), shapes.rows(L, n), L["c_out"])) for l, L in enumerate(NET)]
    recv = orc.reduce_scatter([orc.build_send(NET, gp, 0, facs, [d.numpy() for d in dws2])], gp)[0]
    cached = {l: (v["Ainv"], v["pi"]) for l, v in full["results"][0].items()}
    ref = orc.grefresh_results(NET, gp, 0, recv, gamma, cached)
    rl = st.plan.rank_layers(0)
    for k, l in enumerate(rl["layers"]):
        Ai, Gi = st.inv_views(k)
        dg = shapes.dims(NET[l])[1]
        eg = relerr(Gi.cpu().double().numpy(), ref[l]["Ginv"])
        ee = relerr(st.result(l).cpu().double().numpy(), ref[l]["precond"])
        print(f"layer {l}: G-refresh Ginv err {eg:.2e}, e2e {ee:.2e}")
        assert eg <= 2e-3 and ee <= TOL_PREC
    # A's inverse is untouched by the G refresh: a second stale-A G refresh with the first inputs
    # restores the full step's result
    st.set_grefresh_dw([d.cuda() for d in dws])
    st.run_grefresh([g.cuda() for g in gys], gamma)
    torch.cuda.synchronize()
    for l in range(len(NET)):
        assert relerr(st.result(l).cpu().double().numpy(), full["results"][0][l]["precond"]) <= TOL_PREC
