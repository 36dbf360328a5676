"""GPU parity: the CUDA path (through the C-ABI) against the fp64 oracle on the
same seeded inputs.

Tolerances (BASELINE.json north_star): relative Frobenius error vs fp64
  factors (half inputs, fp32 accumulate)      <= 2e-3
  damped inverse (vs fp64 inverse of the same fp32 damped matrix) <= 1e-5
  preconditioned gradient                     <= 2e-3
Layouts / ownership are bit-exact (tests/test_abi.py).
"""
import numpy as np
import pytest
import torch

from synth import inputs, shapes

pytestmark = pytest.mark.gpu

TOL_FACTOR, TOL_INV, TOL_PREC = 2e-3, 1e-5, 2e-3


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


def unpack_f32(p, d):
    M = np.zeros((d, d))
    iu = np.triu_indices(d)
    M[iu] = p
    M = M + M.T - np.diag(np.diag(M))
    return M


def gpu_factor(K, layer, t, n, which, alpha):
    d_a, d_g = shapes.dims(layer)
    d = d_a if which == 0 else d_g
    out = torch.full((d * (d + 1) // 2,), float("nan"), dtype=torch.float32, device="cuda")
    wsb = K.factor_ws_bytes(layer, n, which)
    ws = torch.empty(max(wsb, 16), dtype=torch.uint8, device="cuda")
    f = K.factor_A if which == 0 else K.factor_G
    f(layer, t.cuda(), n, alpha, out, ws)
    torch.cuda.synchronize()
    return out.cpu().double().numpy()


GEOMS = {  # name: (layer, n) -- each exercises one staging path / edge case
    "config1_im2col_c16_bias": (shapes.single_conv()[0], 32),
    "im2col_c64_3x3": (shapes.conv("c", 64, 64, 3, 1, 1, 9), 3),
    "im2col_c32_3x3_s2": (shapes.conv("c", 32, 48, 3, 2, 1, 11), 4),
    "im2col_c128_1x1_s2": (shapes.conv("c", 128, 256, 1, 2, 0, 14), 2),
    "tiled_1x1_multitile_splitk": (shapes.conv("c", 256, 64, 1, 1, 0, 28), 16),
    "gather_stem_c3_7x7_s2": (shapes.conv("c", 3, 64, 7, 2, 3, 30), 2),
    "fc_bias_c1000": (shapes.linear("fc", 1000, 1000), 8),
    "fc_c10_gather": (shapes.linear("fc", 200, 10), 5),
    "ragged_rows_d_not_128": (shapes.conv("c", 48, 40, 3, 1, 1, 5), 3),
    # 5-D slot-merged boxes: 7x7 outputs -> 8-wide boxes, 8 images per chunk (phantom images)
    "im2col_c256_3x3_7x7_phantom": (shapes.conv("c", 256, 64, 3, 1, 1, 7), 3),
    "im2col_c64_3x3_14x14": (shapes.conv("c", 64, 32, 3, 1, 1, 14), 2),
    # 16-channel slots: 16 boxes per 256-feature operand (the owned-box list at its limit)
    "tiled_c304_cb16_many_boxes": (shapes.linear("fc", 304, 24, bias=0), 100),
    # two 256-tiles per side: diagonal (multi-unit stages) and off-diagonal items
    "tiled_c512_two_tiles": (shapes.conv("c", 512, 40, 1, 1, 0, 6), 3),
}


@pytest.mark.parametrize("name", list(GEOMS))
@pytest.mark.parametrize("dtype", ["bf16", "fp16"])
def test_factor_parity(K, orc, name, dtype):
    layer, n = GEOMS[name]
    x = inputs.layer_x(layer, 0, n, dtype=dtype, stem=layer["c_in"] == 3)
    gy = inputs.layer_gy(layer, 0, n, dtype=dtype)
    rows = shapes.rows(layer, n)
    d_a, d_g = shapes.dims(layer)
    A = orc.factor_A(layer, inputs.half_bits(x), n, fmt=dtype)
    G = orc.factor_G(inputs.half_bits(gy), rows, d_g, fmt=dtype)
    pa = gpu_factor(K, layer, x, n, 0, 1.0 / rows)
    pg = gpu_factor(K, layer, gy, n, 1, 1.0 / rows)
    assert np.all(np.isfinite(pa)) and np.all(np.isfinite(pg))
    ea = relerr(unpack_f32(pa, d_a), A)
    eg = relerr(unpack_f32(pg, d_g), G)
    print(f"{name} {dtype}: A err {ea:.2e}  G err {eg:.2e}")
    assert ea <= TOL_FACTOR and eg <= TOL_FACTOR
    assert ea <= 1e-5 and eg <= 1e-5  # fp32 accumulation of exact half products


@pytest.mark.parametrize("name", ["im2col_c64_3x3", "im2col_c32_3x3_s2", "tiled_1x1_multitile_splitk"])
def test_factor_gather_matches_tma(K, orc, monkeypatch, name):
    """The generic gather producer and the TMA producers agree (their K chunking differs, so the
    fp32 accumulation order differs: agreement to accumulation rounding, and both match the oracle)."""
    layer, n = GEOMS[name]
    x = inputs.layer_x(layer, 0, n)
    rows = shapes.rows(layer, n)
    d_a, _ = shapes.dims(layer)
    a = gpu_factor(K, layer, x, n, 0, 1.0 / rows)
    monkeypatch.setenv("KFAC_FORCE_GATHER", "1")
    b = gpu_factor(K, layer, x, n, 0, 1.0 / rows)
    A = orc.factor_A(layer, inputs.half_bits(x), n)
    assert relerr(unpack_f32(a, d_a), unpack_f32(b, d_a)) <= 1e-6
    assert relerr(unpack_f32(b, d_a), A) <= 1e-5


def test_factor_deterministic(K):
    layer, n = GEOMS["tiled_1x1_multitile_splitk"]
    x = inputs.layer_x(layer, 0, n)
    rows = shapes.rows(layer, n)
    a = gpu_factor(K, layer, x, n, 0, 1.0 / rows)
    b = gpu_factor(K, layer, x, n, 0, 1.0 / rows)
    assert np.array_equal(a, b)


# --------------------------------------------------------------- full step
def _run_step(K, layers, n, gamma, world=1, rank=0, policy=0, dws=None, seed=1811):
    st = K.KfacStep(layers, n, rank=rank, world=world, policy=policy)
    xs = [inputs.layer_x(l, i, n, rank, seed).cuda() for i, l in enumerate(layers)]
    gys = [inputs.layer_gy(l, i, n, rank, seed).cuda() for i, l in enumerate(layers)]
    if dws is None:
        dws = [inputs.layer_dw(l, i, rank, seed) for i, l in enumerate(layers)]
    st.set_dw([d.cuda() for d in dws])
    st.run(xs, gys, gamma)
    torch.cuda.synchronize()
    return st, xs, gys, dws


@pytest.mark.parametrize("gamma", [2.5e-2, 2.5e-4])
def test_step_config1_end_to_end(K, orc, gamma):
    layers, n = shapes.config("single_conv")
    st, xs, gys, dws = _run_step(K, layers, n, gamma)
    rin = [([inputs.half_bits(x.cpu()) for x in xs], [inputs.half_bits(g.cpu()) for g in gys],
            [d.numpy() for d in dws], n)]
    ref = orc.kfac_step(layers, rin, 1, gamma)
    res = ref["results"][0][0]
    # stage-wise: RS result (world 1 = copy of the send buffer)
    dW, pa, pg = st.recv_views(0)
    d_a, d_g = shapes.dims(layers[0])
    assert relerr(unpack_f32(pa.cpu().double().numpy(), d_a), res["A"]) <= TOL_FACTOR
    assert relerr(unpack_f32(pg.cpu().double().numpy(), d_g), res["G"]) <= TOL_FACTOR
    assert np.array_equal(dW.cpu().numpy(), dws[0].numpy())
    assert st.dev_status.cpu().tolist() == [0, 0]
    assert abs(st.pi[0].item() - res["pi"]) <= 1e-6 * res["pi"]
    # inverse vs fp64 inverse of the SAME fp32 damped matrix the GPU saw
    Ai, Gi = st.inv_views(0)
    A32 = unpack_f32(pa.cpu().double().numpy(), d_a)
    G32 = unpack_f32(pg.cpu().double().numpy(), d_g)
    Ad, Gd, _ = orc.damp(A32, G32, gamma)
    ea = relerr(Ai.cpu().double().numpy(), orc.inverse(Ad)[0])
    eg = relerr(Gi.cpu().double().numpy(), orc.inverse(Gd)[0])
    print(f"inverse err A {ea:.2e} G {eg:.2e}")
    assert ea <= TOL_INV and eg <= TOL_INV
    # precondition vs oracle on the same fp32 inverses
    pre_ref = orc.precondition(Gi.cpu().double().numpy(), Ai.cpu().double().numpy(), dW.cpu().double().numpy())
    ep = relerr(st.result(0).cpu().double().numpy(), pre_ref)
    assert ep <= TOL_PREC and ep <= 1e-5
    # end to end vs the all-fp64 oracle from the same half inputs
    e2e = relerr(st.result(0).cpu().double().numpy(), res["precond"])
    print(f"precond err {ep:.2e} e2e {e2e:.2e}")
    assert e2e <= TOL_PREC


def test_step_multilayer_end_to_end(K, orc):
    """A small multi-layer network touching every staging path, world 1."""
    layers = [shapes.conv("stem", 3, 16, 7, 2, 3, 20), shapes.conv("a", 16, 32, 3, 1, 1, 10, bias=1),
              shapes.conv("b", 32, 64, 1, 2, 0, 10), shapes.conv("c", 64, 64, 3, 1, 1, 5),
              shapes.linear("fc", 64, 10)]
    n, gamma = 4, 2.5e-2
    st, xs, gys, dws = _run_step(K, layers, n, gamma)
    rin = [([inputs.half_bits(x.cpu()) for x in xs], [inputs.half_bits(g.cpu()) for g in gys],
            [d.numpy() for d in dws], n)]
    ref = orc.kfac_step(layers, rin, 1, gamma)
    assert st.dev_status.cpu().abs().sum().item() == 0
    for l in range(len(layers)):
        e = relerr(st.result(l).cpu().double().numpy(), ref["results"][0][l]["precond"])
        print(f"layer {l}: e2e {e:.2e}")
        assert e <= TOL_PREC


@pytest.mark.parametrize("prec", [1, 2])  # INV_FP64, INV_INT8
def test_inverse_reports_not_pd(K, orc, prec):
    layers = [shapes.linear("fc", 7, 5, bias=0)]
    st = K.KfacStep(layers, 1, inv_precision=prec)
    dW, pa, pg = None, None, None
    # hand-made recv: A = -I (not PD after damping 0.1*pi), G = I
    d_a, d_g = 7, 5
    A = np.eye(d_a)
    A[0, 0], A[1, 1] = 5.0, -1.0  # positive trace (pi real), not PD at pivot 1
    G = np.eye(d_g)
    _, pa, pg = st.recv_views(0)
    pa.copy_(torch.as_tensor(orc.pack(A), dtype=torch.float32))
    pg.copy_(torch.as_tensor(orc.pack(G), dtype=torch.float32))
    st.inverse(1e-2)
    torch.cuda.synchronize()
    _, want = orc.inverse(orc.damp(A, G, 1e-2)[0])
    assert st.dev_status.cpu().tolist() == [want, 0]
    assert want == 2


@pytest.mark.parametrize("prec", [0, 1])  # INV_AUTO (per-matrix bound), INV_FP64
@pytest.mark.parametrize("n", [64, 65, 130, 300, 513, 1153])
def test_inverse_ill_conditioned(K, orc, n, prec):
    """Rank-deficient ReLU-like factors at small damping (kappa ~ 1e4): the sweep meets 1e-5 with
    fp64 updates and with the per-matrix choice (R-12)."""
    rng = np.random.default_rng(n)
    X = np.maximum(rng.standard_normal((n // 3, n)), 0)
    A = (X.T @ X / X.shape[0]).astype(np.float32).astype(np.float64)
    G = np.eye(4)
    layers = [shapes.linear("fc", n, 4, bias=0)]
    st = K.KfacStep(layers, 1, inv_precision=prec)
    _, pa, pg = st.recv_views(0)
    pa.copy_(torch.as_tensor(orc.pack(A), dtype=torch.float32))
    pg.copy_(torch.as_tensor(orc.pack(G), dtype=torch.float32))
    st.inverse(2.5e-4)
    torch.cuda.synchronize()
    Ad, _, _ = orc.damp(A, G, 2.5e-4)
    ref, s = orc.inverse(Ad)
    Ai, _ = st.inv_views(0)
    e = relerr(Ai.cpu().double().numpy(), ref)
    print(f"n={n} cond={np.linalg.cond(Ad):.1e} err={e:.2e} report={st.inverse_report()}")
    assert s == 0 and st.dev_status.cpu().tolist() == [0, 0]
    assert e <= TOL_INV


@pytest.mark.timeout(300)
@pytest.mark.parametrize("prec", [1, 2])  # INV_FP64, INV_INT8
def test_inverse_batched_dataflow(K, orc, prec):
    """Several owned matrices of mixed sizes (ragged tails, 1x1, multi-step) in ONE persistent
    dataflow launch, one of them not PD mid-sweep (pivot 400 of 1000: its tasks stop, the others
    must complete and stay exact -- no deadlock on the skipped tasks' stamps)."""
    layers = [shapes.linear("a", 700, 17, bias=0), shapes.linear("b", 129, 300, bias=0),
              shapes.linear("c", 1000, 1, bias=0), shapes.linear("d", 128, 65, bias=0)]
    st = K.KfacStep(layers, 1, inv_precision=prec)
    rng = np.random.default_rng(7)
    mats = []
    for k, l in enumerate(layers):
        d_a, d_g = shapes.dims(l)
        pair = []
        for d in (d_a, d_g):
            X = np.maximum(rng.standard_normal((max(d // 2, 1), d)), 0)
            M = (X.T @ X / X.shape[0] + 0.05 * np.eye(d)).astype(np.float32).astype(np.float64)
            pair.append(M)
        if k == 2:
            pair[0][400, 400] = -10.0  # not PD: the LDL^T pivot 400 is negative
        _, pa, pg = st.recv_views(k)
        pa.copy_(torch.as_tensor(orc.pack(pair[0]), dtype=torch.float32))
        pg.copy_(torch.as_tensor(orc.pack(pair[1]), dtype=torch.float32))
        mats.append(pair)
    st.inverse(2.5e-3)
    torch.cuda.synchronize()
    status = st.dev_status.cpu().tolist()
    for k in range(len(layers)):
        Ad, Gd, _ = orc.damp(mats[k][0], mats[k][1], 2.5e-3)
        Ai, Gi = st.inv_views(k)
        for which, (Md, Mi) in enumerate(((Ad, Ai), (Gd, Gi))):
            ref, s_ref = orc.inverse(Md)
            assert status[2 * k + which] == s_ref, (k, which, status)
            if s_ref == 0:
                e = relerr(Mi.cpu().double().numpy(), ref)
                assert e <= TOL_INV, (k, which, e)
    assert status[4] == 401


@pytest.mark.timeout(300)
@pytest.mark.parametrize("prec", [0, 1, 2])
@pytest.mark.parametrize("n", [2049, 4608])
def test_fullsize_inverse_residual(K, n, prec):
    """BASELINE config 5's largest factors (FC 2049, conv 4608; 17 / 36 sweep steps, merged
    two-step updates, odd and even step counts).  A rigorous bound on the relative error of the
    returned fp32 inverse X from its fp64 residual R = M X - I:
    ||X - M^-1||_F = ||M^-1 R||_F <= ||R||_F / lambda_min(M), and ||M^-1||_F >= ||X||_F - that."""
    g = 64
    layers = [shapes.linear("fc", n, g, bias=0)]
    st = K.KfacStep(layers, 1, inv_precision=prec)
    gen = torch.Generator(device="cuda").manual_seed(n)
    X = torch.relu(torch.randn(n // 2, n, generator=gen, device="cuda", dtype=torch.float64))
    A = (X.T @ X / X.shape[0]).float()
    iu = torch.triu_indices(n, n, device="cuda")
    _, pa, pg = st.recv_views(0)
    pa.copy_(A[iu[0], iu[1]])
    pg.copy_(torch.eye(g, device="cuda")[torch.triu_indices(g, g, device="cuda").unbind()])
    gamma = 2.5e-3
    st.inverse(gamma)
    torch.cuda.synchronize()
    assert st.dev_status.cpu().tolist() == [0, 0]
    # the damping the library applied (R-1): pi from the traces, A_d = A + pi sqrt(gamma) I
    A64 = A.double()
    pi = float(np.sqrt((torch.trace(A64).item() / n) / 1.0))
    Ad = A64 + pi * np.sqrt(gamma) * torch.eye(n, device="cuda", dtype=torch.float64)
    Ai, _ = st.inv_views(0)
    Xi = Ai.double()
    res = torch.linalg.norm(Ad @ Xi - torch.eye(n, device="cuda", dtype=torch.float64)).item()
    lam_min = torch.linalg.eigvalsh(Ad)[0].item()
    err_abs = res / lam_min
    err_rel = err_abs / (torch.linalg.norm(Xi).item() - err_abs)
    print(f"n={n} prec={prec} residual {res:.2e} lambda_min {lam_min:.2e} relative error <= {err_rel:.2e} "
          f"report {st.inverse_report()}")
    assert 0 < err_rel <= TOL_INV
    assert torch.allclose(Xi, Xi.T)


# --------------------------------------------------------------- full-size, sampled
@pytest.mark.parametrize("cfg", ["resnet50"])
def test_fullsize_factors_sampled(K, orc, cfg):
    """BASELINE config 3 at full size, in the bench's launch configuration (kfac_factor_all):
    sampled packed entries vs the oracle's entries, one by one."""
    layers, n = shapes.config(cfg)
    st = K.KfacStep(layers, n)
    xs = [inputs.layer_x(l, i, n) for i, l in enumerate(layers)]
    gys = [inputs.layer_gy(l, i, n) for i, l in enumerate(layers)]
    st.factors([x.cuda() for x in xs], [g.cuda() for g in gys])
    torch.cuda.synchronize()
    rng = np.random.default_rng(0)
    errs = []
    for l, layer in enumerate(layers):
        d_a, d_g = shapes.dims(layer)
        rows = shapes.rows(layer, n)
        for which, d in ((0, d_a), (1, d_g)):
            m = 24
            ij = np.stack([rng.integers(0, d, m), rng.integers(0, d, m)], 1)
            ij[:4] = [[0, 0], [d - 1, d - 1], [0, d - 1], [d // 2, d // 2]]
            ij = np.sort(ij, 1)
            got = st.send_factor_view(l, which).cpu().double().numpy()
            g = got[ij[:, 0] * d - ij[:, 0] * (ij[:, 0] - 1) // 2 + (ij[:, 1] - ij[:, 0])]
            if which == 0:
                ref = orc.factor_A_entries(layer, inputs.half_bits(xs[l]), n, ij)
                scale = np.sqrt(np.abs(orc.factor_A_entries(layer, inputs.half_bits(xs[l]), n,
                                                            np.stack([ij[:, 0], ij[:, 0]], 1)) *
                                       orc.factor_A_entries(layer, inputs.half_bits(xs[l]), n,
                                                            np.stack([ij[:, 1], ij[:, 1]], 1))))
            else:
                ref = orc.factor_G_entries(inputs.half_bits(gys[l]), rows, d, ij)
                scale = np.sqrt(np.abs(orc.factor_G_entries(inputs.half_bits(gys[l]), rows, d,
                                                            np.stack([ij[:, 0], ij[:, 0]], 1)) *
                                       orc.factor_G_entries(inputs.half_bits(gys[l]), rows, d,
                                                            np.stack([ij[:, 1], ij[:, 1]], 1))))
            # entry error relative to sqrt(A_ii A_jj) (the Cauchy-Schwarz scale of the entry): an
            # entrywise form of the north-star relative error bound 2e-3
            err = np.max(np.abs(g - ref) / np.maximum(scale, 1e-30))
            errs.append((err, layer["name"], "AG"[which]))
    errs.sort(reverse=True)
    print(f"{cfg}: worst sampled entry errors {[(f'{e:.1e}', n, w) for e, n, w in errs[:6]]}")
    assert errs[0][0] <= TOL_FACTOR, errs[:3]


@pytest.mark.parametrize("gamma", [2.5e-2, 2.5e-4])
def test_inverse_report(K, orc, gamma):
    """kfac_inverse_report: the a-priori bound tr(M_d)/delta of every matrix (R-12) against the
    host's own trace arithmetic, and the precision each mode assigns (AUTO: int8 slices iff the
    bound is <= 3e6)."""
    layers = [shapes.linear("a", 300, 40, bias=0), shapes.linear("b", 129, 7, bias=0)]
    rng = np.random.default_rng(3)
    mats = []
    for l in layers:
        pair = []
        for d in shapes.dims(l):
            X = np.maximum(rng.standard_normal((max(d // 4, 1), d)), 0)
            pair.append((X.T @ X / X.shape[0]).astype(np.float32).astype(np.float64))
        mats.append(pair)
    for prec in (0, 1, 2):
        st = K.KfacStep(layers, 1, inv_precision=prec)
        for k, (A, G) in enumerate(mats):
            _, pa, pg = st.recv_views(k)
            pa.copy_(torch.as_tensor(orc.pack(A), dtype=torch.float32))
            pg.copy_(torch.as_tensor(orc.pack(G), dtype=torch.float32))
        st.inverse(gamma)
        rep = st.inverse_report()
        for k, (A, G) in enumerate(mats):
            _, _, pi = orc.damp(A, G, gamma)
            for which, (M, add) in enumerate(((A, pi * np.sqrt(gamma)), (G, np.sqrt(gamma) / pi))):
                want = (np.trace(M) + M.shape[0] * add) / add
                got = rep[k][0][which]
                assert abs(got - want) <= 1e-6 * want, (k, which, got, want)
                sl = rep[k][1][which]
                assert sl == {0: 5 if want <= 3e6 else 0, 1: 0, 2: 5}[prec], (prec, k, which, want, sl)
        assert st.dev_status.cpu().abs().sum().item() == 0
