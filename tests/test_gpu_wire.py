"""GPU parity of the fp16 factor wire (NEXT-4(ii); reading R-23) through the C-ABI
(kfac_plan_set_wire + kfac_reduce_scatter_factors_ws), world 1 here (world 2 / 4 in tests/mp_parity.py).

* the wire round trip (pack -> fp16 -> unpack) against oracle.reduce_scatter(wire=...) on the same fp32
  send buffer: BIT-EXACT, including round-to-nearest-even ties, overflow to inf, fp16 subnormals and
  flush to zero, under non-unit power-of-two scales, with and without send == recv aliasing, ragged
  segment tails, and the stale (dW-only, no staging) and G-refresh layouts;
* a full step with the fp16 wire: the factors the owner receives are exactly the wire values of the
  factors the GPU computed, and 𝒢 end to end against oracle.kfac_step(wire=...) (2e-3).
"""
import numpy as np
import pytest
import torch

from synth import inputs, shapes

pytestmark = pytest.mark.gpu

NET = [shapes.conv("stem", 3, 16, 7, 2, 3, 20), shapes.conv("a", 16, 32, 3, 1, 1, 10, bias=1),
       shapes.conv("b", 32, 64, 1, 2, 0, 10), shapes.conv("c", 64, 64, 3, 1, 1, 5), shapes.linear("fc", 64, 10),
       shapes.linear("odd", 37, 5, bias=1)]  # odd dims: ragged packed tails


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


def _send(orc, pl, layers, seed):
    """A seeded fp32 send buffer: values over 2^-40 .. 2^20, zero padding, and crafted fp16 edge cases
    (ties, overflow, subnormals) at the start of each factor segment."""
    rng = np.random.default_rng(seed)
    n = pl["rs_chunk"]
    send = np.zeros(n, dtype=np.float32)
    edge = np.array([1 + 2 ** -11, 1 + 3 * 2 ** -11, 2049, 2051, 65504, 70000, 2 ** -25, 3 * 2 ** -26,
                     2 ** -24, -(1 + 2 ** -11), 0.1, -0.0], dtype=np.float64)
    for l, (o_w, o_a, o_g) in pl["local"][0].items():
        a, g = orc.dims(layers[l])
        segs = [(o_w, g * a, 1.0)] + [(o, m * (m + 1) // 2, s) for o, m, s in ((o_a, a, 2.0 ** 3), (o_g, g, 2.0 ** -2))
                                      if o is not None]
        for o, ln, s in segs:
            v = rng.standard_normal(ln) * np.exp2(rng.integers(-40, 20, ln))
            k = min(ln, len(edge))
            v[:k] = edge[:k] / s  # the edge cases land on them after scaling
            send[o:o + ln] = v.astype(np.float32)
    return send


@pytest.mark.parametrize("layout", ["full", "grefresh", "stale"])
@pytest.mark.parametrize("alias", [False, True])
def test_wire_roundtrip_bit_exact(K, orc, layout, alias):
    sc = (2.0 ** 3, 2.0 ** -2)
    full = K.Plan(NET, 1, 4, K.RR)
    full.set_wire(K.WIRE_FP16, *sc)
    plan = {"full": full, "grefresh": full.grefresh_plan(), "stale": full.stale_plan()}[layout]
    q = plan.query()
    pl = orc.plan(NET, 1, orc.POLICY_RR, stale=layout == "stale", g_only=layout == "grefresh")
    assert pl["rs_chunk"] == q["rs_chunk"]
    send = _send(orc, pl, NET, 7)
    d_send = torch.from_numpy(send).cuda()
    d_recv = d_send if alias else torch.zeros_like(d_send)  # padding is left untouched (zero on both sides)
    ws = torch.zeros(max(q["ws_bytes"], 16), dtype=torch.uint8, device="cuda")
    K.reduce_scatter_factors(None, plan, d_send, d_recv, ws=ws)
    torch.cuda.synchronize()
    got = d_recv.cpu().numpy().astype(np.float64)
    want = orc.reduce_scatter([send.astype(np.float64)], pl, wire=sc, layers=NET)[0]
    assert np.array_equal(got, want, equal_nan=True), \
        f"{int(np.sum(got != want))} elements differ, first at {int(np.argmax(got != want))}"
    if layout != "stale":  # the factor segments really went through fp16 (else this test proves nothing)
        assert np.isinf(got).any() and not np.array_equal(got, send.astype(np.float64))
    # kfac_reduce_scatter_factors without a workspace refuses a plan that needs staging
    if layout != "stale":
        with pytest.raises(K.KfacError):
            K.reduce_scatter_factors(None, plan, d_send, d_recv)
    else:
        K.reduce_scatter_factors(None, plan, d_send, d_recv)


def test_wire_scale_validation(K):
    plan = K.Plan(NET, 1, 4, K.RR)
    for bad in (3.0, 0.0, -2.0, float("inf"), 2.0 ** 70):
        with pytest.raises(K.KfacError):
            plan.set_wire(K.WIRE_FP16, bad, 1.0)
    with pytest.raises(K.KfacError):
        plan.set_wire(7, 1.0, 1.0)
    b = plan.query()["ws_bytes"]
    plan.set_wire(K.WIRE_FP16, 1.0, 1.0)
    assert plan.query()["ws_bytes"] >= b
    plan.set_wire(K.WIRE_FP32, 1.0, 1.0)
    assert plan.query()["ws_bytes"] == b


@pytest.mark.parametrize("cfg", ["small", "resnet18_cifar"])
def test_step_with_fp16_wire(K, orc, cfg):
    if cfg == "small":
        layers, n = NET, 4
    else:
        layers, n = shapes.config(cfg)
    gamma, sc = 2.5e-2, (1.0, 1.0)
    xs = [inputs.layer_x(l, i, n) for i, l in enumerate(layers)]
    gys = [inputs.layer_gy(l, i, n) for i, l in enumerate(layers)]
    dws = [inputs.layer_dw(l, i) for i, l in enumerate(layers)]
    ref32 = K.KfacStep(layers, n)  # the same step with the fp32 wire: the factors before the wire
    ref32.set_dw([d.cuda() for d in dws])
    ref32.run([x.cuda() for x in xs], [g.cuda() for g in gys], gamma)
    st = K.KfacStep(layers, n, wire=K.WIRE_FP16, wire_scale=sc)
    st.rs_recv = torch.zeros_like(st.rs_send)  # keep the fp32 factors in rs_send for the check below
    st.set_dw([d.cuda() for d in dws])
    st.run([x.cuda() for x in xs], [g.cuda() for g in gys], gamma)
    torch.cuda.synchronize()
    assert st.dev_status.abs().sum().item() == 0
    pl = orc.plan(layers, 1, orc.POLICY_RR)
    # stage 3: the received factors are exactly the wire values of the GPU's own fp32 factors
    sent = st.rs_send.cpu().numpy().astype(np.float64)
    want = orc.reduce_scatter([sent], pl, wire=sc, layers=layers)[0]
    got = st.rs_recv.cpu().numpy().astype(np.float64)
    for l, (o_w, o_a, o_g) in pl["local"][0].items():
        a, g = orc.dims(layers[l])
        for o, ln in ((o_w, g * a), (o_a, a * (a + 1) // 2), (o_g, g * (g + 1) // 2)):
            assert np.array_equal(got[o:o + ln], want[o:o + ln])
    # the fp32-wire step's factors are the same fp32 values (same kernels, same inputs)
    assert torch.equal(ref32.rs_send, st.rs_send)
    # end to end against the oracle step with the fp16 wire
    ref = orc.kfac_step(layers, [([inputs.half_bits(x) for x in xs], [inputs.half_bits(g) for g in gys],
                                  [d.numpy() for d in dws], n)], 1, gamma, wire=sc)
    err = 0.0
    for l in range(len(layers)):
        da, dg = shapes.dims(layers[l])
        err = max(err, relerr(st.result(l).cpu().numpy(), ref["results"][0][l]["precond"]))
    print(f"{cfg}: fp16 wire end-to-end max err {err:.2e}")
    assert err <= 2e-3
