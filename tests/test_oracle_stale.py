"""Pins for the oracle's stale-Fisher functions (NEXT-1).

refresh_interval / refresh against the paper's printed schedules and SPEC's
worked examples (tests/golden/stale_schedule.json); fim_diff against closed
forms (scaled identities, a single symmetric off-diagonal perturbation);
the stale wire layout against the layout invariants and the SPEC invariant
"stale iterations carry strictly fewer bytes in stage 3"; a stale
step against the full step it must reproduce when the factors are unchanged
(the always-fresh identity).
"""
import json
import math
import os

import numpy as np
import pytest

from synth import shapes, inputs

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "stale_schedule.json")))


def test_refresh_interval_tables(orc):
    for sched in ("rampup", "step13"):
        for e, iv in GOLD[sched].items():
            assert orc.refresh_interval(int(e), sched) == iv, (sched, e)
    with pytest.raises(ValueError):
        orc.refresh_interval(0, "nope")


def test_refresh_examples(orc):
    for ex in GOLD["refresh_examples"]:
        got = orc.refresh(ex["t"], ex["epoch"], ex["schedule"], ex["fresh_floor"])
        assert got == ex["expected"], ex["cite"]
    with pytest.raises(ValueError):
        orc.refresh(10, 0, interval=0)
    # fresh_floor = inf and interval 1: always fresh
    assert all(orc.refresh(t, 30, fresh_floor=10 ** 9) for t in range(50))
    assert all(orc.refresh(t, 30, interval=1, fresh_floor=0) for t in range(50))


def test_fim_diff_closed_forms(orc):
    n = 7
    I = np.eye(n)
    assert orc.fim_diff(I, I) == 0.0
    assert orc.fim_diff(2 * I, I) == pytest.approx(1.0, rel=1e-15)
    assert orc.fim_diff(0.25 * I, I) == pytest.approx(0.75, rel=1e-15)
    # one symmetric off-diagonal pair (both triangle halves count): sqrt(2)/sqrt(n)
    X = I.copy()
    X[1, 4] = X[4, 1] = 1.0
    assert orc.fim_diff(X, I) == pytest.approx(math.sqrt(2.0 / n), rel=1e-15)
    # a diagonal perturbation counts once: 1/sqrt(n)
    Y = I.copy()
    Y[3, 3] = 2.0
    assert orc.fim_diff(Y, I) == pytest.approx(1.0 / math.sqrt(n), rel=1e-15)
    assert orc.fim_diff(I, np.zeros((n, n))) is None
    with pytest.raises(ValueError):
        orc.fim_diff(np.eye(3), np.eye(4))


def test_diff_percentiles(orc):
    ex = GOLD["percentile_example"]
    p = orc.diff_percentiles(ex["diffs"])
    assert p[50] == pytest.approx(ex["p50"], abs=1e-15)
    rng = np.random.default_rng(5)
    v = rng.random(23)
    p = orc.diff_percentiles(list(v) + [None])
    for q in (5, 25, 50, 75, 95):
        assert p[q] == pytest.approx(float(np.percentile(v, q)), rel=1e-14)  # numpy's default (linear)
    assert orc.diff_percentiles([None])[50] is None


@pytest.mark.parametrize("cfg", ["single_conv", "resnet18_cifar", "resnet50", "stress"])
@pytest.mark.parametrize("P", [1, 2, 4, 8])
@pytest.mark.parametrize("policy", [0, 1])
def test_stale_layout_invariants(orc, cfg, P, policy):
    layers, _ = shapes.config(cfg)
    full = orc.plan(layers, P, policy)
    st = orc.plan(layers, P, policy, stale=True)
    assert np.array_equal(full["owner"], st["owner"]) and full["owned"] == st["owned"]
    assert np.array_equal(full["ag_off"], st["ag_off"]) and full["ag_chunk"] == st["ag_chunk"]
    assert st["rs_chunk"] < full["rs_chunk"]  # stale steps move strictly fewer bytes
    assert (st["seg_off"][:, 1:] == -1).all()
    for r in range(P):
        end = 0
        for l in st["owned"][r]:
            o_w, o_a, o_g = st["local"][r][l]
            a, g = orc.dims(layers[l])
            assert o_a is None and o_g is None and o_w % 16 == 0 and o_w >= end
            end = o_w + a * g
        assert end <= st["rs_chunk"]
    pay = sum(orc.dims(l)[0] * orc.dims(l)[1] for l in layers)
    assert st["rs_chunk"] * P >= pay


def test_stale_step_reproduces_full_step(orc):
    """A stale step with the inverses of a full step on the same factors and the
    same ∇W gives the full step's 𝒢 bitwise."""
    layers, n = shapes.config("single_conv")
    layers = layers + [shapes.conv("c2", 8, 16, 1, 1, 0, 8), shapes.linear("fc", 24, 10, 1)]
    P, gamma = 2, 2.5e-2
    rank_inputs = []
    for r in range(P):
        xs, gys, dws = [], [], []
        for i, l in enumerate(layers):
            xs.append(inputs.half_bits(inputs.layer_x(l, i, 4, rank=r, stem=False)))
            gys.append(inputs.half_bits(inputs.layer_gy(l, i, 4, rank=r)))
            dws.append(inputs.layer_dw(l, i, rank=r).numpy())
        rank_inputs.append((xs, gys, dws, 4))
    full = orc.kfac_step(layers, rank_inputs, P, gamma)
    st = orc.plan(layers, P, 0, stale=True)
    sends = [orc.build_send(layers, st, r, None, rank_inputs[r][2]) for r in range(P)]
    recvs = orc.reduce_scatter(sends, st)
    for r in range(P):
        cached = {l: (v["Ainv"], v["Ginv"]) for l, v in full["results"][r].items()}
        got = orc.stale_results(layers, st, r, recvs[r], cached)
        for l, v in got.items():
            assert np.array_equal(v["dW"], full["results"][r][l]["dW"])
            assert np.array_equal(v["precond"], full["results"][r][l]["precond"])


def test_refresh_kinds(orc):
    """A refreshes with its interval multiplied ('A-multiplier 2, G interval 10 -> A every 20')."""
    for t in range(500, 700):
        ra, rg = orc.refresh_kinds(t, 20, "step13", 500, a_multiple=2)  # interval 20
        assert rg == (t % 20 == 0) and ra == (t % 40 == 0)
        assert not ra or rg  # A implies G
    assert orc.refresh_kinds(3, 0, "rampup", 50, a_multiple=4) == (True, True)  # fresh floor: both
    with pytest.raises(ValueError):
        orc.refresh_kinds(3, 0, a_multiple=0)


@pytest.mark.parametrize("cfg", ["single_conv", "resnet50", "stress"])
@pytest.mark.parametrize("P", [1, 2, 8])
def test_grefresh_layout_invariants(orc, cfg, P):
    layers, _ = shapes.config(cfg)
    full, st = orc.plan(layers, P, 1), orc.plan(layers, P, 1, stale=True)
    gp = orc.plan(layers, P, 1, g_only=True)
    assert st["rs_chunk"] < gp["rs_chunk"] < full["rs_chunk"]
    assert (gp["seg_off"][:, 1] == -1).all() and (gp["seg_off"][:, 2] >= 0).all()
    assert np.array_equal(gp["owner"], full["owner"]) and np.array_equal(gp["ag_off"], full["ag_off"])
    for r in range(P):
        end = 0
        for l in gp["owned"][r]:
            o_w, o_a, o_g = gp["local"][r][l]
            a, g = orc.dims(layers[l])
            assert o_a is None and o_w % 16 == 0 and o_g % 16 == 0 and o_w >= end and o_g >= o_w + g * a
            end = o_g + g * (g + 1) // 2
        assert end <= gp["rs_chunk"]


def test_grefresh_step_reproduces_full_step(orc):
    """A G refresh with the same factors, the full step's π and A_d⁻¹ gives the full step's 𝒢 (R-20)."""
    layers, n = shapes.config("single_conv")
    layers = layers + [shapes.conv("c2", 8, 16, 1, 1, 0, 8), shapes.linear("fc", 24, 10, 1)]
    P, gamma = 2, 2.5e-2
    rank_inputs = []
    for r in range(P):
        xs = [inputs.half_bits(inputs.layer_x(l, i, 4, rank=r, stem=False)) for i, l in enumerate(layers)]
        gys = [inputs.half_bits(inputs.layer_gy(l, i, 4, rank=r)) for i, l in enumerate(layers)]
        dws = [inputs.layer_dw(l, i, rank=r).numpy() for i, l in enumerate(layers)]
        rank_inputs.append((xs, gys, dws, 4))
    full = orc.kfac_step(layers, rank_inputs, P, gamma)
    gp = orc.plan(layers, P, 0, g_only=True)
    sends = []
    for r in range(P):
        xs, gys, dws, nl = rank_inputs[r]
        facs = [(None, orc.factor_G(gys[l], orc.rows(L, nl), L["c_out"])) for l, L in enumerate(layers)]
        sends.append(orc.build_send(layers, gp, r, facs, dws))
    recvs = orc.reduce_scatter(sends, gp)
    for r in range(P):
        cached = {l: (v["Ainv"], v["pi"]) for l, v in full["results"][r].items()}
        got = orc.grefresh_results(layers, gp, r, recvs[r], gamma, cached)
        for l, v in got.items():
            want = full["results"][r][l]
            assert np.array_equal(v["G"], want["G"])
            assert np.allclose(v["G_d"], want["G_d"], rtol=1e-15, atol=0)
            assert np.allclose(v["precond"], want["precond"], rtol=1e-12, atol=1e-15)
