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
