"""Pins for the oracle's post-AllGather update (NEXT-3).

Table 3's BS=4,096 row and SPEC's derived spot values (tests/golden/update_examples.json),
SPEC's two-step hand trace of Eq. paramupdate, the trivial special cases (m = 0, η = 0),
and the normalizing-weights closed forms (target norm, idempotence, the ε guard).
"""
import json
import math
import os

import numpy as np
import pytest

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "update_examples.json")))
T3 = GOLD["table3_bs4096"]


def test_learning_rate_and_momentum(orc):
    lr = lambda e: orc.learning_rate(T3["eta0"], T3["e_start"], T3["e_end"], T3["p_decay"], e)  # noqa: E731
    assert lr(GOLD["lr_e27"]["epoch"]) == pytest.approx(GOLD["lr_e27"]["expected"], rel=1e-12)
    assert lr(T3["e_start"]) == T3["eta0"] and lr(0) == T3["eta0"]  # clamp before e_start
    assert lr(T3["e_end"]) == 0.0 and lr(80) == 0.0
    vals = [lr(e / 4) for e in range(0, 4 * 60)]
    assert all(a >= b for a, b in zip(vals, vals[1:]))
    m27 = orc.momentum(T3["m0"], T3["eta0"], lr(27))
    assert m27 == pytest.approx(GOLD["momentum_e27"]["expected"], rel=1e-12)
    assert orc.momentum(T3["m0"], T3["eta0"], T3["eta0"]) == pytest.approx(T3["m0"], rel=1e-15)
    for e in (1.5, 10, 30, 52):  # m / eta constant
        assert orc.momentum(T3["m0"], T3["eta0"], lr(e)) / lr(e) == pytest.approx(T3["m0"] / T3["eta0"], rel=1e-14)


def test_apply_update_cases(orc):
    rng = np.random.default_rng(3)
    w, wp, G = (rng.standard_normal((5, 7)) for _ in range(3))
    new, keep = orc.apply_update(w, wp, G, 0.3, 0.0)  # m = 0: plain step
    assert np.array_equal(new, w - 0.3 * G) and np.array_equal(keep, w)
    new, _ = orc.apply_update(w, wp, G, 0.0, 1.0)  # eta = 0, m = 1: the velocity repeats
    assert np.allclose(new - w, w - wp, rtol=0, atol=1e-15)
    tr = GOLD["two_step_trace"]
    w1, k1 = orc.apply_update([tr["w0"]], [tr["w_m1"]], [tr["grads"][0]], tr["eta"], tr["m"])
    w2, _ = orc.apply_update(w1, k1, [tr["grads"][1]], tr["eta"], tr["m"])
    assert w1[0] == pytest.approx(tr["w1"], abs=1e-15) and w2[0] == pytest.approx(tr["w2"], abs=1e-15)
    with pytest.raises(ValueError):
        orc.apply_update(w, wp[:, :3], G, 0.1, 0.1)


def test_rescale_weights(orc):
    ex = GOLD["rescale_dout8_norm2"]
    w = np.zeros((8, 3))
    w[0, 0], w[5, 2] = 1.2, 1.6  # ||w|| = 2
    r = orc.rescale_weights(w, ex["d_out"])
    assert np.linalg.norm(r) == pytest.approx(ex["norm_out"], rel=1e-9)
    assert np.allclose(r, 2.0 * w, rtol=1e-9)
    assert np.allclose(orc.rescale_weights(r, 8), r, rtol=1e-9, atol=0)  # idempotent
    assert np.array_equal(orc.rescale_weights(np.zeros((4, 4)), 4), np.zeros((4, 4)))  # eps guard
    with pytest.raises(ValueError):
        orc.rescale_weights(w, 0)


def test_update_layer_bias_not_rescaled(orc):
    rng = np.random.default_rng(4)
    dg, da = 6, 10  # 9 weight columns + the bias column
    w, wp, G = (rng.standard_normal((dg, da)) for _ in range(3))
    new, keep = orc.update_layer(w, wp, G, 0.05, 0.9, has_bias=True)
    plain, _ = orc.apply_update(w, wp, G, 0.05, 0.9)
    assert np.array_equal(new[:, -1], plain[:, -1])
    assert np.linalg.norm(new[:, :-1]) == pytest.approx(math.sqrt(2 * dg), rel=1e-9)
    assert np.array_equal(keep, w)
    new2, _ = orc.update_layer(w, wp, G, 0.05, 0.9, has_bias=False)
    assert np.linalg.norm(new2) == pytest.approx(math.sqrt(2 * dg), rel=1e-9)
    new3, _ = orc.update_layer(w, wp, G, 0.05, 0.9, has_bias=True, rescale=False)
    assert np.array_equal(new3, plain)
