"""Pins for the oracle's ownership/layout and simulated collectives."""
import json
import os

import numpy as np
import pytest

from synth import shapes, inputs

SPEC = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def _layers(n):
    return [shapes.conv(f"c{i}", 8 * (i % 3 + 1), 4 * (i % 2 + 1), 3, 1, 1, 6) for i in range(n)]


def test_assign_spec_examples(orc):
    e = SPEC["assign_3_2"]
    pl = orc.plan(_layers(e["L"]), e["P"], orc.POLICY_RR)
    assert pl["owned"] == e["owned"]
    e = SPEC["assign_2_5"]
    pl = orc.plan(_layers(e["L"]), e["P"], orc.POLICY_RR)
    assert all(len(o) >= 1 for o in pl["owned"])
    for l in range(e["L"]):
        assert sum(l in o for o in pl["owned"]) >= 2


@pytest.mark.parametrize("cfg", ["single_conv", "resnet18_cifar", "resnet50", "stress"])
@pytest.mark.parametrize("P", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("policy", [0, 1])
def test_layout_invariants(orc, cfg, P, policy):
    L, _ = shapes.config(cfg)
    pl = orc.plan(L, P, policy)
    # every layer has exactly one primary owner, which owns it
    for l in range(len(L)):
        assert l in pl["owned"][pl["owner"][l]]
    # segments aligned, non-overlapping, inside the owner's chunk
    for r in range(P):
        spans = []
        for l, offs in pl["local"][r].items():
            a, g = orc.dims(L[l])
            for o, n in zip(offs, (g * a, orc.packed_len(a), orc.packed_len(g))):
                assert o % 16 == 0
                spans.append((o, o + n))
        spans.sort()
        for (a0, a1), (b0, b1) in zip(spans, spans[1:]):
            assert a1 <= b0
        if spans:
            assert spans[-1][1] <= pl["rs_chunk"]
    if policy == 1:
        cost = [orc.layer_cost(l) for l in L]
        load = [sum(cost[l] for l in range(len(L)) if pl["owner"][l] == r) for r in range(P)]
        assert max(load) <= sum(cost) / P + max(cost)  # Graham's LPT bound (weak form)


def test_reduce_scatter_spec_example(orc):
    e = SPEC["reduce_scatter_2"]
    layer = shapes.linear("fc", 1, 1, bias=1)  # dW has dG*dA = 2 values
    pl = orc.plan([layer], 2, orc.POLICY_RR)
    # put the layer at owner 1 by using two layers and looking at layer 1
    pl = orc.plan([layer, layer], 2, orc.POLICY_RR)
    sends = []
    for vals in e["values"]:
        s = np.zeros(2 * pl["rs_chunk"])
        o = pl["seg_off"][1][0]
        s[o:o + 2] = vals
        sends.append(s)
    recv = orc.reduce_scatter(sends, pl)
    o_local = pl["local"][1][1][0]
    assert recv[1][o_local:o_local + 2].tolist() == e["expected"]
    assert pl["owner"][1] == 1 and 1 not in pl["local"][0]


@pytest.mark.parametrize("P", [2, 3, 4])
def test_rs_then_ag_is_mean_allreduce(orc, P):
    """ReduceScatterV ∘ AllGatherV = mean AllReduce, bitwise, rank-ordered sum."""
    rng = np.random.default_rng(P)
    pl = orc.plan(_layers(5), P)
    c = pl["rs_chunk"]
    sends = [rng.standard_normal(P * c) for _ in range(P)]
    recv = orc.reduce_scatter(sends, pl)
    full = orc.all_gather(recv, pl)
    direct = np.zeros(P * c)
    for s in sends:
        direct = direct + s
    direct = direct * (1.0 / P)
    for f in full:
        assert np.array_equal(f, direct)


def test_kfac_step_worker_count_invariance(orc):
    """The whole oracle step gives the same 𝒢 for P = 1, 2, 4 on one global batch."""
    layers = [shapes.conv("a", 8, 8, 3, 1, 1, 4, bias=1), shapes.conv("b", 8, 16, 1, 2, 0, 4),
              shapes.linear("fc", 16, 5)]
    n_glob = 4
    dws = [inputs.layer_dw(l, i, rank=0) for i, l in enumerate(layers)]
    ref = None
    for P in (1, 2, 4):
        nl = n_glob // P
        rin = []
        for r in range(P):
            xs = [inputs.half_bits(inputs.layer_x(l, i, nl, rank=r)) for i, l in enumerate(layers)]
            gys = [inputs.half_bits(inputs.layer_gy(l, i, nl, rank=r)) for i, l in enumerate(layers)]
            rin.append((xs, gys, [d.numpy() for d in dws], nl))
        out = orc.kfac_step(layers, rin, P, 2.5e-2)
        pl = out["plan"]
        got = []
        for l in range(len(layers)):
            a, g = orc.dims(layers[l])
            o = pl["ag_off"][l]
            got.append(out["gathered"][0][o:o + g * a].reshape(g, a))
            for r in range(1, P):
                assert np.array_equal(out["gathered"][r], out["gathered"][0])  # replica consistency
        if ref is None:
            ref = got
        else:
            for a, b in zip(got, ref):
                assert np.linalg.norm(a - b) <= 1e-12 * np.linalg.norm(b)


def test_redundant_owners_identical(orc):
    """L < P: redundant owners compute bitwise-identical 𝒢 (R-16)."""
    layers = [shapes.conv("a", 8, 8, 3, 1, 1, 4, bias=1), shapes.linear("fc", 16, 5)]
    P = 5
    rin = []
    for r in range(P):
        xs = [inputs.half_bits(inputs.layer_x(l, i, 1, rank=r)) for i, l in enumerate(layers)]
        gys = [inputs.half_bits(inputs.layer_gy(l, i, 1, rank=r)) for i, l in enumerate(layers)]
        rin.append((xs, gys, [inputs.layer_dw(l, i, rank=r).numpy() for i, l in enumerate(layers)], 1))
    out = orc.kfac_step(layers, rin, P, 2.5e-2)
    for l in range(len(layers)):
        copies = [out["results"][r][l]["precond"] for r in range(P) if l in out["results"][r]]
        assert len(copies) >= 2
        for c in copies[1:]:
            assert np.array_equal(c, copies[0])


LPT = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "lpt_examples.json")))


@pytest.mark.parametrize("name", [k for k in LPT if k.startswith("cost")])
def test_lpt_hand_worked_costs(orc, monkeypatch, name):
    """R-15's LPT policy on hand-worked cost lists (tests/golden/lpt_examples.json):
    the exact owner list and loads.  Descending order, the (-cost, l) key and the lowest-rank
    tie-break each change the result of at least one example."""
    e = LPT[name]
    layers = [shapes.linear(f"l{i}", 1, 1, bias=0) for i in range(len(e["costs"]))]
    cost = {id(layer): c for layer, c in zip(layers, e["costs"])}
    monkeypatch.setattr(orc, "layer_cost", lambda layer: cost[id(layer)])
    pl = orc.plan(layers, e["P"], orc.POLICY_LPT)
    assert pl["owner"].tolist() == e["owner"]
    load = [sum(c for c, o in zip(e["costs"], e["owner"]) if o == r) for r in range(e["P"])]
    assert load == e["load"]


def test_lpt_hand_worked_fc_dims(orc):
    """The same policy with the real cost model (R-15) on hand-computed FC costs."""
    e = LPT["fc_dims_P3"]
    layers = [shapes.linear(f"fc{i}", a, g, bias=0) for i, (a, g) in enumerate(e["dims"])]
    assert [orc.layer_cost(l) for l in layers] == e["costs"]
    pl = orc.plan(layers, e["P"], orc.POLICY_LPT)
    assert pl["owner"].tolist() == e["owner"]
    assert pl["owned"] == [[l for l in range(len(layers)) if e["owner"][l] == r] for r in range(e["P"])]
