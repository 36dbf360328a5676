"""CPU tests of the C-ABI library: it loads, exports every symbol include/kfac.h
declares, and its host-side plan (stage a0) is bit-exact with the oracle's
independent implementation."""
import os
import re

import numpy as np
import pytest

from synth import shapes

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def K():
    from conftest import build_lib
    build_lib()
    from paper_1811_12019_b200 import kfac
    return kfac


def test_exports_every_declared_symbol(K):
    hdr = open(os.path.join(ROOT, "include", "kfac.h")).read()
    declared = sorted(set(re.findall(r"KFAC_API [^;]*?\b(kfac_\w+)\s*\(", hdr)))
    assert len(declared) >= 17
    for name in declared:
        assert hasattr(K._lib, name), name
    assert set(K.EXPORTS) <= set(declared)
    assert "sm_100a" in K.version()


def test_library_is_sm100a_with_tcgen05():
    import subprocess
    lib = os.path.join(ROOT, "paper_1811_12019_b200", "libkfac.so")
    out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
    assert "UTCHMMA" in out and "UTMALDG" in out and "LDTM" in out  # tcgen05.mma / TMA / tcgen05.ld
    assert "sm_100a" in subprocess.run(["cuobjdump", "-lelf", lib], capture_output=True, text=True).stdout


@pytest.mark.parametrize("cfg", ["single_conv", "resnet18_cifar", "resnet50", "stress"])
@pytest.mark.parametrize("P", [1, 2, 3, 4, 5, 8])
@pytest.mark.parametrize("policy", [0, 1])
def test_plan_bit_exact_vs_oracle(K, orc, cfg, P, policy):
    L, n = shapes.config(cfg)
    plan = K.Plan(L, P, n, policy)
    q = plan.query()
    ref = orc.plan(L, P, policy)
    assert q["owner"] == ref["owner"].tolist()
    assert q["rs_chunk"] == ref["rs_chunk"] and q["ag_chunk"] == ref["ag_chunk"]
    assert np.array_equal(np.array(q["seg_off"]), ref["seg_off"])
    assert q["ag_off"] == ref["ag_off"].tolist()
    for r in range(P):
        rl = plan.rank_layers(r)
        assert rl["layers"] == ref["owned"][r]
        assert [tuple(o) for o in rl["local_off"]] == [ref["local"][r][l] for l in ref["owned"][r]]
        # inverse workspace: disjoint, in range
        spans = []
        for l, (a, g) in zip(rl["layers"], rl["inv_off"]):
            da, dg = orc.dims(L[l])
            spans += [(a, a + da * da), (g, g + dg * dg)]
        spans.sort()
        assert all(x[1] <= y[0] for x, y in zip(spans, spans[1:]))
        assert spans[-1][1] <= rl["inv_floats"]
    assert q["ws_bytes"] > 0


def test_plan_errors(K):
    L, n = shapes.config("single_conv")
    with pytest.raises(K.KfacError, match="ERR_ARG"):
        K.Plan(L, 0, n)
    with pytest.raises(K.KfacError, match="ERR_ARG"):
        K.Plan(L, 2, n, policy=7)
    bad = dict(L[0], c_in=0)
    with pytest.raises(K.KfacError, match="ERR_SHAPE"):
        K.Plan([bad], 1, n)
    bad = dict(L[0], kind=3)
    with pytest.raises(K.KfacError, match="ERR_SHAPE"):
        K.Plan([bad], 1, n)
    with pytest.raises(K.KfacError, match="ERR_ARG"):
        K.factor_ws_bytes(L[0], 0, 0)


def test_factor_ws_bytes_split_k(K):
    # large-K / small-d problems are split along K (deterministic fix-up needs scratch)
    L = shapes.resnet50()
    assert K.factor_ws_bytes(L[1], 32, 0) > 0  # l1b0c1: dA=64, 100k rows
    assert K.factor_ws_bytes(L[-1], 32, 0) == 256  # fc: 32 rows -> no partials, only the work-item counter


@pytest.mark.parametrize("cfg", ["single_conv", "resnet50", "stress"])
@pytest.mark.parametrize("P", [1, 2, 5, 8])
@pytest.mark.parametrize("policy", [0, 1])
def test_stale_plan_bit_exact_vs_oracle(K, orc, cfg, P, policy):
    """kfac_plan_create_stale: dW-only layout, bit-exact against oracle.plan(stale=True) (R-20)."""
    L, n = shapes.config(cfg)
    full = K.Plan(L, P, n, policy)
    st = full.stale_plan()
    assert st.stale and not full.stale
    q, qf = st.query(), full.query()
    ref = orc.plan(L, P, policy, stale=True)
    assert q["owner"] == ref["owner"].tolist() == qf["owner"]
    assert q["rs_chunk"] == ref["rs_chunk"] < qf["rs_chunk"]
    assert np.array_equal(np.array(q["seg_off"]), ref["seg_off"])
    assert q["ag_off"] == qf["ag_off"] and q["ag_chunk"] == qf["ag_chunk"] and q["ws_bytes"] == qf["ws_bytes"]
    for r in range(P):
        rl, rf = st.rank_layers(r), full.rank_layers(r)
        assert rl["layers"] == rf["layers"] == ref["owned"][r]
        assert rl["inv_off"] == rf["inv_off"] and rl["inv_floats"] == rf["inv_floats"]
        assert [tuple(-1 if v is None else v for v in ref["local"][r][l]) for l in ref["owned"][r]] == \
            [tuple(o) for o in rl["local_off"]]
    with pytest.raises(K.KfacError, match="ERR_STATE"):
        K.Plan(L, P, n, stale_of=st)


def test_refresh_controller_vs_oracle(K, orc):
    """kfac_refresh_interval / kfac_refresh against the oracle's schedules (pinned to P:705-711)."""
    for sched, name in ((K.RAMPUP, "rampup"), (K.STEP13, "step13")):
        for e in range(0, 60):
            assert K.refresh_interval(sched, e) == orc.refresh_interval(e, name)
            for t in (0, 3, 499, 500, 501, 520, 1000, 1001, 1234):
                for floor in (0, 50, 500):
                    assert K.refresh(t, e, sched, floor) == orc.refresh(t, e, name, floor)
    assert K.refresh(30, 40, K.RAMPUP, 0, interval=3) == orc.refresh(30, 40, fresh_floor=0, interval=3)
    assert K.refresh_interval(9, 0) == -1 and K.refresh_interval(0, -1) == -1
    with pytest.raises(ValueError):
        K.refresh(-1, 0)


@pytest.mark.parametrize("cfg", ["single_conv", "resnet50"])
@pytest.mark.parametrize("P", [1, 2, 5])
def test_grefresh_plan_bit_exact_vs_oracle(K, orc, cfg, P):
    """kfac_plan_create_grefresh: the [dW, G] layout, bit-exact against oracle.plan(g_only=True)."""
    L, n = shapes.config(cfg)
    full = K.Plan(L, P, n, 1)
    gp = full.grefresh_plan()
    assert gp.kind == 1 and full.kind == 0 and full.stale_plan().kind == 2
    q = gp.query()
    ref = orc.plan(L, P, 1, g_only=True)
    assert q["rs_chunk"] == ref["rs_chunk"] and np.array_equal(np.array(q["seg_off"]), ref["seg_off"])
    for r in range(P):
        rl = gp.rank_layers(r)
        assert [tuple(-1 if v is None else v for v in ref["local"][r][l]) for l in ref["owned"][r]] == \
            [tuple(o) for o in rl["local_off"]]
        assert rl["inv_off"] == full.rank_layers(r)["inv_off"]
    with pytest.raises(K.KfacError, match="ERR_STATE"):
        K.Plan(L, P, n, grefresh_of=gp)


def test_plan_lpt_hand_worked(K):
    """plan.cpp's LPT owners on the hand-worked example of tests/golden/lpt_examples.json (R-15)."""
    import json
    e = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "lpt_examples.json")))["fc_dims_P3"]
    layers = [shapes.linear(f"fc{i}", a, g, bias=0) for i, (a, g) in enumerate(e["dims"])]
    assert K.Plan(layers, e["P"], 1, 1).query()["owner"] == e["owner"]
