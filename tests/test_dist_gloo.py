"""world_size-2 gloo tests of the multi-rank host logic (CPU, no GPU).

Two processes each build the library plan (kfac_plan_create) for the same
layers, exchange it, and run the ReduceScatterV / AllGatherV of the plan's
owner-major wire layout with torch.distributed (gloo) on CPU buffers shaped
exactly like the device buffers.  The result must equal the oracle's simulated
collectives (R-11, R-16) -- this pins the layout semantics the NCCL
path relies on: rank r's recv chunk = mean over ranks of chunk r, and the AG
buffer holds every layer's result at ag_off.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cfg, policy, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from paper_1811_12019_b200 import kfac
        from synth import shapes
        layers, n = shapes.config(cfg)
        plan = kfac.Plan(layers, world, n, policy)
        qd = plan.query()
        # every rank computed the same plan
        gathered = [None] * world
        dist.all_gather_object(gathered, (qd["owner"], qd["seg_off"], qd["rs_chunk"], qd["ag_off"], qd["ag_chunk"]))
        assert all(g == gathered[0] for g in gathered)
        ref = oracle.plan(layers, world, policy)
        assert qd["owner"] == ref["owner"].tolist() and qd["rs_chunk"] == ref["rs_chunk"]
        # ReduceScatterV over the wire layout: rank-dependent send buffers
        c = qd["rs_chunk"]
        rng = np.random.default_rng(100 + rank)
        send = torch.from_numpy(rng.standard_normal(world * c).astype(np.float64))
        recv = torch.empty(c, dtype=torch.float64)
        dist.reduce_scatter_tensor(recv, send, op=dist.ReduceOp.SUM)
        recv /= world
        sends = [torch.empty_like(send) for _ in range(world)]
        dist.all_gather(sends, send)
        want = oracle.reduce_scatter([s.numpy() for s in sends], ref)[rank]
        assert np.allclose(recv.numpy(), want, rtol=1e-14, atol=1e-14)
        # layers this rank owns live in its chunk at the plan's local offsets
        rl = plan.rank_layers(rank)
        assert rl["layers"] == ref["owned"][rank]
        # AllGatherV: every rank contributes its ag slot, everyone gets all slots
        a = qd["ag_chunk"]
        slot = torch.full((a,), float(rank + 1), dtype=torch.float64)
        full = torch.empty(world * a, dtype=torch.float64)
        dist.all_gather_into_tensor(full, slot)
        for l, off in enumerate(qd["ag_off"]):
            assert full[off].item() == float(qd["owner"][l] + 1)
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("cfg,policy", [("resnet50", 1), ("stress", 0), ("single_conv", 0)])
def test_two_rank_layout_collectives(cfg, policy):
    from conftest import build_lib
    build_lib()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, cfg, policy, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res


def _stale_worker(rank, world, port, cfg, policy, q):
    """Stale steps (R-20): each rank places its dW at the library's stale-plan offsets, the gloo
    ReduceScatter of the dW-only layout must deliver the oracle's stale recv chunk, and every owned
    layer's dW there must be the rank mean."""
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from paper_1811_12019_b200 import kfac
        from synth import inputs, shapes
        layers, n = shapes.config(cfg)
        st = kfac.Plan(layers, world, n, policy).stale_plan()
        qd = st.query()
        ref = oracle.plan(layers, world, policy, stale=True)
        dws = [inputs.layer_dw(l, i, rank).double() for i, l in enumerate(layers)]
        send = torch.zeros(world * qd["rs_chunk"], dtype=torch.float64)
        for l, d in enumerate(dws):
            o = qd["seg_off"][l][0]
            send[o:o + d.numel()] = d.reshape(-1)
        recv = torch.empty(qd["rs_chunk"], dtype=torch.float64)
        dist.reduce_scatter_tensor(recv, send, op=dist.ReduceOp.SUM)
        recv /= world
        all_dws = [None] * world
        dist.all_gather_object(all_dws, [d.numpy() for d in dws])
        want = oracle.reduce_scatter([oracle.build_send(layers, ref, r, None, all_dws[r]) for r in range(world)],
                                     ref)[rank]
        assert np.allclose(recv.numpy(), want, rtol=1e-14, atol=1e-14)
        rl = st.rank_layers(rank)
        for k, l in enumerate(rl["layers"]):
            o = rl["local_off"][k][0]
            mean = sum(a[l] for a in all_dws) / world
            assert np.allclose(recv[o:o + mean.size].numpy(), mean.reshape(-1), rtol=1e-14, atol=1e-14)
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("cfg,policy", [("resnet18_cifar", 1), ("resnet50", 0)])
def test_two_rank_stale_layout(cfg, policy):
    from conftest import build_lib
    build_lib()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_stale_worker, args=(r, 2, port, cfg, policy, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res
