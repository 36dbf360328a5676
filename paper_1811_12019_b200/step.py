"""One distributed K-FAC step (Algorithm 1 body, minus
forward/backward and the update) driven through the C-ABI.

Plumbing only: torch allocates the caller-owned buffers the C-ABI asks for
(kfac_plan_query sizes) and supplies the stream; every stage runs in
libkfac.so kernels / NCCL.
"""
from __future__ import annotations

import torch

from . import kfac


class KfacStep:
    """Caller-owned buffers of one rank + the six stages.

    stale=True also prepares the steps that reuse stale factors (NEXT-1,
    P:701-711; R-20): a stale plan (dW-only ReduceScatter layout) with its own
    send/recv buffers, and a second recv chunk so that kfac_factor_diff can
    compare the factors of two consecutive refreshes.
    """

    def __init__(self, layers, n_local, rank=0, world=1, policy=kfac.RR, comm=None, device=None, stale=False,
                 inv_precision=kfac.INV_AUTO, rs_mode=kfac.RS_PER_OWNER, wire=kfac.WIRE_FP32, wire_scale=(1.0, 1.0)):
        self.layers = list(layers)
        self.rank, self.world, self.n_local = int(rank), int(world), int(n_local)
        self.comm = comm
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.plan = kfac.Plan(self.layers, world, n_local, policy)
        self.plan.set_inverse_precision(inv_precision)
        self.plan.set_rs_mode(rs_mode)
        self.plan.set_wire(wire, *wire_scale)  # before the query: the fp16 wire stages in ws
        q = self.plan.query()
        self.q = q
        self.rl = self.plan.rank_layers(rank)
        dev = self.device
        self.rs_send = torch.zeros(world * q["rs_chunk"], dtype=torch.float32, device=dev)
        # world 1: the mean ReduceScatter is the identity, so the receive buffer IS the send buffer
        # (kfac_reduce_scatter_factors does nothing when send == recv)
        self.rs_recv = self.rs_send if world == 1 else torch.zeros(q["rs_chunk"], dtype=torch.float32, device=dev)
        self.ag_buf = torch.zeros(world * q["ag_chunk"], dtype=torch.float32, device=dev)
        self.inv_ws = torch.zeros(max(self.rl["inv_floats"], 1), dtype=torch.float32, device=dev)
        self.ws = torch.zeros(max(q["ws_bytes"], 16), dtype=torch.uint8, device=dev)
        n_owned = len(self.rl["layers"])
        self.dev_status = torch.zeros(max(2 * n_owned, 1), dtype=torch.int32, device=dev)
        self.pi = torch.zeros(max(n_owned, 1), dtype=torch.float32, device=dev)
        self.splan = None
        if stale:
            self.splan = self.plan.stale_plan()
            self.sq = self.splan.query()
            self.s_send = torch.zeros(world * self.sq["rs_chunk"], dtype=torch.float32, device=dev)
            self.s_recv = torch.zeros(self.sq["rs_chunk"], dtype=torch.float32, device=dev)
            self.rs_recv_prev = torch.zeros_like(self.rs_recv)  # the previous refresh's factors
            self.diff = torch.full((max(2 * n_owned, 1),), float("nan"), dtype=torch.float64, device=dev)
            self.refreshes = 0
            self.gplan = self.plan.grefresh_plan()  # G refresh, A kept stale
            self.gq = self.gplan.query()
            self.g_send = torch.zeros(world * self.gq["rs_chunk"], dtype=torch.float32, device=dev)
            self.g_recv = torch.zeros(self.gq["rs_chunk"], dtype=torch.float32, device=dev)

    # ---- views (zero-copy: the caller's dW lives in the send buffer)
    def dims(self, l):
        L = self.layers[l]
        return L["c_in"] * L["kh"] * L["kw"] + (1 if L["has_bias"] else 0), L["c_out"]

    def dw_view(self, l):
        da, dg = self.dims(l)
        o = self.q["seg_off"][l][0]
        return self.rs_send[o:o + dg * da].view(dg, da)

    def set_dw(self, dws):
        for l, d in enumerate(dws):
            self.dw_view(l).copy_(d, non_blocking=True)

    def stale_dw_view(self, l):
        da, dg = self.dims(l)
        o = self.sq["seg_off"][l][0]
        return self.s_send[o:o + dg * da].view(dg, da)

    def set_stale_dw(self, dws):
        for l, d in enumerate(dws):
            self.stale_dw_view(l).copy_(d, non_blocking=True)

    def send_factor_view(self, l, which):
        da, dg = self.dims(l)
        o = self.q["seg_off"][l][1 + which]
        n = da if which == 0 else dg
        return self.rs_send[o:o + n * (n + 1) // 2]

    def recv_views(self, k):
        """(dW, A packed, G packed) of the k-th owned layer in rs_recv."""
        l = self.rl["layers"][k]
        da, dg = self.dims(l)
        o = self.rl["local_off"][k]
        return (self.rs_recv[o[0]:o[0] + dg * da].view(dg, da), self.rs_recv[o[1]:o[1] + da * (da + 1) // 2],
                self.rs_recv[o[2]:o[2] + dg * (dg + 1) // 2])

    def inv_views(self, k):
        l = self.rl["layers"][k]
        da, dg = self.dims(l)
        a, g = self.rl["inv_off"][k]
        return self.inv_ws[a:a + da * da].view(da, da), self.inv_ws[g:g + dg * dg].view(dg, dg)

    def result(self, l):
        da, dg = self.dims(l)
        o = self.q["ag_off"][l]
        return self.ag_buf[o:o + dg * da].view(dg, da)

    # ---- the six stages
    def factors(self, xs, gys, alphaA=None, alphaG=None, stream=None):
        kfac.factor_all(self.plan, xs, gys, self.rs_send, self.ws, alphaA, alphaG, stream)

    def reduce_scatter(self, stream=None):
        kfac.reduce_scatter_factors(self.comm, self.plan, self.rs_send, self.rs_recv, stream, ws=self.ws)

    def inverse(self, gamma, stream=None):
        kfac.damped_inverse(self.plan, self.rank, self.rs_recv, gamma, self.inv_ws, self.dev_status, self.pi,
                            self.ws, stream)

    def inverse_report(self, stream=None):
        """Per owned layer k: ((bound_A, bound_G), (slices_A, slices_G)) of the last inverse."""
        n = len(self.rl["layers"])
        b, s = kfac.inverse_report(self.plan, self.rank, self.ws, n, stream)
        return [((b[2 * k], b[2 * k + 1]), (s[2 * k], s[2 * k + 1])) for k in range(n)]

    def precondition(self, stream=None):
        kfac.precondition(self.plan, self.rank, self.rs_recv, self.inv_ws, self.ag_buf, self.ws, stream)

    def allgather(self, stream=None):
        kfac.allgather_precond(self.comm, self.plan, self.ag_buf, stream)

    def run_stale(self, stream=None, events=None):
        """A step with stale factors (R-20): dW (set_stale_dw) -> ReduceScatter of the dW-only layout ->
        precondition with the inverses cached by the last full step -> AllGather.  No factor, no inverse."""
        stages = (lambda: kfac.factor_all(self.splan, None, None, self.s_send, self.ws, stream=stream),
                  lambda: kfac.reduce_scatter_factors(self.comm, self.splan, self.s_send, self.s_recv, stream,
                                                      ws=self.ws),
                  lambda: None,
                  lambda: kfac.precondition(self.splan, self.rank, self.s_recv, self.inv_ws, self.ag_buf, self.ws,
                                            stream),
                  lambda: self.allgather(stream))
        for i, f in enumerate(stages):
            f()
            if events is not None:
                events[i].record(stream)

    def grefresh_dw_view(self, l):
        da, dg = self.dims(l)
        o = self.gq["seg_off"][l][0]
        return self.g_send[o:o + dg * da].view(dg, da)

    def set_grefresh_dw(self, dws):
        for l, d in enumerate(dws):
            self.grefresh_dw_view(l).copy_(d, non_blocking=True)

    def run_grefresh(self, gys, gamma, stream=None, events=None):
        """A step that refreshes G but keeps A stale (R-20): G factors only, ReduceScatter of [dW, G],
        G_d^-1 with the pi of the last full step (self.pi), the cached A_d^-1 and its split, AllGather."""
        stages = (lambda: kfac.factor_all(self.gplan, None, gys, self.g_send, self.ws, stream=stream),
                  lambda: kfac.reduce_scatter_factors(self.comm, self.gplan, self.g_send, self.g_recv, stream,
                                                      ws=self.ws),
                  lambda: kfac.damped_inverse(self.gplan, self.rank, self.g_recv, gamma, self.inv_ws, self.dev_status,
                                              self.pi, self.ws, stream),
                  lambda: kfac.precondition(self.gplan, self.rank, self.g_recv, self.inv_ws, self.ag_buf, self.ws,
                                            stream),
                  lambda: self.allgather(stream))
        for i, f in enumerate(stages):
            f()
            if events is not None:
                events[i].record(stream)

    def run_refresh(self, xs, gys, gamma, stream=None, events=None):
        """A full step that also measures Diff against the previous refresh: the recv chunks
        ping-pong, and self.diff[2k + {0, 1}] receives the A / G change rate of the k-th owned layer
        (NaN before the second refresh)."""
        self.rs_recv, self.rs_recv_prev = self.rs_recv_prev, self.rs_recv
        self.run(xs, gys, gamma, stream, events)
        self.refreshes += 1
        if self.refreshes >= 2:
            kfac.factor_diff(self.plan, self.rank, self.rs_recv, self.rs_recv_prev, self.diff, self.ws, stream)

    def update(self, w, w_prev, lr, momentum, rescale=True, eps=1e-9, stream=None):
        """NEXT-3: Eq. paramupdate + Normalizing Weights on every layer's [dG, dA] weights."""
        kfac.update(self.plan, self.ag_buf, w, w_prev, lr, momentum, self.ws, rescale, eps, stream)

    def run(self, xs, gys, gamma, stream=None, events=None):
        """Stages 1-6.  `events`: optional list of 6 torch.cuda.Event recorded after each stage."""
        stages = (lambda: self.factors(xs, gys, stream=stream), lambda: self.reduce_scatter(stream),
                  lambda: self.inverse(gamma, stream), lambda: self.precondition(stream),
                  lambda: self.allgather(stream))
        for i, f in enumerate(stages):
            f()
            if events is not None:
                events[i].record(stream)
