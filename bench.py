#!/usr/bin/env python
"""K-FAC hot-path benchmark (BASELINE.json metric: "ResNet-50 K-FAC step ms & factor
TFLOP/s at 1/2/4/8 B200, % roofline").

A step is one pass of the whole hot path -- factors (A, G) + ReduceScatterV +
damped inverse + precondition + AllGatherV (Alg. 1) -- for
every layer of the configuration, on synthetic inputs of the paper's shapes
(ResNet-50/ImageNet, batch 32 per GPU).  One process per GPU; launched with
torchrun for N > 1.  Prints ONE JSON line on rank 0.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config resnet50] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from synth import inputs, shapes  # noqa: E402

METRIC = "ResNet-50 K-FAC step ms & factor TFLOP/s at 1/2/4/8 B200, % roofline"
# derived peaks: 148 SM x lanes x 2 flop x 1.965 GHz
FP64_PEAK_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12   # 37.2 (DFMA)
NVLINK_GBS = 770.0                                   # measured peer copy per direction (B200_PROFILING.md)


def peaks():
    p = dict(hbm_gbs=6650.0, bf16_tflops=1590.0, bf16_tflops_sustained=1400.0, src="fallback (B200_PROFILING.md)")
    f = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(f):
        m = json.load(open(f))
        p = dict(hbm_gbs=m["hbm_gbs"], bf16_tflops=m["bf16_tflops"], bf16_tflops_sustained=m["bf16_tflops_sustained"],
                 src="measured (MEASURED_PEAKS.json)")
    return p


def work(layers, n, plan_q=None, rank_layers=None):
    """Algorithmic work of one step on one rank."""
    fac_flops = fac_bytes = 0
    for l in layers:
        da, dg = shapes.dims(l)
        rows = shapes.rows(l, n)
        fac_flops += rows * (da * (da + 1) + dg * (dg + 1))  # upper triangle, 2 flop / MAC
        ho, wo = shapes.out_hw(l)
        fac_bytes += n * l["h_in"] * l["w_in"] * l["c_in"] * 2 + n * ho * wo * dg * 2  # x, gy read once
        fac_bytes += 4 * (da * (da + 1) // 2 + dg * (dg + 1) // 2)  # packed fp32 out
    inv_flops = prec_flops = 0
    owned = rank_layers if rank_layers is not None else range(len(layers))
    for li in owned:
        da, dg = shapes.dims(layers[li])
        inv_flops += da ** 3 + dg ** 3
        prec_flops += 2 * dg * dg * da + 2 * dg * da * da
    return dict(factor_flops=fac_flops, factor_bytes=fac_bytes, inverse_flops=inv_flops, precond_flops=prec_flops)


class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu):
        self.gpu, self.lines, self.proc = gpu, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.t.join(timeout=2)

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_sample(layers, n, small_dim, threads=0, images=2):
    """Bounded oracle sample, scaled to one full step (ms).  Factors: `images` images of n (rows
    scale linearly); inverse + precondition: layers with max(dA, dG) <= small_dim, scaled by flops.
    Returns (scaled ms, description, threads used, measured s, scale factor)."""
    import numpy as np

    import oracle
    oracle.build()
    t_fac = 0.0
    for i, l in enumerate(layers):
        x = inputs.half_bits(inputs.layer_x(l, i, images))
        gy = inputs.half_bits(inputs.layer_gy(l, i, images))
        t0 = time.perf_counter()
        oracle.factor_A(l, x, images, threads=threads)
        oracle.factor_G(gy, shapes.rows(l, images), l["c_out"], threads=threads)
        t_fac += time.perf_counter() - t0
    t_inv = 0.0
    f_s = f_all = 0
    rng = np.random.default_rng(0)
    for i, l in enumerate(layers):
        da, dg = shapes.dims(l)
        f = da ** 3 + dg ** 3 + 2 * dg * dg * da + 2 * dg * da * da
        f_all += f
        if max(da, dg) > small_dim:
            continue
        f_s += f
        Ba = rng.standard_normal((da, da)) / da
        Bg = rng.standard_normal((dg, dg)) / dg
        A = Ba @ Ba.T + np.eye(da)
        G = Bg @ Bg.T + np.eye(dg)
        dW = rng.standard_normal((dg, da))
        t0 = time.perf_counter()
        Ad, Gd, _ = oracle.damp(A, G, 2.5e-2)
        Ai, _ = oracle.inverse(Ad, threads)
        Gi, _ = oracle.inverse(Gd, threads)
        oracle.precondition(Gi, Ai, dW, threads)
        t_inv += time.perf_counter() - t0
    scaled = (t_fac * n / images + t_inv * (f_all / max(f_s, 1))) * 1e3
    measured = t_fac + t_inv
    desc = (f"oracle factors on {images} of {n} images (x{n / images:g}) + damp/inverse/precondition of layers with dim <= {small_dim} "
            f"({100.0 * f_s / f_all:.1f}% of stage-4/5 flops, scaled by flops); measured {measured:.1f} s")
    used = threads if threads > 0 else oracle.max_threads()
    return scaled, desc, used, measured, scaled / 1e3 / max(measured, 1e-9)


def cpu_full_step(layers, n, xs, gys, dws, gamma, threads=0):
    """One FULL, unsampled oracle step (P:351-376 minus fwd/bwd) on the bench's own inputs at world 1:
    every layer's A and G (explicit patch loops), damping, Cholesky inverses, preconditioning.
    Returns (ms, {stage: s}, threads used)."""
    import oracle
    oracle.build()
    st = {"factors": 0.0, "inverse": 0.0, "precondition": 0.0}
    t_all = time.perf_counter()
    for i, l in enumerate(layers):
        t0 = time.perf_counter()
        A = oracle.factor_A(l, inputs.half_bits(xs[i]), n, threads=threads)
        G = oracle.factor_G(inputs.half_bits(gys[i]), shapes.rows(l, n), l["c_out"], threads=threads)
        t1 = time.perf_counter()
        Ad, Gd, _ = oracle.damp(A, G, gamma)
        Ai, _ = oracle.inverse(Ad, threads)
        Gi, _ = oracle.inverse(Gd, threads)
        t2 = time.perf_counter()
        oracle.precondition(Gi, Ai, dws[i].double().numpy(), threads)
        t3 = time.perf_counter()
        st["factors"] += t1 - t0
        st["inverse"] += t2 - t1
        st["precondition"] += t3 - t2
    ms = (time.perf_counter() - t_all) * 1e3
    return ms, {k: round(v, 2) for k, v in st.items()}, threads if threads > 0 else oracle.max_threads()


def stage_work(l, n):
    """Oracle work per stage of one layer (multiply-adds): factors, inverse, precondition."""
    da, dg = shapes.dims(l)
    return (shapes.rows(l, n) * (da * da + dg * dg), da ** 3 + dg ** 3, dg * da * (da + dg))


def cpu_subset_step(layers, n, subset, gamma, seed=1811, threads=0):
    """The full, unsampled oracle pipeline (all n images) on the layers in `subset`, scaled to the
    whole step stage by stage by the exact work ratio.  Returns (scaled ms, measured s, {stage: s})."""
    import oracle
    oracle.build()
    t = [0.0, 0.0, 0.0]
    for i in subset:
        l = layers[i]
        x = inputs.half_bits(inputs.layer_x(l, i, n, 0, seed))
        gy = inputs.half_bits(inputs.layer_gy(l, i, n, 0, seed))
        dw = inputs.layer_dw(l, i, 0, seed).double().numpy()
        t0 = time.perf_counter()
        A = oracle.factor_A(l, x, n, threads=threads)
        G = oracle.factor_G(gy, shapes.rows(l, n), l["c_out"], threads=threads)
        t1 = time.perf_counter()
        Ad, Gd, _ = oracle.damp(A, G, gamma)
        Ai, _ = oracle.inverse(Ad, threads)
        Gi, _ = oracle.inverse(Gd, threads)
        t2 = time.perf_counter()
        oracle.precondition(Gi, Ai, dw, threads)
        t3 = time.perf_counter()
        t[0] += t1 - t0
        t[1] += t2 - t1
        t[2] += t3 - t2
    w_all = [sum(stage_work(l, n)[q] for l in layers) for q in range(3)]
    w_sub = [sum(stage_work(layers[i], n)[q] for i in subset) for q in range(3)]
    scaled = sum(t[q] * w_all[q] / max(w_sub[q], 1) for q in range(3)) * 1e3
    return scaled, sum(t), {"factors": round(t[0], 2), "inverse": round(t[1], 2), "precondition": round(t[2], 2)}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    layers, n = shapes.config(args.config)
    # each step runs the full oracle pipeline on 1/S of the layers (subsets of similar work mix: layers by
    # descending work, dealt round-robin), scaled stage by stage to the whole step; consecutive steps
    # visit consecutive subsets, so K >= S steps cover every layer
    S = min(8, len(layers))
    order = sorted(range(len(layers)), key=lambda i: -sum(stage_work(layers[i], n)))
    subsets = [sorted(order[j::S]) for j in range(S)]
    for _ in range(args.warmup):
        cpu_subset_step(layers, 1, [order[-1]], args.gamma, args.seed)  # cheap warm-up (library load, page-in)
    import oracle
    vals, meas = [], []
    for st in range(args.steps):
        v, m, _ = cpu_subset_step(layers, n, subsets[st % S], args.gamma, args.seed)
        vals.append(v)
        meas.append(m)
    ms = statistics.mean(vals)
    cores = oracle.max_threads()
    desc = (f"step i = the full oracle pipeline (all {n} images, real inputs) on layer subset i mod {S} "
            f"(~1/{S} of the layers, similar work mix), scaled stage by stage by the exact work ratio")
    out = {"metric": METRIC, "value": round(ms, 3), "unit": "ms", "impl": "reference", "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": False,
           "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": args.config, "global_batch": n * args.gpus, "per_gpu_batch": n},
           "cpu_baseline": {"value": round(ms, 3), "unit": "ms", "cores": cores, "kind": "oracle", "sample": desc,
                            "sampled": True, "measured_s_per_step": round(statistics.mean(meas), 2),
                            "scale": round(ms / 1e3 / max(statistics.mean(meas), 1e-9), 2),
                            "note": "the full unsampled oracle step is the cpu_baseline of the ours arm"},
           "e2e": {"value": round(ms, 3), "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)
    return 0


def flat_views(ts, device=None, pin=False, align=128):
    """One flat buffer holding copies-to-be of the tensors `ts` (same dtype), each view starting on an
    `align`-element boundary; returns (flat, views).  Host buffers are pinned when `pin`."""
    import torch
    offs, off = [], 0
    for t in ts:
        offs.append(off)
        off += (t.numel() + align - 1) // align * align
    flat = torch.empty(off, dtype=ts[0].dtype, device=device)
    if pin:
        flat = flat.pin_memory()
    views = [flat[o:o + t.numel()].view(t.shape) for o, t in zip(offs, ts)]
    if device is None:
        for v, t in zip(views, ts):
            v.copy_(t)
    return flat, views


def run_ours(args):
    import torch
    import torch.distributed as dist

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        if world == 1 and args.gpus > 1:
            print(json.dumps({"error": "--gpus N>1 must be launched with torchrun"}), flush=True)
            return 2
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    import paper_1811_12019_b200 as K

    comm = None
    if world > 1:
        uid = torch.zeros(128, dtype=torch.uint8, device=dev)
        if rank == 0:
            uid.copy_(torch.frombuffer(bytearray(K.comm_unique_id()), dtype=torch.uint8))
        dist.broadcast(uid, 0)
        comm = K.Comm(bytes(uid.cpu().numpy().tobytes()), rank, world, local)

    layers, n = shapes.config(args.config)
    policy = K.LPT if args.policy == "lpt" else K.RR
    st = K.KfacStep(layers, n, rank=rank, world=world, policy=policy, comm=comm, device=dev,
                    stale=not args.no_stale, inv_precision={"auto": K.INV_AUTO, "fp64": K.INV_FP64,
                                                            "int8": K.INV_INT8}[args.inv_precision],
                    rs_mode={"padded": K.RS_PADDED, "per_owner": K.RS_PER_OWNER}[args.rs_mode],
                    wire={"fp32": K.WIRE_FP32, "fp16": K.WIRE_FP16}[args.wire])
    # synthetic inputs of this rank (global-sample seeded), pinned host copies for the e2e leg
    t0 = time.time()
    # x and gy of all layers live in ONE flat buffer (per-layer views 256-byte aligned), host (pinned)
    # and device alike, so a step's input upload is a single large H2D copy
    L_ = len(layers)
    xg_h, xg_views = flat_views([inputs.layer_x(l, i, n, rank, args.seed) for i, l in enumerate(layers)] +
                                [inputs.layer_gy(l, i, n, rank, args.seed) for i, l in enumerate(layers)], pin=True)
    dws_h = [inputs.layer_dw(l, i, rank, args.seed).pin_memory() for i, l in enumerate(layers)]
    gen_s = time.time() - t0
    xg_d, xg_dv = flat_views(xg_views, device=dev)
    xg_d.copy_(xg_h)
    xs, gys = xg_dv[:L_], xg_dv[L_:]
    st.set_dw([d.to(dev) for d in dws_h])
    in_bytes = sum(x.numel() * 2 for x in xs) + sum(g.numel() * 2 for g in gys)
    dw_bytes = sum(d.numel() * 4 for d in dws_h)
    l2_bytes = 126 * 2 ** 20
    flush = torch.empty(0, device=dev)
    if in_bytes < 2 * l2_bytes:
        flush = torch.empty(256 * 2 ** 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()
    nst = 5
    names = ["factors", "reduce_scatter", "inverse", "precondition", "allgather"]

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local])
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        st.run(xs, gys, args.gamma, stream)
    torch.cuda.synchronize()
    status = st.dev_status.cpu().tolist()

    # ---- device-timed region: inputs resident in HBM; clocks sampled while it runs
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(nst + 1)] for _ in range(args.steps)]
    clk = ClockSampler(local).__enter__()
    time.sleep(0.3)  # sampler start-up, outside the timed region
    barrier()
    l0 = K.kfac.launch_count()
    t_start = time.time()
    for s in range(args.steps):
        if flush.numel():
            flush.fill_(s & 0xFF)
        ev[s][0].record(stream)
        st.run(xs, gys, args.gamma, stream, events=ev[s][1:])
    barrier()
    wall_s = time.time() - t_start
    clk.__exit__(None, None, None)
    launches = K.kfac.launch_count() - l0
    step_ms = [e[0].elapsed_time(e[nst]) for e in ev]
    stage_ms = [[e[i].elapsed_time(e[i + 1]) for e in ev] for i in range(nst)]
    mine = torch.tensor([sum(step_ms)] + [sum(x) for x in stage_ms], dtype=torch.float64, device=dev)
    per_rank = [mine.clone() for _ in range(world)]
    if world > 1:
        dist.all_gather(per_rank, mine)  # every rank's own stage split (the critical rank's below)
        dist.all_reduce(mine, op=dist.ReduceOp.MAX)
    tot = mine.cpu().tolist()
    ms = tot[0] / args.steps
    st_ms = {nm: tot[1 + i] / args.steps for i, nm in enumerate(names)}
    # the critical rank: the last to reach the AllGather (longest stages 1-5); its AllGather is the
    # collective's own cost, where stage_ms (the per-stage max over ranks) charges the AllGather of the
    # ranks that arrive early with their wait for it
    pr = [t.cpu().tolist() for t in per_rank]
    crit = max(range(world), key=lambda r: pr[r][0] - pr[r][len(names)])
    crit_ms = {nm: round(pr[crit][1 + i] / args.steps, 3) for i, nm in enumerate(names)}

    # ---- stale-Fisher steps (NEXT-1; R-20): dW-only ReduceScatter, cached inverses, no factor
    # or inverse work; and the Diff kernel a refresh step adds.  Same timing rules.
    stale = None
    if not args.no_stale:
        st.set_stale_dw([d.to(dev) for d in dws_h])
        st.rs_recv_prev.copy_(st.rs_recv).mul_(0.5)
        for _ in range(args.warmup):
            st.run_stale(stream)
            K.factor_diff(st.plan, rank, st.rs_recv, st.rs_recv_prev, st.diff, st.ws, stream)
        sev = [[torch.cuda.Event(enable_timing=True) for _ in range(nst + 1)] for _ in range(args.steps)]
        dev_ev = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(args.steps)]
        barrier()
        for s in range(args.steps):
            if flush.numel():
                flush.fill_(s & 0xFF)
            sev[s][0].record(stream)
            st.run_stale(stream, events=sev[s][1:])
        for s in range(args.steps):
            dev_ev[s][0].record(stream)
            K.factor_diff(st.plan, rank, st.rs_recv, st.rs_recv_prev, st.diff, st.ws, stream)
            dev_ev[s][1].record(stream)
        barrier()
        # G-only refresh steps (A kept stale): G factors, [dW, G] ReduceScatter, G inverses
        st.set_grefresh_dw([d.to(dev) for d in dws_h])
        for _ in range(args.warmup):
            st.run_grefresh(gys, args.gamma, stream)
        gev = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(args.steps)]
        barrier()
        for s in range(args.steps):
            if flush.numel():
                flush.fill_(s & 0xFF)
            gev[s][0].record(stream)
            st.run_grefresh(gys, args.gamma, stream)
            gev[s][1].record(stream)
        barrier()
        gms = torch.tensor([sum(e[0].elapsed_time(e[1]) for e in gev) / args.steps], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(gms, op=dist.ReduceOp.MAX)
        sm = torch.tensor([sum(e[0].elapsed_time(e[nst]) for e in sev)] +
                          [sum(e[i].elapsed_time(e[i + 1]) for e in sev) for i in range(nst)] +
                          [sum(e[0].elapsed_time(e[1]) for e in dev_ev)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(sm, op=dist.ReduceOp.MAX)
        sm = (sm / args.steps).cpu().tolist()
        diff_bytes = 0
        for li in st.rl["layers"]:
            da, dg = shapes.dims(layers[li])
            diff_bytes += 8 * (da * (da + 1) // 2 + dg * (dg + 1) // 2)  # both chunks' packed factors, 4 B each
        dgbs = diff_bytes / (sm[-1] / 1e3) / 1e9
        hbm = peaks()["hbm_gbs"]
        iv = K.refresh_interval(K.RAMPUP, 44)  # the schedule's steady-state interval (20)
        stale = {"step_ms": round(sm[0], 3), "stage_ms": {k: round(sm[1 + i], 3) for i, k in enumerate(names)},
                 "rs_bytes_per_rank": st.sq["rs_chunk"] * 4, "full_rs_bytes_per_rank": st.q["rs_chunk"] * 4,
                 "refresh_interval": iv, "amortized_ms": round((ms + (iv - 1) * sm[0]) / iv, 3),
                 "diff_ms": round(sm[-1], 4),
                 "grefresh_step_ms": round(gms.item(), 3),
                 "grefresh_rs_bytes_per_rank": st.gq["rs_chunk"] * 4,
                 "diff_roofline": {"bound": "hbm", "achieved": round(dgbs, 1), "peak": hbm, "unit": "GB/s",
                                   "frac": round(dgbs / hbm, 4), "traffic": None,
                                   "kernel": "diff_partial_kernel + diff_final_kernel",
                                   "bytes_counting": "8 B per owned packed factor element (cur + prev fp32)"}}

    # ---- the update after the AllGather (NEXT-3): Eq. paramupdate + Normalizing Weights on
    # every layer's weights (replicated on every rank), timed over K launches like the rest.
    upd = None
    if not args.no_stale:
        gw = torch.Generator(device=dev).manual_seed(args.seed)
        w_l = [torch.randn(shapes.dims(l)[1] * shapes.dims(l)[0], generator=gw, device=dev) * 0.05 for l in layers]
        wp_l = [w + 0.01 for w in w_l]
        for _ in range(args.warmup):
            st.update(w_l, wp_l, 8.18e-3, 0.997, stream=stream)
        uev = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(args.steps)]
        barrier()
        for s in range(args.steps):
            uev[s][0].record(stream)
            st.update(w_l, wp_l, 8.18e-3, 0.997, stream=stream)
            uev[s][1].record(stream)
        barrier()
        um = torch.tensor([sum(e[0].elapsed_time(e[1]) for e in uev) / args.steps], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(um, op=dist.ReduceOp.MAX)
        nw = sum(w.numel() for w in w_l)
        ugbs = 20 * nw / (um.item() / 1e3) / 1e9
        hbm = peaks()["hbm_gbs"]
        upd = {"ms": round(um.item(), 4), "weights": nw, "rescale": True,
               "roofline": {"bound": "hbm", "achieved": round(ugbs, 1), "peak": hbm, "unit": "GB/s",
                            "frac": round(ugbs / hbm, 4), "traffic": None,
                            "kernel": "update_step_kernel + update_scale_kernel",
                            "bytes_counting": "20 B per weight (w, w_prev, P read; w, w_prev written)"}}
        del w_l, wp_l

    # ---- the Batch Normalization Fisher (NEXT-2, R-22): per-sample scale / shift gradients of the 53
    # RN50 BN layers (one after every conv) from xhat, gy of the conv-output shape, then the diagonal and
    # the full (Woodbury) preconditioners with gamma_BN = rho_BN * gamma (Table 3: rho_BN = 16).
    bn = None
    if not args.no_stale and args.config == "resnet50":
        convs = [l for l in layers if l["kind"] == 0]
        bc = [l["c_out"] for l in convs]
        bhw = [shapes.out_hw(l)[0] * shapes.out_hw(l)[1] for l in convs]
        gb = torch.Generator(device=dev).manual_seed(args.seed + 7)
        bx = [torch.randn(n, hw, c, generator=gb, device=dev).to(torch.bfloat16) for c, hw in zip(bc, bhw)]
        bg = [(torch.randn(n, hw, c, generator=gb, device=dev) * 0.01).to(torch.bfloat16) for c, hw in zip(bc, bhw)]
        bS = [torch.empty(n, 2 * c, device=dev) for c in bc]
        bgr = [torch.randn(2 * c, generator=gb, device=dev) for c in bc]
        bo = [torch.empty(2 * c, device=dev) for c in bc]
        lam = 16.0 * args.gamma
        bws = torch.empty(K.bn_ws_bytes(bc, n), dtype=torch.uint8, device=dev)

        def bn_run(full):
            K.bn_grads(bc, bhw, bx, bg, n, bS, stream)
            K.bn_precondition(bc, n, bS, bgr, lam, full, bo, bws, stream)

        res = {}
        for full in (0, 1):
            for _ in range(args.warmup):
                bn_run(full)
            bev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
            barrier()
            for s in range(args.steps):
                bev[s][0].record(stream)
                K.bn_grads(bc, bhw, bx, bg, n, bS, stream)
                bev[s][1].record(stream)
                K.bn_precondition(bc, n, bS, bgr, lam, full, bo, bws, stream)
                bev[s][2].record(stream)
            barrier()
            res[full] = (sum(e[0].elapsed_time(e[1]) for e in bev) / args.steps,
                         sum(e[1].elapsed_time(e[2]) for e in bev) / args.steps)
        bbytes = sum(4 * n * hw * c for c, hw in zip(bc, bhw))  # xhat + gy, 2 B each, read once
        ggbs = bbytes / (res[1][0] / 1e3) / 1e9
        hbm = peaks()["hbm_gbs"]
        bn = {"layers": len(bc), "grads_ms": round(res[1][0], 4), "precond_diag_ms": round(res[0][1], 4),
              "precond_full_ms": round(res[1][1], 4),
              "full_fim_bytes_paper": sum(4 * (2 * c) * (2 * c + 1) // 2 for c in bc),
              "full_fim_bytes_woodbury_S": sum(4 * n * 2 * c for c in bc),
              "grads_roofline": {"bound": "hbm", "achieved": round(ggbs, 1), "peak": hbm, "unit": "GB/s",
                                 "frac": round(ggbs / hbm, 4), "traffic": None, "kernel": "bn_grads_kernel",
                                 "bytes_counting": "4 B per (sample, pixel, channel): xhat + gy bf16"}}
        del bx, bg

    # ---- end-to-end through the public API with host buffers (H2D inputs, D2H result).  Every
    # step's inputs are copied from pinned host memory and its result read back inside the timed
    # region; the copies run on their own streams (H2D and D2H directions concurrently) and are
    # double-buffered, so step s+1's upload overlaps step s's compute (a training loop prefetching
    # its next batch).  Dependencies: the dW upload waits for the previous step's ReduceScatter
    # (dW lives in the send buffer), an input set is reused two steps later, the result read-back
    # of step s must finish before step s+1's precondition rewrites the AllGather buffer.
    e2e = None
    if not args.no_e2e:
        out_h = torch.empty(st.ag_buf.numel(), dtype=torch.float32).pin_memory()
        dwv = [st.dw_view(l) for l in range(len(layers))]
        xg_d2, xg_dv2 = flat_views(xg_views, device=dev)
        bufs = [(xg_d, xs, gys), (xg_d2, xg_dv2[:L_], xg_dv2[L_:])]
        up_s, down_s = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)

        def e2e_run(ke):
            E = lambda: torch.cuda.Event()  # noqa: E731
            ev_up, ev_fac, ev_rs, ev_ag, ev_dn = ([E() for _ in range(ke)] for _ in range(5))

            def upload(s):
                # x, gy of step s go into the input buffer step s-2 used (its factors are done); only the
                # dW copy waits for step s-1's ReduceScatter (dW lives in the send buffer), so the
                # uploads run back to back on the copy stream and the PCIe link stays busy
                flat = bufs[s % 2][0]
                if s >= 2:
                    up_s.wait_event(ev_fac[s - 2])
                with torch.cuda.stream(up_s):
                    flat.copy_(xg_h, non_blocking=True)  # every layer's x and gy in one copy
                if s >= 1:
                    up_s.wait_event(ev_rs[s - 1])
                with torch.cuda.stream(up_s):
                    for d, dh in zip(dwv, dws_h):
                        d.copy_(dh, non_blocking=True)
                ev_up[s].record(up_s)

            upload(0)
            for s in range(ke):
                _, X, Gy = bufs[s % 2]
                stream.wait_event(ev_up[s])
                st.factors(X, Gy, stream=stream)
                ev_fac[s].record(stream)
                st.reduce_scatter(stream)
                ev_rs[s].record(stream)
                if s + 1 < ke:
                    upload(s + 1)
                st.inverse(args.gamma, stream)
                if s >= 1:
                    stream.wait_event(ev_dn[s - 1])
                st.precondition(stream)
                st.allgather(stream)
                ev_ag[s].record(stream)
                down_s.wait_event(ev_ag[s])
                with torch.cuda.stream(down_s):
                    out_h.copy_(st.ag_buf, non_blocking=True)
                ev_dn[s].record(down_s)
            stream.wait_event(ev_dn[ke - 1])

        e2e_run(2)
        barrier()
        up_s.wait_stream(stream)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ke = max(2, args.steps)  # the same K as the device-timed region (fill and drain amortised alike)
        e0.record(stream)
        up_s.wait_event(e0)  # the first upload starts inside the timed region
        e2e_run(ke)
        e1.record(stream)
        barrier()
        em = torch.tensor([e0.elapsed_time(e1) / ke], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(em, op=dist.ReduceOp.MAX)
        e2e = {"value": round(em.item(), 3), "unit": "ms", "h2d_bytes_per_step": xg_h.numel() * 2 + dw_bytes,
               "d2h_bytes_per_step": out_h.numel() * 4, "steps": ke,
               "pipelining": "H2D of step s+1 overlaps step s (double-buffered inputs, separate copy streams; "
                             "x / gy uploads back to back, dW after the previous ReduceScatter)"}

    # ---- roofline of the dominant stage (+ the factor kernel, the north-star contraction)
    pk = peaks()
    w = work(layers, n, rank_layers=st.rl["layers"])
    wmax = torch.tensor([w["inverse_flops"], w["precond_flops"]], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(wmax, op=dist.ReduceOp.MAX)
    fac_s = st_ms["factors"] / 1e3
    fac_tflops = w["factor_flops"] / fac_s / 1e12
    fac_roof = {"bound": "tensor", "achieved": round(fac_tflops, 2), "peak": pk["bf16_tflops_sustained"],
                "unit": "TFLOP/s", "frac": round(fac_tflops / pk["bf16_tflops_sustained"], 4), "traffic": None,
                "kernel": "factor_syrk_kernel (+fixup, bias)", "flops_counting": "upper triangle, rows*d*(d+1)",
                "hbm_gbs": round(w["factor_bytes"] / fac_s / 1e9, 1), "peak_src": pk["src"] + " sustained"}
    inv_tf = w["inverse_flops"] / (st_ms["inverse"] / 1e3) / 1e12
    # per-matrix precision of the sweep (kfac_inverse_report, reading R-12): int8-digit matrices run
    # 15 digit-pair MMAs per 128^3 update tile and 21 per panel product on the int8 tensor cores, the
    # others n^3 fp64 flops on DMMA.  Executed int8 ops per matrix of nt blocks: sum over steps of
    # (nt - 1) panels x 21 + nt (nt - 1) / 2 update tiles x 15, times 2 * 128^3.
    rep = st.inverse_report()
    i8_ops, f64_flops, n_i8 = 0, 0, 0
    for k, li in enumerate(st.rl["layers"]):
        for which, d in enumerate(shapes.dims(layers[li])):
            if rep[k][1][which]:
                nt_ = (d + 127) // 128
                i8_ops += nt_ * ((nt_ - 1) * 21 + nt_ * (nt_ - 1) // 2 * 15) * 2 * 128 ** 3
                n_i8 += 1
            else:
                f64_flops += d ** 3
    i8_peak = pk["bf16_tflops_sustained"] * 2.0  # int8 dense = 2x bf16 (B200 nominal 4.5 / 2.25 P)
    i8_tops = i8_ops / (st_ms["inverse"] / 1e3) / 1e12
    prec_peak = pk["bf16_tflops_sustained"] * 0.5 / 3.0
    prec_tf = w["precond_flops"] / (st_ms["precondition"] / 1e3) / 1e12
    rs_bytes = st.q["rs_chunk"] * 4 * (world - 1)
    roofs = {
        "factors": fac_roof,
        "inverse": ({"bound": "tensor", "achieved": round(i8_tops, 2), "peak": round(i8_peak, 1), "unit": "TOPS",
                     "frac": round(i8_tops / i8_peak, 4), "traffic": None,
                     "kernel": "inverse_kernel (persistent block sweep: int8-digit tcgen05 updates / panels, fp64 pivots)",
                     "ops_counting": "executed int8 MMA ops: 15 digit pairs per 128^3 update tile, 21 per panel product",
                     "int8_matrices": n_i8, "fp64_matrices": len(rep) * 2 - n_i8,
                     "fp64_equivalent_tflops": round(inv_tf, 2),
                     "fp64_equivalent_frac_of_dmma_peak": round(inv_tf / FP64_PEAK_TFLOPS, 3),
                     "peak_src": pk["src"] + " bf16 sustained x 2 (int8 dense = 2x bf16)"}
                    if n_i8 else
                    {"bound": "tensor", "achieved": round(inv_tf, 3), "peak": round(FP64_PEAK_TFLOPS, 1),
                     "unit": "TFLOP/s", "frac": round(inv_tf / FP64_PEAK_TFLOPS, 4), "traffic": None,
                     "kernel": "inverse_kernel (persistent fp64 block sweep on DMMA; + pivot, finalize)",
                     "flops_counting": "n^3 per matrix",
                     "peak_src": "derived fp64 148x64x2x1.965GHz (DMMA measured 37.1, scripts/micro/dmma_bench.cu)"}),
        "precondition": {"bound": "tensor", "achieved": round(prec_tf, 3), "peak": round(prec_peak, 1),
                         "unit": "TFLOP/s", "frac": round(prec_tf / prec_peak, 4), "traffic": None,
                         "kernel": "gemm_3xtf32_kernel (tcgen05 kind::tf32, 3 products per fp32 product)",
                         "flops_counting": "2 dG dA (dA + dG) per layer (useful fp32 flops)",
                         "peak_src": pk["src"] + " bf16 sustained x 1/2 (tf32) / 3 (3xTF32)"},
    }
    if world > 1:
        for nm in ("reduce_scatter", "allgather"):
            b = rs_bytes if nm == "reduce_scatter" else st.q["ag_chunk"] * 4 * (world - 1)
            gbs = b / (st_ms[nm] / 1e3) / 1e9
            roofs[nm] = {"bound": "nvlink", "achieved": round(gbs, 1), "peak": NVLINK_GBS, "unit": "GB/s",
                         "frac": round(gbs / NVLINK_GBS, 4), "traffic": None, "kernel": "NCCL"}
    dom = max((k for k in roofs), key=lambda k: st_ms[k])
    # committed ncu traffic per kernel, if a profile summary exists
    tf = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tf):
        tr = json.load(open(tf))
        for k, r in roofs.items():
            if k in tr:
                r["traffic"] = tr[k]

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        # the full, unsampled oracle step on this run's own inputs (all cores) ...
        xs_c = [inputs.layer_x(l, i, n, rank, args.seed) for i, l in enumerate(layers)]
        gys_c = [inputs.layer_gy(l, i, n, rank, args.seed) for i, l in enumerate(layers)]
        dws_c = [inputs.layer_dw(l, i, rank, args.seed) for i, l in enumerate(layers)]
        v, stg, cores = cpu_full_step(layers, n, xs_c, gys_c, dws_c, args.gamma)
        del xs_c, gys_c
        # ... and one thread on a bounded sample (a full single-thread step would take ~cores x longer)
        v1, desc1, _, m1, sc1 = cpu_sample(layers, n, 576, threads=1, images=1)
        cpu = {"value": round(v, 1), "unit": "ms", "cores": cores, "kind": "oracle",
               "sample": f"one full unsampled {args.config} step (all {len(layers)} layers, batch {n}, gamma "
                         f"{args.gamma}) on this run's own inputs, {cores} threads",
               "sampled": False, "measured_s": round(v / 1e3, 2), "scale": 1.0, "stage_s": stg,
               "single_thread": {"value": round(v1, 1), "unit": "ms", "cores": 1, "sampled": True,
                                 "measured_s": round(m1, 2), "scale": round(sc1, 2), "sample": desc1}}

    if rank == 0:
        out = {
            "metric": METRIC, "value": round(ms, 3), "unit": "ms", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": False, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": args.config, "global_batch": n * world, "per_gpu_batch": n,
                       "parallelism": f"dp{world}+layer-sharded inverse/precondition ({args.policy})",
                       "gamma": args.gamma, "rs_mode": args.rs_mode, "wire": args.wire,
                       "inv_precision": args.inv_precision, "l2": ("inputs %.2f GB > 126 MB L2" % (in_bytes / 1e9)) if not flush.numel()
                       else "L2 flushed (256 MB write) between steps"},
            "factor_tflops": round(fac_tflops, 2),
            "images_per_s": round(n * world / (ms / 1e3), 1),
            "stage_ms": {k: round(v, 3) for k, v in st_ms.items()},
            "stage_ms_critical_rank": dict(crit_ms, rank=crit),
            "roofline": dict(roofs[dom], stage=dom),
            "roofline_factors": fac_roof,
            "roofline_stages": roofs,
            "e2e": e2e,
            "stale": stale,
            "update": upd,
            "bn_fisher": bn,
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
            "timed_wall_s": round(wall_s, 3),
            "cpu_baseline": cpu,
            "dev_status_ok": all(v == 0 for v in status),
            "input_gen_s": round(gen_s, 1),
        }
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.barrier(device_ids=[local])
        del comm
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="resnet50", choices=list(shapes.CONFIGS))
    ap.add_argument("--policy", default="lpt", choices=["lpt", "rr"])
    ap.add_argument("--gamma", type=float, default=2.5e-2)  # gamma^(0), Table 3
    ap.add_argument("--seed", type=int, default=1811)
    ap.add_argument("--rs-mode", default="per_owner", choices=["padded", "per_owner"],
                    help="ReduceScatter: one padded ncclReduceScatter or per-owner grouped ncclReduce (kfac_plan_set_rs_mode)")
    ap.add_argument("--wire", default="fp32", choices=["fp32", "fp16"],
                    help="factor wire of the ReduceScatter (kfac_plan_set_wire; fp16 = NEXT-4(ii), scales 1)")
    ap.add_argument("--inv-precision", default="auto", choices=["auto", "fp64", "int8"],
                    help="damped-inverse update precision (kfac_plan_set_inverse_precision, reading R-12)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-stale", action="store_true", help="skip the stale-Fisher step (NEXT-1), update (NEXT-3) and BN Fisher (NEXT-2) timings")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
