"""Multi-GPU parity of the full K-FAC step (launched with torchrun, one rank per GPU).

  torchrun --nproc-per-node P tests/mp_parity.py [config] [policy]

Every rank runs stages 1-6 through the C-ABI on its own shard (NCCL
ReduceScatter / AllGather over NVLink); rank 0 then checks, against the fp64
oracle simulating the same P ranks (oracle.kfac_step):
  * the reduced factors each owner received (stage 3),
  * every layer's preconditioned gradient in the gathered buffer (stage 6),
  * that the AllGather buffers of all ranks are bitwise identical (replica consistency);
then a stale-factor step (NEXT-1, R-20: new dW, dW-only ReduceScatter, the
cached inverses) against oracle.stale_results, replicas again identical; a G-only
refresh against oracle.grefresh_results; and the BN
Fisher across ranks (kfac_bn_exchange + replicated kfac_bn_precondition, R-22).
Exit code 0 on success.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from synth import inputs, shapes  # noqa: E402

NETS = {
    "small": lambda: ([shapes.conv("stem", 3, 16, 7, 2, 3, 20), shapes.conv("a", 16, 32, 3, 1, 1, 10, bias=1),
                       shapes.conv("b", 32, 64, 1, 2, 0, 10), shapes.conv("c", 64, 64, 3, 1, 1, 5),
                       shapes.linear("fc", 64, 10)], 4),
    "one_layer": lambda: ([shapes.conv("a", 16, 32, 3, 1, 1, 8, bias=1)], 4),  # L < P: redundant owners
    "single_conv": lambda: shapes.config("single_conv"),
    # BASELINE configs 4 and 5 at full size (core step only; see main())
    "resnet50": lambda: shapes.config("resnet50"),
    "stress": lambda: shapes.config("stress"),
}
BIG = ("resnet50", "stress")


def relerr(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(np.asarray(b)), 1e-300))


def unpack(p, d):
    M = np.zeros((d, d))
    M[np.triu_indices(d)] = p
    return M + M.T - np.diag(np.diag(M))


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "small"
    policy = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    rs_mode = int(sys.argv[3]) if len(sys.argv) > 3 else 0  # 0 padded ReduceScatter, 1 per-owner grouped Reduce
    wire = int(sys.argv[4]) if len(sys.argv) > 4 else 0  # 1: fp16 factor wire (NEXT-4(ii), R-23)
    wsc = (2.0, 4.0) if wire else None  # non-unit power-of-two scales (oracle: mean of the fp16 wire values, R-23)
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    # rank 0 runs minutes of fp64 oracle work on the full-size configs while the others wait
    import datetime
    dist.init_process_group("nccl", device_id=dev, timeout=datetime.timedelta(minutes=60))
    import paper_1811_12019_b200 as K

    uid = torch.zeros(128, dtype=torch.uint8, device=dev)
    if rank == 0:
        uid.copy_(torch.frombuffer(bytearray(K.comm_unique_id()), dtype=torch.uint8))
    dist.broadcast(uid, 0)
    comm = K.Comm(bytes(uid.cpu().numpy().tobytes()), rank, world, local)
    layers, n = NETS[cfg]()
    gamma = 2.5e-2
    st = K.KfacStep(layers, n, rank=rank, world=world, policy=policy, comm=comm, device=dev, stale=True, rs_mode=rs_mode,
                    wire=wire, wire_scale=wsc or (1.0, 1.0))
    xs = [inputs.layer_x(l, i, n, rank) for i, l in enumerate(layers)]
    gys = [inputs.layer_gy(l, i, n, rank) for i, l in enumerate(layers)]
    dws = [inputs.layer_dw(l, i, rank) for i, l in enumerate(layers)]
    st.set_dw([d.to(dev) for d in dws])
    st.run([x.to(dev) for x in xs], [g.to(dev) for g in gys], gamma)
    torch.cuda.synchronize()
    ok = st.dev_status.abs().sum().item() == 0
    # replica consistency of the gathered buffer
    bufs = [torch.empty_like(st.ag_buf) for _ in range(world)]
    dist.all_gather(bufs, st.ag_buf)
    recvs = [torch.empty_like(st.rs_recv) for _ in range(world)]
    dist.all_gather(recvs, st.rs_recv)
    # every rank ships its inputs to rank 0 for the oracle
    big = cfg in BIG
    if big:  # rank 0 regenerates every rank's seeded inputs (global sample index, rank-local dW)
        allin = None
        if rank == 0:
            allin = [([inputs.half_bits(inputs.layer_x(l, i, n, r)) for i, l in enumerate(layers)],
                      [inputs.half_bits(inputs.layer_gy(l, i, n, r)) for i, l in enumerate(layers)],
                      [inputs.layer_dw(l, i, r).numpy() for i, l in enumerate(layers)], n) for r in range(world)]
    else:
        payload = ([inputs.half_bits(x) for x in xs], [inputs.half_bits(g) for g in gys], [d.numpy() for d in dws], n)
        allin = [None] * world
        dist.all_gather_object(allin, payload)
    err = 0.0
    if rank == 0:
        import oracle
        for b in bufs[1:]:
            ok &= torch.equal(b, bufs[0])
        ref = oracle.kfac_step(layers, allin, world, gamma, policy=policy, wire=wsc)
        pl = ref["plan"]
        for r in range(world):
            rl = st.plan.rank_layers(r)
            for k, l in enumerate(rl["layers"]):
                da, dg = shapes.dims(layers[l])
                o = rl["local_off"][k]
                got = recvs[r].cpu().double().numpy()
                res = ref["results"][r][l]
                err = max(err, relerr(unpack(got[o[1]:o[1] + da * (da + 1) // 2], da), res["A"]),
                          relerr(unpack(got[o[2]:o[2] + dg * (dg + 1) // 2], dg), res["G"]),
                          relerr(got[o[0]:o[0] + dg * da], res["dW"].reshape(-1)))
        stage3 = err
        g = bufs[0].cpu().double().numpy()
        for l in range(len(layers)):
            da, dg = shapes.dims(layers[l])
            off = pl["ag_off"][l]
            owner = pl["owner"][l]
            e = relerr(g[off:off + dg * da], ref["results"][owner][l]["precond"].reshape(-1))
            err = max(err, e)
        print(f"mp_parity {cfg} P={world} policy={policy} rs_mode={rs_mode} wire={wire}: stage3 err {stage3:.2e}, end-to-end max err {err:.2e}, "
              f"replicas identical {ok}", flush=True)
        ok &= err <= 2e-3
    if big:  # the stale / G-refresh / BN legs are covered by the small nets
        flag = torch.tensor([1 if ok else 0], device=dev)
        dist.broadcast(flag, 0)
        del st, comm
        dist.destroy_process_group()
        sys.exit(0 if flag.item() == 1 else 1)
    # ---- a stale step: new dW, cached inverses
    dws2 = [inputs.layer_dw(l, i, rank, seed=4242) for i, l in enumerate(layers)]
    st.set_stale_dw([d.to(dev) for d in dws2])
    st.run_stale()
    torch.cuda.synchronize()
    bufs = [torch.empty_like(st.ag_buf) for _ in range(world)]
    dist.all_gather(bufs, st.ag_buf)
    all_dw2 = [None] * world
    dist.all_gather_object(all_dw2, [d.numpy() for d in dws2])
    if rank == 0:
        import oracle
        for b in bufs[1:]:
            ok &= torch.equal(b, bufs[0])
        sp = oracle.plan(layers, world, policy, stale=True)
        srecvs = oracle.reduce_scatter([oracle.build_send(layers, sp, r, None, all_dw2[r]) for r in range(world)], sp)
        g = bufs[0].cpu().double().numpy()
        serr = 0.0
        for l in range(len(layers)):
            da, dg = shapes.dims(layers[l])
            owner = pl["owner"][l]
            cached = {m: (v["Ainv"], v["Ginv"]) for m, v in ref["results"][owner].items()}
            want = oracle.stale_results(layers, sp, owner, srecvs[owner], cached)[l]["precond"]
            serr = max(serr, relerr(g[pl["ag_off"][l]:pl["ag_off"][l] + dg * da], want.reshape(-1)))
        print(f"mp_parity {cfg} P={world} stale step: end-to-end max err {serr:.2e}, replicas identical {ok}",
              flush=True)
        ok &= serr <= 2e-3
    # ---- a G-only refresh (A kept stale, R-20): new gy and dW, [dW, G] ReduceScatter, cached pi and A_d^-1
    gys3 = [inputs.layer_gy(l, i, n, rank, seed=777) for i, l in enumerate(layers)]
    dws3 = [inputs.layer_dw(l, i, rank, seed=778) for i, l in enumerate(layers)]
    st.set_grefresh_dw([d.to(dev) for d in dws3])
    st.run_grefresh([g.to(dev) for g in gys3], gamma)
    torch.cuda.synchronize()
    bufs = [torch.empty_like(st.ag_buf) for _ in range(world)]
    dist.all_gather(bufs, st.ag_buf)
    all3 = [None] * world
    dist.all_gather_object(all3, ([inputs.half_bits(g) for g in gys3], [d.numpy() for d in dws3]))
    if rank == 0:
        import oracle
        for b in bufs[1:]:
            ok &= torch.equal(b, bufs[0])
        gp = oracle.plan(layers, world, policy, g_only=True)
        sends = []
        for r in range(world):
            facs = [(None, oracle.factor_G(all3[r][0][l], shapes.rows(L, n), L["c_out"])) for l, L in enumerate(layers)]
            sends.append(oracle.build_send(layers, gp, r, facs, all3[r][1]))
        grecvs = oracle.reduce_scatter(sends, gp, wire=wsc, layers=layers)
        g = bufs[0].cpu().double().numpy()
        gerr = 0.0
        for l in range(len(layers)):
            da, dg = shapes.dims(layers[l])
            owner = pl["owner"][l]
            cached = {m: (v["Ainv"], v["pi"]) for m, v in ref["results"][owner].items()}
            want = oracle.grefresh_results(layers, gp, owner, grecvs[owner], gamma, cached)[l]["precond"]
            gerr = max(gerr, relerr(g[pl["ag_off"][l]:pl["ag_off"][l] + dg * da], want.reshape(-1)))
        print(f"mp_parity {cfg} P={world} G refresh: end-to-end max err {gerr:.2e}, replicas identical {ok}",
              flush=True)
        ok &= gerr <= 2e-3

    # ---- BN Fisher across ranks (NEXT-2, R-22): AllGather of S, mean of the BN grads, replicated solve
    bc, bhw = [64, 256, 6], [25, 9, 16]
    gb = torch.Generator().manual_seed(500 + rank)
    bx = [torch.randn(n, hw, c, generator=gb).to(torch.bfloat16) for c, hw in zip(bc, bhw)]
    bg = [(torch.randn(n, hw, c, generator=gb) * 0.05).to(torch.bfloat16) for c, hw in zip(bc, bhw)]
    bgr = [torch.randn(2 * c, generator=gb) for c in bc]
    S_loc = [torch.empty(n, 2 * c, device=dev) for c in bc]
    S_all = [torch.empty(world * n, 2 * c, device=dev) for c in bc]
    gdev = [g.to(dev) for g in bgr]
    K.bn_grads(bc, bhw, [x.to(dev) for x in bx], [g.to(dev) for g in bg], n, S_loc)
    K.bn_exchange(comm, bc, n, S_loc, S_all, gdev)
    bws = torch.empty(K.bn_ws_bytes(bc, world * n), dtype=torch.uint8, device=dev)
    bout = {f: [torch.empty(2 * c, device=dev) for c in bc] for f in (0, 1)}
    for f in (0, 1):
        K.bn_precondition(bc, world * n, S_all, gdev, 0.4, f, bout[f], bws if f else None)
    torch.cuda.synchronize()
    ball = [None] * world
    dist.all_gather_object(ball, ([inputs.half_bits(x) for x in bx], [inputs.half_bits(g) for g in bg],
                                  [g.numpy() for g in bgr]))
    mine = [torch.cat([bout[0][i], bout[1][i]]) for i in range(len(bc))]
    allb = [[torch.empty_like(m) for _ in range(world)] for m in mine]
    for i, m in enumerate(mine):
        dist.all_gather(allb[i], m)
    if rank == 0:
        import oracle
        berr = 0.0
        for i, (c, hw) in enumerate(zip(bc, bhw)):
            ok &= all(torch.equal(b, allb[i][0]) for b in allb[i][1:])  # replicated: identical on every rank
            Sg = np.concatenate([oracle.bn_sample_grads(ball[r][0][i], ball[r][1][i], n, hw, c) for r in range(world)])
            gm = sum(ball[r][2][i].astype(np.float64) for r in range(world)) / world
            got = allb[i][0].cpu().double().numpy()
            for f, mode in ((0, "diag"), (1, "full")):
                want = oracle.bn_precondition(oracle.bn_fisher(Sg, mode), gm, 0.4)
                berr = max(berr, relerr(got[f * 2 * c:(f + 1) * 2 * c], want))
        print(f"mp_parity {cfg} P={world} BN Fisher: max err {berr:.2e}, replicas identical {ok}", flush=True)
        ok &= berr <= 2e-3
    flag = torch.tensor([1 if ok else 0], device=dev)
    dist.broadcast(flag, 0)
    dist.barrier(device_ids=[local])
    del st, comm
    dist.destroy_process_group()
    sys.exit(0 if flag.item() == 1 else 1)


if __name__ == "__main__":
    main()
