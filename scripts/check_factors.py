"""Full check of the grouped factor launch against torch fp64 on the GPU (G for every layer, A for
1x1 convs / FC): check_factors.py [config]; prints per-problem relative errors and the worst tiles."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1811_12019_b200 as K
from synth import shapes, inputs
cfg = sys.argv[1] if len(sys.argv) > 1 else "resnet50"
layers, n = shapes.config(cfg)
st = K.KfacStep(layers, n, device=torch.device("cuda"))
xs = [inputs.layer_x(l, i, n).cuda() for i, l in enumerate(layers)]
gys = [inputs.layer_gy(l, i, n).cuda() for i, l in enumerate(layers)]
st.factors(xs, gys)
torch.cuda.synchronize()
worst = []
for i, l in enumerate(layers):
    da, dg = shapes.dims(l)
    rows = shapes.rows(l, n)
    cases = [(1, gys[i].reshape(rows, -1), dg)]
    if l["kind"] == "linear" or (l["kh"] == 1 and l["stride_h"] == 1 and l["pad_h"] == 0):
        X = xs[i].reshape(rows, -1)
        if l["has_bias"]:
            X = torch.cat([X, torch.ones(rows, 1, dtype=X.dtype, device=X.device)], 1)
        cases.append((0, X, da))
    for which, X, d in cases:
        Xd = X.double()
        ref = (Xd.T @ Xd) / rows
        got = st.send_factor_view(i, which).double()
        M = torch.zeros(d, d, dtype=torch.float64, device="cuda")
        iu = torch.triu_indices(d, d, device="cuda")
        M[iu[0], iu[1]] = got
        D = (M - torch.triu(ref)).abs()
        scale = torch.sqrt(torch.outer(ref.diagonal(), ref.diagonal())).clamp_min(1e-30)
        E = torch.triu(D / scale)
        e = E.max().item()
        if e > 1e-4:
            nt = (d + 255) // 256
            bad = []
            for ti in range(nt):
                for tj in range(ti, nt):
                    t = E[ti * 256:(ti + 1) * 256, tj * 256:(tj + 1) * 256].max().item()
                    if t > 1e-4:
                        bad.append((ti, tj, f"{t:.1e}"))
            print(f"{l['name']} {'AG'[which]} d={d} rows={rows}: max err {e:.2e} bad tiles {bad[:12]}", flush=True)
        worst.append((e, l["name"], "AG"[which]))
worst.sort(reverse=True)
print("worst", [(f"{e:.1e}", a, b) for e, a, b in worst[:5]])
