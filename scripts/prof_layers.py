"""Per-layer timing of the factor kernels (single-problem launches) for a config."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1811_12019_b200 as K
from synth import shapes, inputs

cfg = sys.argv[1] if len(sys.argv) > 1 else "resnet50"
layers, n = shapes.config(cfg)
tot = 0.0
for i, l in enumerate(layers):
    x = inputs.layer_x(l, i, n).cuda()
    gy = inputs.layer_gy(l, i, n).cuda()
    da, dg = shapes.dims(l)
    rows = shapes.rows(l, n)
    res = []
    for which, t, d in ((0, x, da), (1, gy, dg)):
        out = torch.empty(d * (d + 1) // 2, device="cuda")
        wsb = K.factor_ws_bytes(l, n, which)
        ws = torch.empty(max(wsb, 16), dtype=torch.uint8, device="cuda")
        f = K.factor_A if which == 0 else K.factor_G
        for _ in range(2):
            f(l, t, n, 1.0 / rows, out, ws)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        R = 5
        for _ in range(R):
            f(l, t, n, 1.0 / rows, out, ws)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / R
        tot += ms
        tf = rows * d * (d + 1) / (ms / 1e3) / 1e12
        gb = (t.numel() * 2) / (ms / 1e3) / 1e9
        res.append(f"{'AG'[which]} d={d:5d} {ms:8.3f} ms {tf:7.1f} TF/s {gb:7.1f} GB/s")
    print(f"{i:2d} {l['name']:8s} rows={rows:7d} | " + " | ".join(res), flush=True)
print(f"total {tot:.3f} ms")
