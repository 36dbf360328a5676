"""Time one layer's factor kernel: time_factor.py <layer> <A|G> [config]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1811_12019_b200 as K
from synth import shapes, inputs
li, which = int(sys.argv[1]), "AG".index(sys.argv[2])
cfg = sys.argv[3] if len(sys.argv) > 3 else "resnet50"
layers, n = shapes.config(cfg)
l = layers[li]
t = (inputs.layer_x(l, li, n) if which == 0 else inputs.layer_gy(l, li, n)).cuda()
da, dg = shapes.dims(l)
d = da if which == 0 else dg
out = torch.empty(d * (d + 1) // 2, device="cuda")
ws = torch.empty(max(K.factor_ws_bytes(l, n, which), 16), dtype=torch.uint8, device="cuda")
f = K.factor_A if which == 0 else K.factor_G
rows = shapes.rows(l, n)
for _ in range(3):
    f(l, t, n, 1.0 / rows, out, ws)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
for _ in range(10):
    f(l, t, n, 1.0 / rows, out, ws)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print(f"{l['name']} {'AG'[which]} d={d} rows={rows} dbg={os.environ.get('KFAC_DBG_MODE','0')}: {ms*1e3:.1f} us  {rows*d*(d+1)/(ms/1e3)/1e12:.1f} TF/s")
