"""Run one RN50 layer's factor kernel R times (for ncu): one_factor.py <layer> <A|G> [R] [config]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1811_12019_b200 as K
from synth import shapes, inputs
li, which = int(sys.argv[1]), "AG".index(sys.argv[2])
R = int(sys.argv[3]) if len(sys.argv) > 3 else 3
cfg = sys.argv[4] if len(sys.argv) > 4 else "resnet50"
layers, n = shapes.config(cfg)
l = layers[li]
t = (inputs.layer_x(l, li, n) if which == 0 else inputs.layer_gy(l, li, n)).cuda()
da, dg = shapes.dims(l)
d = da if which == 0 else dg
out = torch.empty(d * (d + 1) // 2, device="cuda")
ws = torch.empty(max(K.factor_ws_bytes(l, n, which), 16), dtype=torch.uint8, device="cuda")
f = K.factor_A if which == 0 else K.factor_G
for _ in range(R):
    f(l, t, n, 1.0 / shapes.rows(l, n), out, ws)
torch.cuda.synchronize()
print("ok", l["name"], "AG"[which], d)
