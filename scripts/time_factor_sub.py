"""Time the grouped factor launch over a subset of a config's layers:
time_factor_sub.py <config> <regex on layer name> [A|G|AG]"""
import os, re, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1811_12019_b200 as K
from synth import shapes, inputs
cfg, pat = sys.argv[1], sys.argv[2]
which = sys.argv[3] if len(sys.argv) > 3 else "AG"
layers, n = shapes.config(cfg)
idx = [i for i, l in enumerate(layers) if re.search(pat, l["name"])]
sub = [layers[i] for i in idx]
st = K.KfacStep(sub, n, device=torch.device("cuda"))
xs = [inputs.layer_x(layers[i], i, n).cuda() for i in idx]
gys = [inputs.layer_gy(layers[i], i, n).cuda() for i in idx]
# an "A only" / "G only" run zeroes nothing: it just reports the flops of the chosen factors
for _ in range(3):
    st.factors(xs, gys)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
R = 10
e0.record()
for _ in range(R):
    st.factors(xs, gys)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / R
fl = sum(shapes.rows(l, n) * (d * (d + 1)) for l in sub for d in shapes.dims(l))
print(f"{cfg} [{pat}] {len(sub)} layers factors dbg={os.environ.get('KFAC_DBG_MODE','0')}: {ms*1e3:.1f} us  {fl/(ms/1e3)/1e12:.1f} TF/s", flush=True)
