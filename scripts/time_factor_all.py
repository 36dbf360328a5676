"""Time the grouped factor launch (kfac_factor_all) of a config: time_factor_all.py [config]
KFAC_DBG_MODE=1 drops the MMAs, 2 drops the TMA loads, 5 drops the epilogue stores."""
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
fl = sum(shapes.rows(l, n) * (d * (d + 1)) for l in layers for d in shapes.dims(l))
print(f"{cfg} factors dbg={os.environ.get('KFAC_DBG_MODE','0')}: {ms:.3f} ms  {fl/(ms/1e3)/1e12:.1f} TF/s")
