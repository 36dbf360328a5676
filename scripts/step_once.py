"""Run the full K-FAC step of a config N times (for launch-list profiling): step_once.py [config] [reps]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1811_12019_b200 as K
from synth import shapes, inputs
cfg = sys.argv[1] if len(sys.argv) > 1 else "resnet50"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
layers, n = shapes.config(cfg)
st = K.KfacStep(layers, n, device=torch.device("cuda"), policy=1)
xs = [inputs.layer_x(l, i, n).cuda() for i, l in enumerate(layers)]
gys = [inputs.layer_gy(l, i, n).cuda() for i, l in enumerate(layers)]
st.set_dw([inputs.layer_dw(l, i).cuda() for i, l in enumerate(layers)])
for _ in range(reps):
    st.run(xs, gys, 2.5e-2)
torch.cuda.synchronize()
print("done")
