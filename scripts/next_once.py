"""One RN50 refresh step + Diff + update on cuda:0 (for ncu captures of diff.cu / update.cu)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1811_12019_b200 as K  # noqa: E402
from synth import inputs, shapes  # noqa: E402

layers, n = shapes.config("resnet50")
st = K.KfacStep(layers, n, stale=True)
xs = [inputs.layer_x(l, i, n).cuda() for i, l in enumerate(layers)]
gys = [inputs.layer_gy(l, i, n).cuda() for i, l in enumerate(layers)]
st.set_dw([inputs.layer_dw(l, i).cuda() for i, l in enumerate(layers)])
for _ in range(2):
    st.run_refresh(xs, gys, 2.5e-2)
w = [torch.randn(shapes.dims(l)[0] * shapes.dims(l)[1], device="cuda") for l in layers]
wp = [x + 0.01 for x in w]
st.update(w, wp, 8.18e-3, 0.997)
torch.cuda.synchronize()
print("diff p50", float(st.diff.median()), "status ok", int(st.dev_status.abs().sum()) == 0)
