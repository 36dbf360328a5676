"""Cycles per phase of the 128^2 pivot inversions of one RN50 step (library built with
KFAC_NVCC_EXTRA=-DPIVOT_DBG): pivot_phases.py"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1811_12019_b200 as K
from synth import shapes, inputs
layers, n = shapes.config("resnet50")
st = K.KfacStep(layers, n, device=torch.device("cuda"), policy=1)
xs = [inputs.layer_x(l, i, n).cuda() for i, l in enumerate(layers)]
gys = [inputs.layer_gy(l, i, n).cuda() for i, l in enumerate(layers)]
st.set_dw([inputs.layer_dw(l, i).cuda() for i, l in enumerate(layers)])
st.run(xs, gys, 2.5e-2)
torch.cuda.synchronize()
acc = np.zeros(32, dtype=np.uint64)
K.kfac._lib.kfac_debug_pclk(acc.ctypes.data_as(ctypes.c_void_p))

counts = sum(((a + 127) // 128) for l in layers for a in shapes.dims(l))  # pivots = column blocks per matrix
names = {0: "load S", 20: "loop exit", 21: "final writes"}
for sb in range(4):
    names.update({1 + 4 * sb: f"sb{sb} sweep32", 2 + 4 * sb: f"sb{sb} copy O", 3 + 4 * sb: f"sb{sb} W=QO (DMMA)",
                  4 + 4 * sb: f"sb{sb} S-=O^TW + bands"})
tot = acc.sum()
print(f"pivots {counts}, total {tot / counts / 1965:.1f} us per pivot (1965 MHz)")
for k in sorted(names):
    if acc[k]:
        print(f"  {names[k]:24s} {acc[k] / counts / 1965:6.2f} us")
