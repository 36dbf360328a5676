"""Timeline of the persistent inverse inside one full RN50 step (library built with
KFAC_NVCC_EXTRA=-DINV_TRACE): trace_step.py <out.txt>"""
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
for _ in range(3):
    st.run(xs, gys, 2.5e-2)
torch.cuda.synchronize()
lib = K.kfac._lib
buf = np.zeros((1 << 17) * 24, dtype=np.int32)  # TraceRec: 6 ints + 9 int64 = 96 B
lib.kfac_debug_inverse_trace(buf.ctypes.data_as(ctypes.c_void_p), 1 << 17)
rec = buf.view(np.uint8).reshape(-1, 96)
ints = rec[:, :24].copy().view(np.int32).reshape(-1, 6)
ts = rec[:, 24:].copy().view(np.int64).reshape(-1, 9)
with open(sys.argv[1], "w") as f:
    for i in range(len(ints)):
        if ts[i, 2]:
            f.write(" ".join(map(str, list(ints[i]) + list(ts[i]))) + "\n")
print("records", int((ts[:, 2] != 0).sum()))
if hasattr(lib, "kfac_debug_ozprof"):
    prof = np.zeros(8, dtype=np.uint64)
    lib.kfac_debug_ozprof(prof.ctypes.data_as(ctypes.c_void_p))
    nt = max(int(prof[6]), 1)
    names = ["ring wait", "TMEM-empty wait", "A wait", "TMEM-full wait (warp 1)", "drain (warp 1)", "MMA issue"]
    print("int8 update tasks:", nt, " per task (us @1.9GHz, summed over the 3 runs' last pass counts): " +
          ", ".join(f"{n} {prof[i] / nt / 1900:.2f}" for i, n in enumerate(names)))

if hasattr(lib, "kfac_debug_ozt"):
    t = np.zeros((148, 80), dtype=np.int64)
    lib.kfac_debug_ozt(t.ctypes.data_as(ctypes.c_void_p))
    for c in range(3):
        r = t[c]
        if r[0] == 0:
            continue
        b = r[0]
        print(f"CTA {c} merged task timeline (cycles from issue 0): issue start " + " ".join(str(x - b) for x in r[0:8]))
        print("   issue end " + " ".join(str(x - b) for x in r[8:16]))
        print("   w1 TF done " + " ".join(str(x - b) for x in r[16:24]))
        print("   w1 drain done " + " ".join(str(x - b) for x in r[24:32]))
        print("   w0 drain done " + " ".join(str(x - b) for x in r[32:40]))
        print("   loop top (before TE wait) " + " ".join(str(x - b) for x in r[40:48]))
        print("   TE done " + " ".join(str(x - b) for x in r[48:56]))
        print("   RF done " + " ".join(str(x - b) for x in r[56:64]))
        print("   ring load issued " + " ".join(str(x - b) for x in r[64:72]))
