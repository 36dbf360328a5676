"""Timeline of the persistent inverse for ONE matrix (library built with KFAC_NVCC_EXTRA=-DINV_TRACE):
trace_one.py <n> <out.txt>"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1811_12019_b200 as K
from synth import shapes
n = int(sys.argv[1])
layers = [shapes.linear("fc", n, 64, bias=0)]
st = K.KfacStep(layers, 1)
_, pa, pg = st.recv_views(0)
gen = torch.Generator(device="cuda").manual_seed(0)
X = torch.relu(torch.randn(n // 2, n, generator=gen, device="cuda"))
A = X.T @ X / X.shape[0]
iu = torch.triu_indices(n, n, device="cuda")
pa.copy_(A[iu[0], iu[1]])
pg.copy_(torch.eye(64, device="cuda")[torch.triu_indices(64, 64, device="cuda").unbind()])
for _ in range(3):
    st.inverse(2.5e-2)
torch.cuda.synchronize()
lib = K.kfac._lib
buf = np.zeros((1 << 17) * 16, dtype=np.int32)
lib.kfac_debug_inverse_trace(buf.ctypes.data_as(ctypes.c_void_p), 1 << 17)
rec = buf.view(np.uint8).reshape(-1, 64)
ints = rec[:, :24].copy().view(np.int32).reshape(-1, 6)
ts = rec[:, 24:].copy().view(np.int64).reshape(-1, 5)
with open(sys.argv[2], "w") as f:
    for i in range(len(ints)):
        if ts[i, 2]:
            f.write(" ".join(map(str, list(ints[i]) + list(ts[i]))) + "\n")
print("records", int((ts[:, 2] != 0).sum()))
