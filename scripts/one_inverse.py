"""Run the damped inverse of one synthetic layer (for ncu)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1811_12019_b200 as K
from synth import shapes
n = int(sys.argv[1]) if len(sys.argv) > 1 else 2304
g = int(sys.argv[2]) if len(sys.argv) > 2 else 512
layers = [shapes.linear("fc", n, g, bias=0)]
st = K.KfacStep(layers, 1)
_, pa, pg = st.recv_views(0)
rng = np.random.default_rng(0)
X = np.maximum(rng.standard_normal((n // 2, n)), 0).astype(np.float32)
A = X.T @ X / X.shape[0]
iu = np.triu_indices(n)
pa.copy_(torch.as_tensor(A[iu]))
G = np.eye(g, dtype=np.float32)
pg.copy_(torch.as_tensor(G[np.triu_indices(g)]))
for _ in range(2):
    st.inverse(2.5e-2)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record(); st.inverse(2.5e-2); e1.record(); torch.cuda.synchronize()
print("inverse n=%d: %.3f ms, %.2f TF/s fp64" % (n, e0.elapsed_time(e1), (n**3 + g**3) / (e0.elapsed_time(e1) / 1e3) / 1e12))
