"""The grouped factor launch on a subset of RN50 layers (for ncu): factor_subset.py <subset> [reps]
  tensor   -- the tensor-bound set: 3x3 / 7x7 convs (A is the big contraction)
  all      -- every layer (the bench launch)
Prints the CUDA-event time and the achieved TFLOP/s over rows*d*(d+1) of A and G."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1811_12019_b200 as K
from synth import shapes, inputs
subset = sys.argv[1] if len(sys.argv) > 1 else "tensor"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
layers, n = shapes.config("resnet50")
if subset == "tensor":
    layers = [l for l in layers if l["kh"] > 1]
st = K.KfacStep(layers, n, device=torch.device("cuda"))
xs = [inputs.layer_x(l, i, n).cuda() for i, l in enumerate(layers)]
gys = [inputs.layer_gy(l, i, n).cuda() for i, l in enumerate(layers)]
flops = sum(shapes.rows(l, n) * d * (d + 1) for l in layers for d in shapes.dims(l))
for _ in range(2):
    st.factors(xs, gys)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
for _ in range(reps):
    st.factors(xs, gys)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
print(f"factors[{subset}] {len(layers)} layers: {ms:.3f} ms, {flops / ms / 1e9:.1f} TFLOP/s ({flops / 1e9:.1f} GFLOP)")
