"""Layer shape tables for the benchmark workloads (BASELINE.json `configs`).

Workload description only: this module holds no K-FAC arithmetic. It is shared
by the oracle, the tests and bench.py (the "seeded input generators" module of
its own).

A layer is a plain dict with the fields of the C-ABI descriptor
(include/kfac.h `kfac_layer_desc`):

  kind      0 = conv2d, 1 = linear (fully connected)
  c_in, c_out, kh, kw, stride_h, stride_w, pad_h, pad_w, h_in, w_in, has_bias

Shapes follow the paper's workload: ResNet-50 on ImageNet at 32 images per GPU
(§5.1), 53 conv + 1 FC factorised layers, and
the Fig. 4 memory totals 587/1017 MiB pin this table
(tests/test_shapes_pin.py).  ResNet-50 is v1 (stride on the first 1x1 of a
down-sampling block, Chainer's example; SURVEY R-17).
"""

from __future__ import annotations


def conv(name, c_in, c_out, k, s, p, h_in, bias=0):
    return dict(name=name, kind=0, c_in=c_in, c_out=c_out, kh=k, kw=k,
                stride_h=s, stride_w=s, pad_h=p, pad_w=p, h_in=h_in, w_in=h_in,
                has_bias=bias)


def linear(name, c_in, c_out, bias=1):
    return dict(name=name, kind=1, c_in=c_in, c_out=c_out, kh=1, kw=1,
                stride_h=1, stride_w=1, pad_h=0, pad_w=0, h_in=1, w_in=1,
                has_bias=bias)


def out_hw(layer):
    """Output spatial size of a layer (standard zero-padded convolution)."""
    if layer["kind"] == 1:
        return 1, 1
    ho = (layer["h_in"] + 2 * layer["pad_h"] - layer["kh"]) // layer["stride_h"] + 1
    wo = (layer["w_in"] + 2 * layer["pad_w"] - layer["kw"]) // layer["stride_w"] + 1
    return ho, wo


def dims(layer):
    """(dA, dG): A is over im2col patches (+1 bias coordinate), G over C_out."""
    d_a = layer["c_in"] * layer["kh"] * layer["kw"] + (1 if layer["has_bias"] else 0)
    return d_a, layer["c_out"]


def rows(layer, n):
    ho, wo = out_hw(layer)
    return n * ho * wo


def resnet50(v15: bool = False):
    """ResNet-50 (ImageNet 224x224), the 54 K-FAC layers in forward order."""
    L = [conv("conv1", 3, 64, 7, 2, 3, 224)]
    c_in, h = 64, 56  # after 3x3/2 max-pool
    for stage, (width, blocks) in enumerate([(64, 3), (128, 4), (256, 6), (512, 3)]):
        out = width * 4
        for b in range(blocks):
            s = 2 if (b == 0 and stage > 0) else 1
            pre = f"l{stage + 1}b{b}"
            s1, s2 = (1, s) if v15 else (s, 1)
            L.append(conv(pre + "c1", c_in, width, 1, s1, 0, h))
            h2 = (h - 1) // s1 + 1
            L.append(conv(pre + "c2", width, width, 3, s2, 1, h2))
            h3 = (h2 + 2 - 3) // s2 + 1
            L.append(conv(pre + "c3", width, out, 1, 1, 0, h3))
            if b == 0:
                L.append(conv(pre + "ds", c_in, out, 1, s, 0, h))
            c_in, h = out, h3
    L.append(linear("fc", 2048, 1000))
    return L


def resnet18_cifar():
    """ResNet-18 with the CIFAR stem (3x3/1, no max-pool), 32x32 input, 21 layers."""
    L = [conv("conv1", 3, 64, 3, 1, 1, 32)]
    c_in, h = 64, 32
    for stage, width in enumerate([64, 128, 256, 512]):
        for b in range(2):
            s = 2 if (b == 0 and stage > 0) else 1
            pre = f"l{stage + 1}b{b}"
            L.append(conv(pre + "c1", c_in, width, 3, s, 1, h))
            h2 = (h + 2 - 3) // s + 1
            L.append(conv(pre + "c2", width, width, 3, 1, 1, h2))
            if b == 0 and (s != 1 or c_in != width):
                L.append(conv(pre + "ds", c_in, width, 1, s, 0, h))
            c_in, h = width, h2
    L.append(linear("fc", 512, 10))
    return L


def single_conv():
    """BASELINE config 1: one 3x3 conv, C_in=16, C_out=32, 8x8, with bias (A 145x145)."""
    return [conv("conv", 16, 32, 3, 1, 1, 8, bias=1)]


def stress():
    """BASELINE config 5: 3 x {A 4608, G 512} (3x3 conv 512->512 at 7x7) + FC {A 2049, G 1000}."""
    return [conv(f"l4c2_{i}", 512, 512, 3, 1, 1, 7) for i in range(3)] + [linear("fc", 2048, 1000)]


# name -> (layer list, per-GPU batch, description)
CONFIGS = {
    "single_conv": (single_conv, 32, "single 3x3 conv C_in=16 C_out=32, 8x8, batch 32"),
    "resnet18_cifar": (resnet18_cifar, 128, "ResNet-18 CIFAR-10 shapes, batch 128"),
    "resnet50": (resnet50, 32, "ResNet-50 ImageNet shapes, batch 32/GPU"),
    "stress": (stress, 256, "ResNet-50 stress: 3x{A4608,G512} + FC{A2049,G1000}, batch 256/GPU"),
}


def config(name):
    fn, batch, desc = CONFIGS[name]
    return fn(), batch
