"""Host logic of the persistent dataflow inverse (stage a6): the task-list generator
the device runs (csrc/inverse_tasks.hpp) is compiled for the host by
scripts/check_inverse_tasks.cpp, which checks coverage (every panel once, every tile once per
sweep step, merged two-step tasks only away from the pivot rows) and that every wait the kernel
performs points to an earlier task of the list (deadlock freedom of the in-order persistent
schedule)."""
import os
import subprocess

import pytest

from synth import shapes

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def checker(tmp_path_factory):
    exe = str(tmp_path_factory.mktemp("cit") / "check_inverse_tasks")
    subprocess.check_call(["g++", "-O2", "-std=c++17", "-I", os.path.join(ROOT, "paper_1811_12019_b200", "csrc"),
                           "-I", "/usr/local/cuda/include", os.path.join(ROOT, "scripts", "check_inverse_tasks.cpp"),
                           "-o", exe])
    return exe


def test_exhaustive_small_mixes(checker):
    out = subprocess.run([checker], capture_output=True, text=True)
    assert out.returncode == 0, out.stderr[-2000:]
    assert out.stdout.startswith("OK")


@pytest.mark.parametrize("cfg", ["single_conv", "resnet18_cifar", "resnet50", "stress"])
def test_config_mix(checker, cfg):
    L, _ = shapes.config(cfg)
    nts = []
    for layer in L:
        for d in shapes.dims(layer):
            nts.append((d + 127) // 128)
    out = subprocess.run([checker, *map(str, nts)], capture_output=True, text=True)
    assert out.returncode == 0, out.stderr[-2000:]
