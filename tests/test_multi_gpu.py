"""Multi-GPU parity (NCCL ReduceScatter/AllGather over NVLink) via torchrun; needs >= 2 GPUs."""
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ngpu():
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


# (config, policy, ranks, rs_mode, wire): wire 1 = the fp16 factor wire (NEXT-4(ii), R-23)
@pytest.mark.parametrize("cfg,policy,nproc,rs_mode,wire", [
    ("small", 0, 2, 0, 0), ("small", 1, 2, 0, 0), ("one_layer", 0, 2, 0, 0), ("small", 1, 4, 0, 0),
    ("resnet50", 1, 2, 0, 0), ("resnet50", 1, 4, 0, 0), ("stress", 1, 2, 0, 0), ("stress", 1, 4, 0, 0),
    ("small", 1, 2, 1, 0), ("small", 1, 4, 1, 0), ("resnet50", 1, 4, 1, 0),
    ("small", 1, 2, 1, 1), ("small", 1, 4, 0, 1), ("one_layer", 0, 2, 1, 1), ("resnet50", 1, 4, 1, 1)])
@pytest.mark.timeout(3600)
def test_mp_parity(cfg, policy, nproc, rs_mode, wire):
    if _ngpu() < nproc:
        pytest.skip(f"needs {nproc} GPUs, have {_ngpu()}")
    from conftest import build_lib
    build_lib()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr=127.0.0.1", "--master-port=29631", os.path.join(ROOT, "tests", "mp_parity.py"), cfg,
           str(policy), str(rs_mode), str(wire)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=3000, cwd=ROOT)
    print(r.stdout[-2000:], r.stderr[-2000:])
    assert r.returncode == 0
    assert "mp_parity" in r.stdout
