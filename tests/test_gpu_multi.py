"""Multi-GPU parity of the NCCL expert-parallel / DTD path (needs >= 2 GPUs).

Each case launches tests/mp_layer_check.py under torchrun on the visible GPUs.
"""
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CASES = [  # (world, G_t, G_ep, extra args)
    (2, 1, 2, ["--variants"]),         # + top-2 / random priority / aux loss (NEXT #4)
    (2, 2, 1, ["--variants"]),
    (2, 1, 1, []),                     # pure data parallel: no collectives
    (4, 2, 2, []),
    (4, 1, 4, ["--experts", "16"]),
    (4, 4, 1, []),
    (4, 2, 2, ["--cf", "0.5", "--variants"]),  # drops under DTD
    (8, 2, 4, ["--experts", "16"]),
    (8, 1, 8, ["--experts", "32"]),
    (8, 4, 2, []),
]


@pytest.mark.parametrize("world,gt,gep,extra", CASES)
def test_multi_gpu_parity(world, gt, gep, extra):
    n = torch.cuda.device_count()
    if n < world:
        pytest.skip(f"needs {world} GPUs, have {n}")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(29500 + world * 10 + gt),
           os.path.join(ROOT, "tests", "mp_layer_check.py"), "--gt", str(gt), "--gep", str(gep), *extra]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    print(r.stdout[-4000:], r.stderr[-4000:])
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]


def test_multi_gpu_absent_peer_times_out():
    """Device-side deadline of the window barrier (one process per GPU): a peer that never
    calls moe_forward yields MOE_ERR_TIMEOUT on the other rank, not a hang."""
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", "29611", os.path.join(ROOT, "tests", "mp_timeout_check.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=ROOT)
    print(r.stdout[-3000:], r.stderr[-3000:])
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
