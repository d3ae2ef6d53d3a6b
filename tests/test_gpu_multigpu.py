"""Multi-GPU (NCCL, one process per GPU) coverage of the frame-sharded CUDA path (DESIGN.md §7,
SURVEY §8(e)): two ranks under torchrun demodulate their local stacks with libbosrm.so, rank 0
gathers the maps and compares them bit for bit with one GPU demodulating the whole global
stack — for both reference modes (recomputed on every rank / NCCL broadcast from rank 0).
Skips when fewer than 2 GPUs are visible (the round-end GPU box has one; the CPU gloo tests in
test_sharding.py cover the host logic at world size 2)."""

import json
import os
import socket
import subprocess
import sys

import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(world, mode):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(world),
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(ROOT, "tools", "nccl_shard_check.py"), "--mode", mode]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout
    d = json.loads(lines[0])
    assert d["world"] == world and d["bitwise_equal"] is True, d


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["recompute", "broadcast"])
def test_two_rank_nccl_sharded_stack_bitwise(mode):
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    _run(2, mode)


@pytest.mark.gpu
def test_one_rank_nccl_check_script():
    """The same script at world size 1 (NCCL process group on one GPU): runs wherever a GPU is."""
    _run(1, "broadcast")
