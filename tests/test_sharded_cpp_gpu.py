"""GPU: catalog sharding from C++ with no PyTorch on the path
(tests/cpp/test_sharded.cpp through the C-ABI's lf_comm): two processes
sharing cuda:0 exchange over the peer-memory communicator (CUDA IPC), and one
process over a size-1 NCCL communicator.  Each rank checks its sharded
lse / pos / loss / dX / dE-rows / skip statistics against the unsharded call
(pos bitwise; fp32 rounding of the partial sums elsewhere)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "build", "test_sharded")


def run(*args):
    assert os.path.exists(BIN), f"{BIN} missing: run __graft_entry__.build()"
    p = subprocess.run([BIN, *args], capture_output=True, text=True, timeout=300,
                       env=dict(os.environ, LSEFORGE_PEER_TIMEOUT_MS="20000"))
    print(p.stdout)
    assert p.returncode == 0, p.stdout + p.stderr
    return p.stdout


def test_peer_communicator_two_processes(cuda):
    out = run("peer", "2")
    assert out.count("[rank 0/2]") == 5 and out.count("[rank 1/2]") == 5
    assert "FAIL" not in out


def test_nccl_communicator_world_one(cuda):
    out = run("nccl1")
    assert out.count("[rank 0/1]") == 5 and "FAIL" not in out
