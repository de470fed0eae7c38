"""The multi-GPU code path (AllScanP2P: CUDA-IPC handle exchange, peer stores, flags, acks, epochs)
run by 2 processes sharing this GPU (gloo bootstrap); bitwise equal to the single-process list form."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("P,graph", [(2, False), (3, False), (2, True)])
def test_ipc_allscan_two_processes_one_gpu(P, graph):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={P}",
           "--master-addr", "127.0.0.1", "--master-port", str(29611 + P + 10 * graph),
           os.path.join(ROOT, "scripts", "spmd_ipc_check.py"), "--same-device", "--rounds", "2"] + (["--graph"] if graph else [])
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=400, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    assert "SPMD IPC check OK" in r.stdout


@pytest.mark.parametrize("P", [2, 4])
def test_ipc_cfg3_shape_against_oracle(P):
    """BASELINE config 3 per-rank shape (16,384 tokens/rank, d=128; 2 heads, long-memory gates) through
    ZecoRank / AllScanP2P in P processes, every output and gradient checked against the f64 oracle."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={P}",
           "--master-addr", "127.0.0.1", "--master-port", str(29641 + P),
           os.path.join(ROOT, "scripts", "spmd_ipc_check.py"), "--same-device", "--rounds", "1",
           "--seq", "16384", "--heads", "2", "--oracle"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    assert "SPMD IPC check OK" in r.stdout and r.stdout.count("oracle ") == 5


def test_ipc_overlap_schedule_against_oracle():
    """ZecoRank's head-group overlap schedule (each group's All-Scan on a communication stream under the
    other groups' kernels) over the real CUDA-IPC chain in 3 processes, checked against the f64 oracle."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=3",
           "--master-addr", "127.0.0.1", "--master-port", "29655",
           os.path.join(ROOT, "scripts", "spmd_ipc_check.py"), "--same-device", "--rounds", "2",
           "--seq", "1024", "--heads", "4", "--overlap-groups", "2", "--oracle"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    assert "SPMD IPC check OK" in r.stdout and r.stdout.count("oracle ") == 5


@pytest.mark.parametrize("P,D", [(2, 128), (3, 64)])
def test_ipc_layer_function_against_torch_reference(P, D):
    """The autograd layer function (the GLAModel path) sequence-parallel over P processes with AllScanP2P,
    token-major head-slice inputs, outputs and gradients against the float64 torch GLA on the whole sequence."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={P}",
           "--master-addr", "127.0.0.1", "--master-port", str(29671 + P),
           os.path.join(ROOT, "scripts", "spmd_layer_check.py"), "--same-device", "--seq", "512", "--dim", str(D)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    assert "SPMD layer check OK" in r.stdout, r.stdout[-2000:]


def test_ipc_eight_processes_against_oracle():
    """The north star's P = 8: eight processes over the real CUDA-IPC All-Scan chain (sharing one GPU), bitwise
    equal to the single-process list form and within the bf16 bound of the f64 oracle."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=8",
           "--master-addr", "127.0.0.1", "--master-port", "29701",
           os.path.join(ROOT, "scripts", "spmd_ipc_check.py"), "--same-device", "--rounds", "2",
           "--seq", "256", "--heads", "2", "--oracle"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    assert "SPMD IPC check OK (P=8" in r.stdout and r.stdout.count("oracle ") == 5
