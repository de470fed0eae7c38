"""bench.py contract on the GPU: the N=1 JSON line, and the N>1 path under torchrun (2 processes sharing
this GPU with --same-device, so timings are meaningless but every key of the scaling line is produced:
All-Scan in the step, the isolated All-Scan vs NCCL chain vs all-gather-of-states comparison)."""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def last_json(out):
    lines = [ln for ln in out.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out[-3000:]
    return json.loads(lines[0])


def common_keys(d, n):
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
                "dtype", "config", "roofline", "e2e", "gpu_launches", "clocks"):
        assert key in d, key
    assert d["n_gpus"] == n and d["value"] > 0 and d["gpu_launches"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert 0 < d["roofline"]["frac"] < 1.5


def test_bench_single_gpu_line():
    r = subprocess.run([sys.executable, "bench.py", "--steps", "3", "--warmup", "3", "--e2e-steps", "1",
                        "--no-cpu-baseline"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    d = last_json(r.stdout)
    common_keys(d, 1)
    assert not any(k.endswith("_allscan") for k in d["phase_ms"])  # nothing to report at N=1


def test_bench_torchrun_two_ranks_same_device():
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2", "--master-addr",
           "127.0.0.1", "--master-port", "29677", "bench.py", "--gpus", "2", "--steps", "3", "--warmup", "3",
           "--e2e-steps", "1", "--same-device", "--seq", "2048"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    d = last_json(r.stdout)
    common_keys(d, 2)
    assert d["config"]["global_tokens"] == 2 * 2048
    assert "fwd_allscan" in d["phase_ms"] and "bwd_allscan" in d["phase_ms"]
    a = d["allscan"]
    for key in ("p2p_us", "p2p_bwd_us", "nccl_chain_us", "allgather_states_us", "allgather_over_allscan",
                "tau_min_us", "nvlink_frac", "state_bytes"):
        assert key in a and a[key] > 0, key
    assert a["state_bytes"] == 16 * 128 * 128 * 4
