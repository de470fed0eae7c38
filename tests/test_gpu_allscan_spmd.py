"""The SPMD All-Scan kernel (the one each GPU runs in the multi-GPU path) exercised on one GPU:
P communicator objects are bound to each other's device buffers in-process
(zgla_allscan_bind_local) and every rank's kernel is launched on its own stream, so the
flag / ack / epoch protocol runs exactly as it does over NVLink peer memory, including
back-to-back FWD and BWD calls that reuse the inboxes."""

import ctypes

import numpy as np
import pytest
import torch

from oracle import gla_oracle as orc

pytestmark = pytest.mark.gpu


def make_comms(P, h, dk, dv, max_blocks=8):
    from paper_2507_01004_b200 import _native
    lib = _native.load()
    comms = []
    for r in range(P):
        hdl = ctypes.c_void_p()
        _native.check(lib.zgla_allscan_create(r, P, h, dk, dv, max_blocks, ctypes.byref(hdl)), "create")
        comms.append(hdl)
    for r in range(P):
        nxt = comms[r + 1] if r + 1 < P else None
        prv = comms[r - 1] if r > 0 else None
        _native.check(lib.zgla_allscan_bind_local(comms[r], nxt, prv), "bind_local")
    return lib, comms


def run_round(lib, comms, local, logs, K, direction, streams):
    from paper_2507_01004_b200 import _native
    P = len(comms)
    recv = torch.empty_like(local)
    scanned = torch.empty_like(local)
    # launch in CHAIN order: streams may share a hardware queue (false serialization), and a
    # producer queued behind its own consumer would deadlock; in chain order it can only delay
    order = list(range(P)) if direction == 0 else list(range(P - 1, -1, -1))
    for r in order:
        with torch.cuda.stream(streams[r]):
            _native.check(lib.zgla_allscan_run(comms[r], K, direction, ctypes.c_void_p(local[r].data_ptr()),
                                               ctypes.c_void_p(logs[r].data_ptr()),
                                               ctypes.c_void_p(recv[r].data_ptr()),
                                               ctypes.c_void_p(scanned[r].data_ptr()),
                                               ctypes.c_void_p(streams[r].cuda_stream)), "run")
    for s in streams:
        s.synchronize()
    return recv, scanned


@pytest.mark.parametrize("P,K", [(2, 1), (4, 4), (8, 16)])
def test_spmd_allscan_protocol(P, K):
    h, dk, dv = 2, 64, 32
    lib, comms = make_comms(P, h, dk, dv, max_blocks=16)
    streams = [torch.cuda.Stream() for _ in range(P)]
    gen = torch.Generator(device="cuda").manual_seed(P * 10 + K)
    try:
        for rnd in range(3):  # epochs advance; inboxes and acks are reused
            local = torch.rand(P, h, dk, dv, device="cuda", generator=gen) * 2 - 1
            logs = -2 * torch.rand(P, h, dk, device="cuda", generator=gen)
            for direction in (0, 1):
                recv, scanned = run_round(lib, comms, local, logs, K, direction, streams)
                order = list(range(P)) if direction == 0 else list(range(P - 1, -1, -1))
                ln, gn = local.double().cpu().numpy(), logs.double().cpu().numpy()
                want_r, want_s = orc.scan_ranks([ln[r] for r in order], [gn[r] for r in order])
                for pos, r in enumerate(order):
                    np.testing.assert_allclose(recv[r].double().cpu().numpy(), want_r[pos], rtol=1e-5, atol=1e-6)
                    np.testing.assert_allclose(scanned[r].double().cpu().numpy(), want_s[pos], rtol=1e-5, atol=1e-6)
        sent = [lib.zgla_allscan_bytes_sent(c) for c in comms]
        state_bytes = h * dk * dv * 4
        # every rank sends once per direction except the chain sink (3 rounds x 2 directions)
        assert sent[0] == 3 * state_bytes and sent[-1] == 3 * state_bytes
        if P > 2:
            assert all(x == 6 * state_bytes for x in sent[1:-1])
    finally:
        for c in comms:
            lib.zgla_allscan_destroy(c)


def test_spmd_matches_list_form_bitwise():
    """Same device code: the SPMD chain and the list-form kernel give identical bits."""
    from paper_2507_01004_b200 import ops
    P, h, dk, dv = 4, 2, 128, 128
    lib, comms = make_comms(P, h, dk, dv)
    streams = [torch.cuda.Stream() for _ in range(P)]
    try:
        gen = torch.Generator(device="cuda").manual_seed(5)
        local = torch.rand(P, h, dk, dv, device="cuda", generator=gen)
        logs = -torch.rand(P, h, dk, device="cuda", generator=gen)
        r1, s1 = run_round(lib, comms, local, logs, 4, 0, streams)
        r2, s2 = ops.allscan_local(local, logs, 4, 0)
        assert torch.equal(r1, r2) and torch.equal(s1, s2)
    finally:
        for c in comms:
            lib.zgla_allscan_destroy(c)


_DEADLOCK_SCRIPT = r"""
import ctypes, sys, time
sys.path.insert(0, sys.argv[1])
import torch
from paper_2507_01004_b200 import _native, errors
from tests.test_gpu_allscan_spmd import make_comms
lib, comms = make_comms(2, 2, 64, 32)
local = torch.rand(2, 2, 64, 32, device="cuda")
logs = -torch.rand(2, 2, 64, device="cuda")
recv, scanned = torch.empty_like(local), torch.empty_like(local)
t0 = time.time()
# only rank 1 runs: its predecessor never stores, so the chain wait must time out (no trap, no hang)
_native.check(lib.zgla_allscan_run(comms[1], 4, 0, ctypes.c_void_p(local[1].data_ptr()),
                                   ctypes.c_void_p(logs[1].data_ptr()), ctypes.c_void_p(recv[1].data_ptr()),
                                   ctypes.c_void_p(scanned[1].data_ptr()), None), "run")
try:
    _native.check(lib.zgla_allscan_status(comms[1], 1), "status")
    print("NO-ERROR")
except errors.DeadlockError as e:
    print("DEADLOCK", round(time.time() - t0, 2))
# the CUDA context is still usable after the timed-out kernel
x = torch.ones(4, device="cuda") * 3
print("CTX-OK", float(x.sum()))
try:  # and the communicator refuses further calls
    _native.check(lib.zgla_allscan_run(comms[1], 4, 0, ctypes.c_void_p(local[1].data_ptr()),
                                       ctypes.c_void_p(logs[1].data_ptr()), ctypes.c_void_p(recv[1].data_ptr()),
                                       ctypes.c_void_p(scanned[1].data_ptr()), None), "run")
    print("RERUN-ACCEPTED")
except errors.DeadlockError:
    print("RERUN-REFUSED")
"""


def test_spmd_timeout_raises_deadlock_not_trap(tmp_path):
    """A chain wait that never completes reports ZGLA_ERR_DEADLOCK -> DeadlockError (SURVEY §5:
    bounded-spin timeout -> error code, not a hang) and leaves the CUDA context usable."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = tmp_path / "dl.py"
    script.write_text(_DEADLOCK_SCRIPT)
    env = dict(os.environ, ZGLA_ALLSCAN_TIMEOUT_MS="300", PYTHONPATH=root)
    out = subprocess.run([sys.executable, str(script), root], capture_output=True, text=True, timeout=240, env=env,
                         cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    assert "DEADLOCK" in out.stdout, out.stdout
    assert "CTX-OK 12.0" in out.stdout and "RERUN-REFUSED" in out.stdout, out.stdout
