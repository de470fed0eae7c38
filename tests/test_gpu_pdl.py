"""Programmatic dependent launch (on by default) must not change results: the same config-2 step
run with ZGLA_PDL=1 and ZGLA_PDL=0 (read once per process, hence two subprocesses) is bit-identical,
eagerly and replayed from a CUDA graph."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import hashlib, math, sys, torch
sys.path.insert(0, sys.argv[1])
from paper_2507_01004_b200 import ops
torch.manual_seed(0)
h, L, D = 16, 16384, 128
q, k, v, do = ((torch.rand(h, L, D, device="cuda") * 2 - 1).to(torch.bfloat16) for _ in range(4))
g = torch.rand(h, L, D, device="cuda") * (math.log(0.999) - math.log(0.9)) + math.log(0.9)
sh = ops.ZecoShard(h, L, D, D, 64, torch.bfloat16)
o = torch.empty_like(q)
grads = (torch.empty_like(q), torch.empty_like(k), torch.empty_like(v), torch.empty_like(g))
def step():
    sh.fwd_local(k, v, g)
    sh.fwd_output(q, k, v, g, None, out=o)
    sh.bwd_local(q, g, do)
    sh.bwd_output(q, k, v, g, do, None, None, grads=grads)
def digest():
    torch.cuda.synchronize()
    hsh = hashlib.sha256()
    for t in (o,) + grads:
        hsh.update(t.contiguous().view(torch.uint8).cpu().numpy().tobytes())
    return hsh.hexdigest()
step(); eager = digest()
for t in (o,) + grads: t.zero_()
s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    step()
torch.cuda.current_stream().wait_stream(s)
graph = torch.cuda.CUDAGraph()
with torch.cuda.graph(graph):
    step()
for t in (o,) + grads: t.zero_()
graph.replay(); graph.replay()
print(eager, digest())
"""


def run(pdl, early="0"):
    env = dict(os.environ, ZGLA_PDL=pdl, ZGLA_EARLY_INPUTS=early)
    out = subprocess.run([sys.executable, "-c", SCRIPT, ROOT], env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    return out.stdout.split()[-2:]


def test_pdl_launch_is_bit_identical():
    on, off = run("1"), run("0")
    assert on[0] == on[1], "graph replay differs from the eager step (PDL on)"
    assert off[0] == off[1], "graph replay differs from the eager step (PDL off)"
    assert on == off


def test_early_inputs_bit_identical():
    """Early inputs (the output kernels stream q/k/v/g/dO before waiting for the preceding grid) change only
    the launch overlap, never the results."""
    early, plain = run("1", "1"), run("1", "0")
    assert early[0] == early[1], "graph replay differs from the eager step (early inputs)"
    assert early == plain
