"""Per-CTA timeline of one list-form All-Scan call (diagnostics): start / first batch polled /
first batch stored / exit, per virtual rank, in us since the first CTA started."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2507_01004_b200 import _native, ops
P, h, d = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (8, 4, 64)))
lib = _native.load()
local = torch.rand(P, h, d, d, device="cuda"); logs = -torch.rand(P, h, d, device="cuda")
recv, sc = torch.empty_like(local), torch.empty_like(local)
buf = torch.zeros(4 * 8192, dtype=torch.int64, device="cuda")
a = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16)
import time
t_end = time.time() + 0.5
while time.time() < t_end:  # warm the clocks up (an idle B200 sits at 120 MHz)
    a @ a
torch.cuda.synchronize()
for it in range(4):
    if it == 3:
        _native.call("zgla_set_trace", ctypes.c_void_p(buf.data_ptr()), 0)
    _native.check(lib.zgla_allscan_local(P, h, d, d, _native.ZGLA_F32, 1, 0, ops._p(local), ops._p(logs), ops._p(recv),
                                         ops._p(sc), ops._stream()), "x")
    if it < 3:
        torch.cuda.synchronize()
    else:
        for _ in range(50):
            a @ a  # keep the SMs busy (and the clocks up) right behind the traced call
        torch.cuda.synchronize()
_native.call("zgla_set_trace", None, 0)
t = buf.view(-1, 4).cpu()
n = int((t[:, 0] > 0).sum()); per = n // P
t = t[:n]; t0 = int(t[:, 0].min())
for r in range(P):
    rows = t[r * per:(r + 1) * per]
    f = lambda c: [(int(x) - t0) / 1000 for x in rows[:, c] if int(x) > 0]
    st, po, sd, ex = f(0), f(1), f(2), f(3)
    print(f"rank {r}: ctas {per} start {min(st):.2f}-{max(st):.2f} polled {min(po) if po else float('nan'):.2f}-{max(po) if po else float('nan'):.2f} stored {min(sd):.2f}-{max(sd):.2f} exit {min(ex):.2f}-{max(ex):.2f}")
