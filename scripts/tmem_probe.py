import ctypes, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2507_01004_b200 import _native
out = torch.zeros(1, dtype=torch.int64, device="cuda"); sink = torch.zeros(1, device="cuda")
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
for mode, name in ((0, "ld x32 + wait"), (1, "2 x ld x32, 1 wait"), (2, "st x32 + wait")):
    for nw in (1, 2, 4, 8, 16):
        iters = 256
        _native.call("zgla_selftest_tmem", nw, iters, mode, ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(sink.data_ptr()), st)
        torch.cuda.synchronize()
        cyc = int(out.item())
        byts = nw * iters * 32 * 32 * 4
        print(f"{name:20s} warps={nw:2d}: {cyc/iters:7.1f} cyc/iter/warp, {byts/cyc:7.1f} B/cycle/SM")
