"""tcgen05 SS MMA issue rate by shape (zgla_selftest_mma_rate): SM cycles per M x N x 16 bf16 MMA."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2507_01004_b200 import _native

ctas = 148
out = torch.zeros(ctas, dtype=torch.int64, device="cuda")
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
for M, N in ((128, 64), (128, 128), (128, 256), (64, 64), (64, 128), (64, 256)):
    for a_mn, b_mn in ((0, 0), (1, 1), (2, 0), (2, 1)):  # a_mn 2: A from TMEM
        for c in (1, ctas):
            _native.call("zgla_selftest_mma_rate", M, N, a_mn, b_mn, 512, c, ctypes.c_void_p(out.data_ptr()), st)
            torch.cuda.synchronize()
            cyc = out[:c].double().mean().item() / 1000
            macs = M * N * 16
            print(f"M={M:3d} N={N:3d} a_mn={a_mn} b_mn={b_mn} ctas={c:3d}: {cyc:6.1f} cycles/MMA, {macs / cyc:7.0f} MAC/cycle/SM")
