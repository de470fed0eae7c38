"""TMA streaming-rate probe: achievable GB/s vs stages / tensors per stage / L2 prefetch (disjoint data)."""
import ctypes, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2507_01004_b200 import _native
rows = 16 * 16384 * 8   # 2M rows x 256 B = 512 MiB
x = torch.randn(rows, 128, device="cuda").to(torch.bfloat16)
ctas = 148
for tensors in (1, 2, 3, 4, 5):
    for ns in (2, 3, 4, 6):
        for pf in (0,):
            if 1024 + ns * tensors * 16384 + 256 > 227 * 1024:
                continue
            tpc = rows // tensors // 64 // ctas
            args = (ctypes.c_void_p(x.data_ptr()), rows, tpc, ns, tensors, pf, ctas, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
            _native.call("zgla_selftest_stream", *args)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            for _ in range(5):
                _native.call("zgla_selftest_stream", *args)
            e1.record(); torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 5
            gb = ctas * tpc * tensors * 16384 / 1e9
            print(f"tensors/stage={tensors} ({tensors*16}KB) stages={ns} prefetch={pf}: {gb/ms*1e3:7.1f} GB/s  ({ms*1e3:.1f} us)")
