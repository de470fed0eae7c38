"""Per-group timeline of the host-buffer pipeline (ZGLA_HOST_TRACE=1)."""
import os, sys, math, time
os.environ["ZGLA_HOST_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2507_01004_b200 import distributed as zd
H, L, D = 16, 16384, 128
G = int(sys.argv[1]) if len(sys.argv) > 1 else 8
mk = lambda dt: torch.rand((H, L, D)).to(dt).pin_memory()
host_in = [mk(torch.bfloat16), mk(torch.bfloat16), mk(torch.bfloat16), (torch.rand((H, L, D)) * -0.1 - 0.001).pin_memory(), mk(torch.bfloat16)]
host_out = [torch.empty((H, L, D), dtype=dt).pin_memory() for dt in [torch.bfloat16] * 4 + [torch.float32]]
layer = zd.ZecoRank(H, L, D, 64, torch.bfloat16)
for it in range(2):
    t = time.perf_counter()
    layer.forward_backward_host(host_in, host_out, head_groups=G)
    torch.cuda.synchronize()
    print(f"G={G} call {it}: {1e3 * (time.perf_counter() - t):.2f} ms wall (incl. trace sync)", flush=True)
