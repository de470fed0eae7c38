import sys, math, torch
sys.path.insert(0, ".")
from paper_2507_01004_b200 import distributed as zd
H, L, D = 16, 16384, 128
q, k, v = (torch.rand(H, L, D, device="cuda").to(torch.bfloat16) for _ in range(3))
g = torch.rand(H, L, D, device="cuda") * (math.log(0.999) - math.log(0.9)) + math.log(0.9)
r = zd.ZecoRank(H, L, D, 64, torch.bfloat16)
o = torch.empty_like(q)
for save in (True, False, True, False):
    for _ in range(3): r.forward(q, k, v, g, out=o, save_states=save)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20): r.forward(q, k, v, g, out=o, save_states=save)
    b.record(); torch.cuda.synchronize()
    print("save_states", save, "forward ms", round(a.elapsed_time(b) / 20, 4))
