"""Save (or compare) the outputs of one fixed cfg2 fwd+bwd step, to check that a kernel variant is
bit-identical to the in-tree build:  ZGLA_LIB=var/X/libzeco_gla.so python scripts/ab_bitwise.py save X;
python scripts/ab_bitwise.py cmp base X"""
import math, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_01004_b200 import ops  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out")
if sys.argv[1] == "save":
    torch.manual_seed(0)
    h, L, D = 16, 16384, 128
    q, k, v, do = ((torch.rand(h, L, D, device="cuda") * 2 - 1).to(torch.bfloat16) for _ in range(4))
    g = torch.rand(h, L, D, device="cuda") * (math.log(0.999) - math.log(0.9)) + math.log(0.9)
    sh = ops.ZecoShard(h, L, D, D, 64, torch.bfloat16)
    sh.fwd_local(k, v, g)
    o = sh.fwd_output(q, k, v, g).clone()
    sh.bwd_local(q, g, do)
    grads = [x.clone() for x in sh.bwd_output(q, k, v, g, do, None, None)]
    torch.save({"o": o.cpu(), "dq": grads[0].cpu(), "dk": grads[1].cpu(), "dv": grads[2].cpu(), "dg": grads[3].cpu()},
               os.path.join(OUT, f"ab_{sys.argv[2]}.pt"))
else:
    a = torch.load(os.path.join(OUT, f"ab_{sys.argv[2]}.pt"))
    b = torch.load(os.path.join(OUT, f"ab_{sys.argv[3]}.pt"))
    for key in a:
        same = torch.equal(a[key], b[key])
        d = (a[key].float() - b[key].float()).abs().max().item()
        print(key, "bitwise" if same else f"DIFF max {d:.3e}")
