"""Layer-level d=64 debugging: GLA core gradients vs the float64 torch reference, per tensor and through
the layer (the per-head RMS norm of near-zero rows amplifies bf16 rounding; see tests/test_gpu_layer.py)."""
import sys, torch
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_01004_b200.layer import GatedLinearAttention, gla_reference, zeco_gla
def rel(a, b):
    a, b = a.double(), b.double(); s = max(a.norm().item(), b.norm().item()); return (a - b).norm().item() / s
torch.manual_seed(1)
layer = GatedLinearAttention(hidden_size=256, num_heads=4, device="cuda")
x = (torch.randn(512, 256, device="cuda") * 0.5).to(torch.bfloat16)
with torch.no_grad():
    q, k, v, g, r = layer.project(x)
print("g range", g.min().item(), g.max().item(), "strides q", q.stride(), "g", g.stride())
w = torch.randn(4, 512, 64, device="cuda", dtype=torch.float64)
res = {}
for name, core, mk in (("zeco", zeco_gla, lambda t: t.detach().clone().requires_grad_(True)),
                       ("zeco_strided", zeco_gla, None), ("ref", gla_reference, None)):
    if mk is None:
        leaves = [t.detach().requires_grad_(True) for t in (q, k, v, g)]  # keep strided views
        if name == "ref":
            leaves = [t.detach().double().requires_grad_(True) for t in (q, k, v, g)]
    else:
        leaves = [mk(t).contiguous().detach().requires_grad_(True) for t in (q, k, v, g)]
    o = core(*leaves)
    (o.double() * w).sum().backward()
    res[name] = [o.detach()] + [t.grad for t in leaves]
for a in ("zeco", "zeco_strided"):
    print(a, [round(rel(x, y), 5) for x, y in zip(res[a], res["ref"])])

# sensitivity of the layer's x.grad to core rounding: reference core in float64 vs float32
def ref32(q, k, v, g, *a):
    return gla_reference(q.float(), k.float(), v.float(), g.float()).to(q.dtype)
outs = {}
for name, core in (("zeco", None), ("ref64", gla_reference), ("ref32", ref32)):
    layer.zero_grad()
    xx = x.clone().requires_grad_(True)
    y = layer(xx, core)
    y.float().square().mean().backward()
    outs[name] = (y.detach(), xx.grad.clone())
for a, b in (("zeco", "ref64"), ("ref32", "ref64")):
    print(a, "vs", b, "y", round(rel(outs[a][0], outs[b][0]), 5), "x.grad", round(rel(outs[a][1], outs[b][1]), 5))

variants = {
    "zeco_dense_in": lambda q, k, v, g, *a: zeco_gla(q.contiguous(), k.contiguous(), v.contiguous(), g.contiguous()),
    "zeco_dense_out": lambda q, k, v, g, *a: zeco_gla(q, k, v, g).contiguous(),
}
for name, core in variants.items():
    layer.zero_grad()
    xx = x.clone().requires_grad_(True)
    y = layer(xx, core)
    y.float().square().mean().backward()
    print(name, "vs ref64 x.grad", round(rel(xx.grad, outs["ref64"][1]), 5))

cap = {}
def wrap(name, core):
    def f(q, k, v, g, *a):
        for n, t in zip("qkvg", (q, k, v, g)):
            t.retain_grad()
        cap[name] = (q, k, v, g)
        o = core(q, k, v, g, *a)
        o.retain_grad()
        cap[name + "_o"] = o
        return o
    return f
for name, core in (("zeco", zeco_gla), ("ref", gla_reference)):
    layer.zero_grad()
    xx = x.clone().requires_grad_(True)
    y = layer(xx, wrap(name, core))
    y.float().square().mean().backward()
print("d_out rel", round(rel(cap["zeco_o"].grad, cap["ref_o"].grad), 5), "|d_out|", cap["ref_o"].grad.abs().max().item())
for i, n in enumerate("qkvg"):
    print("grad", n, round(rel(cap["zeco"][i].grad, cap["ref"][i].grad), 5), "max", cap["ref"][i].grad.abs().max().item())

do_l = cap["ref_o"].grad.detach()
print("d_out dtype", do_l.dtype, "stride", do_l.stride(), "absmax", do_l.abs().max().item(), "absmean", do_l.abs().mean().item())
qq, kk, vv, gg = (t.detach() for t in cap["ref"])
for scale in (1.0, 1e4):
    res2 = {}
    for name, core in (("zeco", zeco_gla), ("ref", gla_reference)):
        leaves = [t.clone().requires_grad_(True) for t in (qq, kk, vv, gg)]
        if name == "ref":
            leaves = [t.double().requires_grad_(True) for t in (qq, kk, vv, gg)]
        o = core(*leaves)
        o.backward((do_l.double() * scale).to(o.dtype))
        res2[name] = [t.grad for t in leaves]
    print("layer d_out x", scale, [round(rel(a, b), 5) for a, b in zip(res2["zeco"], res2["ref"])])
torch.save({"q": qq, "k": kk, "v": vv, "g": gg, "do": do_l}, "gpurun_out/dbg_d64.pt")

oz, orf = cap["zeco_o"].detach().float(), cap["ref_o"].detach().float()
rms_z = oz.pow(2).mean(-1).sqrt()
print("o rel", round(rel(oz, orf), 5), "d_out rel", round(rel(cap["zeco_o"].grad, cap["ref_o"].grad), 5))
print("rms(o) per (head, token): min", rms_z.min().item(), "median", rms_z.median().item())
bad = (rms_z < 1e-3).sum().item()
print("rows with rms < 1e-3:", bad, "of", rms_z.numel())
