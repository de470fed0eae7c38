"""Per-tile pipeline timeline of one CTA of the fused kernels (diagnostics)."""
import ctypes, math, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2507_01004_b200 import ops, _native

H, L, D = 16, 16384, 128
dev = torch.device("cuda")
gen = torch.Generator(device=dev).manual_seed(0)
u = lambda lo, hi, dt: (torch.rand((H, L, D), device=dev, generator=gen) * (hi - lo) + lo).to(dt)
q, k, v, do = (u(-1, 1, torch.bfloat16) for _ in range(4))
g = u(math.log(0.9), math.log(0.999), torch.float32)
sh = ops.ZecoShard(H, L, D, D, 64, torch.bfloat16)
buf = torch.zeros(32 * 512, dtype=torch.int64, device=dev)
cta = int(sys.argv[1]) if len(sys.argv) > 1 else 0
FWD_EV = ["tma", "prep", "mma1", "mma24", "mma3", "st_afull", "st_mask", "st_kvfull", "st_upd", "st_ofull", "st_epi", "mma_wait_s_o", "prep_start"]
BWD_EV = ["tma", "prep", "mma_sc", "mma_wait3", "mma_grads", "st_scfull", "st_dp", "st_prologue", "st_gfull", "st_epi", "prep_g", "prep_full"]
for it in range(3):
    s_loc, g_tot = sh.fwd_local(k, v, g)
    if it == 2:
        _native.call("zgla_set_trace", ctypes.c_void_p(buf.data_ptr()), cta)
    sh.fwd_output(q, k, v, g, None)
    torch.cuda.synchronize()
    if it == 2:
        fwd_tr = buf.view(32, 512).cpu().clone(); buf.zero_()
    d0 = sh.bwd_local(q, g, do)
    sh.bwd_output(q, k, v, g, do, None, None)
    torch.cuda.synchronize()
    if it == 2:
        bwd_tr = buf.view(32, 512).cpu().clone()
        _native.call("zgla_set_trace", None, 0)

def show(tr, names, title):
    t0 = min(int(x) for x in tr[:len(names)].flatten() if int(x) > 0)
    print(f"== {title}: columns are tiles, values us since first event")
    nt = int((tr[0] > 0).sum())
    for e, name in enumerate(names):
        row = [(int(tr[e, n]) - t0) / 1000 if int(tr[e, n]) > 0 else float('nan') for n in range(nt)]
        print(f"{name:14s}" + " ".join(f"{x:7.1f}" for x in row[:14]), " ... last", f"{row[-1]:.1f}")
show(fwd_tr, FWD_EV, f"fwd_out_kernel CTA {cta}")
show(bwd_tr, BWD_EV, f"bwd_out_kernel CTA {cta}")

def steady(tr, names, pairs, title):
    """mean durations (us) over the steady tiles 2..nt-2 for (name, from_event, to_event) pairs"""
    nt = int((tr[0] > 0).sum())
    ix = {n: i for i, n in enumerate(names)}
    out = []
    period = (int(tr[ix[pairs[0][2]], nt - 2]) - int(tr[ix[pairs[0][2]], 2])) / (nt - 4) / 1000
    for name, a, b in pairs:
        d = [(int(tr[ix[b], n]) - int(tr[ix[a], n])) / 1000 for n in range(2, nt - 1)]
        out.append(f"{name}={sum(d) / len(d):.2f}")
    print(f"STEADY {title}: period={period:.2f}us " + " ".join(out))

steady(bwd_tr, BWD_EV, [("epi", "st_gfull", "st_epi"), ("mma", "st_dp", "st_gfull"),
                        ("mask_dp", "st_scfull", "st_dp"), ("tma2prep", "tma", "prep")], "bwd")
steady(fwd_tr, FWD_EV, [("epi", "st_ofull", "st_epi"), ("tma2prep", "tma", "prep")], "fwd")


def ctas(tr, title):
    """per-CTA lifetimes (us): spread of start and end across the grid"""
    st, en = tr[26].numpy().astype("int64"), tr[27].numpy().astype("int64")
    n = int((st > 0).sum())
    st, en = st[:n], en[:n]
    t0 = st.min()
    dur = (en - st) / 1000
    print(f"CTAS {title}: n={n} start spread {(st.max() - t0) / 1000:.1f}us, end first {(en.min() - t0) / 1000:.1f} "
          f"last {(en.max() - t0) / 1000:.1f}us; duration min {dur.min():.1f} median {sorted(dur)[n // 2]:.1f} max {dur.max():.1f}")
    slow = sorted(range(n), key=lambda i: -dur[i])[:6]
    print("   slowest:", [(i, round(float(dur[i]), 1), int(tr[28, i])) for i in slow])

ctas(fwd_tr, "fwd_out")
ctas(bwd_tr, "bwd_out")
