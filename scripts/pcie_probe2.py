"""PCIe probe 2: bidirectional copies split into n chunks per direction (same stream per direction)."""
import json, time, torch
N = 402653184
dev = torch.device("cuda")
hin = torch.empty(N, dtype=torch.uint8).pin_memory(); hout = torch.empty(N, dtype=torch.uint8).pin_memory()
din = torch.empty(N, dtype=torch.uint8, device=dev); dout = torch.empty(N, dtype=torch.uint8, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
busy = torch.empty(2 * 1024 ** 3, dtype=torch.uint8, device=dev)
def run(n, kernels=False):
    c = N // n
    torch.cuda.synchronize(); t = time.perf_counter()
    for i in range(n):
        with torch.cuda.stream(s1): din[i * c:(i + 1) * c].copy_(hin[i * c:(i + 1) * c], non_blocking=True)
        with torch.cuda.stream(s2): hout[i * c:(i + 1) * c].copy_(dout[i * c:(i + 1) * c], non_blocking=True)
        if kernels: busy[: 1024 ** 3].copy_(busy[1024 ** 3:])
    torch.cuda.synchronize(); return (time.perf_counter() - t) * 1e3
out = {}
for n in (1, 8, 40, 80, 160):
    run(n); out[f"n{n}"] = round(min(run(n) for _ in range(3)), 3)
for n in (40, 80):
    run(n, True); out[f"n{n}_with_hbm_kernels"] = round(min(run(n, True) for _ in range(3)), 3)
print(json.dumps(out))
