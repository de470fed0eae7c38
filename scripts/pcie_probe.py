"""PCIe copy-rate probe: H2D, D2H, both directions concurrently (pinned host memory)."""
import torch, time, json
n = 402653184 // 4
dev = torch.device("cuda")
hs = [torch.empty(n, dtype=torch.float32).pin_memory() for _ in range(2)]
ds = [torch.empty(n, dtype=torch.float32, device=dev) for _ in range(2)]
s1, s2, s3 = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
def timeit(fn, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize(); t = time.perf_counter(); fn(); torch.cuda.synchronize(); best = min(best, time.perf_counter() - t)
    return best
def h2d():
    with torch.cuda.stream(s1): ds[0].copy_(hs[0], non_blocking=True)
def d2h():
    with torch.cuda.stream(s2): hs[1].copy_(ds[1], non_blocking=True)
def both():
    h2d(); d2h()
def h2d_split():
    h = n // 2
    with torch.cuda.stream(s1): ds[0][:h].copy_(hs[0][:h], non_blocking=True)
    with torch.cuda.stream(s3): ds[0][h:].copy_(hs[0][h:], non_blocking=True)
out = {}
for name, fn in (("h2d", h2d), ("d2h", d2h), ("both", both), ("h2d_2streams", h2d_split)):
    t = timeit(fn)
    out[name] = {"ms": t * 1e3, "GBps_per_dir": 402653184 / t / 1e9}
print(json.dumps(out))
