"""development: pinned host <-> device copy bandwidth (each way and both at once)"""
import json, time, torch
n = 4 << 30  # bytes
h1 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d1 = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(f):
    torch.cuda.synchronize(); t0 = time.perf_counter(); f(); torch.cuda.synchronize(); return time.perf_counter() - t0
for _ in range(2):
    h2d = t(lambda: d1.copy_(h1, non_blocking=True))
    d2h = t(lambda: h2.copy_(d2, non_blocking=True))
    def both():
        with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
        with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
    bi = t(both)
print(json.dumps({"h2d_GBs": n / h2d / 1e9, "d2h_GBs": n / d2h / 1e9, "bidir_GBs_each": n / bi / 1e9}))
