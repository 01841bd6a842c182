import torch, time, json
n = 1 << 28  # 256M int32 = 1 GiB
h = torch.empty(n, dtype=torch.int32).pin_memory(); d = torch.empty(n, dtype=torch.int32, device="cuda")
h2 = torch.empty(n, dtype=torch.int32).pin_memory(); d2 = torch.empty(n, dtype=torch.int32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for _ in range(2): d.copy_(h, non_blocking=True); h.copy_(d, non_blocking=True)
torch.cuda.synchronize()
def t(f):
    torch.cuda.synchronize(); t0 = time.perf_counter(); f(); torch.cuda.synchronize(); return time.perf_counter() - t0
r = {}
r["h2d_GBs"] = 4 * n / t(lambda: d.copy_(h, non_blocking=True)) / 1e9
r["d2h_GBs"] = 4 * n / t(lambda: h.copy_(d, non_blocking=True)) / 1e9
def both():
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
r["duplex_GBs_total"] = 8 * n / t(both) / 1e9
def two_h2d():
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): d2.copy_(h2, non_blocking=True)
r["two_h2d_GBs_total"] = 8 * n / t(two_h2d) / 1e9
print(json.dumps({k: round(v, 1) for k, v in r.items()}))
