"""cuBLAS DGEMM / int ops reference throughput (torch.matmul float64) — the
library denominator for the fp64 (+,x) roofline."""
import json, torch
res = {}
for n in (8192, 16384):
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    c = torch.empty_like(a)
    for _ in range(2):
        torch.matmul(a, b, out=c)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 5 if n == 8192 else 3
    e0.record()
    for _ in range(reps):
        torch.matmul(a, b, out=c)
    e1.record(); torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 1e3 / reps
    res[f"cublas_dgemm_n{n}_tflops"] = 2 * n ** 3 / t / 1e12
print(json.dumps(res))
