"""Library int8 tensor-core peak on this B200: torch._int_mm (cuBLASLt, int8 x int8 -> int32),
best of 10 (burst) and back-to-back for ~4 s (sustained), CUDA events -- the int8 analogue
of MEASURED_PEAKS.json's bf16 torch.matmul figures.  Writes profiles/r01_int8_peak.json."""
import json, os, sys, time
import torch
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
out = {}
for n in (8192, 16384):
    a = torch.randint(-128, 128, (n, n), dtype=torch.int8, device="cuda")
    b = torch.randint(-128, 128, (n, n), dtype=torch.int8, device="cuda")
    torch._int_mm(a, b)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); torch._int_mm(a, b); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    reps, t0 = 0, time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    while time.perf_counter() - t0 < 4.0:
        for _ in range(8):
            torch._int_mm(a, b)
        reps += 8
        torch.cuda.synchronize()
    e1.record(); torch.cuda.synchronize()
    sus = e0.elapsed_time(e1) / reps
    out[f"int_mm_n{n}_burst_tops"] = 2 * n ** 3 / best / 1e9
    out[f"int_mm_n{n}_sustained_tops"] = 2 * n ** 3 / sus / 1e9
out["how"] = "torch._int_mm (cuBLASLt) int8 x int8 -> int32, square n; burst = best of 10, sustained = back to back ~4 s"
print(json.dumps(out))
json.dump(out, open(os.path.join(REPO, "profiles", "r01_int8_peak.json"), "w"), indent=1)
