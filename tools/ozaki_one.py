"""One warm-up + one timed Ozaki-II execute at n (for ncu launch lists)."""
import sys, os
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1911_05328_b200 import _lib
n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
emu = (sys.argv[2] != "dmma") if len(sys.argv) > 2 else True
g = torch.Generator(device="cuda"); g.manual_seed(3)
A = torch.randn(n, n, generator=g, dtype=torch.float64, device="cuda")
B = torch.randn(n, n, generator=g, dtype=torch.float64, device="cuda")
C = torch.rand(n, n, generator=g, dtype=torch.float64, device="cuda")
flags = _lib.F_FP64_EMU if emu else 0
plan = _lib.Plan(_lib.SR_FP64, "co2", "pooled", n, n, n, 64, 148, -1, 0, flags)
s = torch.cuda.current_stream().cuda_stream
for _ in range(2):
    plan.execute(C.data_ptr(), n, A.data_ptr(), n, B.data_ptr(), n, s)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); plan.execute(C.data_ptr(), n, A.data_ptr(), n, B.data_ptr(), n, s); e1.record()
torch.cuda.synchronize()
print("path", _lib.PATH_NAMES.get(plan.stats()["path"]), "ms", round(e0.elapsed_time(e1), 3),
      "tflops", round(2 * n ** 3 / e0.elapsed_time(e1) / 1e9, 1))
