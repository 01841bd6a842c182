"""One plan, a few executes: a target for ncu captures of a single kernel variant.
  python tools/one_mm.py <semiring> <algo> <n> <ksplit|-1> [reps]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1911_05328_b200 as sm  # noqa: E402
from paper_1911_05328_b200 import _lib  # noqa: E402

sid, algo, n, ks = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 3
s = sm.get_semiring(sid)
g = torch.Generator(device="cuda")
g.manual_seed(1)
if s.torch_dtype == torch.float64:
    A = torch.randn(n, n, generator=g, device="cuda", dtype=torch.float64)
    B = torch.randn(n, n, generator=g, device="cuda", dtype=torch.float64)
else:
    A = torch.randint(0, 100, (n, n), generator=g, device="cuda").to(s.torch_dtype)
    B = torch.randint(0, 100, (n, n), generator=g, device="cuda").to(s.torch_dtype)
C = torch.zeros(n, n, dtype=s.torch_dtype, device="cuda")
p = _lib.Plan(s.sr_id, algo, "pooled", n, n, n, 64, 148, ks, 0, _lib.F_ALLOW_NONPOW2)
for _ in range(reps):
    p.execute(C.data_ptr(), n, A.data_ptr(), n, B.data_ptr(), n, torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
st = p.stats()
print(sid, algo, n, ks, st["path_name"], "S", st["ksplit"], "cluster", st["cluster_size"],
      "balanced", st["balanced_workers"])
p.close()
