"""One cuBLAS DGEMM (torch.matmul float64, n=8192) -- for an ncu capture of the
library kernel we compare the DMMA tile kernel against."""
import torch
n = 8192
a = torch.randn(n, n, dtype=torch.float64, device="cuda")
b = torch.randn(n, n, dtype=torch.float64, device="cuda")
for _ in range(3):
    c = a @ b
torch.cuda.synchronize()
