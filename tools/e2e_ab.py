"""A/B timing of the host-buffer path (starmm_execute_host): block_rows sweep.

  python tools/e2e_ab.py [n] [float|int] [block_rows ...]"""
import os, sys, time, json
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1911_05328_b200 as sm
n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
sid = sys.argv[2] if len(sys.argv) > 2 else "float"
brs = [int(x) for x in sys.argv[3:]] or [0, 4096, 1024]
s = sm.get_semiring(sid)
if sid == "int":
    A = torch.randint(-16, 17, (n, n), dtype=torch.int64).pin_memory()
    B = torch.randint(-16, 17, (n, n), dtype=torch.int64).pin_memory()
else:
    A = torch.randn(n, n, dtype=torch.float64).pin_memory()
    B = torch.randn(n, n, dtype=torch.float64).pin_memory()
C = torch.zeros(n, n, dtype=s.torch_dtype).pin_memory()
res = {}
with sm.Executor(sm.Config(base_dim=64, workers=148)) as ex:
    for br in brs:
        ex.execute_host("star", C, A, B, s, block_rows=br)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(3):
            ex.execute_host("star", C, A, B, s, block_rows=br)
        t = (time.perf_counter() - t0) / 3
        res[f"block_rows={br}"] = {"ms": t * 1e3, "tops": 2 * n ** 3 / t / 1e12}
    t0 = time.perf_counter(); Ad = A.to("cuda", non_blocking=True); torch.cuda.synchronize()
    res["h2d_GBps"] = A.numel() * A.element_size() / (time.perf_counter() - t0) / 1e9
    t0 = time.perf_counter(); A.copy_(Ad, non_blocking=True); torch.cuda.synchronize()
    res["d2h_GBps"] = A.numel() * A.element_size() / (time.perf_counter() - t0) / 1e9
res["kchunk"] = os.environ.get("STARMM_HOST_KCHUNK", "1")
print(json.dumps(res))
