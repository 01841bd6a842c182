"""Throughput of the reference's own float64 (min,+) semiring on non-integer data (general
DADD+DMNMX kernel) and on integer-valued data (exact narrow paths)."""
import sys, os, time, json, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1911_05328_b200 as sm
n = 8192
s = sm.TROPICAL
res = {}
for kind in ("fractional", "integer"):
    A = torch.rand(n, n, dtype=torch.float64, device="cuda") * 100
    B = torch.rand(n, n, dtype=torch.float64, device="cuda") * 100
    if kind == "integer":
        A, B = A.floor(), B.floor()
    C = torch.full((n, n), float("inf"), dtype=torch.float64, device="cuda")
    with sm.Executor(sm.Config(base_dim=64, workers=148)) as ex:
        M, Am, Bm = sm.Matrix(C, s), sm.Matrix(A, s), sm.Matrix(B, s)
        sm.run_algorithm(ex, "star", M, Am, Bm, s); torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(3):
            sm.run_algorithm(ex, "star", M, Am, Bm, s)
        torch.cuda.synchronize(); t = (time.perf_counter() - t) / 3
        res[kind] = {"ms": round(t * 1e3, 2), "tops": round(2 * n ** 3 / t / 1e12, 2),
                     "path": ex.last_stats["path_name"]}
print(json.dumps(res))
