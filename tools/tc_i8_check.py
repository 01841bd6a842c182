"""Quick correctness + timing check of the opt-in tcgen05 int8 path (exact int64)."""
import sys, os, time, json
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1911_05328_b200 as sm
from oracle import oracle as O
res = {}
for n in [int(x) for x in (sys.argv[1:] or ["256", "512", "1000", "4096"])]:
    rng = np.random.default_rng(n)
    A = rng.integers(-16, 17, (n, n), dtype=np.int64)
    B = rng.integers(-16, 17, (n, n), dtype=np.int64)
    C0 = rng.integers(-50, 50, (n, n), dtype=np.int64)
    s = sm.INT_RING
    cfg = sm.Config(base_dim=64, workers=148, int_tensor_cores=True, allow_nonpow2=True)
    with sm.Executor(cfg) as ex:
        C = sm.Matrix(C0, s); Am, Bm = sm.Matrix(A, s), sm.Matrix(B, s)
        sm.run_algorithm(ex, "star", C, Am, Bm, s)
        path = ex.last_stats["path_name"]
        got = C.numpy()
        rows = slice(0, min(n, 256))
        want = C0[rows].copy()
        O.gemm_fold(O.SR_INT64, want, np.ascontiguousarray(A[rows]), B, par=True)
        ok = bool(np.array_equal(got[rows], want))
        torch.cuda.synchronize(); t = time.perf_counter()
        for _ in range(5):
            sm.run_algorithm(ex, "star", C, Am, Bm, s)
        torch.cuda.synchronize(); t = (time.perf_counter() - t) / 5
    res[n] = {"path": path, "exact_first_rows": ok, "ms": round(t * 1e3, 3),
              "tops": round(2 * n ** 3 / t / 1e12, 1)}
    print(json.dumps({n: res[n]}), flush=True)
