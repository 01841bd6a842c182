import sys, numpy as np, torch
sys.path.insert(0, ".")
import paper_1911_05328_b200 as sm
rng = np.random.default_rng(77); n = 512; s = sm.INT_RING
cfg = sm.Config(base_dim=64, workers=148, int_tensor_cores=True)
with sm.Executor(cfg) as ex:
    for lo, hi in [(-5, 6), (-2 ** 40, 2 ** 40), (-2 ** 40, 2 ** 40), (-5, 6)]:
        A = rng.integers(lo, hi, (n, n), dtype=np.int64); B = rng.integers(lo, hi, (n, n), dtype=np.int64)
        C = sm.Matrix(np.zeros((n, n), np.int64), s)
        sm.run_algorithm(ex, "star", C, sm.Matrix(A, s), sm.Matrix(B, s), s)
        st = ex.last_stats
        print(hi, st["path_name"], st["guard_syncs"], st["candidates"], st["executes"])
