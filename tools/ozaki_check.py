"""Accuracy + timing of the opt-in Ozaki-II fp64 emulation against DMMA and an exact
reference (Python integers on sampled entries, correctly rounded once).

  python tools/ozaki_check.py [n ...]      (config 4 distributions: N(0,1) x N(0,1), C0 U[-1,1))
"""
import sys, os, time, json
from fractions import Fraction
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1911_05328_b200 as sm


def exact_entry(a, b, c0):
    ma, ea = np.frexp(a); mb, eb = np.frexp(b)
    ia = (ma * 2.0 ** 53).astype(np.int64); ib = (mb * 2.0 ** 53).astype(np.int64)
    ex = (ea.astype(np.int64) - 53) + (eb.astype(np.int64) - 53)
    e0 = int(ex.min())
    tot = 0
    for x, y, e in zip(ia.tolist(), ib.tolist(), ex.tolist()):
        tot += (x * y) << (e - e0)
    return float(Fraction(tot) * Fraction(2) ** e0 + Fraction(c0)) if e0 < 0 else float(tot * 2 ** e0 + Fraction(c0))


def run(n, emu, A, B, C0, reps):
    s = sm.FLOAT_RING
    cfg = sm.Config(base_dim=64, workers=148, fp64_emulation=emu, allow_nonpow2=True)
    with sm.Executor(cfg) as ex:
        C = sm.Matrix(C0.copy(), s); Am, Bm = sm.Matrix(A, s), sm.Matrix(B, s)
        sm.run_algorithm(ex, "star", C, Am, Bm, s)
        path = ex.last_stats["path_name"]
        out = C.numpy().copy()
        torch.cuda.synchronize(); t = time.perf_counter()
        for _ in range(reps):
            sm.run_algorithm(ex, "star", C, Am, Bm, s)
        torch.cuda.synchronize(); t = (time.perf_counter() - t) / max(1, reps)
    return out, path, t


res = {}
for n in [int(x) for x in (sys.argv[1:] or ["300", "1024", "4096"])]:
    rng = np.random.default_rng(3)
    A = rng.standard_normal((n, n)); B = rng.standard_normal((n, n)); C0 = rng.uniform(-1, 1, (n, n))
    reps = 3 if n >= 8192 else 5
    got_d, path_d, t_d = run(n, False, A, B, C0, reps)
    got_e, path_e, t_e = run(n, True, A, B, C0, reps)
    idx = [(int(i), int(j)) for i, j in zip(rng.integers(0, n, 24), rng.integers(0, n, 24))]
    ulp_d, ulp_e, rel_d, rel_e = [], [], [], []
    absab = None
    for i, j in idx:
        x = exact_entry(A[i], B[:, j], C0[i, j])
        u = np.spacing(abs(x)) if x != 0 else np.spacing(0.0)
        scale = float(np.abs(A[i]) @ np.abs(B[:, j]))
        ulp_d.append(abs(got_d[i, j] - x) / u); ulp_e.append(abs(got_e[i, j] - x) / u)
        rel_d.append(abs(got_d[i, j] - x) / scale); rel_e.append(abs(got_e[i, j] - x) / scale)
    res[n] = {"dmma": {"path": path_d, "ms": round(t_d * 1e3, 3), "tflops": round(2 * n ** 3 / t_d / 1e12, 1),
                       "max_ulp": round(max(ulp_d), 2), "max_err_over_absAB": float(max(rel_d))},
              "ozaki2": {"path": path_e, "ms": round(t_e * 1e3, 3), "tflops": round(2 * n ** 3 / t_e / 1e12, 1),
                         "max_ulp": round(max(ulp_e), 2), "max_err_over_absAB": float(max(rel_e))},
              "emu_vs_dmma_max_rel": float(np.max(np.abs(got_e - got_d) / np.maximum(np.abs(got_d), 1e-300)))}
    print(json.dumps({n: res[n]}), flush=True)

# non-finite inputs must fall back to DMMA with IEEE results
n = 256
rng = np.random.default_rng(5)
A = rng.standard_normal((n, n)); B = rng.standard_normal((n, n)); A[3, 7] = np.nan; B[9, 11] = np.inf
got_d, path_d, _ = run(n, False, A, B, np.zeros((n, n)), 0)
got_e, path_e, _ = run(n, True, A, B, np.zeros((n, n)), 0)
fin = np.isfinite(got_d)
print(json.dumps({"nonfinite": {"path": path_e,
                                "same_pattern": bool(np.array_equal(np.isnan(got_d), np.isnan(got_e)) and
                                                     np.array_equal(np.isinf(got_d), np.isinf(got_e))),
                                "finite_close": bool(np.allclose(got_d[fin], got_e[fin], rtol=1e-12, atol=1e-12))}}))
