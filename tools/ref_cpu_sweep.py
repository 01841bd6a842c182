"""The reference's own CPU path, swept on the GPU box's host cores:
star_mm (classic.py:314-316) from the UNMODIFIED package in baseline/_ref under
Config(base_dim=b, workers=W) for W in {1, os.cpu_count()}, n = 256, 512, ... doubling
after a small-n JIT warm-up, stopping at the first run over the cap (600 s) -- a run
whose predicted time (8x the previous) exceeds 1.5x the cap is recorded as skipped
rather than burnt.  Writes profiles/r02_ref_cpu_sweep.json (largest n completed per
semiring and W, Gop/s at every n).

  python tools/ref_cpu_sweep.py [--cap 600] [--semirings float,int,tropical]
  python tools/ref_cpu_sweep.py --native-matmul     # the reference's own leaf kernel,
        Semiring.matmul (semiring.py:92-94, numba _mm_*), single-threaded, n = 512..2048
        -> profiles/r02_ref_native_matmul.json
"""
import argparse
import json
import os
import subprocess
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import os, sys, time, json
sys.dont_write_bytecode = True
sys.path.insert(0, os.path.join(%(repo)r, "baseline", "_ref"))
sys.path.insert(0, %(repo)r)
import numpy as np
import starmm as ref
from bench_configs import make_inputs, to_reference
cid, n, W, b = %(cid)d, %(n)d, %(W)d, %(b)d
s = ref.get_semiring(%(sid)r)
A, B, C = make_inputs(cid, n)
Am = ref.Matrix(to_reference(cid, A), s)
Bm = Am if B is A else ref.Matrix(to_reference(cid, B), s)
Cm = ref.Matrix(to_reference(cid, C).copy(), s)
t0 = time.perf_counter()
ref.star_mm(Cm, Am, Bm, s, ref.Config(base_dim=b, workers=W))
print(json.dumps({"seconds": time.perf_counter() - t0}))
"""

CID_OF = {"float": 4, "int": 2, "tropical": 5}

NATIVE = r"""
import os, sys, time, json
sys.dont_write_bytecode = True
sys.path.insert(0, os.path.join(%(repo)r, "baseline", "_ref"))
sys.path.insert(0, %(repo)r)
import numpy as np
import starmm as ref
from bench_configs import make_inputs, to_reference
cid, n = %(cid)d, %(n)d
s = ref.get_semiring(%(sid)r)
A, B, C = make_inputs(cid, n)
A = to_reference(cid, A); B = A if B is A else to_reference(cid, B)
s.matmul(A[:64, :64].copy(), B[:64, :64].copy())          # JIT
t0 = time.perf_counter()
s.matmul(A, B)
print(json.dumps({"seconds": time.perf_counter() - t0}))
"""


def native_matmul(out_name):
    env = dict(os.environ, NUMBA_CACHE_DIR="/tmp/starmm_ref_numba_cache", NUMBA_NUM_THREADS="1",
               OMP_NUM_THREADS="1", OPENBLAS_NUM_THREADS="1", MKL_NUM_THREADS="1")
    out = {"host_cores": os.cpu_count(), "threads": 1, "rows": [],
           "how": "reference Semiring.matmul (baseline/_ref, unmodified; numba leaf kernels / numpy "
                  "matmul as the reference chooses), one call on the BASELINE config distributions"}
    for sid in ("float", "int", "tropical"):
        for n in (512, 1024, 2048):
            code = NATIVE % {"repo": REPO, "cid": CID_OF[sid], "n": n, "sid": sid}
            p = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=900, env=env)
            if p.returncode != 0:
                out["rows"].append({"semiring": sid, "n": n, "status": "error", "stderr": p.stderr[-300:]})
                continue
            sec = json.loads(p.stdout.strip().splitlines()[-1])["seconds"]
            out["rows"].append({"semiring": sid, "n": n, "seconds": sec, "gops": 2.0 * n ** 3 / sec / 1e9})
            print(out["rows"][-1], flush=True)
    json.dump(out, open(os.path.join(REPO, "profiles", out_name), "w"), indent=1)


def run_one(sid, n, W, b, cap):
    code = CHILD % {"repo": REPO, "cid": CID_OF[sid], "n": n, "W": W, "b": b, "sid": sid}
    env = dict(os.environ, NUMBA_CACHE_DIR="/tmp/starmm_ref_numba_cache")
    t0 = time.perf_counter()
    try:
        p = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=cap,
                           env=env)
    except subprocess.TimeoutExpired:
        return {"n": n, "status": f"over {cap:.0f} s (killed)", "seconds": time.perf_counter() - t0}
    if p.returncode != 0:
        return {"n": n, "status": "error", "stderr": p.stderr[-400:]}
    sec = json.loads(p.stdout.strip().splitlines()[-1])["seconds"]
    return {"n": n, "status": "ok", "seconds": sec, "gops": 2.0 * n ** 3 / sec / 1e9}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cap", type=float, default=600.0)
    ap.add_argument("--semirings", default="float,int,tropical")
    ap.add_argument("--workers", default="")
    ap.add_argument("--out", default="r02_ref_cpu_sweep.json")
    ap.add_argument("--native-matmul", action="store_true")
    args = ap.parse_args()
    if args.native_matmul:
        native_matmul("r02_ref_native_matmul.json")
        return
    cores = os.cpu_count() or 1
    Ws = [int(x) for x in args.workers.split(",")] if args.workers else sorted({1, cores})
    out = {"host_cores": cores, "cap_seconds": args.cap, "series": [], "largest_n": {},
           "how": "reference star_mm (baseline/_ref, unmodified), Config(base_dim=b, workers=W); "
                  "b = 32 up to n = 512, else 64; inputs = the BASELINE config distributions "
                  "(bench_configs.make_inputs: float -> config 4, int -> config 2, tropical -> "
                  "config 5's weights up-cast to float64)"}
    path = os.path.join(REPO, "profiles", args.out)
    for sid in args.semirings.split(","):
        run_one(sid, 64, 1, 32, args.cap)                       # numba JIT into the cache
        for W in Ws:
            rows, n, prev = [], 256, None
            while True:
                b = 32 if n <= 512 else 64
                if prev is not None and prev * 8 > 1.5 * args.cap:
                    rows.append({"n": n, "status": f"skipped: predicted {prev * 8:.0f} s > 1.5 x cap"})
                    break
                r = run_one(sid, n, W, b, args.cap)
                rows.append(r)
                print(sid, W, r, flush=True)
                if r["status"] != "ok" or r["seconds"] > args.cap:
                    break
                prev = r["seconds"]
                n *= 2
            done = [r for r in rows if r["status"] == "ok" and r["seconds"] <= args.cap]
            out["series"].append({"semiring": sid, "workers": W, "runs": rows})
            out["largest_n"][f"{sid}:W{W}"] = max((r["n"] for r in done), default=None)
            json.dump(out, open(path, "w"), indent=1)        # after every series
    print(json.dumps(out["largest_n"]))


if __name__ == "__main__":
    main()
