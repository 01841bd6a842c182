"""Command-line front end (declared at pyproject.toml:18-19 but
absent from the reference package).

  python -m paper_1911_05328_b200 run    --algo star --semiring int --n 64 --b 8 [--seed 1]
  python -m paper_1911_05328_b200 bench  --algos co2,co3,tar,sar,star --n 2048,4096 --b 64 --reps 5 --out t.csv
  python -m paper_1911_05328_b200 verify [--suite correctness|space|all]

Exit codes: 0 ok, 1 verification failure, 2 invalid input.
`run` and `verify` check every schedule against an INDEPENDENT plain-PyTorch
product (the role of ``naive_mm``, kernels.py:28-32, which on this build would run
the same tile kernels as the schedules): torch.matmul in float64 and int64 (wraps
mod 2^64) on the CPU, and a broadcast (min,+) reduction in the k order of the
reference for the tropical semirings -- exactly for int / (min,+) and within rel
1e-9 for float.  `verify --suite pool` is the allocator's property
test (one fresh block per size, LIFO re-issue order) on the DEVICE
pool; `--sabotage-lifo` runs every suite with the device pool in FIFO order, the
reference's negative control (pool.py:70-74), and must exit 1.  `bench` reports the paper's speedup formula
(t_peer / t_algo - 1) * 100% against CO2 and CO3, with one
shared base kernel and one b per comparison set (the fairness rule,
PAPER.md:1464-1467).  `analyze` and `simulate` belong to the analysis engine,
which is out of scope for this build: they exit 2.
"""
from __future__ import annotations

import argparse
import csv
import json
import os
import statistics
import sys
import time

import numpy as np

from .errors import StarMMError
from .matrix import Config, Matrix, matrices_equal, random_matrix
from .registry import ALGORITHMS, CLASSICAL, run_algorithm
from .runtime import Executor
from .semiring import get_semiring

EXIT_OK, EXIT_MISMATCH, EXIT_INVALID = 0, 1, 2


def _torch_fold_product(s, C0, A, B):
    """fold_add(C0, A (x) B) in plain PyTorch on the CPU, independent of libstarmm's
    kernels: the checker of `run` / `verify`.  (min,+): first minimum over k in
    increasing k order (semiring.py:56-58), then np.minimum's tie rule (the second
    operand, the product, wins a tie) -- so signed zeros agree too."""
    import torch
    C0, A, B = (x.detach().cpu() for x in (C0, A, B))
    if s.id in ("int", "float"):
        return C0 + A @ B                       # int64 wraps mod 2^64 like _mm_int
    if s.id == "tropical_i32":
        a, b = A.to(torch.int64), B.to(torch.int64)
        inf = 2 ** 31 - 1
        v = (a[:, :, None] + b[None, :, :]).clamp(-2 ** 31, inf)
        v = torch.where((a[:, :, None] == inf) | (b[None, :, :] == inf), torch.full_like(v, inf), v)
        return torch.minimum(C0.to(torch.int64), v.min(dim=1).values).to(torch.int32)
    out = torch.full(C0.shape, float("inf"), dtype=C0.dtype)
    for kk in range(A.shape[1]):               # "if v < out": NaN never wins, first zero kept
        v = A[:, kk:kk + 1] + B[kk:kk + 1, :]
        out = torch.where(v < out, v, out)
    res = torch.where(C0 < out, C0, out)       # np.minimum(C0, out): a tie keeps out
    return torch.where(torch.isnan(C0), C0, res)


def _one(algo, sid, n, b, p, seed, mode="pooled", ksplit=None):
    """Run `algo` once on the reference fixture generator; compare with naive_mm."""
    s = get_semiring(sid)
    A = random_matrix(n, s, seed)
    B = random_matrix(n, s, seed + 1)
    C0 = random_matrix(n, s, seed + 2)
    C = Matrix(C0.data.clone(), s)
    cfg = Config(base_dim=b, workers=p, ksplit=ksplit)
    with Executor(cfg) as ex:
        run_algorithm(ex, algo, C, A, B, s, mode=mode)
        snap = ex.metrics.snapshot(ex.pool).to_dict()
    want = Matrix(_torch_fold_product(s, C0.data, A.data, B.data), s)
    ok = matrices_equal(C, want) if sid != "float" else matrices_equal(
        C.numpy(), want.numpy(), tol=1e-9)
    diff = None
    if not ok:
        a, w = C.numpy().astype(np.float64), want.numpy().astype(np.float64)
        with np.errstate(invalid="ignore"):
            bad = ~((a == w) | (np.isnan(a) & np.isnan(w)))
        diff = {"mismatches": int(bad.sum()), "first": [int(x) for x in np.argwhere(bad)[0]]}
    return ok, snap, diff


def cmd_run(args) -> int:
    try:
        ok, snap, diff = _one(args.algo, args.semiring, args.n, args.b, args.p, args.seed,
                              args.mode, args.ksplit)
    except StarMMError as e:
        print(json.dumps({"status": "error", "error": type(e).__name__, "message": str(e)}))
        return EXIT_INVALID
    except KeyError as e:
        print(json.dumps({"status": "error", "error": "KeyError", "message": str(e)}))
        return EXIT_INVALID
    print(json.dumps({"status": "ok" if ok else "mismatch", "algo": args.algo,
                      "semiring": args.semiring, "n": args.n, "b": args.b, "p": args.p,
                      "metrics": snap, "diff": diff}))
    return EXIT_OK if ok else EXIT_MISMATCH


def _time_one(algo, s, n, b, p, reps, seed):
    import torch
    A = random_matrix(n, s, seed)
    B = random_matrix(n, s, seed + 1)
    C = random_matrix(n, s, seed + 2)
    with Executor(Config(base_dim=b, workers=p)) as ex:
        run_algorithm(ex, algo, C, A, B, s)           # warm-up (plan, arena, JIT-free)
        times = []
        for _ in range(reps):
            torch.cuda.synchronize()
            t0 = time.perf_counter_ns()
            run_algorithm(ex, algo, C, A, B, s)
            times.append(time.perf_counter_ns() - t0)
    return statistics.median(times)


def cmd_bench(args) -> int:
    algos = args.algos.split(",")
    for a in algos:
        if a not in CLASSICAL:
            print(f"bench: unknown or out-of-scope algorithm {a!r}", file=sys.stderr)
            return EXIT_INVALID
    s = get_semiring(args.semiring)
    rows = []
    for n in [int(x) for x in args.n.split(",")]:
        med = {a: _time_one(a, s, n, args.b, args.p, args.reps, args.seed) for a in algos}
        for a in algos:
            row = {"algo": a, "n": n, "b": args.b, "p": args.p, "median_ns": int(med[a])}
            for peer in ("co2", "co3"):
                row[f"speedup_vs_{peer}_pct"] = (
                    round((med[peer] / med[a] - 1.0) * 100.0, 3) if peer in med else "")
            rows.append(row)
    out = open(args.out, "w", newline="") if args.out else sys.stdout
    w = csv.DictWriter(out, fieldnames=["algo", "n", "b", "p", "median_ns", "speedup_vs_co2_pct",
                                        "speedup_vs_co3_pct"])
    w.writeheader()
    w.writerows(rows)
    if args.out:
        out.close()
    return EXIT_OK


def _pool_suite():
    """SPEC.md:562 on the device pool: a released block is the next one issued for its
    size (one fresh allocation however often it cycles), and two released blocks come
    back newest first; sizes are independent of each other."""
    import torch
    from . import _lib
    dev = torch.cuda.current_device()
    fresh, order_ok = 0, True
    sizes = [3 << 20, 5 << 20]                 # sizes no schedule of this run asks for
    for nb in sizes:
        a, f = _lib.pool_acquire(dev, nb)
        fresh += f
        for _ in range(100):                   # release / acquire cycles: always `a`
            _lib.pool_release(dev, a)
            a2, f = _lib.pool_acquire(dev, nb)
            fresh += f
            order_ok &= a2 == a
            a = a2
        b, f = _lib.pool_acquire(dev, nb)
        fresh += f
        _lib.pool_release(dev, a)
        _lib.pool_release(dev, b)
        x, _ = _lib.pool_acquire(dev, nb)
        y, _ = _lib.pool_acquire(dev, nb)
        order_ok &= (x, y) == (b, a)           # LIFO re-issue (pool.py:97)
        _lib.pool_release(dev, y)
        _lib.pool_release(dev, x)
    return {"fresh_allocations": int(fresh), "fresh_allowed": 2 * len(sizes),
            "lifo_reissue_order": bool(order_ok)}


def cmd_verify(args) -> int:
    """Acceptance suites, GPU analogues."""
    import torch
    from . import _lib
    report = {"suites": {}}
    failed = False
    dev = torch.cuda.current_device()
    if args.sabotage_lifo:
        _lib.pool_set_discipline(dev, True)
        report["sabotage"] = "device pool in FIFO order"
    try:
        failed = _verify_suites(args, report)
    finally:
        if args.sabotage_lifo:
            _lib.pool_set_discipline(dev, False)
    report["status"] = "fail" if failed else "ok"
    print(json.dumps(report))
    return EXIT_MISMATCH if failed else EXIT_OK


def _verify_suites(args, report) -> bool:
    failed = False
    if args.suite in ("pool", "all"):
        res = _pool_suite()
        report["suites"]["pool"] = res
        failed |= not (res["lifo_reissue_order"] and res["fresh_allocations"] <= res["fresh_allowed"])
    if args.suite in ("correctness", "all"):
        res = []
        for sid in ("int", "tropical", "float"):
            for algo in CLASSICAL:
                for b in (2, 32):
                    for mult in (1, 2, 4, 8, 16):
                        for seed in range(args.seeds):
                            ok, _, diff = _one(algo, sid, b * mult, b, args.p, 100 * seed + mult)
                            res.append(ok)
                            if not ok:
                                failed = True
                                report.setdefault("failures", []).append(
                                    {"algo": algo, "semiring": sid, "n": b * mult, "b": b,
                                     "seed": seed, "diff": diff})
        report["suites"]["correctness"] = {"cases": len(res), "passed": int(sum(res))}
    if args.suite in ("space", "all"):
        rows = {}
        n, b = 512, 32
        for algo, ks in (("tar", 2), ("sar", 0), ("sar", 1), ("star", 2)):
            _, snap, _ = _one(algo, "int", n, b, args.p, 7, ksplit=ks)
            rows[f"{algo}_ksplit{ks}"] = {k: snap[k] for k in (
                "pool_high_water_bytes", "lazy_temp_acquires", "tile_serializations",
                "pair_transitions", "pair_count", "base_case_max")}
        sar_serial = rows["sar_ksplit0"]["lazy_temp_acquires"] == 0
        pairs_ok = rows["sar_ksplit1"]["pair_transitions"] == 2 * rows["sar_ksplit1"]["pair_count"]
        report["suites"]["space"] = {"bounds": rows, "sar_serial_zero_temps": sar_serial,
                                     "pair_transitions_2_per_pair": pairs_ok}
        failed |= not (sar_serial and pairs_ok)
    return failed


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_1911_05328_b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    r = sub.add_parser("run")
    r.add_argument("--algo", default="star")
    r.add_argument("--semiring", default="int")
    r.add_argument("--n", type=int, default=64)
    r.add_argument("--b", type=int, default=8)
    r.add_argument("--p", type=int, default=1)
    r.add_argument("--seed", type=int, default=1)
    r.add_argument("--mode", default="pooled")
    r.add_argument("--ksplit", type=int, default=None)
    bn = sub.add_parser("bench")
    bn.add_argument("--algos", default=",".join(CLASSICAL))
    bn.add_argument("--semiring", default="float")
    bn.add_argument("--n", default="2048")
    bn.add_argument("--b", type=int, default=64)
    bn.add_argument("--p", type=int, default=148)
    bn.add_argument("--reps", type=int, default=5)
    bn.add_argument("--seed", type=int, default=1)
    bn.add_argument("--out", default=None)
    v = sub.add_parser("verify")
    v.add_argument("--suite", default="all", choices=["correctness", "space", "pool", "all"])
    v.add_argument("--sabotage-lifo", action="store_true",
                   help="negative control: run with the device pool in FIFO order (must exit 1)")
    v.add_argument("--seeds", type=int, default=2)
    v.add_argument("--p", type=int, default=4)
    for name in ("analyze", "simulate"):
        sub.add_parser(name)
    args = ap.parse_args(argv)
    if hasattr(args, "p") and os.environ.get("STAR_MM_THREADS"):   # SPEC.md:552 overrides p
        args.p = int(os.environ["STAR_MM_THREADS"])
    if args.cmd in ("analyze", "simulate"):
        print(f"{args.cmd}: the analysis engine (recurrences, DAG, cache simulator) is out of "
              "scope for the B200 build (SURVEY.md §2)", file=sys.stderr)
        return EXIT_INVALID
    if args.cmd == "run" and args.algo not in ALGORITHMS:
        print(json.dumps({"status": "error", "error": "KeyError", "message": args.algo}))
        return EXIT_INVALID
    return {"run": cmd_run, "bench": cmd_bench, "verify": cmd_verify}[args.cmd](args)

