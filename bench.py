#!/usr/bin/env python
"""Benchmark: semiring MM ops/s (2n^3/t) on B200 -- BASELINE.json's metric.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--algo star]
  python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N
  python bench.py --impl reference ...     # the reference CPU path (oracle port)

Workload: one step = one STAR-MM C <- C (+) A (x) B
over the whole configured problem, inputs resident in HBM.  The default
workload is BASELINE config 4 (fp64 (+,x), n = 16384, A,B ~ N(0,1), C ~
U[-1,1)): the largest single-GPU config quoted at 1/2/4/8 B200 and the one
the >=70%-of-roofline target names (n >= 16384).  Configs 2, 3, 5 run with
--config; config 1 (n=256) is the parity gate, not a bench line.

Multi-GPU: 2D output tiling (pr x pc) and, for config 5, a k-split whose
partial minima are combined by one NCCL reduce-scatter; value = 2n^3 / max
over ranks of the device time.  Inputs are generated on device with torch's
Philox generator (same distributions as bench_configs.py; the tests use the
numpy generators) and are all larger than the 126 MB L2, so no explicit
flush is needed between steps.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np
import torch
import torch.distributed as dist

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

from bench_configs import CONFIGS, device_gen_spec, tolerance  # noqa: E402

# ---- roofline denominators ---------------------------
SM_COUNT_NOMINAL = 148


def _measured(name, key, default):
    p = os.path.join(REPO, "profiles", name)
    try:
        return json.load(open(p)).get(key, default)
    except Exception:
        return default


def _measured_peaks(key, default):
    """A figure from the driver-written MEASURED_PEAKS.json (repo root), else `default`."""
    try:
        return float(json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json"))).get(key, default))
    except Exception:
        return default


def _packed(op_prefix, default):
    p = os.path.join(REPO, "profiles", "r01_packed_ops_microbench.jsonl")
    try:
        for line in open(p):
            d = json.loads(line)
            if d["op"].startswith(op_prefix):
                return d["terms_per_s"]
    except Exception:
        pass
    return default


def peaks(sm_max_mhz: float):
    """Roofline denominators in ops/s (1 term = 2 ops), all measured on this pool's B200s
    (profiles/r01_*); 'issue' is BASELINE's nominal CUDA-core roofline."""
    dmma = 2 * _measured("r01_peaks_microbench.json", "dmma_terms_per_s_b8", 1.8551e13)
    cublas = 1e12 * _measured("r01_cublas_dgemm.json", "cublas_dgemm_n16384_tflops", 36.08)
    issue = SM_COUNT_NOMINAL * 128 * sm_max_mhz * 1e6          # BASELINE: 2 instr / term
    vmin = 2 * _measured("r01_peaks_microbench.json", "viaddmnmx_terms_per_s_b8", 1.8471e13)
    return {"fp64_tensor": max(dmma, cublas), "fp64_dmma_ubench": dmma, "cublas_dgemm": cublas,
            "issue": issue, "viaddmnmx_ubench": vmin,
            "idp4a_ubench": 2 * _packed("dp4a", 7.4066e13),
            "viaddmnmx_s16x2_ubench": 2 * _packed("viaddmnmx_s16x2", 3.6974e13),
            # library int8 GEMM on this pool (tools/int8_peak.py -> profiles/r01_int8_peak.json)
            "int8_tensor_burst": 1e12 * _measured("r01_int8_peak.json", "int_mm_n8192_burst_tops", 3053.9),
            "int8_tensor_sustained": 1e12 * _measured("r01_int8_peak.json", "int_mm_n16384_sustained_tops",
                                                      2061.5)}


# path -> (roofline key, instruction mix) for the dominant kernel
PATH_PEAK = {
    "dmma_f64": ("fp64_tensor", "DMMA.8x8x4 (FP64 tensor core)"),
    "simt_i64_dp4a": ("idp4a_ubench", "IDP.4A: 4 int8 terms per lane-op"),
    "simt_f32_s16x2_viaddmnmx": ("viaddmnmx_s16x2_ubench", "VIADDMNMX.S16x2: 2 terms per lane-op"),
    "simt_i32_s16x2_viaddmnmx": ("viaddmnmx_s16x2_ubench", "VIADDMNMX.S16x2: 2 terms per lane-op"),
    "tcgen05_i8_umma": ("int8_tensor", "tcgen05.mma.cta_group::2 kind::i8 (UTCIMMA.2CTA), s32 in TMEM"),
    "ozaki2_fp64_tcgen05_i8x16": ("int8_tensor", "16 x tcgen05.mma.cta_group::2 kind::i8 residue passes + "
                                  "exact CRT epilogue (Ozaki scheme II)"),
    "tcgen05_i8_radix256_int64": ("int8_tensor", "8 digit-group tcgen05.mma kind::i8 GEMMs per K chunk: "
                                  "36 signed radix-256 digit products per int64 term (mod 2^64)"),
}
INT8_PASSES = {"tcgen05_i8_umma": 1, "ozaki2_fp64_tcgen05_i8x16": 16, "tcgen05_i8_radix256_int64": 36}


# ---- clocks during the timed region ----------------------------------------
class ClockSampler:
    def __init__(self, device_index: int, period=0.2):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self._dev = device_index
        self._period = period
        self._t = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self._h = pynvml.nvmlDeviceGetHandleByIndex(self._dev)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
            self._nv = pynvml
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        except Exception as e:  # pragma: no cover
            self.error = str(e)
        return self

    def _run(self):
        nv = self._nv
        names = {
            "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4,
            "hw_slowdown": 0x8, "sync_boost": 0x10, "sw_thermal_slowdown": 0x20,
            "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80,
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for k, bit in names.items():
                    if r & bit and k != "gpu_idle":
                        self.reasons.add(k)
            except Exception:
                pass
            self._stop.wait(self._period)

    def __exit__(self, *exc):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "samples": len(self.samples),
                "reasons": sorted(self.reasons)}


# ---- device input generation -------------------------------------------------
def gen_panel(cid: int, what: str, rows: int, cols: int, r0: int, c0: int, device):
    """Rows [r0, r0+rows) x cols [c0, c0+cols) of the config's matrix `what`, generated on
    the device by the library's counter-based generator (paper_1911_05328_b200.generate):
    every rank makes exactly its own panels, no collective, and the oracle can regenerate
    any panel bit for bit (the post-run parity check does)."""
    from paper_1911_05328_b200 import generate_panel, get_semiring
    s = get_semiring(CONFIGS[cid]["semiring"])
    spec = device_gen_spec(cid, what)
    if spec == "zeros":
        return torch.zeros(rows, cols, dtype=s.torch_dtype, device=device)
    return generate_panel(s, rows=rows, cols=cols, row0=r0, col0=c0, device=device, **spec)


def host_panel(cid: int, what: str, rows: int, cols: int, r0: int, c0: int):
    """The same panel regenerated on the host by the oracle's restatement (checker only)."""
    from oracle import oracle as O
    sr = O.SR_BY_NAME[CONFIGS[cid]["semiring"]]
    spec = device_gen_spec(cid, what)
    if spec == "zeros":
        return np.zeros((rows, cols), dtype=O.DTYPES[sr])
    spec = dict(spec)
    spec["stream"] = spec.pop("stream_id")
    return O.generate(sr, rows=rows, cols=cols, row0=r0, col0=c0, **spec)


def parity_check(cid: int, n: int, out: torch.Tensor, lo: int, hi: int, c0: int, c1: int,
                 rank: int, tiles: int = 8):
    """Seeded random output tiles of this rank's reduced rows [lo, hi) x [c0, c1),
    recomputed on the host from regenerated panels: fold_add(C0[tile], A[rows, :] (x)
    B[:, cols]) over the FULL k range.  Bit-exact for integer and
    (min,+) configs, rel 1e-10*sqrt(n) for fp64."""
    from oracle import oracle as O
    sr = O.SR_BY_NAME[CONFIGS[cid]["semiring"]]
    tol = tolerance(cid, n)
    rng = np.random.default_rng(7919 + rank)
    worst, ok, checked = 0.0, True, 0
    t0 = time.perf_counter()
    for _ in range(tiles):
        if hi <= lo or c1 <= c0:
            break
        i0 = int(rng.integers(lo, max(lo + 1, hi - 127)))
        j0 = int(rng.integers(c0, max(c0 + 1, c1 - 127)))
        r, c = min(128, hi - i0), min(128, c1 - j0)
        want = host_panel(cid, "C", r, c, i0, j0)
        O.gemm_fold(sr, want, host_panel(cid, "A", r, n, i0, 0), host_panel(cid, "B", n, c, 0, j0), par=True)
        got = out[i0 - lo:i0 - lo + r, j0 - c0:j0 - c0 + c].cpu().numpy()
        if tol == 0.0:
            u = {8: np.uint64, 4: np.uint32}[got.dtype.itemsize]
            same = (got.view(u) == want.view(u))
            if got.dtype.kind == "f":
                same |= np.isnan(got) & np.isnan(want)
            ok &= bool(same.all())
        else:
            err = np.abs(got - want) / np.maximum(1.0, np.maximum(np.abs(got), np.abs(want)))
            worst = max(worst, float(err.max()))
            ok &= bool((err <= tol).all())
        checked += 1
    return {"ok": bool(ok), "tiles": checked, "tile": 128, "rule": "bitwise" if tol == 0.0 else
            f"rel {tol:.3g}", "max_rel_err": worst if tol else 0.0,
            "checker": "oracle/starmm_oracle.c on host-regenerated panels",
            "seconds": round(time.perf_counter() - t0, 2)}


# ---- the reference's own CPU path (UNMODIFIED package under baseline/_ref) ----------
def reference_package():
    """Import the reference package installed (unmodified) into baseline/_ref -- git-ignored,
    it travels to the GPU box with the snapshot.  None when absent."""
    path = os.path.join(REPO, "baseline", "_ref")
    if not os.path.isdir(os.path.join(path, "starmm")):
        return None
    os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join("/tmp", "starmm_ref_numba_cache"))
    sys.dont_write_bytecode = True
    if path not in sys.path:
        sys.path.insert(0, path)
    import starmm  # noqa: E402
    return starmm


def reference_star_sample(cid: int, target_s: float, steps: int = 1, warmup: int = 1, workers=None):
    """The reference's public star_mm (classic.py:314-316) under Config(base_dim=b,
    workers=W) (runtime.py:60-79, numba leaf kernels semiring.py:22-60), W = all host
    threads, on the config's distributions at the largest power-of-two n <= the config's
    whose step fits `target_s` (a bounded sample: the reference is GIL-bound at 1-4 Gop/s,
    config 4 would take ~1 h per step).  Returns a dict or None."""
    ref = reference_package()
    if ref is None:
        return None
    from bench_configs import make_inputs, to_reference
    cfg = CONFIGS[cid]
    s = ref.get_semiring(cfg["ref_semiring"])
    W = workers or os.cpu_count() or 1
    b = cfg["b"]

    def inputs(n):
        A, B, C = make_inputs(cid, n)
        Am = ref.Matrix(to_reference(cid, A), s)
        Bm = Am if B is A else ref.Matrix(to_reference(cid, B), s)
        return Am, Bm, to_reference(cid, C).copy()

    def run(n, Am, Bm, C0, reps):
        ts = []
        for _ in range(reps):
            C = ref.Matrix(C0.copy(), s)
            t0 = time.perf_counter()
            ref.star_mm(C, Am, Bm, s, ref.Config(base_dim=b, workers=W))
            ts.append(time.perf_counter() - t0)
        return ts

    Am, Bm, C0 = inputs(2 * b)
    run(2 * b, Am, Bm, C0, 1)                      # numba JIT (cached under NUMBA_CACHE_DIR)
    n = 512
    Am, Bm, C0 = inputs(n)
    t = run(n, Am, Bm, C0, 1)[0]
    while 2 * n <= cfg["n"] and t * 8 <= target_s:  # a step costs ~8x per doubling
        n *= 2
        t *= 8
    Am, Bm, C0 = inputs(n)
    if warmup:
        run(n, Am, Bm, C0, warmup)
    ts = run(n, Am, Bm, C0, steps)
    tm = sum(ts) / len(ts)
    return {"value": 2.0 * n ** 3 / tm / 1e12, "unit": "Tops/s", "cores": W, "kind": "reference",
            "n": n, "seconds_per_step": tm,
            "sample": f"reference star_mm (baseline/_ref, unmodified) n={n} b={b} workers={W}, "
                      f"{cfg['ref_semiring']} semiring on config {cid}'s distributions"}


def cpu_baseline(cid, n, device, port_seconds):
    """cpu_baseline of the bench line (rank 0, N=1): the reference's own star_mm on a
    bounded sample, plus the oracle port (C, all threads) on a row panel of the full
    problem as a second figure, plus the committed largest-n sweep if present."""
    Ah, Bh = host_panels_for_baseline(cid, n, device)
    v, desc, cores, secs = cpu_sample(cid, Ah, Bh, port_seconds)
    port = {"value": v / 1e12, "unit": "Tops/s", "cores": cores, "kind": "port",
            "sample": desc + f" ({secs:.1f} s), oracle/starmm_oracle.c"}
    ref = reference_star_sample(cid, target_s=8.0)
    sweep = None
    sp = os.path.join(REPO, "profiles", "r02_ref_cpu_sweep.json")
    if os.path.exists(sp):
        try:
            sweep = {"file": "profiles/r02_ref_cpu_sweep.json",
                     "largest_n": json.load(open(sp)).get("largest_n")}
        except Exception:
            sweep = None
    if ref is None:
        port["reference"] = "baseline/_ref not installed"
        return port
    ref["port"] = port
    if sweep:
        ref["sweep"] = sweep
    return ref


# ---- CPU baseline (the reference path's oracle port) --------------------------
def cpu_sample(cid: int, A_host_rows, B_host, target_s: float):
    """Time the oracle port (oracle/starmm_oracle.c, all host threads) on a bounded
    row panel: rows x n x n terms.  Returns (ops_per_s, desc, cores, seconds)."""
    from oracle import oracle as O
    sr = O.SR_BY_NAME[CONFIGS[cid]["semiring"]]
    n = B_host.shape[0]
    cores = O.num_threads()
    rows = min(cores, A_host_rows.shape[0])
    C = np.zeros((rows, B_host.shape[1]), dtype=B_host.dtype)
    t0 = time.perf_counter()
    O.gemm_fold(sr, C, np.ascontiguousarray(A_host_rows[:rows]), B_host, par=True)
    t = time.perf_counter() - t0
    want = max(rows, min(A_host_rows.shape[0], int(rows * target_s / max(t, 1e-3)) // cores * cores))
    if want > rows:
        rows = want
        C = np.zeros((rows, B_host.shape[1]), dtype=B_host.dtype)
        t0 = time.perf_counter()
        O.gemm_fold(sr, C, np.ascontiguousarray(A_host_rows[:rows]), B_host, par=True)
        t = time.perf_counter() - t0
    ops = 2.0 * rows * n * B_host.shape[1]
    return ops / t, f"{rows}x{n} (x) {n}x{B_host.shape[1]} row panel of config {cid}", cores, t


def host_panels_for_baseline(cid, n, device):
    """A row panel and the full B on the host (the oracle's inputs)."""
    rows = min(n, 4096)
    A = gen_panel(cid, "A", rows, n, 0, 0, device).cpu().numpy()
    B = gen_panel(cid, "B", n, n, 0, 0, device).cpu().numpy()
    return A, B


# ---- main -------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=4, choices=[2, 3, 4, 5])
    ap.add_argument("--algo", default="star", choices=["co2", "co3", "tar", "sar", "star"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--size", type=int, default=None, help="override n (smoke runs only)")
    ap.add_argument("--ksplit-gpus", type=int, default=None)
    ap.add_argument("--combine", default="fused", choices=["fused", "nccl"],
                    help="k-split combine across GPUs (only when the grid has ks > 1)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--int-tensor", action="store_true",
                    help="opt-in: small-range int64 on tcgen05 kind::i8 (config 2; DESIGN.md §5c)")
    ap.add_argument("--fp64-emu", action="store_true",
                    help="opt-in: fp64 (+,x) as Ozaki-II over 16 int8 tcgen05 GEMMs (config 4; DESIGN.md §5d)")
    ap.add_argument("--no-opt-in", action="store_true",
                    help="skip the secondary measurement of the opt-in tensor-core path")
    ap.add_argument("--no-fastpath", action="store_true",
                    help="the general (unguarded) kernels: int64 64-bit MAD, fp32 / int32 / fp64 "
                         "(min,+) without the range-guarded narrow encodings (DESIGN.md §7)")
    ap.add_argument("--parity-tiles", type=int, default=8,
                    help="sampled output tiles each rank checks against the oracle after timing")
    ap.add_argument("--ref-step-seconds", type=float, default=8.0,
                    help="--impl reference: target seconds per star_mm step (sets its n)")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: plumbing check with several ranks on fewer GPUs (timings invalid)")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return reference_arm(args, world, rank)

    local_rank = local_rank % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local_rank)
    device = torch.device("cuda", local_rank)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=device)
        else:
            dist.init_process_group("gloo")

    import paper_1911_05328_b200 as sm
    from paper_1911_05328_b200 import _lib
    from paper_1911_05328_b200.distributed import DistributedMM, choose_grid, ks_groups

    cid = args.config
    cfg = CONFIGS[cid]
    n = args.size or cfg["n"]
    s = sm.get_semiring(cfg["semiring"])
    ks = args.ksplit_gpus or (2 if (cid == 5 and world >= 8) else 1)
    grid = choose_grid(world, ks)
    group_ks = ks_groups(grid) if world > 1 else None
    sms = torch.cuda.get_device_properties(device).multi_processor_count
    dmm = DistributedMM(n, s, grid, rank, algo=args.algo, base_dim=cfg["b"], workers=sms,
                        group_ks=group_ks, device=local_rank, time_kernel=True,
                        combine=args.combine, int_tensor=args.int_tensor, fp64_emu=args.fp64_emu,
                        fastpath=not args.no_fastpath, async_exec=True)

    # ---- input distribution: each rank generates its own panels on its device ----
    # (counter-based, no collective: DESIGN.md §8c); timed separately from the steps
    for w in ("A", "B", "C"):          # load the generator's kernels before timing it
        gen_panel(cid, w, 1, 1, 0, 0, device)
    torch.cuda.synchronize()
    g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    g0.record()
    A = gen_panel(cid, "A", dmm.m, dmm.k, dmm.r0, dmm.k0, device)
    B = A if (cid in (3, 5) and dmm.r0 == dmm.k0 and dmm.m == dmm.k and dmm.c0 == dmm.k0
              and dmm.nn == dmm.k) else gen_panel(cid, "B", dmm.k, dmm.nn, dmm.k0, dmm.c0, device)

    def fresh_c():
        # every k-split member holds C0 of its (I, J) block (the owner folds it once)
        return gen_panel(cid, "C", dmm.m, dmm.nn, dmm.r0, dmm.c0, device)

    C = fresh_c()
    g1.record()
    torch.cuda.synchronize()
    dist_ms = torch.tensor([g0.elapsed_time(g1)], dtype=torch.float64, device=device)
    if world > 1:
        dist.all_reduce(dist_ms, op=dist.ReduceOp.MAX)
    gen_bytes = (A.numel() + (0 if B is A else B.numel()) + C.numel()) * A.element_size()

    def step():
        dmm.step(C, A, B)

    import time as _time
    torch.cuda.synchronize()
    _w0 = _time.perf_counter()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    warm_s = (_time.perf_counter() - _w0) / max(1, args.warmup)
    # NVML sampling period: ~20 samples over the timed region, between 5 and 200 ms (polling
    # at 100 Hz cost config 4 0.25%; a fixed 200 ms gave config 2's 12-24 ms region 1 sample)
    clk_period = min(0.2, max(0.005, warm_s * args.steps / 20.0))
    dmm.plan.reset_stats()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank, clk_period) as clk:
        e0.record()
        for _ in range(args.steps):
            step()
        e1.record()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t_local = e0.elapsed_time(e1) / 1e3 / args.steps
    st = dmm.plan.stats()
    kern_s_local = st["main_kernel_ns"] / 1e9 / max(1, st["main_kernel_launches"])
    tt = torch.tensor([t_local, kern_s_local], dtype=torch.float64, device=device)
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    t_step, kern_s = float(tt[0]), float(tt[1])
    total_ops = 2.0 * n ** 3
    value = total_ops / t_step

    # ---- e2e through the public API with pinned host buffers ----
    e2e = None
    if not args.no_e2e:
        e2e = e2e_run(args, sm, s, cid, dmm, A, B, C, device, world, grid, group_ks)

    # ---- parity of this run: one more (untimed) step from a fresh C0, then sampled
    # tiles of this rank's reduced rows against the oracle on regenerated panels ----
    parity = None
    if args.parity_tiles > 0:
        C = fresh_c()
        out = dmm.step(C, A, B)
        torch.cuda.synchronize()
        lo, hi = dmm.owned_rows()
        parity = parity_check(cid, n, out, lo, hi, dmm.c0, dmm.c1, rank, args.parity_tiles)
        if world > 1:
            pt = torch.tensor([0 if parity["ok"] else 1, parity["tiles"]], dtype=torch.float64, device=device)
            dist.all_reduce(pt, op=dist.ReduceOp.SUM)
            parity["ok"] = bool(pt[0] == 0)
            parity["tiles"] = int(pt[1])
            parity["ranks"] = world

    # ---- roofline of the dominant kernel ----
    clocks = clk.summary()
    pk = peaks(clocks["sm_max_mhz"] or 1965.0)
    roof, mix = roofline(pk, st["path_name"], 2.0 * dmm.m * dmm.nn * dmm.k, kern_s)
    # the committed ncu capture is of the full-size single-GPU launch: no figure for a
    # sharded (N > 1) or size-overridden launch
    roof["traffic"] = _ncu_traffic(cid, st["path_name"]) if (world == 1 and args.size is None) else None
    roof["kernel_share_of_step"] = kern_s / t_step

    # ---- the opt-in tensor-core path of this config, measured as a secondary line ----
    opt_in = None
    if world == 1 and not args.no_opt_in and not (args.fp64_emu or args.int_tensor) and cid in (2, 4):
        opt_in = opt_in_run(args, s, cid, n, grid, rank, sms, local_rank, A, B, C, pk)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(cid, n, device, args.cpu_seconds)

    if rank == 0:
        line = {
            "metric": "semiring MM ops/s (2n^3/t)", "value": value / 1e12, "unit": "Tops/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": t_step * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None,
            "dtype": {"float": "f64", "int": "int64", "tropical_f32": "f32",
                      "tropical_i32": "int32"}[s.id],
            "data": "synthetic (library generator: Philox4x32-10 per element, BASELINE config distributions)",
            "config": {"workload": cfg["name"] + ("_general_kernels" if args.no_fastpath else ""),
                       "baseline_config": cid, "n": n, "semiring": s.id,
                       "algo": args.algo, "base_dim": cfg["b"], "workers": sms,
                       "grid": [grid.pr, grid.pc, grid.ks], "path": st["path_name"],
                       "fastpath": not args.no_fastpath,
                       "combine": dmm.combine_mode if grid.ks > 1 else "none",
                       "ksplit_per_tile": st["ksplit"], "l2": "inputs larger than L2 (no flush)"},
            "parity": parity,
            "distribution": {"ms": float(dist_ms[0]), "bytes_per_rank": int(gen_bytes),
                             "method": "counter-based device generation of each rank's own "
                                       "A/B/C panels (generate_panel), no collective; max over ranks"},
            "roofline": roof,
            "opt_in_tensor_path": opt_in,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(st["kernel_launches"]) * args.steps,
            "clocks": clocks,
        }
        print(json.dumps(line))
    dmm.close()
    if world > 1:
        dist.destroy_process_group()


def roofline(pk, path, local_ops, kern_s):
    achieved = local_ops / kern_s
    key, mix = PATH_PEAK.get(path, ("issue", "1 lane-op per term (FADD2+FMNMX3 / "
                                          "VIADDMNMX / IMAD), 64 terms/clk/SM"))
    if key == "int8_tensor":
        passes = INT8_PASSES[path]
        # denominator: the larger of cuBLASLt's measured int8 burst (profiles/r01_int8_peak.json)
        # and twice MEASURED_PEAKS.json's dense bf16 burst (int8 issues at 2x bf16); our
        # long kernels outrun cuBLASLt's power-capped SUSTAINED figure, so that one is not
        # a ceiling.  NVIDIA's nominal dense int8 (4.5 POPS) is reported beside it.
        bf16 = 2e12 * _measured_peaks("bf16_tflops", 1664.4)
        peak = max(pk["int8_tensor_burst"], bf16)
        roof = {"bound": "tensor", "achieved": passes * achieved / 1e12, "peak": peak / 1e12,
                "unit": "int8 Tops/s", "peak_source": "max(measured cuBLASLt int8 burst n=8192 "
                "(profiles/r01_int8_peak.json), 2 x MEASURED_PEAKS.json bf16_tflops)",
                "nominal_dense_int8": 4500.0, "int8_ops_per_semiring_op": passes}
        if path == "ozaki2_fp64_tcgen05_i8x16":
            roof["emulated_fp64_tflops"] = achieved / 1e12
            roof["vs_fp64_tensor_peak"] = achieved / pk["fp64_tensor"]
        if path == "tcgen05_i8_radix256_int64":
            roof["vs_cuda_core_general_int64"] = "7.0 Tops/s (simt_i64, profiles/r02e_bench_c2_general.json)"
    elif key == "fp64_tensor":
        roof = {"bound": "tensor", "achieved": achieved / 1e12, "peak": pk[key] / 1e12,
                "unit": "TFLOP/s", "peak_source": "measured: max(DMMA.8x8x4 ubench, cuBLAS DGEMM) "
                "profiles/r01_peaks_microbench.json, r01_cublas_dgemm.json (MEASURED_PEAKS.json "
                "has no fp64 entry)"}
    else:
        roof = {"bound": "issue", "achieved": achieved / 1e12, "peak": pk[key] / 1e12,
                "unit": "Tops/s", "peak_source": ("measured instruction-mix peak, "
                "profiles/r01_packed_ops_microbench.jsonl / r01_peaks_microbench.json"
                if key != "issue" else "BASELINE issue roofline: 148 SMs x 128 lanes x sm_max_mhz")}
        roof["baseline_issue_roofline"] = pk["issue"] / 1e12
        roof["frac_of_baseline_issue_roofline"] = achieved / pk["issue"]
    roof["instruction_mix"] = mix
    roof["frac"] = roof["achieved"] / roof["peak"]
    roof["kernel_ms"] = kern_s * 1e3
    return roof, mix


def opt_in_run(args, s, cid, n, grid, rank, sms, local_rank, A, B, C, pk):
    """Secondary measurement (N=1) of the config's OPT-IN tensor-core path: int64 on
    tcgen05 kind::i8 (config 2) or fp64 via Ozaki-II (config 4).  Same inputs, own
    copy of C, same timing rules; the headline line above stays the default path."""
    from paper_1911_05328_b200.distributed import DistributedMM
    cfg = CONFIGS[cid]
    dmm = DistributedMM(n, s, grid, rank, algo=args.algo, base_dim=cfg["b"], workers=sms,
                        device=local_rank, time_kernel=True, combine=args.combine,
                        int_tensor=(cid == 2), fp64_emu=(cid == 4), async_exec=True)
    C2 = C.clone()
    steps, warm = max(1, min(args.steps, 3)), max(1, min(args.warmup, 2))
    for _ in range(warm):
        dmm.step(C2, A, B)
    torch.cuda.synchronize()
    dmm.plan.reset_stats()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        dmm.step(C2, A, B)
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 1e3 / steps
    st = dmm.plan.stats()
    kern_s = st["main_kernel_ns"] / 1e9 / max(1, st["main_kernel_launches"])
    roof, _ = roofline(pk, st["path_name"], 2.0 * n ** 3, kern_s)
    dmm.close()
    del C2
    return {"flag": "--fp64-emu" if cid == 4 else "--int-tensor", "path": st["path_name"],
            "value": 2.0 * n ** 3 / t / 1e12, "unit": "Tops/s", "ms_per_step": t * 1e3, "steps": steps,
            "roofline": roof, "note": "opt-in (DESIGN.md §5c/§5d); exactness / error bound in "
            "tests/test_gpu_fp64_emulation.py and test_gpu_parity.py"}


def _ncu_traffic(cid, path):
    p = os.path.join(REPO, "profiles", "ncu_traffic.json")
    try:
        return json.load(open(p)).get(f"{cid}:{path}")
    except Exception:
        return None


def e2e_run(args, sm, s, cid, dmm, A, B, C, device, world, grid, group_ks):
    """Public-API end to end with pinned HOST buffers, every step: N=1 goes through
    host_mm-style Executor.execute_host (starmm_execute_host streams row blocks, copies
    overlapped with the tile kernels); N>1 runs DistributedMM.step_host on each rank's
    pinned panels (the same overlapped host path without a k-split; with one, the
    panels go up, the combine runs on the device and the owned rows come back)."""
    Ah = A.cpu().pin_memory()
    Bh = Ah if B is A else B.cpu().pin_memory()
    Ch0 = C.cpu().pin_memory()
    Ch = Ch0.clone().pin_memory()
    cfg = sm.Config(base_dim=CONFIGS[cid]["b"], workers=torch.cuda.get_device_properties(device)
                    .multi_processor_count, allow_nonpow2=True, int_tensor_cores=args.int_tensor,
                    fp64_emulation=args.fp64_emu)
    ex = sm.Executor(cfg) if world == 1 else None
    out = None
    if world > 1:
        lo, hi = dmm.owned_rows()
        out = torch.empty((hi - lo, dmm.nn), dtype=Ch.dtype).pin_memory()

    def one():
        if world == 1:
            ex.execute_host(args.algo, Ch, Ah, Bh, s)
        else:
            dmm.step_host(Ch, Ah, Bh, out)

    one()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    steps = max(1, min(args.steps, 3))
    t0 = time.perf_counter()   # host-side API with internal streams: wall time of the blocking call
    for _ in range(steps):
        one()
    torch.cuda.synchronize()
    t = torch.tensor([(time.perf_counter() - t0) / steps], dtype=torch.float64, device=device)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if ex is not None:
        ex.close()
    es = Ah.element_size()
    c_up = Ch.numel()
    if world > 1 and dmm.combine_mode == "fused":     # only the owner's C0 rows go up
        lo, hi = dmm.owned_rows()
        c_up = (hi - lo) * dmm.nn
    h2d = (Ah.numel() + (0 if Bh is Ah else Bh.numel()) + c_up) * es
    d2h = (Ch.numel() if world == 1 else out.numel()) * es
    return {"value": 2.0 * dmm.n ** 3 / float(t[0]) / 1e12, "unit": "Tops/s",
            "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
            "steps": steps, "timer": "host wall clock around the blocking API call",
            "api": "Executor.execute_host (starmm_execute_host: pinned host C, A, B)" if world == 1
            else "DistributedMM.step_host with per-rank pinned panels"}


def reference_arm(args, world, rank):
    """--impl reference: the reference's OWN CPU implementation of the path -- the
    unmodified package in baseline/_ref, public star_mm -- on the box's host cores,
    rank 0 only (other ranks exit 0), same metric and config; each step is one star_mm
    at the largest power-of-two n whose step fits --ref-step-seconds (the reference is
    GIL-bound; config 4's n=16384 would take about an hour per step).  Without the
    installed package, the oracle port (C restatement, all threads) on a row panel."""
    if rank != 0:
        return
    cid = args.config
    cfg = CONFIGS[cid]
    n = args.size or cfg["n"]
    dtype = {"float": "f64", "int": "int64", "tropical_f32": "f32", "tropical_i32": "int32"}[cfg["semiring"]]
    line = {"metric": "semiring MM ops/s (2n^3/t)", "unit": "Tops/s", "impl": "reference",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": dtype,
            "data": "synthetic (numpy PCG64, BASELINE config distributions)",
            "config": {"workload": cfg["name"], "baseline_config": cid, "n": n,
                       "semiring": cfg["semiring"], "algo": "star"}}
    res = reference_star_sample(cid, args.ref_step_seconds, steps=max(1, args.steps),
                                warmup=args.warmup)
    if res is not None:
        v = res["value"]
        line.update({"value": v, "ms_per_step": res["seconds_per_step"] * 1e3})
        line["config"]["reference_n"] = res["n"]
        line["cpu_baseline"] = {k: res[k] for k in ("value", "unit", "cores", "kind", "sample")}
    else:
        v, t, desc, cores = _port_arm(args, cid, n)
        line.update({"value": v, "ms_per_step": t * 1e3})
        line["cpu_baseline"] = {"value": v, "unit": "Tops/s", "cores": cores, "kind": "port",
                                "sample": desc + " (baseline/_ref absent)"}
    line["e2e"] = {"value": line["value"], "unit": "Tops/s", "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}
    print(json.dumps(line))


def _port_arm(args, cid, n):
    """The oracle port on a row panel per step (all host threads); returns
    (Tops/s, seconds per step, description, cores)."""
    from oracle import oracle as O
    cfg = CONFIGS[cid]
    rng = np.random.default_rng(cfg["seed"])
    dt = cfg["dtype"]
    if cid == 4:
        Ar = rng.standard_normal((256, n))
        B = rng.standard_normal((n, n))
    elif cid == 2:
        Ar = rng.integers(-16, 17, (256, n), dtype=np.int64)
        B = rng.integers(-16, 17, (n, n), dtype=np.int64)
    elif cid == 3:
        B = rng.integers(1, 101, (n, n), dtype=np.int32).astype(np.float32)
        B[rng.random((n, n), dtype=np.float32) >= 0.1] = np.inf
        np.fill_diagonal(B, 0.0)
        Ar = B[:256]
    else:
        B = rng.integers(1, 10 ** 6 + 1, (n, n), dtype=np.int32)
        np.fill_diagonal(B, 0)
        Ar = B[:256]
    Ar = np.ascontiguousarray(Ar.astype(dt))
    B = np.ascontiguousarray(B.astype(dt))
    sr = O.SR_BY_NAME[cfg["semiring"]]
    cores = O.num_threads()
    rows = cores
    C = np.zeros((rows, n), dtype=dt)
    t0 = time.perf_counter()
    O.gemm_fold(sr, C, Ar[:rows], B, par=True)
    t1 = time.perf_counter() - t0
    rows = int(max(cores, min(Ar.shape[0], rows * 2.0 / max(t1, 1e-3))) // cores * cores)
    C = np.zeros((rows, n), dtype=dt)
    for _ in range(args.warmup):
        O.gemm_fold(sr, C, Ar[:rows], B, par=True)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        O.gemm_fold(sr, C, Ar[:rows], B, par=True)
    t = (time.perf_counter() - t0) / args.steps
    return (2.0 * rows * n * n / t / 1e12, t,
            f"{rows}x{n} (x) {n}x{n} row panel per step, oracle/starmm_oracle.c", cores)


if __name__ == "__main__":
    main()
