"""GPU parity: the CUDA path (through the C ABI, via the drop-in API) vs the
reference's golden outputs and the pinned CPU oracle.

Bar: bit-exact for int64 (+,x) and every (min,+) semiring; float64 (+,x)
within the relative tolerance of matrices_equal (matrix.py:182-193) -- 1e-9
for the SPEC property tests, 1e-12 for PR1 (BASELINE config 1),
1e-10*sqrt(n) for config 4.  FMA (DMMA) rounding is why fp64 is not bitwise.
"""
import os

import numpy as np
import pytest
from _bits import same_bits, diff_count  # noqa: F401
import torch

import paper_1911_05328_b200 as sm
from oracle import oracle as O
from _host_schedule import host_phase1

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden")
SMALL = np.load(os.path.join(GOLD, "ref_small.npz"))
CASES = [(2, 2), (2, 8), (4, 16), (8, 32), (32, 64)]
ALGOS = {"co2": sm.co2, "co3": sm.co3, "tar": sm.tar_mm, "sar": sm.sar_mm, "star": sm.star_mm}
SR_OF = {"int": O.SR_INT64, "float": O.SR_FP64, "tropical": O.SR_TROP_F64,
         "tropical_f32": O.SR_TROP_F32, "tropical_i32": O.SR_TROP_I32}


def run(algo, s, C0, A, B, cfg, mode=None):
    C, Am, Bm = sm.Matrix(C0, s), sm.Matrix(A, s), sm.Matrix(B, s)
    if mode is None:
        ALGOS[algo](C, Am, Bm, s, cfg)
    else:
        ALGOS[algo](C, Am, Bm, s, cfg, mode=mode)
    return C.numpy()


def assert_match(sid, got, want, tol=1e-9):
    if sid == "float":
        bound = tol * np.maximum(1.0, np.maximum(np.abs(got), np.abs(want)))
        assert np.all(np.abs(got - want) <= bound), float(np.max(np.abs(got - want)))
    else:
        assert same_bits(got, want)


# ---- the reference's own fixtures, every schedule -------------------------
@pytest.mark.parametrize("algo", list(ALGOS))
@pytest.mark.parametrize("sid", ["int", "float", "tropical"])
@pytest.mark.parametrize("b,n", CASES)
@pytest.mark.parametrize("workers", [1, 16])
def test_schedules_vs_reference_golden(algo, sid, b, n, workers):
    key = f"{sid}_n{n}_b{b}"
    s = sm.get_semiring(sid)
    got = run(algo, s, SMALL[key + "_C0"], SMALL[key + "_A"], SMALL[key + "_B"],
              sm.Config(base_dim=b, workers=workers))
    assert_match(sid, got, SMALL[f"{key}_{algo}"])


@pytest.mark.parametrize("algo", ["co2", "co3", "tar", "sar", "star"])
@pytest.mark.parametrize("ksplit", [0, 1, 2, 3])
@pytest.mark.parametrize("sid", ["int", "float", "tropical", "tropical_f32", "tropical_i32"])
def test_split_protocols_vs_oracle(algo, ksplit, sid):
    """Force k-splits so every write-back protocol (fold / store+merge / atomic /
    pair+lock) runs, at a size with several tiles and a ragged edge."""
    n = 256
    s = sm.get_semiring(sid)
    rng = np.random.default_rng(ksplit * 10 + len(algo))
    if sid in ("int",):
        A = rng.integers(-50, 50, (n, n)).astype(np.int64)
        B = rng.integers(-50, 50, (n, n)).astype(np.int64)
        C0 = rng.integers(-50, 50, (n, n)).astype(np.int64)
    elif sid == "float":
        A, B, C0 = rng.standard_normal((n, n)), rng.standard_normal((n, n)), rng.standard_normal((n, n))
    else:
        A = rng.integers(0, 100, (n, n)).astype(s.dtype)
        B = rng.integers(0, 100, (n, n)).astype(s.dtype)
        C0 = rng.integers(0, 400, (n, n)).astype(s.dtype)
        inf = O.I32_INF if sid == "tropical_i32" else np.inf
        A[rng.random(A.shape) < 0.2] = inf
        B[rng.random(B.shape) < 0.2] = inf
    want = C0.copy()
    O.gemm_fold(SR_OF[sid], want, A, B)
    cfg = sm.Config(base_dim=16, workers=4, ksplit=ksplit)
    got = run(algo, s, C0, A, B, cfg)
    assert_match(sid, got, want)


# ---- SPEC oracle-equality property and determinism --
@pytest.mark.parametrize("algo", list(ALGOS))
@pytest.mark.parametrize("sid", ["int", "float", "tropical"])
def test_spec_oracle_equality_property(algo, sid):
    """Every algorithm, n in {b, 2b, 4b, 8b, 16b}, 10 seeds: int / tropical exact,
    float within rel 1e-9 (matrices_equal), against the pinned oracle."""
    b = 8
    s = sm.get_semiring(sid)
    for n in (b, 2 * b, 4 * b, 8 * b, 16 * b):
        for seed in range(10):
            rng = np.random.default_rng(1000 * n + seed)
            if sid == "int":
                A, B, C0 = (rng.integers(-100, 100, (n, n)).astype(np.int64) for _ in range(3))
            elif sid == "float":
                A, B, C0 = (rng.uniform(-1, 1, (n, n)) for _ in range(3))
            else:
                A, B, C0 = (rng.integers(0, 50, (n, n)).astype(np.float64) for _ in range(3))
                A[rng.random(A.shape) < 0.1] = np.inf
            want = C0.copy()
            O.gemm_fold(SR_OF[sid], want, A, B)
            got = run(algo, s, C0, A, B, sm.Config(base_dim=b, workers=1 + seed % 4 * 5))
            assert_match(sid, got, want)


@pytest.mark.parametrize("sid", ["int", "tropical", "tropical_f32", "tropical_i32"])
@pytest.mark.parametrize("algo,ksplit", [("tar", 3), ("sar", 3), ("star", 3), ("co3", 2), ("star", None)])
def test_integer_and_minplus_results_deterministic(sid, algo, ksplit):
    """Integer and (min,+) values do not depend on the concurrent schedule: repeated
    runs with concurrent k-slices (atomics, pair states) give identical bits."""
    n = 384
    s = sm.get_semiring(sid)
    rng = np.random.default_rng(7)
    A = rng.integers(-60 if sid == "int" else 0, 60, (n, n)).astype(s.dtype)
    B = rng.integers(-60 if sid == "int" else 0, 60, (n, n)).astype(s.dtype)
    C0 = rng.integers(0, 200, (n, n)).astype(s.dtype)
    cfg = sm.Config(base_dim=32, workers=148, ksplit=ksplit, allow_nonpow2=True)
    outs = [run(algo, s, C0, A, B, cfg) for _ in range(4)]
    for o in outs[1:]:
        assert same_bits(o.view(np.uint8), outs[0].view(np.uint8))


@pytest.mark.parametrize("sid", ["int", "tropical_i32"])
@pytest.mark.parametrize("algo", ["tar", "star"])
@pytest.mark.parametrize("store", [False, True])
def test_balanced_slices_exact(sid, algo, store):
    """Balanced (stream-K) k-slices: at n = 2560 (400 tiles = 1.35 waves of 296 CTAs)
    the planner spreads the flattened (tile, k-stage) space evenly; tiles shared by
    two CTAs merge with the atomic-madd.  Exact vs the oracle, with C folded or
    overwritten (STARMM_F_INIT_IDENTITY), and identical bits with the mode disabled."""
    n = 2560
    s = sm.get_semiring(sid)
    rng = np.random.default_rng(33)
    lo, hi = (0, 10 ** 5) if sid == "tropical_i32" else (-16, 17)
    A = rng.integers(lo, hi, (n, n)).astype(s.dtype)
    B = rng.integers(lo, hi, (n, n)).astype(s.dtype)
    C0 = rng.integers(lo, hi, (n, n)).astype(s.dtype)
    want = (np.full((n, n), O.I32_INF, np.int32) if sid == "tropical_i32" else
            np.zeros((n, n), np.int64)) if store else C0.copy()
    O.gemm_fold(SR_OF[sid], want, A, B, par=True)
    outs = []
    for disable in ("0", "1"):
        os.environ["STARMM_NO_BALANCED"] = disable
        try:
            C = torch.from_numpy(C0.copy()).cuda()
            with sm.Executor(sm.Config(base_dim=64, workers=148, allow_nonpow2=True)) as ex:
                st = ex.execute(algo, C, torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), s,
                                flags=0x4 if store else 0)
            assert (st["balanced_workers"] > 0) == (disable == "0"), st
            outs.append(C.cpu().numpy())
        finally:
            del os.environ["STARMM_NO_BALANCED"]
    assert same_bits(outs[0], want)
    assert same_bits(outs[1], want)


@pytest.mark.parametrize("sid", ["float", "int"])
def test_spec_soft_throughput_gate(sid):
    """SPEC.md:568's soft gate on the schedules, GPU analogue: at n = 2048, b = 64 and
    >= 8 workers, TAR <= 1.15 x CO2 and SAR <= 1.15 x CO3 (median of 7 timed runs)."""
    n = 2048
    s = sm.get_semiring(sid)
    g = torch.Generator(device="cuda").manual_seed(5)
    if sid == "float":
        A = torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g)
        B = torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g)
    else:
        A = torch.randint(-16, 17, (n, n), dtype=torch.int64, device="cuda", generator=g)
        B = torch.randint(-16, 17, (n, n), dtype=torch.int64, device="cuda", generator=g)
    med = {}
    with sm.Executor(sm.Config(base_dim=64, workers=148)) as ex:
        for algo in ("co2", "co3", "tar", "sar"):
            C = sm.Matrix(torch.zeros(n, n, dtype=s.torch_dtype, device="cuda"), s)
            Am, Bm = sm.Matrix(A, s), sm.Matrix(B, s)
            ts = []
            for it in range(9):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                sm.run_algorithm(ex, algo, C, Am, Bm, s)
                e1.record()
                torch.cuda.synchronize()
                if it >= 2:
                    ts.append(e0.elapsed_time(e1))
            med[algo] = sorted(ts)[len(ts) // 2]
    assert med["tar"] <= 1.15 * med["co2"], med
    assert med["sar"] <= 1.15 * med["co3"], med


def test_dmma_wave_gate_with_concurrent_launches(monkeypatch):
    """Two gated DMMA launches on two streams at once (neither grid fully co-resident):
    the bounded gate wait turns itself off instead of stalling, results stay correct.
    (The gate is opt-in, STARMM_DMMA_GATE=1, for the one-CTA-per-SM kernel.)"""
    monkeypatch.setenv("STARMM_DMMA_GATE", "1")
    n = 4096
    s = sm.FLOAT_RING
    g = torch.Generator(device="cuda").manual_seed(9)
    A = torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g)
    B = torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g)
    want = A @ B
    from paper_1911_05328_b200 import _lib
    plans = [_lib.Plan(s.sr_id, "co2", "pooled", n, n, n, 64, 148, -1, 0, _lib.F_INIT_IDENTITY | _lib.F_ASYNC)
             for _ in range(2)]
    outs = [torch.empty(n, n, dtype=torch.float64, device="cuda") for _ in range(2)]
    streams = [torch.cuda.Stream() for _ in range(2)]
    torch.cuda.synchronize()
    import time
    t0 = time.perf_counter()
    for p, o, st in zip(plans, outs, streams):
        p.execute(o.data_ptr(), n, A.data_ptr(), n, B.data_ptr(), n, st.cuda_stream)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    for p in plans:
        p.close()
    for o in outs:
        assert torch.allclose(o, want, rtol=1e-10, atol=1e-9)
    assert dt < 1.0, dt      # 2 x 0.137 Tflop ~ 8 ms of work; a stalled gate would take seconds


# ---- BASELINE config 1 (PR1) ----------------------------------------------
def test_pr1_star_fp64_vs_reference():
    from bench_configs import make_inputs
    A, B, C0 = make_inputs(1)
    want = np.load(os.path.join(GOLD, "ref_pr1.npz"))["star"]
    got = run("star", sm.FLOAT_RING, C0, A, B, sm.Config(base_dim=32, workers=1))
    assert sm.matrices_equal(got, want, tol=1e-12)


# ---- the exact narrow paths and their fallbacks ---------------------------
def _path_of(algo, s, C0, A, B, cfg):
    with sm.Executor(cfg) as ex:
        C, Am, Bm = sm.Matrix(C0, s), sm.Matrix(A, s), sm.Matrix(B, s)
        sm.run_algorithm(ex, algo, C, Am, Bm, s)
        return C.numpy(), ex.last_stats["path_name"]


@pytest.mark.parametrize("lo,hi,expect", [(-16, 17, "simt_i64_dp4a"),
                                          (-127, 128, "simt_i64_dp4a"),
                                          (-1000, 1001, "simt_i64_narrow_i32"),
                                          (-2 ** 40, 2 ** 40, "simt_i64")])
def test_int64_paths_bitexact(lo, hi, expect):
    n = 384
    rng = np.random.default_rng(5)
    A = rng.integers(lo, hi, (n, n), dtype=np.int64)
    B = rng.integers(lo, hi, (n, n), dtype=np.int64)
    C0 = rng.integers(lo, hi, (n, n), dtype=np.int64)
    want = C0.copy()
    O.gemm_fold(O.SR_INT64, want, A, B)
    got, path = _path_of("co2", sm.INT_RING, C0, A, B, sm.Config(base_dim=32, allow_nonpow2=True))
    assert path == expect
    assert same_bits(got, want)


def test_int64_wraps_mod_2_64():
    A = np.full((2, 2), 2 ** 62, np.int64)
    B = np.full((2, 2), 4, np.int64)
    got = run("co2", sm.INT_RING, np.zeros((2, 2), np.int64), A, B, sm.Config(base_dim=2))
    assert got.tolist() == [[0, 0], [0, 0]]


@pytest.mark.parametrize("hi,expect", [(1000, "simt_i32_s16x2_viaddmnmx"),
                                       (4096, "simt_i32_s16x2_viaddmnmx"),
                                       (100000, "simt_i32_via_f32_carrier"),
                                       (1 << 26, "simt_i32_viaddmnmx"),
                                       (1 << 30, "simt_i32_saturating")])
def test_i32_tropical_paths_bitexact(hi, expect):
    n = 320
    rng = np.random.default_rng(9)
    A = rng.integers(-hi, hi, (n, n), dtype=np.int32)
    B = rng.integers(-hi, hi, (n, n), dtype=np.int32)
    A[rng.random(A.shape) < 0.15] = O.I32_INF
    B[rng.random(B.shape) < 0.15] = O.I32_INF
    C0 = rng.integers(-hi, hi, (n, n), dtype=np.int32)
    want = C0.copy()
    O.gemm_fold(O.SR_TROP_I32, want, A, B)
    got, path = _path_of("co2", sm.TROPICAL_I32, C0, A, B, sm.Config(base_dim=32, allow_nonpow2=True))
    assert path == expect
    assert same_bits(got, want)


@pytest.mark.parametrize("kind,expect", [("int_small", "simt_f32_s16x2_viaddmnmx"),
                                         ("int_4096", "simt_f32_s16x2_viaddmnmx"),
                                         ("int_large", "simt_f32_fadd2_fmnmx3"),
                                         ("fractional", "simt_f32_fadd2_fmnmx3"),
                                         ("neg_inf", "simt_f32_fadd2_fmnmx3")])
def test_f32_tropical_paths_bitexact(kind, expect):
    n = 288
    rng = np.random.default_rng(13)
    hi = {"int_small": 100, "int_4096": 4096, "int_large": 5000}.get(kind, 100)
    A = rng.integers(-hi, hi + 1, (n, n)).astype(np.float32)
    B = rng.integers(-hi, hi + 1, (n, n)).astype(np.float32)
    if kind == "fractional":
        A += 0.25
    if kind == "neg_inf":
        A[3, 5] = -np.inf
    A[rng.random(A.shape) < 0.2] = np.inf
    B[rng.random(B.shape) < 0.2] = np.inf
    C0 = rng.integers(-2 * hi, 2 * hi, (n, n)).astype(np.float32)
    C0[rng.random(C0.shape) < 0.1] = np.inf
    want = C0.copy()
    O.gemm_fold(O.SR_TROP_F32, want, A, B)
    got, path = _path_of("co2", sm.TROPICAL_F32, C0, A, B, sm.Config(base_dim=32, allow_nonpow2=True))
    assert path == expect
    assert same_bits(got, want)


@pytest.mark.parametrize("hi,frac,expect", [(50, False, "simt_f64trop_s16x2_viaddmnmx"),
                                            (100000, False, "simt_f64trop_via_f32_carrier"),
                                            (1 << 24, False, "simt_f64_min"),
                                            (50, True, "simt_f64_min")])
def test_reference_tropical_f64_paths_bitexact(hi, frac, expect):
    """The reference's own float64 (min,+) semiring: integer-valued inputs take the exact
    narrow kernels, anything else the float64 kernel -- identical bits either way."""
    n = 272
    rng = np.random.default_rng(17)
    A = rng.integers(-hi, hi + 1, (n, n)).astype(np.float64)
    B = rng.integers(-hi, hi + 1, (n, n)).astype(np.float64)
    if frac:
        B += 0.5
    A[rng.random(A.shape) < 0.1] = np.inf
    B[rng.random(B.shape) < 0.1] = np.inf
    C0 = rng.integers(-hi, hi + 1, (n, n)).astype(np.float64)
    want = C0.copy()
    O.gemm_fold(O.SR_TROP_F64, want, A, B)
    got, path = _path_of("co2", sm.TROPICAL, C0, A, B, sm.Config(base_dim=16, allow_nonpow2=True))
    assert path == expect
    assert same_bits(got, want)


def test_tropical_nan_in_C_propagates_like_np_minimum():
    s = sm.TROPICAL
    A = np.array([[1.0, 2.0], [3.0, 4.0]])
    B = np.array([[0.0, np.inf], [1.0, 0.0]])
    C0 = np.array([[np.nan, 5.0], [0.5, np.inf]])
    want = C0.copy()
    O.gemm_fold(O.SR_TROP_F64, want, A, B)
    got = run("co2", s, C0, A, B, sm.Config(base_dim=2))
    assert same_bits(got, want, equal_nan=True)


# ---- ragged / non-power-of-two / region-strided ---------------------------
@pytest.mark.parametrize("n", [1, 3, 130, 200])
@pytest.mark.parametrize("sid", ["int", "float", "tropical_f32", "tropical_i32"])
def test_nonpow2_sizes(n, sid):
    s = sm.get_semiring(sid)
    rng = np.random.default_rng(n)
    A = rng.integers(0, 30, (n, n)).astype(s.dtype)
    B = rng.integers(0, 30, (n, n)).astype(s.dtype)
    C0 = rng.integers(0, 60, (n, n)).astype(s.dtype)
    want = C0.copy()
    O.gemm_fold(SR_OF[sid], want, A, B)
    got = run("star", s, C0, A, B, sm.Config(base_dim=1, workers=8, allow_nonpow2=True))
    assert_match(sid, got, want)


def test_pow2_precondition_kept_by_default():
    s = sm.FLOAT_RING
    with pytest.raises(sm.InvalidSplit):
        run("star", s, np.zeros((48, 48)), np.zeros((48, 48)), np.zeros((48, 48)), sm.Config())


def test_base_kernel_and_madd_on_regions():
    s = sm.INT_RING
    rng = np.random.default_rng(3)
    M = rng.integers(0, 10, (8, 8)).astype(np.int64)
    C = sm.Matrix(M.copy(), s)
    A = sm.Matrix(rng.integers(0, 10, (8, 8)).astype(np.int64), s)
    B = sm.Matrix(rng.integers(0, 10, (8, 8)).astype(np.int64), s)
    cfg = sm.Config(base_dim=4)
    cq, aq, bq = C.region().quadrant(1, 0), A.region().quadrant(0, 1), B.region().quadrant(1, 1)
    sm.base_kernel(cq, aq, bq, s, cfg)
    want = M.copy()
    want[4:, :4] += A.numpy()[:4, 4:] @ B.numpy()[4:, 4:]
    assert same_bits(C.numpy(), want)
    with pytest.raises(sm.NotBaseCase):
        sm.base_kernel(C, A, B, s, cfg)
    sm.madd(C.region().quadrant(0, 0), A.region().quadrant(1, 1), s)
    want[:4, :4] += A.numpy()[4:, 4:]
    assert same_bits(C.numpy(), want)


def test_naive_mm_and_semiring_hooks():
    s = sm.INT_RING
    out = sm.naive_mm(sm.Matrix(np.array([[1, 2], [3, 4]]), s), sm.Matrix(np.array([[5, 6], [7, 8]]), s), s)
    assert out.numpy().tolist() == [[19, 22], [43, 50]]
    t = sm.TROPICAL.matmul(np.array([[0.0, 1.0], [2.0, 3.0]]), np.array([[0.0, 4.0], [1.0, 0.0]]))
    assert t.tolist() == [[0, 1], [2, 3]]
    # rectangular panels (sampled-tile protocol)
    rng = np.random.default_rng(1)
    A = rng.standard_normal((37, 91))
    B = rng.standard_normal((91, 53))
    assert np.allclose(sm.FLOAT_RING.matmul(A, B), A @ B, rtol=1e-12, atol=1e-12)
    C = np.ones((2, 2))
    sm.TROPICAL.fold_add(C, np.array([[0.5, 2.0], [np.inf, -1.0]]))
    assert C.tolist() == [[0.5, 1.0], [1.0, -1.0]]


def test_atomic_accumulate():
    s = sm.FLOAT_RING
    C = sm.Matrix(np.ones((64, 64)), s)
    P = sm.Matrix(np.full((32, 32), 2.0), s)
    sm.atomic_accumulate(C.region().quadrant(1, 1), P.region(), s,
                         table=sm.TileExclusionTable(64, 64, 32))
    want = np.ones((64, 64))
    want[32:, 32:] += 2.0
    assert same_bits(C.numpy(), want)
    with pytest.raises(sm.DimMismatch):
        sm.atomic_accumulate(C.region(), P.region(), s)


# ---- space / busy-leaves bookkeeping (SPEC.md:562-566 analogues) ----------
def _stats(algo, ksplit, workers=4, n=512, mode="pooled"):
    s = sm.FLOAT_RING
    rng = np.random.default_rng(0)
    A, B = rng.standard_normal((n, n)), rng.standard_normal((n, n))
    cfg = sm.Config(base_dim=32, workers=workers, ksplit=ksplit)
    with sm.Executor(cfg) as ex:
        C = sm.Matrix(np.zeros((n, n)), s)
        sm.run_algorithm(ex, algo, C, sm.Matrix(A, s), sm.Matrix(B, s), s, mode=mode)
        return ex.last_stats, ex.metrics.snapshot(ex.pool), ex.pool.snapshot_counts()


def test_tar_scratch_high_water_bounded_by_workers(monkeypatch):
    # the global-memory protocols (the DMMA cluster merge has its own tests in
    # test_gpu_round2.py)
    monkeypatch.setenv("STARMM_DMMA_CLUSTER", "0")
    st, snap, pool = _stats("tar", ksplit=2)
    tile_bytes = 128 * 128 * 8
    assert st["tar_levels"] == 2
    assert 0 < st["pool_high_water_bytes"] <= st["workers"] * tile_bytes
    assert st["tile_serializations"] == st["tasks"]


def test_sar_serial_buys_no_temporaries():
    st, snap, _ = _stats("sar", ksplit=0)
    assert st["lazy_temp_acquires"] == 0 and st["ksplit"] == 1


def test_sar_pairs_transition_and_lazy_temps(monkeypatch):
    monkeypatch.setenv("STARMM_DMMA_CLUSTER", "0")
    st, snap, _ = _stats("sar", ksplit=1)
    pairs = st["pair_count"]
    tiles = st["tasks"] // st["ksplit"]
    assert st["ksplit"] == 2 and pairs == tiles
    # every first half makes Empty->FirstRunning and FirstRunning->FirstDone
    assert st["pair_transitions"] == 2 * pairs
    assert st["tile_serializations"] == st["tasks"]
    assert 0 <= st["lazy_temp_acquires"] <= pairs
    assert snap.base_case_max <= torch.cuda.get_device_properties(0).multi_processor_count


def test_star_switch_depth_levels():
    st, _, _ = _stats("star", ksplit=3, workers=16)    # switch_depth(16) = 2
    assert st["tar_levels"] == 2 and st["ksplit"] == 8


def test_co3_pooled_reuses_and_raw_allocates():
    s = sm.INT_RING
    n = 256
    A = np.ones((n, n), np.int64)
    cfg = sm.Config(base_dim=32, ksplit=1)
    with sm.Executor(cfg) as ex:
        for _ in range(3):
            C = sm.Matrix(np.zeros((n, n), np.int64), s)
            sm.run_algorithm(ex, "co3", C, sm.Matrix(A, s), sm.Matrix(A, s), s, mode="pooled")
            assert np.all(C.numpy() == n)
        c = ex.pool.snapshot_counts()
        # the workspace comes from the device pool, shared with every earlier plan: the
        # first call may already find a block of its size
        assert c["fresh_count"] + c["reuse_count"] >= 3 and c["reuse_count"] >= 2
        C = sm.Matrix(np.zeros((n, n), np.int64), s)
        sm.run_algorithm(ex, "co3", C, sm.Matrix(A, s), sm.Matrix(A, s), s, mode="raw")
        assert np.all(C.numpy() == n)
        assert ex.metrics.snapshot().raw_alloc_count == 1


def test_errors_map_to_reference_exceptions():
    s = sm.FLOAT_RING
    with pytest.raises(sm.DimMismatch):
        sm.co2(sm.Matrix(np.zeros((4, 4)), s), sm.Matrix(np.zeros((4, 8)), s),
               sm.Matrix(np.zeros((8, 4)), s), s, sm.Config(base_dim=2))
    with pytest.raises(sm.ContractViolation):
        with sm.Executor(sm.Config(base_dim=2)) as ex:
            z = sm.Matrix(np.zeros((4, 4)), s)
            sm.run_algorithm(ex, "tar", z, z, z, s, mode="raw")
    with pytest.raises(KeyError):
        with sm.Executor(sm.Config(base_dim=2)) as ex:
            z = sm.Matrix(np.zeros((4, 4)), s)
            sm.run_algorithm(ex, "bogus", z, z, z, s)


# ---- host-buffer entry point (starmm_execute_host) ------------------------
@pytest.mark.parametrize("sid", ["int", "float", "tropical_f32", "tropical_i32"])
@pytest.mark.parametrize("pinned,block_rows", [(True, 0), (True, 128), (False, 200)])
def test_host_path_streams_row_blocks(sid, pinned, block_rows):
    n = 512
    s = sm.get_semiring(sid)
    rng = np.random.default_rng(21)
    A = rng.integers(-20, 20, (n, n)).astype(s.dtype)
    B = rng.integers(-20, 20, (n, n)).astype(s.dtype)
    C0 = rng.integers(-20, 20, (n, n)).astype(s.dtype)
    want = C0.copy()
    O.gemm_fold(SR_OF[sid], want, A, B)
    At, Bt, Ct = (torch.from_numpy(x.copy()) for x in (A, B, C0))
    if pinned:
        At, Bt, Ct = At.pin_memory(), Bt.pin_memory(), Ct.pin_memory()
    with sm.Executor(sm.Config(base_dim=32, workers=148)) as ex:
        ex.execute_host("star", Ct, At, Bt, s, block_rows=block_rows)
        if block_rows:
            # phase-1 k-chunks over all rows + one execute per phase-2 row block
            nb = -(-n // block_rows)
            assert ex.last_stats["executes"] == (len(host_phase1(n, n, n, sid)) - 1) + nb
    assert_match(sid, Ct.numpy(), want)


@pytest.mark.parametrize("sid", ["int", "float", "tropical_f32", "tropical_i32"])
@pytest.mark.parametrize("n", [512, 640, 1024, 1408])
@pytest.mark.parametrize("aliased", [False, True])
@pytest.mark.parametrize("phase1", ["1", "0"])
def test_host_path_two_phase_schedule(sid, n, aliased, phase1, monkeypatch):
    """Both phases of the host schedule: k-outer chunks (first one stores, C0 folded
    from its staging buffer at the end) and row blocks; A aliasing B uploads each
    element once through the cross / bottom-right regions."""
    monkeypatch.setenv("STARMM_HOST_PHASE1", phase1)
    s = sm.get_semiring(sid)
    rng = np.random.default_rng(n + aliased)
    lo, hi = (1, 100) if sid.startswith("tropical") else (-30, 30)
    A = rng.integers(lo, hi, (n, n)).astype(s.dtype)
    B = A if aliased else rng.integers(lo, hi, (n, n)).astype(s.dtype)
    C0 = rng.integers(lo, hi, (n, n)).astype(s.dtype)
    want = C0.copy()
    O.gemm_fold(SR_OF[sid], want, A, B, par=True)
    At = torch.from_numpy(A.copy()).pin_memory()
    Bt = At if aliased else torch.from_numpy(B.copy()).pin_memory()
    Ct = torch.from_numpy(C0.copy()).pin_memory()
    with sm.Executor(sm.Config(base_dim=64, workers=148, allow_nonpow2=True)) as ex:
        ex.execute_host("star", Ct, At, Bt, s)
        nq = len(host_phase1(n, n, n, sid, aliased)) - 1
        assert nq == (0 if phase1 == "0" else (1 if n < 1024 else 2))
        assert ex.last_stats["executes"] >= nq + 1
    assert_match(sid, Ct.numpy(), want)


def test_host_path_store_flag_ignores_c0():
    """STARMM_F_INIT_IDENTITY through the host path: C <- A (x) B (C0 never uploaded)."""
    n = 1024
    s = sm.INT_RING
    rng = np.random.default_rng(5)
    A = rng.integers(-9, 9, (n, n))
    B = rng.integers(-9, 9, (n, n))
    want = np.zeros((n, n), np.int64)
    O.gemm_fold(O.SR_INT64, want, A, B, par=True)
    for ph in ("1", "0"):
        os.environ["STARMM_HOST_PHASE1"] = ph
        try:
            Ct = torch.full((n, n), 7, dtype=torch.int64).pin_memory()
            with sm.Executor(sm.Config(base_dim=64, workers=148)) as ex:
                ex.execute_host("star", Ct, torch.from_numpy(A).pin_memory(),
                                torch.from_numpy(B).pin_memory(), s, flags=0x4)
            assert same_bits(Ct.numpy(), want), ph
        finally:
            del os.environ["STARMM_HOST_PHASE1"]


def test_host_path_aliased_operands_and_public_api():
    n = 384
    s = sm.TROPICAL_I32
    rng = np.random.default_rng(4)
    W = rng.integers(1, 10 ** 6, (n, n), dtype=np.int32)
    np.fill_diagonal(W, 0)
    C = W.copy()
    sm.host_mm("star", C, W, W, s, sm.Config(base_dim=64, workers=148, allow_nonpow2=True))
    want = W.copy()
    O.gemm_fold(O.SR_TROP_I32, want, W, W)
    assert same_bits(C, want)
    with pytest.raises(sm.InvalidSplit):
        sm.host_mm("star", C, W, W, s, sm.Config(base_dim=64))


@pytest.mark.parametrize("sid", ["int", "float", "tropical_i32"])
@pytest.mark.parametrize("rank", [0, 3])
def test_distributed_step_host_2d_block(sid, rank):
    """DistributedMM.step_host without a k-split: rank (I, J) of a 2 x 2 grid runs its
    block through the overlapped host path on strided views of pinned full matrices."""
    from paper_1911_05328_b200.distributed import DistributedMM, Grid
    n = 1536
    s = sm.get_semiring(sid)
    rng = np.random.default_rng(40 + rank)
    lo, hi = (1, 1000) if sid == "tropical_i32" else (-40, 40)
    A = rng.integers(lo, hi, (n, n)).astype(s.dtype)
    B = rng.integers(lo, hi, (n, n)).astype(s.dtype)
    C0 = rng.integers(lo, hi, (n, n)).astype(s.dtype)
    dmm = DistributedMM(n, s, Grid(2, 2, 1), rank, base_dim=64, workers=148, device=0)
    Ah, Bh = torch.from_numpy(A).pin_memory(), torch.from_numpy(B).pin_memory()
    Ch = torch.from_numpy(C0.copy()).pin_memory()
    out = dmm.step_host(dmm.c_block(Ch), dmm.a_panel(Ah), dmm.b_panel(Bh))
    dmm.close()
    want = C0[dmm.r0:dmm.r1, dmm.c0:dmm.c1].copy()
    O.gemm_fold(SR_OF[sid], want, np.ascontiguousarray(A[dmm.r0:dmm.r1]),
                np.ascontiguousarray(B[:, dmm.c0:dmm.c1]), par=True)
    assert_match(sid, out.numpy(), want)
    rest = np.ones((n, n), bool)
    rest[dmm.r0:dmm.r1, dmm.c0:dmm.c1] = False
    assert same_bits(Ch.numpy()[rest], C0[rest])   # only the rank's block was written


# ---- fused k-split combine (starmm_plan_set_peers), emulated on one GPU -----
@pytest.mark.parametrize("sid,extra", [("int", 0), ("float", 0), ("tropical_f32", 0), ("tropical_i32", 0),
                                       ("int", 0x20), ("float", 0x40)])
@pytest.mark.parametrize("ks", [2, 4])
def test_fused_ksplit_combine_single_gpu_emulation(sid, extra, ks):
    """Exactly the kernel path of DistributedMM(combine="fused"): ks 'virtual ranks',
    each with its own k-slice plan, fold their partial tiles with the atomic-madd into
    the owners' row chunks (here local buffers instead of NVLink-mapped peers).  The
    virtual ranks run one after another, so nothing waits on anything."""
    from paper_1911_05328_b200 import _lib
    from paper_1911_05328_b200.distributed import block_bounds
    n = 256 * ks          # every virtual rank gets a non-empty, 128-aligned k-slice
    s = sm.get_semiring(sid)
    rng = np.random.default_rng(ks)
    A = rng.integers(-30, 30, (n, n)).astype(s.dtype)
    B = rng.integers(-30, 30, (n, n)).astype(s.dtype)
    C0 = rng.integers(-30, 30, (n, n)).astype(s.dtype)
    want = C0.copy()
    O.gemm_fold(SR_OF[sid], want, A, B)
    chunk = -(-n // ks)
    owned = [torch.from_numpy(np.ascontiguousarray(C0[j * chunk:(j + 1) * chunk])).cuda()
             for j in range(ks)]
    Ad, Bd = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    scratch = torch.empty((n, n), dtype=s.torch_dtype, device="cuda")
    for K in range(ks):
        k0, k1 = block_bounds(n, ks, K)
        plan = _lib.Plan(s.sr_id, "star", "pooled", n, n, k1 - k0, 32, 148, -1, 0,
                         _lib.F_ALLOW_NONPOW2 | extra)
        plan.set_peers([t.data_ptr() for t in owned], n, chunk)
        Ap = Ad[:, k0:k1]
        Bp = Bd[k0:k1]
        plan.execute(scratch.data_ptr(), n, Ap.data_ptr(), Ap.stride(0), Bp.data_ptr(),
                     Bp.stride(0), torch.cuda.current_stream().cuda_stream)
        if extra:   # the opt-in tensor-core paths fold through the same remote epilogue
            assert _lib.PATH_NAMES[plan.stats()["path"]] in ("tcgen05_i8_umma", "ozaki2_fp64_tcgen05_i8x16")
        plan.close()
    got = torch.cat(owned, 0).cpu().numpy()
    assert_match(sid, got, want)


# ---- CLI ---------------------------------------------------
def test_cli_run_verify_bench(tmp_path, capsys):
    from paper_1911_05328_b200.cli import main
    assert main(["run", "--algo", "co2", "--n", "64", "--b", "8", "--semiring", "int", "--seed", "1"]) == 0
    assert main(["run", "--algo", "strassen", "--semiring", "tropical"]) == 2   # NoAdditiveInverse
    assert main(["run", "--algo", "tar", "--n", "3", "--b", "1"]) == 2          # InvalidSplit
    assert main(["verify", "--suite", "space"]) == 0
    assert main(["verify", "--suite", "correctness", "--seeds", "1"]) == 0
    out = tmp_path / "b.csv"
    assert main(["bench", "--algos", "co2,co3,tar,star", "--n", "512", "--b", "64", "--reps",
                 "2", "--out", str(out)]) == 0
    rows = out.read_text().strip().split("\n")
    assert rows[0] == "algo,n,b,p,median_ns,speedup_vs_co2_pct,speedup_vs_co3_pct"
    assert len(rows) == 1 + 4


# ---- the Strassen family (strassen.py): rings only, C <- A (x) B ------------
STRASSEN = {"strassen": sm.strassen_parallel, "sar-strassen": sm.sar_strassen,
            "star-strassen-1": sm.star_strassen_1, "star-strassen-2": sm.star_strassen_2}


@pytest.mark.parametrize("algo", list(STRASSEN))
@pytest.mark.parametrize("sid", ["int", "float"])
@pytest.mark.parametrize("n,leaf,workers", [(256, 32, 1), (512, 64, 16), (1024, 128, 4)])
def test_strassen_family_overwrites_with_product(algo, sid, n, leaf, workers):
    s = sm.get_semiring(sid)
    rng = np.random.default_rng(n + len(algo))
    if sid == "int":
        A = rng.integers(-2 ** 40, 2 ** 40, (n, n), dtype=np.int64)   # products wrap mod 2^64
        B = rng.integers(-2 ** 40, 2 ** 40, (n, n), dtype=np.int64)
    else:
        A, B = rng.standard_normal((n, n)), rng.standard_normal((n, n))
    want = O.naive_mm(SR_OF[sid], A, B)
    C = sm.Matrix(np.full((n, n), 7, dtype=s.dtype), s)          # overwritten, not folded
    cfg = sm.Config(base_dim=16, workers=workers, strassen_leaf=leaf)
    STRASSEN[algo](C, sm.Matrix(A, s), sm.Matrix(B, s), s, cfg)
    if sid == "int":
        assert same_bits(C.numpy(), want)
    else:
        assert sm.matrices_equal(C.numpy(), want, tol=1e-9 * n)


def test_strassen_space_straightforward_vs_sar():
    """straightforward keeps up to 17 half-size blocks live per level; sar three."""
    n, leaf = 512, 128
    s = sm.INT_RING
    A = sm.Matrix(np.ones((n, n), np.int64), s)
    hw = {}
    for algo in ("strassen", "sar-strassen"):
        with sm.Executor(sm.Config(base_dim=16, strassen_leaf=leaf)) as ex:
            C = sm.Matrix(np.zeros((n, n), np.int64), s)
            sm.run_algorithm(ex, algo, C, A, A, s)
            assert np.all(C.numpy() == n)
            hw[algo] = ex.last_stats["pool_high_water_bytes"]
    half = (n // 2) ** 2 * 8
    assert hw["sar-strassen"] < hw["strassen"]
    assert hw["strassen"] <= 17 * half + 17 * (n // 4) ** 2 * 8
    with pytest.raises(sm.NoAdditiveInverse):
        T = sm.Matrix(np.zeros((8, 8)), sm.TROPICAL)
        sm.sar_strassen(T, T, T, sm.TROPICAL, sm.Config(base_dim=2))


def _fused_two_process_worker(rank, world, port, sid, n, q, host=False):
    import os
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import numpy as np
        import torch
        import paper_1911_05328_b200 as sm
        from oracle import oracle as O
        from paper_1911_05328_b200.distributed import DistributedMM, choose_grid, ks_groups
        torch.cuda.set_device(0)
        s = sm.get_semiring(sid)
        rng = np.random.default_rng(3)
        A = rng.integers(-40, 40, (n, n)).astype(s.dtype)
        B = rng.integers(-40, 40, (n, n)).astype(s.dtype)
        C0 = rng.integers(-40, 40, (n, n)).astype(s.dtype)
        grid = choose_grid(world, ks=2)                    # 1 x 1 x 2: pure k-split
        dmm = DistributedMM(n, s, grid, rank, algo="star", base_dim=32, workers=148,
                            group_ks=ks_groups(grid), device=0, combine="fused")
        assert dmm.combine_mode == "fused"
        if host:   # host panels: strided views of pinned full matrices, k-streamed
            Ah, Bh, Ch = (torch.from_numpy(x).pin_memory() for x in (A, B, C0))
            out = dmm.step_host(dmm.c_block(Ch), dmm.a_panel(Ah), dmm.b_panel(Bh)).numpy()
        else:
            Cb = torch.from_numpy(np.ascontiguousarray(dmm.c_block(C0))).cuda()
            Ap = torch.from_numpy(np.ascontiguousarray(dmm.a_panel(A))).cuda()
            Bp = torch.from_numpy(np.ascontiguousarray(dmm.b_panel(B))).cuda()
            out = dmm.step(Cb, Ap, Bp).cpu().numpy()
        want = C0.copy()
        O.gemm_fold(O.SR_BY_NAME[sid], want, A, B)
        lo, hi = dmm.owned_rows()
        q.put((rank, bool(same_bits(out, want[lo:hi])), lo, hi))
        dmm.close()
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e), -1, -1))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("sid", ["int", "tropical_i32", "tropical_f32"])
@pytest.mark.parametrize("host", [False, True])
def test_fused_combine_two_processes_cuda_ipc(sid, host):
    """The real DistributedMM(combine='fused') path -- owner rows shared through CUDA IPC
    (torch reduce_tensor / rebuild), tile epilogues folding into the peer's buffer -- run
    as two processes on ONE GPU.  Host collectives go over gloo; no kernel waits on any
    other, so sharing the device is safe (B200_PROFILING.md)."""
    import torch.multiprocessing as mp
    n, world = 768 if host else 512, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 31000 + hash(sid) % 1000 + (500 if host else 0)
    procs = [ctx.Process(target=_fused_two_process_worker, args=(r, world, port, sid, n, q, host))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert all(r[1] is True for r in res), res
    assert sorted((r[2], r[3]) for r in res) == [(0, n // 2), (n // 2, n)]


# ---- raw C-ABI edge cases ------------------------------------------------------
@pytest.mark.parametrize("sid", ["int", "float", "tropical", "tropical_f32", "tropical_i32"])
def test_abi_strided_leading_dimensions(sid):
    """C, A, B as column windows of wider buffers (ld > cols) through starmm_execute."""
    from paper_1911_05328_b200 import _lib
    s = sm.get_semiring(sid)
    n, pad = 200, 37
    rng = np.random.default_rng(8)
    big = lambda: rng.integers(0, 60, (n, n + pad)).astype(s.dtype)   # noqa: E731
    Ab, Bb, Cb = big(), big(), big()
    A, B, C0 = Ab[:, 5:5 + n], Bb[:, 11:11 + n], Cb[:, 3:3 + n]
    want = np.ascontiguousarray(C0).copy()
    O.gemm_fold(SR_OF[sid], want, np.ascontiguousarray(A), np.ascontiguousarray(B))
    Ad, Bd, Cd = (torch.from_numpy(x).cuda() for x in (Ab, Bb, Cb))
    es = Ad.element_size()
    plan = _lib.Plan(s.sr_id, "star", "pooled", n, n, n, 8, 16, -1, 0, _lib.F_ALLOW_NONPOW2)
    plan.execute(Cd.data_ptr() + 3 * es, n + pad, Ad.data_ptr() + 5 * es, n + pad,
                 Bd.data_ptr() + 11 * es, n + pad, torch.cuda.current_stream().cuda_stream)
    plan.close()
    got = Cd.cpu().numpy()
    assert_match(sid, got[:, 3:3 + n], want)
    assert same_bits(got[:, :3], Cb[:, :3]) and same_bits(got[:, 3 + n:], Cb[:, 3 + n:])


def test_abi_error_paths():
    from paper_1911_05328_b200 import _lib
    s = sm.FLOAT_RING
    plan = _lib.Plan(s.sr_id, "co2", "pooled", 64, 64, 64, 8, 1, -1, 0, 0)
    t = torch.zeros(64 * 64 + 1, dtype=torch.float64, device="cuda")
    stream = torch.cuda.current_stream().cuda_stream
    with pytest.raises(sm.AlignmentError):        # 4-byte offset into a float64 buffer
        plan.execute(t.data_ptr() + 4, 64, t.data_ptr(), 64, t.data_ptr(), 64, stream)
    with pytest.raises(sm.DimMismatch):           # ld < cols
        plan.execute(t.data_ptr(), 32, t.data_ptr(), 64, t.data_ptr(), 64, stream)
    with pytest.raises(sm.ContractViolation):     # NULL operand
        plan.execute(0, 64, t.data_ptr(), 64, t.data_ptr(), 64, stream)
    plan.close()
    # the host path: classical schedules only
    h = torch.zeros(64, 64, dtype=torch.float64).pin_memory()
    sp = _lib.Plan(s.sr_id, "strassen", "pooled", 64, 64, 64, 8, 1, -1, 0, 0)
    with pytest.raises(sm.ContractViolation):
        sp.execute_host(h.data_ptr(), 64, h.data_ptr(), 64, h.data_ptr(), 64, stream)
    sp.close()


def test_int64_extreme_values_wrap():
    n = 128
    lo, hi = np.iinfo(np.int64).min, np.iinfo(np.int64).max
    rng = np.random.default_rng(2)
    A = rng.choice(np.array([lo, hi, -1, 1, 0, 2 ** 62], dtype=np.int64), (n, n))
    B = rng.choice(np.array([lo, hi, -1, 3, 2 ** 33], dtype=np.int64), (n, n))
    C0 = rng.choice(np.array([lo, hi, 0], dtype=np.int64), (n, n))
    want = C0.copy()
    O.gemm_fold(O.SR_INT64, want, A, B)
    for algo in ("co2", "tar", "star"):
        got = run(algo, sm.INT_RING, C0, A, B, sm.Config(base_dim=16, workers=16, ksplit=1))
        assert same_bits(got, want), algo


@pytest.mark.parametrize("sid", ["tropical", "tropical_f32"])
def test_tropical_nan_and_neg_inf_operands(sid):
    """NaN candidates are ignored by the reference product ("if v < out"), -inf wins, and
    +inf + -inf (NaN) is ignored too (semiring.py:48-60)."""
    s = sm.get_semiring(sid)
    n = 96
    rng = np.random.default_rng(5)
    A = rng.integers(0, 50, (n, n)).astype(s.dtype)
    B = rng.integers(0, 50, (n, n)).astype(s.dtype)
    A[rng.random(A.shape) < 0.05] = np.nan
    B[rng.random(B.shape) < 0.05] = np.inf
    A[rng.random(A.shape) < 0.02] = -np.inf
    A[0, :] = np.nan                       # a row of only NaN candidates -> stays +inf/C0
    C0 = rng.integers(0, 90, (n, n)).astype(s.dtype)
    want = C0.copy()
    O.gemm_fold(SR_OF[sid], want, A, B)
    for fast in (True, False):
        got = run("co2", s, C0, A, B, sm.Config(base_dim=8, allow_nonpow2=True, fastpath=fast))
        assert same_bits(got, want, equal_nan=True)


# ---- opt-in tcgen05 kind::i8 path (exact small-range int64) -----------------------
@pytest.mark.parametrize("n", [128, 300, 1024, 2048])
@pytest.mark.parametrize("algo", ["co2", "star", "tar"])
def test_tcgen05_int8_path_bitexact(n, algo):
    rng = np.random.default_rng(n)
    A = rng.integers(-127, 128, (n, n), dtype=np.int64)
    B = rng.integers(-127, 128, (n, n), dtype=np.int64)
    C0 = rng.integers(-2 ** 62, 2 ** 62, (n, n), dtype=np.int64)
    want = C0.copy()
    O.gemm_fold(O.SR_INT64, want, A, B, par=True)
    cfg = sm.Config(base_dim=16, workers=16, int_tensor_cores=True, allow_nonpow2=True)
    with sm.Executor(cfg) as ex:
        C = sm.Matrix(C0, sm.INT_RING)
        sm.run_algorithm(ex, algo, C, sm.Matrix(A, sm.INT_RING), sm.Matrix(B, sm.INT_RING), sm.INT_RING)
        assert ex.last_stats["path_name"] == "tcgen05_i8_umma"
    assert same_bits(C.numpy(), want)


def test_tcgen05_guard_falls_back_exactly():
    """Values beyond int8 (or K*max^2 >= 2^31) must leave the single int8 GEMM: with
    int_tensor_cores they take the radix-256 digit GEMMs (exact for any int64)."""
    n = 256
    rng = np.random.default_rng(0)
    A = rng.integers(-127, 128, (n, n), dtype=np.int64)
    B = rng.integers(-127, 128, (n, n), dtype=np.int64)
    A[7, 9] = 128                                    # one value out of int8 range
    want = O.naive_mm(O.SR_INT64, A, B)
    cfg = sm.Config(base_dim=16, int_tensor_cores=True)
    with sm.Executor(cfg) as ex:
        C = sm.Matrix(np.zeros((n, n), np.int64), sm.INT_RING)
        sm.run_algorithm(ex, "co2", C, sm.Matrix(A, sm.INT_RING), sm.Matrix(B, sm.INT_RING), sm.INT_RING)
        assert ex.last_stats["path_name"] == "tcgen05_i8_radix256_int64"
    assert same_bits(C.numpy(), want)
