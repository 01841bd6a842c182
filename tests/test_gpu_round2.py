"""GPU tests of the round-2 boundary work (all through the C ABI / drop-in API):

* signed zeros: the reference's tropical results, sign of zero included, bit for bit
  (tests/golden/ref_signed_zero.npz was computed by the reference itself), on every
  schedule, through the fast paths (C0 holds -0.0) and the ordered kernel (A or B does);
* the device-side range-guard verdict: a plan's later calls never wait for the guard on
  the host, stay exact when the data range changes under them, and STARMM_F_ASYNC holds;
* the per-device block pool: LIFO re-issue, FIFO sabotage, cross-stream ordering, plan
  create/destroy without device-wide synchronisation or cudaFree, Semiring.matmul cost;
* instrumentation: the live leaf gauge, STAR's space bound.
"""
import ctypes
import os
import time

import numpy as np
import pytest
import torch

import paper_1911_05328_b200 as sm
from paper_1911_05328_b200 import _lib
from _bits import same_bits, diff_count
from oracle import oracle as O

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden")
SZ = np.load(os.path.join(GOLD, "ref_signed_zero.npz"))
SZ_CASES = [(1, 4), (2, 8), (4, 16), (8, 32), (16, 32), (32, 32)]
ALGOS = {"co2": sm.co2, "co3": sm.co3, "tar": sm.tar_mm, "sar": sm.sar_mm, "star": sm.star_mm}


def _run(algo, s, C0, A, B, cfg):
    C = sm.Matrix(C0, s)
    with sm.Executor(cfg) as ex:
        sm.run_algorithm(ex, algo, C, sm.Matrix(A, s), sm.Matrix(B, s), s)
        st = ex.last_stats
    return C.numpy(), st


# ---- signed zeros ------------------------------------------------------------------
@pytest.mark.parametrize("algo", list(ALGOS))
@pytest.mark.parametrize("b,n", SZ_CASES)
@pytest.mark.parametrize("workers", [1, 148])
def test_signed_zero_schedules_vs_reference_golden(algo, b, n, workers):
    """+-0.0-heavy operands: every schedule equals the reference bit for bit (the
    guard sees -0.0 and runs the ordered kernel at the plan's leaf size)."""
    key = f"n{n}_b{b}"
    got, st = _run(algo, sm.TROPICAL, SZ[key + "_C0"], SZ[key + "_A"], SZ[key + "_B"],
                   sm.Config(base_dim=b, workers=workers))
    assert st["path_name"] == "minplus_ordered_leaf_order"
    assert same_bits(got, SZ[f"{key}_{algo}"]), diff_count(got, SZ[f"{key}_{algo}"])


@pytest.mark.parametrize("b,n", SZ_CASES)
def test_signed_zero_naive_matmul_and_madd_vs_reference_golden(b, n):
    key = f"n{n}_b{b}"
    s = sm.TROPICAL
    got = sm.naive_mm(sm.Matrix(SZ[key + "_A"], s), sm.Matrix(SZ[key + "_B"], s), s).numpy()
    assert same_bits(got, SZ[key + "_naive"])
    assert same_bits(s.matmul(SZ[key + "_A"], SZ[key + "_B"]), SZ[key + "_naive"])
    C = SZ[key + "_C0"].copy()
    s.fold_add(C, SZ[key + "_A"])
    assert same_bits(C, SZ[key + "_madd"])


@pytest.mark.parametrize("sid", ["tropical", "tropical_f32"])
@pytest.mark.parametrize("algo", ["co2", "co3", "sar", "star"])
@pytest.mark.parametrize("b", [16, 64, 256])
def test_signed_zero_operands_take_ordered_kernel(sid, algo, b):
    """Integer-valued data (the s16x2 fast path's range) with -0.0 sprinkled into A and
    B: the ordered kernel runs and equals the oracle's serial schedule (leaf order of
    the reference) bit for bit."""
    n = 256
    s = sm.get_semiring(sid)
    dt = s.dtype
    rng = np.random.default_rng(b + len(algo))
    A = rng.integers(0, 4, (n, n)).astype(dt)       # minima are mostly zeros of either sign
    B = rng.integers(0, 4, (n, n)).astype(dt)
    for M in (A, B):
        z = rng.random(M.shape) < 0.3
        M[z] = np.where(rng.random(z.sum()) < 0.5, dt.type(0.0), dt.type(-0.0))
        M[rng.random(M.shape) < 0.05] = np.inf
    C0 = rng.integers(0, 2, (n, n)).astype(dt)
    C0[C0 == 0] = np.where(rng.random((C0 == 0).sum()) < 0.5, dt.type(0.0), dt.type(-0.0))
    want = C0.copy()
    O.schedule_mm(O.SR_BY_NAME[sid], algo, want, A, B, b)
    got, st = _run(algo, s, C0, A, B, sm.Config(base_dim=b, workers=148))
    assert st["path_name"] == "minplus_ordered_leaf_order"
    assert same_bits(got, want), diff_count(got, want)
    assert np.any(np.signbit(got) & (got == 0)) and np.any(~np.signbit(got) & (got == 0))


@pytest.mark.parametrize("sid,expect", [("tropical", "simt_f64trop_s16x2_viaddmnmx"),
                                        ("tropical_f32", "simt_f32_s16x2_viaddmnmx")])
def test_signed_zero_in_C0_only_keeps_fast_path(sid, expect):
    """-0.0 only in C0: the packed fast kernels never see it, and the fold keeps
    np.minimum's tie rule (C0 = -0.0 folded with a +0.0 product gives +0.0)."""
    n = 256
    s = sm.get_semiring(sid)
    dt = s.dtype
    rng = np.random.default_rng(3)
    A = rng.integers(-2, 3, (n, n)).astype(dt)
    B = rng.integers(0, 3, (n, n)).astype(dt)
    A[rng.random(A.shape) < 0.3] = np.inf
    C0 = np.where(rng.random((n, n)) < 0.5, dt.type(-0.0), dt.type(0.0)).astype(dt)
    want = C0.copy()
    O.schedule_mm(O.SR_BY_NAME[sid], "co2", want, A, B, 64)
    got, st = _run("co2", s, C0, A, B, sm.Config(base_dim=64, workers=148))
    assert st["path_name"] == expect
    assert same_bits(got, want), diff_count(got, want)


def test_signed_zero_host_path_matches_device_path():
    """The host-buffer schedule (k-chunks, C0 folded between them) keeps the
    reference's fold order: C0 first (madd in reverse order)."""
    n = 1024
    s = sm.TROPICAL_F32
    rng = np.random.default_rng(11)
    A = rng.integers(-2, 3, (n, n)).astype(np.float32)
    B = rng.integers(-2, 3, (n, n)).astype(np.float32)
    for M in (A, B):
        M[rng.random(M.shape) < 0.4] = np.float32(-0.0)
    C0 = np.where(rng.random((n, n)) < 0.5, np.float32(-0.0), np.float32(0.0))
    want = C0.copy()
    O.schedule_mm(O.SR_TROP_F32, "star", want, A, B, 64)
    for phase1 in ("1", "0"):
        os.environ["STARMM_HOST_PHASE1"] = phase1
        try:
            Ct = torch.from_numpy(C0.copy()).pin_memory()
            with sm.Executor(sm.Config(base_dim=64, workers=148)) as ex:
                ex.execute_host("star", Ct, torch.from_numpy(A).pin_memory(),
                                torch.from_numpy(B).pin_memory(), s)
        finally:
            del os.environ["STARMM_HOST_PHASE1"]
        assert same_bits(Ct.numpy(), want), (phase1, diff_count(Ct.numpy(), want))


# ---- the device-side guard verdict ---------------------------------------------------
def _plan(sr, n, flags=0, algo="star", b=64):
    return _lib.Plan(sr, algo, "pooled", n, n, n, b, 148, -1, torch.cuda.current_device(), flags)


def _exec(p, C, A, B):
    p.reset_stats()
    p.execute(C.data_ptr(), C.stride(0), A.data_ptr(), A.stride(0), B.data_ptr(), B.stride(0),
              torch.cuda.current_stream().cuda_stream)
    return p.stats()


def test_guard_verdict_moves_to_the_device_and_tracks_the_data():
    """1st call: host reads the guard (narrowest path).  Later calls: no host wait,
    the device picks the first guess or the exact fallback -- results stay bit-exact
    when the data range changes under the plan, and the next call adapts."""
    n = 512
    p = _plan(_lib.SR_INT64, n)
    rng = np.random.default_rng(0)
    small = [torch.from_numpy(rng.integers(-9, 10, (n, n))).cuda() for _ in range(2)]
    big = [torch.from_numpy(rng.integers(-2 ** 40, 2 ** 40, (n, n))).cuda() for _ in range(2)]
    seq = [(small, "simt_i64_dp4a", 1), (small, "simt_i64_dp4a", 0),
           (big, "simt_i64", 0),          # guess dp4a is wrong: the device runs the general kernel
           (big, "simt_i64", 0),          # the hint moved: the general kernel is the first guess
           (small, "simt_i64", 0)]        # a wider path is always exact (narrows next call)
    try:
        for i, (ops, path, syncs) in enumerate(seq):
            A, B = ops
            C = torch.zeros((n, n), dtype=torch.int64, device="cuda")
            st = _exec(p, C, A, B)
            want = np.zeros((n, n), np.int64)
            O.gemm_fold(O.SR_INT64, want, A.cpu().numpy(), B.cpu().numpy(), par=True)
            assert same_bits(C.cpu().numpy(), want), i
            assert st["guard_syncs"] == syncs, (i, st)
            assert st["path_name"] == path, (i, st["path_name"])
        assert st["candidates"] >= 1
        C = torch.zeros((n, n), dtype=torch.int64, device="cuda")
        st = _exec(p, C, *small)                       # narrowed again
        assert st["path_name"] == "simt_i64_dp4a" and st["guard_syncs"] == 0
    finally:
        p.close()


@pytest.mark.parametrize("sid", ["tropical_i32", "tropical_f32", "tropical"])
def test_guard_device_fallbacks_exact_for_minplus(sid):
    """(min,+) chains: a plan primed on small integers meets -0.0 (float) or huge values
    (int32) -- the device verdict picks the ordered / saturating kernel, bit-exact."""
    n = 512
    s = sm.get_semiring(sid)
    rng = np.random.default_rng(5)
    p = _plan(s.sr_id, n, flags=_lib.F_ALLOW_NONPOW2, algo="co2", b=128)
    try:
        for it in range(3):
            A = rng.integers(0, 50, (n, n)).astype(s.dtype)
            B = rng.integers(0, 50, (n, n)).astype(s.dtype)
            if it == 1:
                if sid == "tropical_i32":
                    A[0, 0] = 2 ** 30
                else:
                    A[rng.random(A.shape) < 0.3] = -0.0
                    B[rng.random(B.shape) < 0.3] = -0.0
            C0 = rng.integers(0, 80, (n, n)).astype(s.dtype)
            want = C0.copy()
            O.schedule_mm(O.SR_BY_NAME[sid], "co2", want, A, B, 128)
            C = torch.from_numpy(C0.copy()).cuda()
            st = _exec(p, C, torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda())
            assert same_bits(C.cpu().numpy(), want), (it, st["path_name"])
            if it == 1:
                assert st["path_name"] in ("minplus_ordered_leaf_order", "simt_i32_saturating")
                assert st["guard_syncs"] == 0
    finally:
        p.close()


def test_async_flag_never_waits_for_the_guard():
    n = 1024
    rng = np.random.default_rng(1)
    A = torch.from_numpy(rng.integers(-100, 100, (n, n)).astype(np.int32)).cuda()
    C0 = A.clone()
    p = _plan(_lib.SR_TROPICAL_I32, n, flags=_lib.F_ASYNC)
    try:
        C = C0.clone()
        st = _exec(p, C, A, A)                 # first call of the plan, asynchronous
        assert st["guard_syncs"] == 0 and st["candidates"] >= 2
        torch.cuda.synchronize()
        want = C0.cpu().numpy().copy()
        O.gemm_fold(O.SR_TROP_I32, want, A.cpu().numpy(), A.cpu().numpy(), par=True)
        assert same_bits(C.cpu().numpy(), want)
    finally:
        p.close()


# ---- the device block pool ---------------------------------------------------------
def test_device_pool_lifo_reissue_and_contracts():
    p = sm.Pool(2, device="cuda")
    h1 = p.acquire(0, 1 << 17)
    p.release(h1)
    h2 = p.acquire(0, 1 << 17)
    assert h2 is h1                                 # LIFO reuse (pool.py:97)
    c = p.snapshot_counts()
    assert c["reuse_count"] >= 1 and c["fresh_count"] <= 1
    with pytest.raises(sm.ContractViolation):
        p.release(h2, worker=1)
    m = h2.as_matrix(64, sm.FLOAT_RING)
    m.data.fill_(2.5)
    assert float(m.data.sum()) == 2.5 * 64 * 64
    p.release(h2)
    with pytest.raises(sm.ContractViolation):
        p.release(h2)                               # double release
    a, b = p.acquire(0, 1 << 16), p.acquire(1, 1 << 16)
    p.release(a)
    p.release(b)
    assert p.acquire(0, 1 << 16) is b               # newest first
    p.close()


def test_fifo_sabotage_reaches_the_device_pool_and_verify_fails(capsys):
    from paper_1911_05328_b200.cli import main
    f = sm.Pool(1, discipline="fifo", device="cuda")
    try:
        w = 12345                                   # a size class nothing else uses
        a, b = f.acquire(0, w), f.acquire(0, w)
        f.release(a)
        f.release(b)
        assert f.acquire(0, w) is a                 # the oldest: FIFO on the device pool
    finally:
        f.close()
    assert main(["verify", "--suite", "pool"]) == 0
    assert main(["verify", "--suite", "pool", "--sabotage-lifo"]) == 1
    capsys.readouterr()


def test_pool_reuse_across_streams_is_ordered_on_the_device():
    """A block released on a busy stream is not handed to another stream while the pool
    has room (a fresh block instead: streams are not chained through the pool); at its
    limit the pool reuses it, ordered by an event wait on the device."""
    dev = torch.cuda.current_device()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    nb = (64 << 20) + 1792                          # a size class nothing else uses
    ptr, _ = _lib.pool_acquire(dev, nb, s1.cuda_stream)
    buf = torch.as_tensor(sm.pool._DeviceBytes(ptr, nb), device="cuda").view(torch.float32)
    with torch.cuda.stream(s1):
        torch.cuda._sleep(50_000_000)               # s1 still busy when the block is freed
        buf.fill_(1.0)
    _lib.pool_release(dev, ptr, s1.cuda_stream)
    other, fresh = _lib.pool_acquire(dev, nb, s2.cuda_stream)
    assert other != ptr and fresh                   # room left: no cross-stream chaining
    _lib.pool_release(dev, other, s2.cuda_stream)
    torch.cuda.synchronize()
    # at the limit: a block still in use on s1 is reused by s2 behind an event wait
    x, _ = _lib.pool_acquire(dev, nb, s1.cuda_stream)
    bx = torch.as_tensor(sm.pool._DeviceBytes(x, nb), device="cuda").view(torch.float32)
    with torch.cuda.stream(s1):
        torch.cuda._sleep(50_000_000)
        bx.fill_(1.0)
    _lib.pool_release(dev, x, s1.cuda_stream)
    before = _lib.pool_counts(dev)
    old = _lib.pool_set_limit(dev, before["allocated_bytes"])
    got = []
    try:
        for _ in range(4):                          # ready blocks first, then x
            p2, fresh = _lib.pool_acquire(dev, nb, s2.cuda_stream)
            assert not fresh
            got.append(p2)
            if p2 == x:
                break
        assert got[-1] == x
        with torch.cuda.stream(s2):
            bx.fill_(2.0)                           # must run after s1's fill
        torch.cuda.synchronize()
        assert float(bx.min()) == 2.0
        assert _lib.pool_counts(dev)["cross_stream_waits"] == before["cross_stream_waits"] + 1
    finally:
        for p2 in got:
            _lib.pool_release(dev, p2, s2.cuda_stream)
        _lib.pool_set_limit(dev, old)


def test_plan_lifecycle_reuses_the_device_pool():
    """Creating, running and destroying plans allocates once: later plans of the same
    shape reuse the pool's blocks (no cudaMalloc / cudaFree per plan)."""
    dev = torch.cuda.current_device()
    n = 512
    A = torch.randn(n, n, dtype=torch.float64, device="cuda")
    _exec_once = lambda: sm.star_mm(sm.Matrix(torch.zeros_like(A), sm.FLOAT_RING),
                                    sm.Matrix(A, sm.FLOAT_RING), sm.Matrix(A, sm.FLOAT_RING),
                                    sm.FLOAT_RING, sm.Config(base_dim=64, workers=148))
    _exec_once()
    before = _lib.pool_counts(dev)
    for _ in range(20):
        _exec_once()                                # an Executor + plan per call
    after = _lib.pool_counts(dev)
    assert after["fresh_count"] == before["fresh_count"]
    assert after["allocated_bytes"] == before["allocated_bytes"]
    assert after["trims"] == before["trims"]


def test_semiring_matmul_per_call_cost_is_microseconds(capsys):
    """10k Semiring.matmul calls at 64x64 (the reference's numba kernel is called per
    leaf): cached plans, pooled staging, device-side guard -- per-call cost in us."""
    s = sm.INT_RING
    A = torch.randint(-5, 5, (64, 64), dtype=torch.int64, device="cuda")
    B = torch.randint(-5, 5, (64, 64), dtype=torch.int64, device="cuda")
    want = (A.cpu() @ B.cpu()).numpy()
    for _ in range(50):
        s.matmul(A, B)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    calls = 10_000
    for _ in range(calls):
        out = s.matmul(A, B)
    torch.cuda.synchronize()
    us = (time.perf_counter() - t0) / calls * 1e6
    assert same_bits(out.cpu().numpy(), want)
    with capsys.disabled():
        print(f"\n[Semiring.matmul 64x64 int64] {us:.1f} us per call over {calls} calls")
    assert us < 500.0


# ---- instrumentation -------------------------------------------------------------
@pytest.mark.parametrize("algo", ["tar", "star", "sar", "co2"])
def test_live_leaf_gauge_is_measured_and_bounded(algo):
    """Busy-leaves: the leaves observed in flight at once never exceed
    the persistent workers, over repeated runs; and the gauge is an observation
    (>= 1), not the grid formula."""
    n = 1024
    rng = np.random.default_rng(2)
    A = rng.integers(-20, 20, (n, n)).astype(np.int64)
    for rep in range(10):
        _, st = _run(algo, sm.INT_RING, np.zeros((n, n), np.int64), A, A,
                     sm.Config(base_dim=64, workers=148, ksplit=None if rep % 2 else 2))
        assert 1 <= st["live_leaves_max"] <= st["workers"], st
    with sm.Executor(sm.Config(base_dim=64, workers=148)) as ex:
        C = sm.Matrix(np.zeros((n, n), np.int64), sm.INT_RING)
        sm.run_algorithm(ex, "star", C, sm.Matrix(A, sm.INT_RING), sm.Matrix(A, sm.INT_RING), sm.INT_RING)
        snap = ex.metrics.snapshot()
        assert snap.base_case_max == ex.last_stats["live_leaves_max"]


@pytest.mark.parametrize("p", [1, 4, 16])
def test_star_space_bound(p):
    """STAR temp high-water <= ceil(n^2/3) + p*b^2 elements, n = 16b, with
    the GPU's leaf (the output tile a CTA owns) as b^2 and p the persistent workers."""
    b = 32
    n = 16 * b
    rng = np.random.default_rng(p)
    A = rng.integers(-20, 20, (n, n)).astype(np.int64)
    for ks in (None, 1, 2, 3):
        _, st = _run("star", sm.INT_RING, np.zeros((n, n), np.int64), A, A,
                     sm.Config(base_dim=b, workers=p, ksplit=ks))
        tile = 128 * 128                            # CUDA-core leaf tile (int64 path)
        bound = (-(-n * n // 3) + st["workers"] * tile) * 8
        assert st["pool_high_water_bytes"] <= bound, (ks, st)


# ---- counter-based input generation ---------------------------
@pytest.mark.parametrize("cid", [1, 2, 3, 4, 5])
@pytest.mark.parametrize("what", ["A", "B", "C"])
def test_device_generator_matches_oracle_regeneration(cid, what):
    """generate_panel on the GPU equals the oracle's host restatement bit for bit, for
    every config's matrices, at panel offsets (so the bench's sampled-tile check can
    regenerate any rank's panels)."""
    from bench_configs import CONFIGS, device_gen_spec
    spec = device_gen_spec(cid, what)
    if spec == "zeros":
        pytest.skip("all-zero matrix")
    s = sm.get_semiring(CONFIGS[cid]["semiring"])
    dev = sm.generate_panel(s, rows=300, cols=260, row0=4093, col0=4000, **spec).cpu().numpy()
    spec = dict(spec)
    spec["stream"] = spec.pop("stream_id")
    host = O.generate(O.SR_BY_NAME[CONFIGS[cid]["semiring"]], rows=300, cols=260, row0=4093,
                      col0=4000, **spec)
    assert same_bits(dev, host), diff_count(dev, host)


def test_generated_config_panel_product_vs_oracle():
    """End to end on generated inputs: a config-4-distributed 1024^3 STAR product's
    sampled tiles vs the oracle on host-regenerated panels."""
    from bench_configs import device_gen_spec
    n = 1024
    s = sm.FLOAT_RING
    A = sm.generate_panel(s, rows=n, cols=n, **device_gen_spec(4, "A"))
    B = sm.generate_panel(s, rows=n, cols=n, **device_gen_spec(4, "B"))
    C = sm.generate_panel(s, rows=n, cols=n, **device_gen_spec(4, "C"))
    C0 = C.cpu().numpy()
    sm.star_mm(sm.Matrix(C, s), sm.Matrix(A, s), sm.Matrix(B, s), s, sm.Config(base_dim=64, workers=148))
    want = C0.copy()
    O.gemm_fold(O.SR_FP64, want, A.cpu().numpy(), B.cpu().numpy(), par=True)
    got = C.cpu().numpy()
    assert np.all(np.abs(got - want) <= 1e-10 * np.sqrt(n) * np.maximum(1, np.abs(want)))


# ---- DMMA split-k on thread-block clusters (DSMEM merge) ----------------------------
@pytest.mark.parametrize("algo", ["tar", "sar", "star"])
@pytest.mark.parametrize("ksplit", [1, 2, 3])
def test_dmma_cluster_split_exact_and_deterministic(algo, ksplit):
    """The S k-slices of each tile run on one cluster and merge through DSMEM in rank
    order: within tolerance of the oracle, bit-identical from run to run (no atomics),
    and no tile locks / pair states / lazy global scratch."""
    n = 768                                           # ragged: 3 x 12 tiles of 256 x 64
    rng = np.random.default_rng(ksplit)
    A, B, C0 = rng.standard_normal((n, n)), rng.standard_normal((n, n)), rng.uniform(-1, 1, (n, n))
    want = C0.copy()
    O.gemm_fold(O.SR_FP64, want, A, B, par=True)
    outs = []
    for _ in range(2):
        got, st = _run(algo, sm.FLOAT_RING, C0, A, B,
                       sm.Config(base_dim=64, workers=148, ksplit=ksplit, allow_nonpow2=True))
        assert st["cluster_size"] == 1 << ksplit and st["ksplit"] == 1 << ksplit
        assert st["pair_count"] == 0 and st["tile_serializations"] == 3 * 12
        assert st["lazy_temp_acquires"] == 3 * 12 * ((1 << ksplit) - 1)
        assert np.all(np.abs(got - want) <= 1e-12 * n * np.maximum(1, np.abs(want)))
        outs.append(got)
    assert same_bits(outs[0], outs[1])


def test_dmma_cluster_store_flag_and_protocol_fallback(monkeypatch):
    """C <- A (x) B (init identity) through the cluster merge, and the same split with
    the global-memory protocols (STARMM_DMMA_CLUSTER=0) agree within rounding."""
    n = 512
    rng = np.random.default_rng(9)
    A, B = rng.standard_normal((n, n)), rng.standard_normal((n, n))
    s = sm.FLOAT_RING
    At, Bt = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    p = _lib.Plan(_lib.SR_FP64, "sar", "pooled", n, n, n, 64, 148, 2, 0, _lib.F_INIT_IDENTITY)
    C = torch.full((n, n), 7.0, dtype=torch.float64, device="cuda")
    st = _exec(p, C, At, Bt)
    p.close()
    assert st["cluster_size"] == 4
    want = A @ B
    assert np.allclose(C.cpu().numpy(), want, rtol=1e-12, atol=1e-10)
    monkeypatch.setenv("STARMM_DMMA_CLUSTER", "0")
    got, st = _run("sar", s, np.zeros((n, n)), A, B, sm.Config(base_dim=64, workers=148, ksplit=2))
    assert st["cluster_size"] == 0 and st["pair_count"] > 0
    assert np.allclose(got, want, rtol=1e-12, atol=1e-10)


# ---- general int64 in two passes (low products, then cross terms) ---------------------
@pytest.mark.parametrize("algo", ["co2", "co3", "tar", "sar", "star"])
@pytest.mark.parametrize("ksplit", [0, 1, 2])
def test_general_int64_two_pass_wraps_bitexact(algo, ksplit):
    """Full-range int64 (wraps mod 2^64) through the general kernel's two passes under
    every write-back protocol, bit-exact against the oracle."""
    n = 384
    rng = np.random.default_rng(40 + ksplit)
    A = rng.integers(-2 ** 62, 2 ** 62, (n, n), dtype=np.int64)
    B = rng.integers(-2 ** 62, 2 ** 62, (n, n), dtype=np.int64)
    C0 = rng.integers(-2 ** 62, 2 ** 62, (n, n), dtype=np.int64)
    want = C0.copy()
    O.gemm_fold(O.SR_INT64, want, A, B, par=True)
    got, st = _run(algo, sm.INT_RING, C0, A, B,
                   sm.Config(base_dim=32, workers=148, ksplit=ksplit, allow_nonpow2=True))
    assert st["path_name"] == "simt_i64"
    assert same_bits(got, want)


@pytest.mark.parametrize("algo", ["tar", "star"])
@pytest.mark.parametrize("store", [False, True])
def test_dmma_balanced_slices(algo, store):
    """n = 2048 fp64 (256 tiles on 148 SMs): tar / star run balanced k-slices on the
    DMMA path (whole tiles folded exclusively, shared pieces by red.add.f64)."""
    n = 2048
    rng = np.random.default_rng(5)
    A, B = rng.standard_normal((n, n)), rng.standard_normal((n, n))
    C0 = rng.uniform(-1, 1, (n, n))
    flags = _lib.F_INIT_IDENTITY if store else 0
    p = _plan(_lib.SR_FP64, n, flags=flags, algo=algo)
    try:
        C = torch.from_numpy(C0.copy()).cuda()
        st = _exec(p, C, torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda())
    finally:
        p.close()
    assert st["balanced_workers"] > 0 and st["path_name"] == "dmma_f64"
    want = np.zeros((n, n)) if store else C0.copy()
    O.gemm_fold(O.SR_FP64, want, A, B, par=True)
    got = C.cpu().numpy()
    assert np.all(np.abs(got - want) <= 1e-10 * np.sqrt(n) * np.maximum(1, np.abs(want)))


# ---- k-outer chunked launches (L2-sized panels) --------------------------------------
@pytest.mark.parametrize("sid,lo,hi", [("int", -100, 100), ("int", -9, 10), ("tropical_i32", 0, 100000),
                                       ("tropical_f32", 0, 1000), ("tropical", 0, 50)])
@pytest.mark.parametrize("store", [False, True])
def test_k_chunked_launches_bitexact(sid, lo, hi, store, monkeypatch):
    """STARMM_K_CHUNKS forces the k-outer chunking (auto only for panels > 2x L2, e.g.
    config 5): every chunk folds whole tiles into C, bit-exact against the oracle."""
    monkeypatch.setenv("STARMM_K_CHUNKS", "3")
    n = 640
    s = sm.get_semiring(sid)
    rng = np.random.default_rng(hi)
    A = rng.integers(lo, hi, (n, n)).astype(s.dtype)
    B = rng.integers(lo, hi, (n, n)).astype(s.dtype)
    C0 = rng.integers(lo, hi, (n, n)).astype(s.dtype)
    want = np.full((n, n), s.zero, dtype=s.dtype) if store else C0.copy()
    O.gemm_fold(O.SR_BY_NAME[sid], want, A, B, par=True)
    flags = _lib.F_ALLOW_NONPOW2 | (_lib.F_INIT_IDENTITY if store else 0)
    p = _lib.Plan(s.sr_id, "co2", "pooled", n, n, n, 64, 148, -1, 0, flags)
    try:
        C = torch.from_numpy(C0.copy()).cuda()
        st = _exec(p, C, torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda())
    finally:
        p.close()
    assert st["k_chunks"] == 3, st
    assert same_bits(C.cpu().numpy(), want)


# ---- opt-in: any int64 as radix-256 digit GEMMs on the int8 tensor cores ---------------
@pytest.mark.parametrize("m,n,k", [(256, 256, 256), (512, 384, 1000), (300, 520, 8192), (256, 256, 17000)])
@pytest.mark.parametrize("store", [False, True])
def test_int64_radix256_tensor_path_wraps_bitexact(m, n, k, store):
    """Full-range int64 (wraps mod 2^64) on tcgen05 kind::i8 as 8 digit-group GEMMs per
    K chunk (<= 8192): bit-exact against the oracle, ragged shapes, several K chunks."""
    rng = np.random.default_rng(m + k)
    A = rng.integers(-2 ** 63, 2 ** 63 - 1, (m, k), dtype=np.int64)
    B = rng.integers(-2 ** 63, 2 ** 63 - 1, (k, n), dtype=np.int64)
    A[0, :4] = [-2 ** 63, 2 ** 63 - 1, -1, 0]
    C0 = rng.integers(-2 ** 63, 2 ** 63 - 1, (m, n), dtype=np.int64)
    want = np.zeros((m, n), np.int64) if store else C0.copy()
    O.gemm_fold(O.SR_INT64, want, A, B, par=True)
    flags = _lib.F_ALLOW_NONPOW2 | _lib.F_INT_TENSOR | (_lib.F_INIT_IDENTITY if store else 0)
    p = _lib.Plan(_lib.SR_INT64, "star", "pooled", m, n, k, 64, 148, -1, 0, flags)
    try:
        C = torch.from_numpy(C0.copy()).cuda()
        At, Bt = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
        p.reset_stats()
        p.execute(C.data_ptr(), n, At.data_ptr(), k, Bt.data_ptr(), n, torch.cuda.current_stream().cuda_stream)
        st = p.stats()
    finally:
        p.close()
    assert st["path_name"] == "tcgen05_i8_radix256_int64"
    assert same_bits(C.cpu().numpy(), want)


def test_int64_radix256_through_the_public_api_and_guard():
    """Config(int_tensor_cores=True): small ranges keep the single int8 GEMM, wide ranges
    take the digit GEMMs -- first call on the host guard, later calls on the device; a
    call whose data outgrows the first guess runs the CUDA-core fallback (cheap to queue
    predicated off) and the next call starts from the digit GEMMs."""
    n = 512
    rng = np.random.default_rng(77)
    s = sm.INT_RING
    cfg = sm.Config(base_dim=64, workers=148, int_tensor_cores=True)
    with sm.Executor(cfg) as ex:
        for lo, hi, path in [(-5, 6, "tcgen05_i8_umma"), (-2 ** 40, 2 ** 40, "simt_i64"),
                             (-2 ** 40, 2 ** 40, "tcgen05_i8_radix256_int64"), (-5, 6, "tcgen05_i8_radix256_int64")]:
            A = rng.integers(lo, hi, (n, n), dtype=np.int64)
            B = rng.integers(lo, hi, (n, n), dtype=np.int64)
            C = sm.Matrix(np.zeros((n, n), np.int64), s)
            sm.run_algorithm(ex, "star", C, sm.Matrix(A, s), sm.Matrix(B, s), s)
            want = np.zeros((n, n), np.int64)
            O.gemm_fold(O.SR_INT64, want, A, B, par=True)
            assert same_bits(C.numpy(), want), path
            assert ex.last_stats["path_name"] == path


# ---- vectorised exclusive epilogue of the CUDA-core tile kernel ----------------------
# (writeback.cuh epilogue_row_vec: 16-byte pieces, even/odd lanes swap pieces so a warp
# access covers whole sectors; taken for full tiles whose rows are 16-byte aligned)
SR_IDS = O.SR_BY_NAME
EPI_CASES = [  # (semiring, value range hi, expected kernel path prefix)
    ("int", 17, "simt_i64_dp4a"),            # 32-byte fragments (4 x int64): paired pieces
    ("int", 1000, "simt_i64_narrow_i32"),        # 32-byte fragments from int32 accumulators
    ("int", 2 ** 40, "simt_i64"),            # 16-byte fragments (2 x int64)
    ("tropical_f32", 100, "simt_f32_s16x2_viaddmnmx"),     # 8 x float = 32 bytes, two outputs per lane-op
    ("tropical_f32", 10 ** 5, "simt_f32_fadd2_fmnmx3"),  # 2 x float = 8-byte fragments
    ("tropical_i32", 100, "simt_i32_s16x2_viaddmnmx"),
    ("tropical_i32", 10 ** 5, "simt_i32_via_f32_carrier"),
    ("tropical_i32", 2 ** 26, "simt_i32_viaddmnmx"),  # 4 x int32 = 16 bytes
    ("tropical", 100, "simt_f64trop_s16x2_viaddmnmx"),        # 8 x double = 64-byte fragments (4 pieces)
    ("tropical", 10 ** 5, "simt_f64trop_via_f32_carrier"),   # 2 x double = 16 bytes
]


@pytest.mark.parametrize("sid,hi,path", EPI_CASES)
@pytest.mark.parametrize("algo,store", [("star", False), ("star", True), ("co3", False)])
def test_vector_epilogue_windows(sid, hi, path, algo, store):
    """C as a column window of a wider buffer, at offsets that leave its rows 16-byte
    aligned (vector epilogue, ld != cols) and misaligned (generic element epilogue), folded
    and overwritten (STARMM_F_INIT_IDENTITY), and co3 with a forced 2-way split (slice 1
    stores into the workspace, whose merge folds into C).  n = 640: five full tile rows;
    the two-outputs-per-lane policies (256-column tiles) end on a ragged tile column.  The
    bytes outside the window must not change."""
    s = sm.get_semiring(sid)
    n, pad = 640, 24
    rng = np.random.default_rng(hi % 1000 + n)
    gen = lambda shape: rng.integers(0 if sid != "int" else -hi + 1, hi, shape).astype(s.dtype)  # noqa: E731
    A, B = gen((n, n)), gen((n, n))
    es = np.dtype(s.dtype).itemsize
    for off in (16 // es, 1, 0):                       # aligned window, misaligned, no offset
        Cb = gen((n, n + pad))
        want = np.ascontiguousarray(Cb[:, off:off + n]).copy()
        Cd = torch.from_numpy(Cb).cuda()
        Ad, Bd = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
        plan = _lib.Plan(s.sr_id, algo, "pooled", n, n, n, 64, 148, 1 if algo == "co3" else -1, 0,
                         _lib.F_ALLOW_NONPOW2 | (_lib.F_INIT_IDENTITY if store else 0))
        plan.execute(Cd.data_ptr() + off * es, n + pad, Ad.data_ptr(), n, Bd.data_ptr(), n,
                     torch.cuda.current_stream().cuda_stream)
        st = plan.stats()
        plan.close()
        assert st["path_name"] == path, st["path_name"]
        if store:
            want = _identity_like(sid, want)
        O.gemm_fold(SR_IDS[sid], want, A, B, par=True)
        got = Cd.cpu().numpy()
        assert same_bits(got[:, off:off + n], want), (off, diff_count(got[:, off:off + n], want))
        assert same_bits(got[:, :off], Cb[:, :off]) and same_bits(got[:, off + n:], Cb[:, off + n:]), off


def _identity_like(sid, x):
    if sid == "int":
        return np.zeros_like(x)
    if sid == "tropical_i32":
        return np.full_like(x, O.I32_INF)
    return np.full_like(x, np.inf)


# ---- the k-stage ring at its edges ----------------------------------------------------
@pytest.mark.parametrize("sid,hi,path", [("int", 17, "simt_i64_dp4a"),                 # cross-stage ring, 4 stages
                                         ("tropical_i32", 100, "simt_i32_s16x2_viaddmnmx"),
                                         ("tropical_i32", 10 ** 5, "simt_i32_via_f32_carrier")])
@pytest.mark.parametrize("algo", ["co2", "tar"])
def test_stage_ring_short_and_ragged_k(sid, hi, path, algo):
    """Rectangular products whose k extent is 1 .. 7 k-stages of the policy (and not a
    multiple of the stage), on 3 x 3 output tiles: the copy ring's prologue, its
    cross-stage fragment prefetch and the early start of the next tile see every short
    case; tar adds forced and balanced k-slices (pieces of 1 .. few stages).  Each case
    runs three times (a race would be timing dependent) and must equal the oracle."""
    s = sm.get_semiring(sid)
    m = n = 384
    rng = np.random.default_rng(hi % 97 + len(algo))
    for k in (64, 96, 128, 192, 200, 256, 320, 448):
        A = rng.integers(0 if sid != "int" else -hi + 1, hi, (m, k)).astype(s.dtype)
        B = rng.integers(0 if sid != "int" else -hi + 1, hi, (k, n)).astype(s.dtype)
        C0 = rng.integers(0, hi, (m, n)).astype(s.dtype)
        want = C0.copy()
        O.gemm_fold(SR_IDS[sid], want, A, B, par=True)
        Ad, Bd = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
        for ks in ((-1,) if algo == "co2" else (-1, 1)):
            plan = _lib.Plan(s.sr_id, algo, "pooled", m, n, k, 32, 148, ks, 0, _lib.F_ALLOW_NONPOW2)
            for rep in range(3):
                Cd = torch.from_numpy(C0.copy()).cuda()
                plan.execute(Cd.data_ptr(), n, Ad.data_ptr(), k, Bd.data_ptr(), n,
                             torch.cuda.current_stream().cuda_stream)
                got = Cd.cpu().numpy()
                assert same_bits(got, want), (k, ks, rep, diff_count(got, want))
            assert plan.stats()["path_name"] == path, plan.stats()["path_name"]
            plan.close()
