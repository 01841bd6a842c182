"""Opt-in fp64 (+,x) emulation on the int8 tensor cores (Ozaki scheme II,
csrc/ozaki.cuh) against EXACT references.

The reference computes float64 A @ B with per-step rounding (semiring.py:35-45);
the DMMA default path rounds per FMA in its own order, so neither is bitwise
reproducible.  Here the bar is an error bound against the exact value
C0 + sum_k a_ik b_kj, computed with Python integers on sampled entries:
    |got - exact| <= 2^(1-t) k max_k|a_ik| max_k|b_kj| + 2^-52 |exact|
(input truncation to t bits per row/column + two roundings), and, on BASELINE
config-4 data, the DGEMM-grade bound 4u (sum|a||b| + |C0|).
"""
import math
from fractions import Fraction

import numpy as np
import pytest
from _bits import same_bits, diff_count  # noqa: F401
import torch

import paper_1911_05328_b200 as sm
from paper_1911_05328_b200 import _lib

pytestmark = pytest.mark.gpu

MODULI = [256, 255, 253, 251, 247, 241, 239, 233, 229, 227, 223, 217, 211, 199, 197, 193]
EMU = "ozaki2_fp64_tcgen05_i8x16"


def t_bits(k):
    lm = sum(math.log2(m) for m in MODULI)
    return min(62, int(math.floor((lm - math.log2(k) - 2) / 2)))


def exact(a, b, c0):
    """C0 + a . b exactly, rounded once to float64."""
    tot = Fraction(c0)
    ma, ea = np.frexp(a)
    mb, eb = np.frexp(b)
    ia = (ma * 2.0 ** 53).astype(np.int64).tolist()
    ib = (mb * 2.0 ** 53).astype(np.int64).tolist()
    ex = ((ea.astype(np.int64) - 53) + (eb.astype(np.int64) - 53)).tolist()
    e0 = min(ex)
    acc = 0
    for x, y, e in zip(ia, ib, ex):
        acc += (x * y) << (e - e0)
    return float(tot + Fraction(acc) * Fraction(2) ** e0)


def run_emu(A, B, C0, algo="star", flags_extra=0, init_identity=False):
    m, k = A.shape
    n = B.shape[1]
    Ad, Bd = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    Cd = torch.from_numpy(C0.copy()).cuda()
    flags = _lib.F_ALLOW_NONPOW2 | _lib.F_FP64_EMU | flags_extra
    if init_identity:
        flags |= _lib.F_INIT_IDENTITY
    plan = _lib.Plan(_lib.SR_FP64, algo, "pooled", m, n, k, 64, 148, -1, 0, flags)
    plan.execute(Cd.data_ptr(), n, Ad.data_ptr(), k, Bd.data_ptr(), n, torch.cuda.current_stream().cuda_stream)
    path = _lib.PATH_NAMES[plan.stats()["path"]]
    plan.close()
    return Cd.cpu().numpy(), path


def check_bound(A, B, C0, got, samples, t, rng):
    k = A.shape[1]
    amax = np.max(np.abs(A), axis=1)
    bmax = np.max(np.abs(B), axis=0)
    for i, j in zip(rng.integers(0, A.shape[0], samples), rng.integers(0, B.shape[1], samples)):
        x = exact(A[i], B[:, j], C0[i, j])
        bound = 2.0 ** (1 - t) * k * amax[i] * bmax[j] + 2.0 ** -52 * abs(x)
        assert abs(got[i, j] - x) <= bound, (i, j, got[i, j], x, bound)


@pytest.mark.parametrize("n", [64, 256, 1000, 2048])
def test_config4_data_dgemm_grade(n):
    """BASELINE config 4 distributions: A, B ~ N(0,1), C ~ U[-1,1)."""
    rng = np.random.default_rng(3)
    A = rng.standard_normal((n, n))
    B = rng.standard_normal((n, n))
    C0 = rng.uniform(-1, 1, (n, n))
    got, path = run_emu(A, B, C0)
    assert path == EMU
    for i, j in zip(rng.integers(0, n, 24), rng.integers(0, n, 24)):
        x = exact(A[i], B[:, j], C0[i, j])
        scale = float(np.abs(A[i]) @ np.abs(B[:, j])) + abs(C0[i, j])
        assert abs(got[i, j] - x) <= 4 * 2.0 ** -53 * scale, (i, j)
    # and the config-4 tolerance against the oracle's float64 product
    want = C0 + A @ B
    assert np.all(np.abs(got - want) <= 1e-10 * math.sqrt(n) * np.maximum(1.0, np.abs(want)))


def test_wide_dynamic_range_zero_rows_and_columns():
    n, k = 384, 520
    rng = np.random.default_rng(11)
    A = rng.standard_normal((n, k)) * 2.0 ** rng.integers(-300, 300, (n, 1))
    B = rng.standard_normal((k, n)) * 2.0 ** rng.integers(-300, 300, (1, n))
    A[:, :7] *= 2.0 ** -40            # small entries inside large rows get truncated
    A[5] = 0.0
    B[:, 9] = 0.0
    C0 = rng.uniform(-1, 1, (n, n))
    Ad, Bd, Cd = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), torch.from_numpy(C0.copy()).cuda()
    plan = _lib.Plan(_lib.SR_FP64, "co2", "pooled", n, n, k, 64, 148, -1, 0,
                     _lib.F_ALLOW_NONPOW2 | _lib.F_FP64_EMU)
    plan.execute(Cd.data_ptr(), n, Ad.data_ptr(), k, Bd.data_ptr(), n, torch.cuda.current_stream().cuda_stream)
    assert _lib.PATH_NAMES[plan.stats()["path"]] == EMU
    plan.close()
    got = Cd.cpu().numpy()
    assert same_bits(got[5], C0[5]) and same_bits(got[:, 9], C0[:, 9])
    check_bound(A, B, C0, got, 40, t_bits(k), rng)


def test_nonfinite_inputs_fall_back_to_dmma():
    n = 256
    rng = np.random.default_rng(5)
    A = rng.standard_normal((n, n))
    B = rng.standard_normal((n, n))
    A[3, 7] = np.nan
    B[9, 11] = np.inf
    C0 = rng.uniform(-1, 1, (n, n))
    got, path = run_emu(A, B, C0, algo="co2")
    assert path == "dmma_f64"
    Cd = torch.from_numpy(C0.copy()).cuda()
    Ad, Bd = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()   # keep alive across the call
    plan = _lib.Plan(_lib.SR_FP64, "co2", "pooled", n, n, n, 64, 148, -1, 0, 0)
    plan.execute(Cd.data_ptr(), n, Ad.data_ptr(), n, Bd.data_ptr(), n, torch.cuda.current_stream().cuda_stream)
    plan.close()
    dm = Cd.cpu().numpy()
    assert same_bits(got, dm, equal_nan=True)
    assert np.all(np.isnan(got[3])) and not np.isfinite(got[:, 11]).any()


def test_init_identity_overwrites():
    n = 320
    rng = np.random.default_rng(2)
    A = rng.uniform(-3, 3, (n, n))
    B = rng.uniform(-3, 3, (n, n))
    junk = np.full((n, n), 7.5)
    got, path = run_emu(A, B, junk, init_identity=True)
    assert path == EMU
    check_bound(A, B, np.zeros((n, n)), got, 24, t_bits(n), rng)


def test_deterministic_across_schedules_and_runs():
    """No atomics on the local path: every schedule gives the same bits, every run."""
    n = 512
    rng = np.random.default_rng(4)
    A = rng.standard_normal((n, n))
    B = rng.standard_normal((n, n))
    C0 = rng.uniform(-1, 1, (n, n))
    outs = [run_emu(A, B, C0, algo=a)[0] for a in ("co2", "co3", "tar", "sar", "star", "star")]
    for o in outs[1:]:
        assert same_bits(o, outs[0])


def test_large_k_stays_on_dmma():
    """k >= 2^17 would overflow the int32 per-modulus accumulators: DMMA instead."""
    m, n, k = 64, 64, 1 << 17
    rng = np.random.default_rng(9)
    A = rng.standard_normal((m, k))
    B = rng.standard_normal((k, n))
    Ad, Bd = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    Cd = torch.zeros((m, n), dtype=torch.float64, device="cuda")
    plan = _lib.Plan(_lib.SR_FP64, "co2", "pooled", m, n, k, 64, 148, -1, 0,
                     _lib.F_ALLOW_NONPOW2 | _lib.F_FP64_EMU)
    plan.execute(Cd.data_ptr(), n, Ad.data_ptr(), k, Bd.data_ptr(), n, torch.cuda.current_stream().cuda_stream)
    assert _lib.PATH_NAMES[plan.stats()["path"]] == "dmma_f64"
    plan.close()
    assert np.allclose(Cd.cpu().numpy(), A @ B, rtol=1e-9, atol=1e-9)


def test_drop_in_config_flag():
    n = 256
    rng = np.random.default_rng(1)
    A, B, C0 = (rng.standard_normal((n, n)) for _ in range(3))
    cfg = sm.Config(base_dim=32, workers=16, fp64_emulation=True)
    with sm.Executor(cfg) as ex:
        C = sm.Matrix(C0, sm.FLOAT_RING)
        sm.run_algorithm(ex, "star", C, sm.Matrix(A, sm.FLOAT_RING), sm.Matrix(B, sm.FLOAT_RING), sm.FLOAT_RING)
        assert ex.last_stats["path_name"] == EMU
    assert sm.matrices_equal(C.numpy(), C0 + A @ B, tol=1e-12)
