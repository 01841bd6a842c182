"""CPU: pin the oracle (oracle/starmm_oracle.c) against the REFERENCE's own outputs.

tests/golden/* were produced by importing the reference package itself
(oracle/gen_golden.py).  The oracle must reproduce them bit for bit -- for
the float64 schedules too, since it restates the reference's loop order
without FMA contraction.
"""
import hashlib
import json
import os

import numpy as np
import pytest

from bench_configs import CONFIGS, make_inputs
from oracle import oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")
SMALL = np.load(os.path.join(GOLD, "ref_small.npz"))
SPEC = json.load(open(os.path.join(GOLD, "ref_spec.json")))
TILES = json.load(open(os.path.join(GOLD, "ref_tiles.json")))
CASES = [(2, 2), (2, 8), (4, 16), (8, 32), (32, 64)]
SIDS = [("int", O.SR_INT64), ("float", O.SR_FP64), ("tropical", O.SR_TROP_F64)]


@pytest.mark.parametrize("sid,sr", SIDS)
@pytest.mark.parametrize("b,n", CASES)
def test_naive_matches_reference(sid, sr, b, n):
    key = f"{sid}_n{n}_b{b}"
    out = O.naive_mm(sr, SMALL[key + "_A"], SMALL[key + "_B"])
    assert np.array_equal(out, SMALL[key + "_naive"])


@pytest.mark.parametrize("algo", ["co2", "co3", "tar", "sar", "star"])
@pytest.mark.parametrize("sid,sr", SIDS)
@pytest.mark.parametrize("b,n", CASES)
def test_schedules_match_reference_bitwise(algo, sid, sr, b, n):
    key = f"{sid}_n{n}_b{b}"
    C = SMALL[key + "_C0"].copy()
    O.schedule_mm(sr, algo, C, SMALL[key + "_A"], SMALL[key + "_B"], b)
    assert np.array_equal(C, SMALL[f"{key}_{algo}"])


def test_spec_known_answers():
    assert O.naive_mm(O.SR_INT64, np.array([[2]], np.int64), np.array([[3]], np.int64)).tolist() \
        == SPEC["naive_1x1"]
    assert O.naive_mm(O.SR_INT64, np.array([[1, 2], [3, 4]], np.int64),
                      np.array([[5, 6], [7, 8]], np.int64)).tolist() == SPEC["naive_2x2"] \
        == [[19, 22], [43, 50]]
    t = O.naive_mm(O.SR_TROP_F64, np.array([[0, 1], [2, 3]], float), np.array([[0, 4], [1, 0]], float))
    assert t.tolist() == SPEC["naive_trop_2x2"] == [[0, 1], [2, 3]]
    C = np.array([[5]], np.int64)
    O.gemm_fold(O.SR_INT64, C, np.array([[2]], np.int64), np.array([[3]], np.int64))
    assert C.tolist() == SPEC["base_kernel_b1"] == [[11]]
    C = np.array([[4.0]])
    O.gemm_fold(O.SR_TROP_F64, C, np.array([[1.0]]), np.array([[2.0]]))
    assert C.tolist() == SPEC["base_kernel_trop_b1"] == [[3.0]]
    C = np.array([[1, 2], [3, 4]], np.int64)
    O.fold(O.SR_INT64, C, np.array([[10, 20], [30, 40]], np.int64))
    assert C.tolist() == SPEC["madd_int"]
    C = np.array([[1.0, 5.0]])
    O.fold(O.SR_TROP_F64, C, np.array([[3.0, 2.0]]))
    assert C.tolist() == SPEC["madd_trop"]
    w = O.naive_mm(O.SR_INT64, np.array([[2 ** 62]], np.int64), np.array([[4]], np.int64))
    assert w.tolist() == SPEC["int_wrap"] == [[0]]


def test_pr1_star_bitwise():
    """BASELINE config 1: the oracle's serial STAR equals the reference star_mm(workers=1)."""
    A, B, C0 = make_inputs(1)
    C = C0.copy()
    O.schedule_mm(O.SR_FP64, "star", C, A, B, 32)
    assert np.array_equal(C, np.load(os.path.join(GOLD, "ref_pr1.npz"))["star"])


def _tile_sha(cid, A, B, C0, i0, j0):
    sr = O.SR_BY_NAME[CONFIGS[cid]["semiring"]]
    Ct = np.ascontiguousarray(C0[i0:i0 + 128, j0:j0 + 128])
    O.gemm_fold(sr, Ct, np.ascontiguousarray(A[i0:i0 + 128]), np.ascontiguousarray(B[:, j0:j0 + 128]),
                par=True)
    return hashlib.sha256(Ct.tobytes()).hexdigest()


@pytest.mark.parametrize("cid", [2, 3])
def test_config_tiles_match_reference(cid):
    A, B, C0 = make_inputs(cid)
    for e in TILES[str(cid)]:
        assert _tile_sha(cid, A, B, C0, e["i0"], e["j0"]) == e["sha256"]


@pytest.mark.slow
@pytest.mark.parametrize("cid", [4, 5])
def test_config_tiles_match_reference_large(cid):
    A, B, C0 = make_inputs(cid)
    for e in TILES[str(cid)]:
        if cid == 4:   # fp64: the oracle restates the reference loop order, so bits match
            assert _tile_sha(cid, A, B, C0, e["i0"], e["j0"]) == e["sha256"]
        else:
            assert _tile_sha(cid, A, B, C0, e["i0"], e["j0"]) == e["sha256"]


def test_parallel_oracle_is_bitwise_serial():
    rng = np.random.default_rng(7)
    A = rng.standard_normal((96, 80))
    B = rng.standard_normal((80, 72))
    assert np.array_equal(O.matmul(O.SR_FP64, A, B, par=False), O.matmul(O.SR_FP64, A, B, par=True))


def test_new_semiring_oracles_agree_with_float64_tropical():
    """fp32 / int32 (min,+) oracles == reference tropical on integer-valued up-casts."""
    rng = np.random.default_rng(11)
    A = rng.integers(0, 1000, (40, 50)).astype(np.float64)
    B = rng.integers(0, 1000, (50, 30)).astype(np.float64)
    A[rng.random(A.shape) < 0.1] = np.inf
    B[rng.random(B.shape) < 0.1] = np.inf
    ref = O.matmul(O.SR_TROP_F64, A, B)
    f32 = O.matmul(O.SR_TROP_F32, A.astype(np.float32), B.astype(np.float32))
    assert np.array_equal(f32.astype(np.float64), ref)
    Ai = np.where(np.isinf(A), O.I32_INF, A).astype(np.int32)
    Bi = np.where(np.isinf(B), O.I32_INF, B).astype(np.int32)
    i32 = O.matmul(O.SR_TROP_I32, Ai, Bi)
    assert np.array_equal(np.where(i32 == O.I32_INF, np.inf, i32.astype(np.float64)), ref)


def test_i32_tropical_saturation():
    big = O.I32_INF - 5
    A = np.array([[big, O.I32_INF]], np.int32)
    B = np.array([[10], [0]], np.int32)
    assert O.matmul(O.SR_TROP_I32, A, B).tolist() == [[O.I32_INF]]
    A = np.array([[-2 ** 31 + 3]], np.int32)
    B = np.array([[-10]], np.int32)
    assert O.matmul(O.SR_TROP_I32, A, B).tolist() == [[-2 ** 31]]


SZ = np.load(os.path.join(GOLD, "ref_signed_zero.npz"))
SZ_CASES = [(1, 4), (2, 8), (4, 16), (8, 32), (16, 32), (32, 32)]


@pytest.mark.parametrize("algo", ["co2", "co3", "tar", "sar", "star"])
@pytest.mark.parametrize("b,n", SZ_CASES)
def test_signed_zero_schedules_bitwise(algo, b, n):
    """+-0.0-heavy tropical operands: the oracle's leaf order (first minimum inside a
    b-leaf, semiring.py:56-58) and np.minimum's second-operand tie (semiring.py:126-127)
    reproduce the reference bit for bit, sign of zero included."""
    from _bits import same_bits
    key = f"n{n}_b{b}"
    C = SZ[key + "_C0"].copy()
    O.schedule_mm(O.SR_TROP_F64, algo, C, SZ[key + "_A"], SZ[key + "_B"], b)
    assert same_bits(C, SZ[f"{key}_{algo}"])


@pytest.mark.parametrize("b,n", SZ_CASES)
def test_signed_zero_naive_and_madd_bitwise(b, n):
    from _bits import same_bits
    key = f"n{n}_b{b}"
    assert same_bits(O.naive_mm(O.SR_TROP_F64, SZ[key + "_A"], SZ[key + "_B"]), SZ[key + "_naive"])
    C = SZ[key + "_C0"].copy()
    O.fold(O.SR_TROP_F64, C, SZ[key + "_A"])
    assert same_bits(C, SZ[key + "_madd"])
    # the golden really exercises both signs of zero
    assert np.any(np.signbit(SZ[key + "_star"]) & (SZ[key + "_star"] == 0))
