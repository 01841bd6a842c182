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


# ---- the input generator's restatement (csrc/generate.cuh) --------------------------
def test_philox4x32_10_known_answers():
    """Random123's published Philox4x32-10 known-answer vectors."""
    assert O.philox4x32_10([0, 0, 0, 0], [0, 0]) == [0x6627e8d5, 0xe169c58d, 0xbc57ac4c, 0x9b00dbd8]
    assert O.philox4x32_10([0xffffffff] * 4, [0xffffffff] * 2) == \
        [0x408f276d, 0x41c83b0e, 0xa20bc7c6, 0x6d5451fd]
    assert O.philox4x32_10([0x243f6a88, 0x85a308d3, 0x13198a2e, 0x03707344], [0xa4093822, 0x299f31d0]) == \
        [0xd16cfe09, 0x94fdcceb, 0x5001e420, 0x24126ea1]


@pytest.mark.parametrize("cid", [1, 2, 3, 4, 5])
def test_generator_is_panel_invariant_and_matches_the_config_distribution(cid):
    """Element (i, j) depends only on (seed, stream, i, j): a panel cut anywhere equals
    the same window of a larger panel; moments match BASELINE's distributions."""
    from bench_configs import device_gen_spec
    sr = O.SR_BY_NAME[CONFIGS[cid]["semiring"]]
    spec = dict(device_gen_spec(cid, "A"))
    spec["stream"] = spec.pop("stream_id")
    big = O.generate(sr, rows=200, cols=300, row0=1000, col0=2000, **spec)
    sub = O.generate(sr, rows=37, cols=51, row0=1100, col0=2222, **spec)
    assert np.array_equal(big[100:137, 222:273], sub)
    x = big.astype(np.float64)
    if cid == 4:
        assert abs(x.mean()) < 0.02 and abs(x.std() - 1.0) < 0.02
    if cid == 1:
        assert x.min() >= -1 and x.max() < 1 and abs(x.mean()) < 0.02
    if cid == 2:
        assert x.min() == -16 and x.max() == 16 and abs(x.mean()) < 0.2
    if cid == 3:
        fin = np.isfinite(x)
        assert abs(fin.mean() - 0.1) < 0.01 and x[fin].min() >= 1 and x[fin].max() <= 100
    if cid == 5:
        assert x.min() >= 1 and x.max() <= 10 ** 6
        d = O.generate(sr, rows=64, cols=64, row0=0, col0=0, **spec)
        assert np.all(np.diag(d) == 0)                  # 0 on the diagonal


def test_generator_normal_is_accurate_box_muller():
    """The + - * / log and cos of the normal transform agree with libm to ~1e-15."""
    import math
    seed, stream = 3, 0
    z = O.generate(O.SR_FP64, "normal", 4, 64, seed=seed, stream=stream)
    for j in range(64):
        x = O.philox4x32_10([j, 0, stream, 0], [seed, 0])
        ua = (x[0] << 21) | (x[1] >> 11)
        ub = (x[2] << 21) | (x[3] >> 11)
        u1, u2 = (ua + 1) * 2.0 ** -53, ub * 2.0 ** -53
        want = math.sqrt(-2.0 * math.log(u1)) * math.cos(2 * math.pi * u2)
        assert abs(z[0, j] - want) <= 1e-13 * max(1.0, abs(want)), (j, z[0, j], want)
