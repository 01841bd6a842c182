"""GPU parity at the BASELINE.json configs' FULL sizes.

Sampled-tile protocol: for 64 seeded random 128x128 output
tiles, expected = fold_add(C0[tile], A[rows,:] (x) B[:,cols]) by the pinned CPU
oracle; the reference's own tile hashes (tests/golden/ref_tiles.json, computed
by the reference package's Semiring objects) are checked too.  Plus
size-independent properties over the whole output:
  int64     checksum of checksums: sum(C) = sum(C0) + colsum(A).rowsum(B) mod 2^64
  fp64      the same checksum within tolerance
  (min,+)   idempotence (C (+) X (+) X = C (+) X) and schedule invariance
"""
import hashlib
import json
import os

import numpy as np
import pytest
from _bits import same_bits, diff_count  # noqa: F401
import torch

import paper_1911_05328_b200 as sm
from bench_configs import CONFIGS, make_inputs, sample_tiles, tolerance
from oracle import oracle as O

pytestmark = pytest.mark.gpu

TILES = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "ref_tiles.json")))


def _run(cid, algo="star", C0=None, A=None, B=None, workers=148, **opt):
    cfg = CONFIGS[cid]
    s = sm.get_semiring(cfg["semiring"])
    if A is None:
        A, B, C0 = make_inputs(cid)
    Am = sm.Matrix(A, s)
    Bm = Am if B is A else sm.Matrix(B, s)
    C = sm.Matrix(C0, s)
    conf = sm.Config(base_dim=cfg["b"], workers=workers, allow_nonpow2=(cid == 5), **opt)
    with sm.Executor(conf) as ex:
        sm.run_algorithm(ex, algo, C, Am, Bm, s)
        st = ex.last_stats
    return A, B, C0, C, Am, Bm, st


def _check_tiles(cid, A, B, C0, Cdev, count):
    sr = O.SR_BY_NAME[CONFIGS[cid]["semiring"]]
    n = A.shape[0]
    tol = tolerance(cid, n)
    tiles = sample_tiles(cid, count=count) + [(e["i0"], e["j0"]) for e in TILES[str(cid)]]
    golden = {(e["i0"], e["j0"]): e["sha256"] for e in TILES[str(cid)]}
    for (i0, j0) in tiles:
        got = Cdev[i0:i0 + 128, j0:j0 + 128].cpu().numpy()
        want = np.ascontiguousarray(C0[i0:i0 + 128, j0:j0 + 128])
        O.gemm_fold(sr, want, np.ascontiguousarray(A[i0:i0 + 128]),
                    np.ascontiguousarray(B[:, j0:j0 + 128]), par=True)
        if tol == 0.0:
            assert same_bits(got, want), (cid, i0, j0)
            if (i0, j0) in golden:
                assert hashlib.sha256(got.tobytes()).hexdigest() == golden[(i0, j0)]
        else:
            bound = tol * np.maximum(1.0, np.maximum(np.abs(got), np.abs(want)))
            assert np.all(np.abs(got - want) <= bound), (cid, i0, j0, np.abs(got - want).max())


def test_config2_int64_n4096():
    A, B, C0, C, Am, Bm, st = _run(2)
    assert st["path_name"] == "simt_i64_dp4a"
    _check_tiles(2, A, B, C0, C.data, count=64)
    # checksum of checksums, exact mod 2^64 (torch int64 arithmetic wraps)
    lhs = C.data.sum()
    rhs = torch.from_numpy(C0).cuda().sum() + (Am.data.sum(0) * Bm.data.sum(1)).sum()
    assert int(lhs) == int(rhs)


def test_config2_general_int64_kernel_full_size():
    """The same config through the general 64-bit kernel (fast path off): bit-identical."""
    cfg = CONFIGS[2]
    A, B, C0 = make_inputs(2)
    s = sm.INT_RING
    ref = _run(2, A=A, B=B, C0=C0)[3].data
    C = sm.Matrix(C0, s)
    with sm.Executor(sm.Config(base_dim=cfg["b"], workers=148, fastpath=False)) as ex:
        sm.run_algorithm(ex, "star", C, sm.Matrix(A, s), sm.Matrix(B, s), s)
        assert ex.last_stats["path_name"] == "simt_i64"
    assert torch.equal(C.data, ref)


def test_config3_tropical_f32_n8192():
    A, B, C0, C, Am, Bm, st = _run(3)
    assert st["path_name"] == "simt_f32_s16x2_viaddmnmx"
    _check_tiles(3, A, B, C0, C.data, count=64)
    # idempotence: folding the same product again changes nothing
    first = C.data.clone()
    s = sm.TROPICAL_F32
    with sm.Executor(sm.Config(base_dim=64, workers=148)) as ex:
        sm.run_algorithm(ex, "star", C, Am, Bm, s)
    assert torch.equal(C.data, first)
    # schedule invariance (exact semiring): co2 and tar give the same bits, and so
    # does the general fp32 FADD2/FMNMX3 kernel (fast path off)
    for algo, fast in (("co2", True), ("tar", True), ("star", False)):
        C2 = sm.Matrix(C0, s)
        with sm.Executor(sm.Config(base_dim=64, workers=148, ksplit=1, fastpath=fast)) as ex:
            sm.run_algorithm(ex, algo, C2, Am, Bm, s)
            if not fast:
                assert ex.last_stats["path_name"] == "simt_f32_fadd2_fmnmx3"
        assert torch.equal(C2.data, first), algo


def test_config4_fp64_n16384():
    A, B, C0, C, Am, Bm, st = _run(4)
    assert st["path_name"] == "dmma_f64"
    _check_tiles(4, A, B, C0, C.data, count=64)
    n = A.shape[0]
    lhs = (C.data.sum() - torch.from_numpy(C0).cuda().sum()).item()
    rhs = (Am.data.sum(0) * Bm.data.sum(1)).sum().item()
    assert abs(lhs - rhs) <= 1e-9 * max(1.0, abs(rhs)) * n


def test_config2_opt_in_tensor_cores_full_size():
    """Opt-in tcgen05 kind::i8 path at config 2's full size: the 64 sampled tiles and
    the reference's tile hashes bit-exact, and bit-identical to the default dp4a path."""
    A, B, C0 = make_inputs(2)
    ref = _run(2, A=A, B=B, C0=C0)[3].data
    _, _, _, C, Am, Bm, st = _run(2, A=A, B=B, C0=C0, int_tensor_cores=True)
    assert st["path_name"] == "tcgen05_i8_umma"
    _check_tiles(2, A, B, C0, C.data, count=64)
    assert torch.equal(C.data, ref)


def test_config4_opt_in_fp64_emulation_full_size():
    """Opt-in Ozaki-II at config 4's full size: sampled tiles within the config-4
    tolerance, the checksum of checksums, and bitwise determinism across runs."""
    A, B, C0, C, Am, Bm, st = _run(4, fp64_emulation=True)
    assert st["path_name"] == "ozaki2_fp64_tcgen05_i8x16"
    _check_tiles(4, A, B, C0, C.data, count=64)
    n = A.shape[0]
    lhs = (C.data.sum() - torch.from_numpy(C0).cuda().sum()).item()
    rhs = (Am.data.sum(0) * Bm.data.sum(1)).sum().item()
    assert abs(lhs - rhs) <= 1e-9 * max(1.0, abs(rhs)) * n
    again = _run(4, A=A, B=B, C0=C0, fp64_emulation=True)[3].data
    assert torch.equal(again, C.data)


def test_config5_tropical_i32_n49152():
    A, B, C0, C, Am, Bm, st = _run(5)
    assert A is B
    assert st["path_name"] == "simt_i32_via_f32_carrier"
    assert st["k_chunks"] > 1              # k-outer chunks keep a wave's panels L2-sized
    _check_tiles(5, A, B, C0, C.data, count=64)
    # idempotence on the full 49152^2 output
    first = C.data.clone()
    with sm.Executor(sm.Config(base_dim=64, workers=148, allow_nonpow2=True)) as ex:
        sm.run_algorithm(ex, "star", C, Am, Bm, sm.TROPICAL_I32)
    assert torch.equal(C.data, first)
