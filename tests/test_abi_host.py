"""CPU: the C-ABI library loads and exports every symbol include/starmm_b200.h
declares; argument validation that needs no GPU; the drop-in host logic
(Config, registry validation order, switch depth, errors) mirrors the reference."""
import ctypes
import json
import os
import re

import numpy as np
import pytest

import paper_1911_05328_b200 as sm
from paper_1911_05328_b200 import _lib

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(REPO, "include", "starmm_b200.h")
SPEC = json.load(open(os.path.join(REPO, "tests", "golden", "ref_spec.json")))


def declared_functions():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(starmm_[a-z_0-9]+)\s*\(", txt)))


def test_header_declares_the_boundary():
    fns = declared_functions()
    for f in ("starmm_plan_create", "starmm_execute", "starmm_plan_stats", "starmm_plan_destroy",
              "starmm_matmul", "starmm_madd", "starmm_atomic_accumulate", "starmm_strerror"):
        assert f in fns


def test_library_exports_every_declared_symbol():
    L = ctypes.CDLL(_lib.LIB_PATH)
    missing = [f for f in declared_functions() if not hasattr(L, f)]
    assert not missing, missing


def test_abi_version_and_strerror():
    L = _lib.lib()
    assert L.starmm_abi_version() == 3
    assert L.starmm_strerror(0) == b"ok"
    assert L.starmm_strerror(2).startswith(b"InvalidSplit")
    assert L.starmm_strerror(1).startswith(b"DimMismatch")


def test_plan_create_validates_before_touching_a_device():
    L = _lib.lib()
    h = ctypes.c_void_p()
    # unknown semiring / algo / mode -> ContractViolation (5)
    assert L.starmm_plan_create(ctypes.byref(h), 9, 0, 0, 64, 64, 64, 32, 1, -1, 0, 0) == 5
    assert L.starmm_plan_create(ctypes.byref(h), 0, 9, 0, 64, 64, 64, 32, 1, -1, 0, 0) == 5
    # raw mode only for co3 (registry.py:34-35)
    assert L.starmm_plan_create(ctypes.byref(h), 0, 2, 1, 64, 64, 64, 32, 1, -1, 0, 0) == 5
    # base_dim must be a power of two (matrix.py:44-45)
    assert L.starmm_plan_create(ctypes.byref(h), 0, 0, 0, 64, 64, 64, 24, 1, -1, 0, 0) == 5
    # check_problem: non-pow2 n -> InvalidSplit (2); n < b -> InvalidSplit
    assert L.starmm_plan_create(ctypes.byref(h), 0, 0, 0, 48, 48, 48, 16, 1, -1, 0, 0) == 2
    assert L.starmm_plan_create(ctypes.byref(h), 0, 0, 0, 16, 16, 16, 32, 1, -1, 0, 0) == 2
    # the fast family needs a ring -> NoAdditiveInverse (7)
    assert L.starmm_plan_create(ctypes.byref(h), 2, 5, 0, 64, 64, 64, 32, 1, -1, 0, 0) == 7
    assert L.starmm_plan_create(ctypes.byref(h), 4, 8, 0, 64, 64, 64, 32, 1, -1, 0, 0) == 7
    # raw mode is accepted by strassen only among the fast family
    assert L.starmm_plan_create(ctypes.byref(h), 0, 6, 1, 64, 64, 64, 32, 1, -1, 0, 0) == 5
    # non-square without ALLOW_NONPOW2 -> DimMismatch (1)
    assert L.starmm_plan_create(ctypes.byref(h), 0, 0, 0, 64, 32, 64, 16, 1, -1, 0, 0) == 1
    # NULL plan pointer
    assert L.starmm_plan_create(None, 0, 0, 0, 64, 64, 64, 16, 1, -1, 0, 0) == 5


def test_status_maps_to_reference_exceptions():
    for code, exc in [(1, sm.DimMismatch), (2, sm.InvalidSplit), (3, sm.NotBaseCase),
                      (4, sm.AllocFailure), (5, sm.ContractViolation), (6, sm.AlignmentError),
                      (8, sm.TooLarge), (9, sm.InternalError), (102, sm.CudaError)]:
        with pytest.raises(exc):
            _lib.check(code)
    _lib.check(0)
    assert issubclass(sm.CudaError, sm.StarMMError)


def test_switch_depth_matches_reference():
    for p, k in SPEC["switch_depth"].items():
        assert sm.switch_depth(int(p)) == k


def test_config_validation_mirrors_reference():
    with pytest.raises(sm.ContractViolation):
        sm.Config(base_dim=24)
    with pytest.raises(sm.ContractViolation):
        sm.Config(workers=0)
    with pytest.raises(sm.ContractViolation):
        sm.Config(cache_size=16, line_size=8)
    with pytest.raises(sm.ContractViolation):
        sm.Config(epsilon=2)
    cfg = sm.Config(base_dim=32)
    with pytest.raises(sm.InvalidSplit):
        cfg.check_problem(48)
    with pytest.raises(sm.InvalidSplit):
        cfg.check_problem(16)
    cfg.check_problem(64)
    sm.Config(allow_nonpow2=True).check_problem(49152)


def _cpu(data, s):
    return sm.Matrix(data, s, device="cpu")


def test_registry_validation_order_without_gpu():
    s = sm.INT_RING
    z = _cpu(np.zeros((4, 4), np.int64), s)
    with sm.Executor(sm.Config(base_dim=2)) as ex:
        with pytest.raises(KeyError):
            sm.run_algorithm(ex, "nope", z, z, z, s)
        with pytest.raises(sm.ContractViolation):
            sm.run_algorithm(ex, "co2", z, z, z, s, mode="weird")
        with pytest.raises(sm.ContractViolation):
            sm.run_algorithm(ex, "star", z, z, z, s, mode="raw")
        with pytest.raises(sm.DimMismatch):
            sm.run_algorithm(ex, "co2", z, _cpu(np.zeros((4, 2), np.int64), s), z, s)
        with pytest.raises(sm.DimMismatch):
            sm.run_algorithm(ex, "co2", z, z, z, sm.FLOAT_RING)
        with pytest.raises(sm.NoAdditiveInverse):
            t = _cpu(np.zeros((4, 4)), sm.TROPICAL)
            sm.run_algorithm(ex, "strassen", t, t, t, sm.TROPICAL)
    with sm.Executor(sm.Config(base_dim=8)) as ex:
        with pytest.raises(sm.InvalidSplit):
            sm.run_algorithm(ex, "co2", z, z, z, s)


def test_regions_and_quadrants():
    s = sm.FLOAT_RING
    M = _cpu(np.arange(16.0).reshape(4, 4), s)
    q = sm.quadrant(M.region(), 0, 1)
    assert (q.row0, q.col0, q.rows, q.cols) == (0, 2, 2, 2)
    assert q.view().tolist() == [[2.0, 3.0], [6.0, 7.0]]
    assert q.data_ptr() == M.data.data_ptr() + 2 * 8
    with pytest.raises(sm.InvalidSplit):
        sm.MatrixRegion(M, 0, 0, 3, 3).quadrant(0, 0)
    with pytest.raises(sm.AlignmentError):
        sm.MatrixRegion(M, 1, 0, 2, 2).tile_range(2)
    with pytest.raises(sm.DimMismatch):
        sm.MatrixRegion(M, 3, 3, 2, 2)


def test_matrices_equal_semantics():
    a = np.array([[1.0, 2.0]])
    assert sm.matrices_equal(a, a + 1e-12)
    assert not sm.matrices_equal(a, a + 1e-6)
    # raw float arrays take the tolerance branch, where inf - inf is NaN: the
    # reference returns False here too (matrix.py:188-191)
    assert not sm.matrices_equal(np.array([[np.inf]]), np.array([[np.inf]]))
    with pytest.raises(sm.DimMismatch):
        sm.matrices_equal(a, np.zeros((2, 2)))


def test_pool_contract_errors_before_any_device_call():
    with pytest.raises(sm.ContractViolation):
        sm.Pool(1, discipline="random")
    with pytest.raises(sm.ContractViolation):
        sm.Pool(1, device="cpu")                    # the pool is the device pool


def test_semiring_elementwise_ops():
    assert sm.INT_RING.add(2, 3) == 5 and sm.INT_RING.mul(2, 3) == 6
    assert sm.TROPICAL.add(2.0, 3.0) == 2.0 and sm.TROPICAL.mul(2.0, 3.0) == 5.0
    assert sm.TROPICAL_I32.mul(np.int32(2 ** 31 - 1), np.int32(-5)) == 2 ** 31 - 1
    assert sm.INT_RING.neg(5) == -5
    with pytest.raises(sm.NoAdditiveInverse):
        sm.TROPICAL.neg(1.0)
    with pytest.raises(KeyError):
        sm.get_semiring("bogus")
    assert sm.get_semiring("tropical_f32").dtype == np.float32


def test_fixture_text_roundtrip_matches_reference_format(tmp_path):
    s = sm.TROPICAL
    M = sm.Matrix(np.array([[0.0, np.inf], [2.0, 3.5]]), s, device="cpu")
    p = tmp_path / "m.txt"
    sm.save_matrix_text(M, p)
    assert p.read_text() == "2 2 tropical\n0 inf\n2 3.5\n"
    back = sm.load_matrix_text(p, device="cpu")
    assert back.semiring is s and np.array_equal(back.numpy(), M.numpy())
    I = sm.Matrix(np.array([[1, -2]], dtype=np.int64), sm.INT_RING, device="cpu")
    sm.save_matrix_text(I, p)
    assert p.read_text() == "1 2 int\n1 -2\n"
    with pytest.raises(sm.DimMismatch):
        p.write_text("2 2 int\n1 2 3\n")
        sm.load_matrix_text(p, device="cpu")


def test_cli_invalid_inputs_exit_2():
    from paper_1911_05328_b200.cli import main
    assert main(["analyze"]) == 2
    assert main(["simulate"]) == 2
    assert main(["run", "--algo", "bogus"]) == 2
    assert main(["bench", "--algos", "strassen"]) == 2


def test_host_schedule_phase1_rule_on_baseline_configs(monkeypatch):
    """The host path's k-outer prologue runs for the compute-bound BASELINE configs
    (3, 4, 5) and not for the PCIe-bound one (config 2: 384 MB up for 1.4 ms of work)."""
    from _host_schedule import host_phase1
    monkeypatch.delenv("STARMM_HOST_PHASE1", raising=False)
    assert host_phase1(4096, 4096, 4096, "int") == [0]
    assert host_phase1(8192, 8192, 8192, "tropical_f32", aliased=True) == [0, 256, 768, 1792, 3840]
    assert host_phase1(16384, 16384, 16384, "float") == [0, 256, 768, 1792, 3840, 7936]
    assert host_phase1(49152, 49152, 49152, "tropical_i32", aliased=True)[-1] == 23040
    assert host_phase1(256, 256, 256, "float") == [0]
    monkeypatch.setenv("STARMM_HOST_PHASE1", "1")
    assert host_phase1(4096, 4096, 4096, "int") == [0, 128, 384, 896, 1920]
    monkeypatch.setenv("STARMM_HOST_PHASE1", "0")
    assert host_phase1(16384, 16384, 16384, "float") == [0]
