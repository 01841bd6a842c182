"""ctypes front-end of the CPU oracle (oracle/starmm_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
CPU-baseline legs of bench.py -- never by the product package.  See the header
of starmm_oracle.c for the reference function each entry point restates.

Semiring ids are the C-ABI ids of include/starmm_b200.h:
  0 "int"  (int64 (+,x), wraps mod 2**64)      semiring.py:130-133
  1 "float" (float64 (+,x))                     semiring.py:135-138
  2 "tropical" (float64 (min,+), +inf zero)     semiring.py:140-143
  3 "tropical_f32" (float32 (min,+))            new id (SURVEY.md finding 1)
  4 "tropical_i32" (int32 (min,+), INT32_MAX = +inf)  new id
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")

SR_INT64, SR_FP64, SR_TROP_F64, SR_TROP_F32, SR_TROP_I32 = range(5)
DTYPES = {SR_INT64: np.int64, SR_FP64: np.float64, SR_TROP_F64: np.float64,
          SR_TROP_F32: np.float32, SR_TROP_I32: np.int32}
SR_BY_NAME = {"int": SR_INT64, "float": SR_FP64, "tropical": SR_TROP_F64,
              "tropical_f32": SR_TROP_F32, "tropical_i32": SR_TROP_I32}
I32_INF = np.iinfo(np.int32).max

_lib = None


def build(force: bool = False) -> str:
    """Compile liboracle.so with the committed Makefile (gcc only)."""
    if force or not os.path.exists(_LIB_PATH) or (
            os.path.getmtime(_LIB_PATH) < os.path.getmtime(os.path.join(_HERE, "starmm_oracle.c"))):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB_PATH)
        i64, vp, ci = ctypes.c_int64, ctypes.c_void_p, ctypes.c_int
        L.oracle_matmul.argtypes = [ci, vp, vp, vp, i64, i64, i64, i64, i64, i64, ci]
        L.oracle_fold.argtypes = [ci, vp, vp, i64, i64, i64, i64]
        L.oracle_gemm_fold.argtypes = [ci, vp, vp, vp, i64, i64, i64, i64, i64, i64, ci]
        L.oracle_serial_mm.argtypes = [ci, vp, vp, vp, i64, i64]
        L.oracle_co3_mm.argtypes = [ci, vp, vp, vp, i64, i64]
        L.oracle_num_threads.restype = ci
        L.oracle_set_threads.argtypes = [ci]
        L.oracle_generate.argtypes = [ci, ci, vp, i64, i64, i64, i64, i64, ctypes.c_uint64,
                                      ctypes.c_uint32, ctypes.c_double, ctypes.c_double,
                                      ctypes.c_double, ci]
        L.oracle_philox4x32_10.argtypes = [ctypes.POINTER(ctypes.c_uint32)] * 3
        L.oracle_philox4x32_10.restype = None
        for f in (L.oracle_matmul, L.oracle_fold, L.oracle_gemm_fold,
                  L.oracle_serial_mm, L.oracle_co3_mm, L.oracle_generate):
            f.restype = ci
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)


def _check2d(a, dt):
    if a.dtype != dt or a.ndim != 2 or a.strides[1] != a.itemsize:
        raise ValueError(f"expected a row-contiguous 2-D {np.dtype(dt)} array")
    return a.strides[0] // a.itemsize


def matmul(sr: int, A: np.ndarray, B: np.ndarray, par: bool = False) -> np.ndarray:
    """Semiring.matmul restated (semiring.py:92-94): A (x) B from the identity."""
    dt = DTYPES[sr]
    lda, ldb = _check2d(A, dt), _check2d(B, dt)
    r, kk = A.shape
    kk2, c = B.shape
    if kk != kk2:
        raise ValueError("inner dimensions differ")
    out = np.empty((r, c), dtype=dt)
    rc = lib().oracle_matmul(sr, _ptr(A), _ptr(B), _ptr(out), r, kk, c, lda, ldb, c, int(par))
    if rc:
        raise RuntimeError(f"oracle_matmul rc={rc}")
    return out


def fold(sr: int, C: np.ndarray, D: np.ndarray) -> None:
    """Semiring.fold_add restated (semiring.py:96-98): C <- C (+) D in place."""
    dt = DTYPES[sr]
    ldc, ldd = _check2d(C, dt), _check2d(D, dt)
    if C.shape != D.shape:
        raise ValueError("shapes differ")
    lib().oracle_fold(sr, _ptr(C), _ptr(D), C.shape[0], C.shape[1], ldc, ldd)


def gemm_fold(sr: int, C: np.ndarray, A: np.ndarray, B: np.ndarray, par: bool = False) -> None:
    """C <- C (+) A (x) B for rectangular panels: the sampled-tile oracle."""
    dt = DTYPES[sr]
    ldc, lda, ldb = _check2d(C, dt), _check2d(A, dt), _check2d(B, dt)
    r, kk = A.shape
    c = B.shape[1]
    if C.shape != (r, c) or B.shape[0] != kk:
        raise ValueError("shape mismatch")
    rc = lib().oracle_gemm_fold(sr, _ptr(C), _ptr(A), _ptr(B), r, kk, c, ldc, lda, ldb, int(par))
    if rc:
        raise RuntimeError(f"oracle_gemm_fold rc={rc}")


def naive_mm(sr: int, A: np.ndarray, B: np.ndarray) -> np.ndarray:
    """kernels.naive_mm restated (kernels.py:28-32)."""
    return matmul(sr, np.ascontiguousarray(A), np.ascontiguousarray(B))


def schedule_mm(sr: int, algo: str, C: np.ndarray, A: np.ndarray, B: np.ndarray, b: int) -> None:
    """The reference schedules at workers=1, bitwise (classic.py:117-236)."""
    dt = DTYPES[sr]
    for M in (C, A, B):
        if M.dtype != dt or not M.flags.c_contiguous:
            raise ValueError("C, A, B must be C-contiguous of the semiring dtype")
    n = C.shape[0]
    fn = lib().oracle_co3_mm if algo == "co3" else lib().oracle_serial_mm
    rc = fn(sr, _ptr(C), _ptr(A), _ptr(B), n, b)
    if rc:
        raise RuntimeError(f"oracle schedule rc={rc}")


def num_threads() -> int:
    return lib().oracle_num_threads()


def set_threads(t: int) -> None:
    lib().oracle_set_threads(int(t))


# ---- the input generator's restatement (csrc/generate.cuh) ---------------------
DIST_IDS = {"uniform_real": 0, "normal": 1, "uniform_int": 2, "graph": 3}


def philox4x32_10(ctr, key):
    """Philox4x32-10 block: 4 x uint32 counter, 2 x uint32 key -> 4 x uint32."""
    c = (ctypes.c_uint32 * 4)(*[int(x) & 0xffffffff for x in ctr])
    k = (ctypes.c_uint32 * 2)(*[int(x) & 0xffffffff for x in key])
    o = (ctypes.c_uint32 * 4)()
    lib().oracle_philox4x32_10(c, k, o)
    return [int(x) for x in o]


def generate(sr: int, dist: str, rows: int, cols: int, row0: int = 0, col0: int = 0, seed: int = 0,
             stream: int = 0, a: float = 0.0, b: float = 1.0, p: float = 0.0,
             zero_diag: bool = False) -> np.ndarray:
    """Host regeneration of a device-generated panel (bit for bit)."""
    out = np.empty((rows, cols), dtype=DTYPES[sr])
    rc = lib().oracle_generate(sr, DIST_IDS[dist], _ptr(out), cols, rows, cols, row0, col0,
                               ctypes.c_uint64(seed), ctypes.c_uint32(stream), ctypes.c_double(a),
                               ctypes.c_double(b), ctypes.c_double(p), 1 if zero_diag else 0)
    if rc:
        raise RuntimeError(f"oracle_generate rc={rc}")
    return out
