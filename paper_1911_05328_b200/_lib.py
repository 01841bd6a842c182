"""ctypes binding of libstarmm_b200.so (include/starmm_b200.h).

The product path has no CPU fallback: if the shared library is missing or
cannot be loaded, every entry point raises (StarMMError subclass
``NativeUnavailable``).  Build it with ``python __graft_entry__.py`` or
``make -C paper_1911_05328_b200/csrc``.
"""
from __future__ import annotations

import ctypes
import os
import threading

from . import errors

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libstarmm_b200.so")

# enums (include/starmm_b200.h)
SR_INT64, SR_FP64, SR_TROPICAL_F64, SR_TROPICAL_F32, SR_TROPICAL_I32 = range(5)
ALGO_IDS = {"co2": 0, "co3": 1, "tar": 2, "sar": 3, "star": 4, "strassen": 5, "sar-strassen": 6,
            "star-strassen-1": 7, "star-strassen-2": 8}
ALLOC_IDS = {"pooled": 0, "raw": 1}
F_ASYNC, F_NO_FASTPATH, F_INIT_IDENTITY, F_ALLOW_NONPOW2, F_TIME_MAIN = 0x1, 0x2, 0x4, 0x8, 0x10
F_INT_TENSOR = 0x20
F_FP64_EMU = 0x40

PATH_NAMES = {1: "dmma_f64", 2: "simt_i64", 3: "simt_i64_narrow_i32", 4: "simt_f32_fadd2_fmnmx3",
              5: "simt_i32_via_f32_carrier", 6: "simt_i32_viaddmnmx", 7: "simt_i32_saturating",
              8: "simt_f64_min", 9: "simt_i64_dp4a", 10: "simt_f32_s16x2_viaddmnmx",
              11: "simt_i32_s16x2_viaddmnmx", 12: "simt_f64trop_s16x2_viaddmnmx",
              13: "simt_f64trop_via_f32_carrier", 14: "tcgen05_i8_umma",
              15: "ozaki2_fp64_tcgen05_i8x16", 16: "minplus_ordered_leaf_order",
              17: "tcgen05_i8_radix256_int64"}
ABI_VERSION = 3


class StarmmStats(ctypes.Structure):
    _fields_ = [(name, ctypes.c_int64) for name in (
        "pool_total_allocated_bytes", "pool_high_water_bytes", "pool_fresh_count",
        "pool_reuse_count", "tile_serializations", "pair_count", "pair_transitions",
        "lazy_temp_acquires", "raw_alloc_count", "raw_alloc_bytes", "tasks", "workers",
        "ksplit", "tar_levels", "kernel_launches", "path", "executes", "main_kernel_ns",
        "main_kernel_launches", "balanced_workers", "live_leaves_max", "guard_syncs",
        "candidates", "cluster_size", "k_chunks")]

    def to_dict(self):
        return {name: int(getattr(self, name)) for name, _ in self._fields_}


class PoolCounts(ctypes.Structure):
    """starmm_pool_counts: the device block pool's counters (pool.py:158-167)."""
    _fields_ = [(name, ctypes.c_int64) for name in (
        "allocated_bytes", "cached_bytes", "issued_bytes", "high_water_bytes", "fresh_count",
        "reuse_count", "cross_stream_waits", "trims")]

    def to_dict(self):
        return {name: int(getattr(self, name)) for name, _ in self._fields_}


_lib = None
_lock = threading.Lock()

# status -> exception class (errors.py:4-41)
_STATUS_EXC = {
    1: errors.DimMismatch, 2: errors.InvalidSplit, 3: errors.NotBaseCase,
    4: errors.AllocFailure, 5: errors.ContractViolation, 6: errors.AlignmentError,
    7: errors.NoAdditiveInverse, 8: errors.TooLarge, 9: errors.InternalError,
}


def lib():
    """Load the native library (once).  Raises NativeUnavailable if absent."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise errors.NativeUnavailable(
                f"{LIB_PATH} is not built; run `make -C {os.path.join(_HERE, 'csrc')}` "
                "(there is no CPU fallback)")
        try:
            L = ctypes.CDLL(LIB_PATH)
        except OSError as e:
            raise errors.NativeUnavailable(f"cannot load {LIB_PATH}: {e}") from e
        i64, vp, ci = ctypes.c_int64, ctypes.c_void_p, ctypes.c_int
        L.starmm_abi_version.restype = ci
        L.starmm_strerror.restype = ctypes.c_char_p
        L.starmm_strerror.argtypes = [ci]
        L.starmm_device_sm_count.argtypes = [ci]
        L.starmm_device_sm_count.restype = ci
        L.starmm_plan_create.argtypes = [ctypes.POINTER(vp), ci, ci, ci, i64, i64, i64, ci, ci,
                                         ci, ci, ci]
        L.starmm_plan_create.restype = ci
        L.starmm_execute.argtypes = [vp, vp, i64, vp, i64, vp, i64, vp]
        L.starmm_execute.restype = ci
        L.starmm_execute_host.argtypes = [vp, vp, i64, vp, i64, vp, i64, vp, i64]
        L.starmm_execute_host.restype = ci
        L.starmm_plan_set_strassen_leaf.argtypes = [vp, i64]
        L.starmm_plan_set_strassen_leaf.restype = ci
        L.starmm_plan_set_peers.argtypes = [vp, ci, ctypes.POINTER(vp), i64, i64]
        L.starmm_plan_set_peers.restype = ci
        L.starmm_ipc_handle.argtypes = [vp, ctypes.c_char_p]
        L.starmm_ipc_handle.restype = ci
        L.starmm_ipc_open.argtypes = [ctypes.c_char_p, ctypes.POINTER(vp)]
        L.starmm_ipc_open.restype = ci
        L.starmm_ipc_close.argtypes = [vp]
        L.starmm_ipc_close.restype = ci
        L.starmm_plan_stats.argtypes = [vp, ctypes.POINTER(StarmmStats)]
        L.starmm_plan_stats.restype = ci
        L.starmm_plan_reset_stats.argtypes = [vp]
        L.starmm_plan_reset_stats.restype = ci
        L.starmm_plan_destroy.argtypes = [vp]
        L.starmm_plan_destroy.restype = None
        L.starmm_matmul.argtypes = [ci, vp, i64, vp, i64, vp, i64, i64, i64, i64, vp, ci]
        L.starmm_matmul.restype = ci
        L.starmm_madd.argtypes = [ci, vp, i64, vp, i64, i64, i64, vp, ci]
        L.starmm_madd.restype = ci
        L.starmm_atomic_accumulate.argtypes = [ci, vp, i64, vp, i64, i64, i64, vp, ci]
        L.starmm_atomic_accumulate.restype = ci
        L.starmm_generate.argtypes = [ci, ci, vp, i64, i64, i64, i64, i64, ctypes.c_uint64,
                                      ctypes.c_uint32, ctypes.c_double, ctypes.c_double,
                                      ctypes.c_double, ci, vp]
        L.starmm_generate.restype = ci
        L.starmm_pool_acquire.argtypes = [ci, i64, vp, ctypes.POINTER(vp), ctypes.POINTER(ci)]
        L.starmm_pool_acquire.restype = ci
        L.starmm_pool_release.argtypes = [ci, vp, vp]
        L.starmm_pool_release.restype = ci
        L.starmm_pool_counts_get.argtypes = [ci, ctypes.POINTER(PoolCounts)]
        L.starmm_pool_counts_get.restype = ci
        L.starmm_pool_reset.argtypes = [ci]
        L.starmm_pool_reset.restype = ci
        L.starmm_pool_set_limit.argtypes = [ci, i64, ctypes.POINTER(i64)]
        L.starmm_pool_set_limit.restype = ci
        L.starmm_pool_set_discipline.argtypes = [ci, ci]
        L.starmm_pool_set_discipline.restype = ci
        if L.starmm_abi_version() != ABI_VERSION:
            raise errors.NativeUnavailable("libstarmm_b200.so ABI version mismatch")
        _lib = L
    return _lib


def check(status: int, what: str = "") -> None:
    """Raise the reference exception class matching a C-ABI status."""
    if status == 0:
        return
    msg = lib().starmm_strerror(status).decode()
    if what:
        msg = f"{what}: {msg}"
    if status >= 100:
        raise errors.CudaError(msg)
    raise _STATUS_EXC.get(status, errors.InternalError)(msg)


class Plan:
    """Owns one starmm_plan (Executor + Config analogue for one problem shape)."""

    def __init__(self, sr: int, algo: str, mode: str, m: int, n: int, k: int, base_dim: int,
                 workers: int, ksplit_log2: int, device: int, flags: int):
        self._h = ctypes.c_void_p()
        check(lib().starmm_plan_create(ctypes.byref(self._h), sr, ALGO_IDS[algo], ALLOC_IDS[mode],
                                       m, n, k, base_dim, workers, ksplit_log2, device, flags),
              "starmm_plan_create")
        self.sr, self.algo, self.mode = sr, algo, mode
        self.m, self.n, self.k, self.device, self.flags = m, n, k, device, flags

    def execute(self, C_ptr: int, ldc: int, A_ptr: int, lda: int, B_ptr: int, ldb: int,
                stream: int) -> None:
        check(lib().starmm_execute(self._h, C_ptr, ldc, A_ptr, lda, B_ptr, ldb, stream),
              "starmm_execute")

    def execute_host(self, C_ptr: int, ldc: int, A_ptr: int, lda: int, B_ptr: int, ldb: int,
                     stream: int, block_rows: int = 0) -> None:
        check(lib().starmm_execute_host(self._h, C_ptr, ldc, A_ptr, lda, B_ptr, ldb, stream,
                                        block_rows), "starmm_execute_host")

    def set_strassen_leaf(self, leaf: int) -> None:
        check(lib().starmm_plan_set_strassen_leaf(self._h, int(leaf)), "starmm_plan_set_strassen_leaf")

    def set_peers(self, bases, ld: int, rows_per_part: int) -> None:
        """Route every tile's atomic-madd to the owner part's buffer (fused k-split combine)."""
        arr = (ctypes.c_void_p * max(1, len(bases)))(*[ctypes.c_void_p(b) for b in bases])
        check(lib().starmm_plan_set_peers(self._h, len(bases), arr, ld, rows_per_part),
              "starmm_plan_set_peers")

    def stats(self) -> dict:
        st = StarmmStats()
        check(lib().starmm_plan_stats(self._h, ctypes.byref(st)), "starmm_plan_stats")
        d = st.to_dict()
        d["path_name"] = PATH_NAMES.get(d["path"], "none")
        return d

    def reset_stats(self) -> None:
        check(lib().starmm_plan_reset_stats(self._h), "starmm_plan_reset_stats")

    def close(self) -> None:
        if self._h:
            lib().starmm_plan_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):  # pragma: no cover - best effort
        try:
            self.close()
        except Exception:
            pass


def ipc_handle(ptr: int) -> bytes:
    buf = ctypes.create_string_buffer(64)
    check(lib().starmm_ipc_handle(ptr, buf), "starmm_ipc_handle")
    return buf.raw


def ipc_open(handle: bytes) -> int:
    out = ctypes.c_void_p()
    check(lib().starmm_ipc_open(handle, ctypes.byref(out)), "starmm_ipc_open")
    return int(out.value)


def ipc_close(ptr: int) -> None:
    check(lib().starmm_ipc_close(ptr), "starmm_ipc_close")


# ---- the device block pool (starmm_pool_*, csrc/arena.h) ----------------------
def pool_acquire(device: int, nbytes: int, stream: int = 0):
    """(device pointer, fresh) of an exact-size block from the device's pool."""
    out = ctypes.c_void_p()
    fresh = ctypes.c_int(0)
    check(lib().starmm_pool_acquire(device, nbytes, stream, ctypes.byref(out), ctypes.byref(fresh)),
          "starmm_pool_acquire")
    return int(out.value), bool(fresh.value)


def pool_release(device: int, ptr: int, stream: int = 0) -> None:
    check(lib().starmm_pool_release(device, ptr, stream), "starmm_pool_release")


def pool_counts(device: int) -> dict:
    c = PoolCounts()
    check(lib().starmm_pool_counts_get(device, ctypes.byref(c)), "starmm_pool_counts_get")
    return c.to_dict()


def pool_reset(device: int) -> None:
    check(lib().starmm_pool_reset(device), "starmm_pool_reset")


def pool_set_discipline(device: int, fifo: bool) -> None:
    check(lib().starmm_pool_set_discipline(device, 1 if fifo else 0), "starmm_pool_set_discipline")


def pool_set_limit(device: int, nbytes: int) -> int:
    """Set the pool's owned-bytes limit; returns the previous one."""
    old = ctypes.c_int64(0)
    check(lib().starmm_pool_set_limit(device, nbytes, ctypes.byref(old)), "starmm_pool_set_limit")
    return int(old.value)
