"""Executor: owns the device plans, the block pool and the metrics (runtime.py:57-249).

The reference runs its task trees on p Python worker threads with work
stealing.  Here the workers are persistent CTAs on the GPU (one per SM) and
the task tree is flattened into leaf tasks (output tile x k-slice) inside
libstarmm_b200; the Executor keeps the reference's surface -- context
manager, ``run``, ``parallel``, ``acquire_temp``/``release_temp``, ``pool``,
``metrics`` -- and caches one native plan per problem shape, so a long-lived
Executor reuses its device arena across calls the way the reference pool
survives until ``reset`` (pool.py:148-156).
"""
from __future__ import annotations

import threading

import torch

from . import _lib
from .errors import ContractViolation, DimMismatch
from .matrix import Matrix
from .metrics import Metrics
from .pool import Pool

__all__ = ["Executor", "current_worker_index"]

_tls = threading.local()


def current_worker_index():
    """Index of the worker executing the calling task (0 outside the pool)."""
    return getattr(_tls, "worker", 0)


class Executor:
    """Owns the native plans, the block pool, metrics and the CUDA stream binding."""

    def __init__(self, cfg, pool_discipline="lifo", tracer=None):
        if tracer is not None:
            # element-granularity CPU traces feed the LRU simulator, which is out of
            # scope for the GPU path (trace.py / cachesim.py OUT)
            raise ContractViolation("access tracing is not supported by the GPU executor")
        self.cfg = cfg
        self.p = cfg.workers
        self.device = cfg.device if cfg.device is not None else (
            torch.cuda.current_device() if torch.cuda.is_available() else 0)
        self._pool_discipline = pool_discipline
        self._pool = None            # the device pool's per-worker view, made on first use
        if pool_discipline not in ("lifo", "fifo"):
            raise ContractViolation(f"unknown pool discipline {pool_discipline!r}")
        self.metrics = Metrics()
        self.tracer = None
        self._plans = {}
        self._closed = False
        self.last_stats = {}

    @property
    def pool(self):
        """Pool view of the device block pool (pool.py:67-167); FIFO while this executor
        lives if it was built with pool_discipline="fifo" (the sabotage hook)."""
        if self._pool is None:
            self._pool = Pool(self.p, discipline=self._pool_discipline, device=f"cuda:{self.device}")
        return self._pool

    # -- lifecycle --------------------------------------------------------
    def close(self):
        if self._closed:
            return
        self._closed = True
        for plan in self._plans.values():
            plan.close()
        self._plans.clear()
        if self._pool is not None:
            self._pool.close()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- task execution (reference surface) --------------------------------
    def run(self, fn):
        """Execute `fn` as the root task and block until it completes."""
        self.metrics.running = True
        try:
            fn()
        finally:
            self.metrics.running = False

    def parallel(self, thunks):
        """Run zero-argument callables as sibling tasks (host-level; the GPU schedules
        never go through here -- their parallelism is the CUDA grid)."""
        for fn in thunks:
            fn()

    def current_worker(self):
        return current_worker_index()

    # -- native plans ------------------------------------------------------
    def plan(self, s, algo, mode, m, n, k, flags):
        cfg = self.cfg
        ks = -1 if cfg.ksplit is None else int(cfg.ksplit)
        if not cfg.fastpath:
            flags |= _lib.F_NO_FASTPATH
        if cfg.allow_nonpow2:
            flags |= _lib.F_ALLOW_NONPOW2
        if cfg.int_tensor_cores:
            flags |= _lib.F_INT_TENSOR
        if cfg.fp64_emulation:
            flags |= _lib.F_FP64_EMU
        key = (s.sr_id, algo, mode, m, n, k, flags, ks)
        p = self._plans.get(key)
        if p is None:
            p = _lib.Plan(s.sr_id, algo, mode, m, n, k, cfg.base_dim, cfg.workers, ks,
                          self.device, flags)
            if cfg.strassen_leaf is not None:
                p.set_strassen_leaf(cfg.strassen_leaf)
            self._plans[key] = p
        return p

    def execute(self, algo, C, A, B, s, mode="pooled", flags=0):
        """C <- C (+) A (x) B through the C ABI on the current stream (blocking)."""
        Cd, Ad, Bd = (x.data if isinstance(x, Matrix) else x for x in (C, A, B))
        m, n = Cd.shape
        k = Ad.shape[1]
        plan = self.plan(s, algo, mode, m, n, k, flags)
        plan.reset_stats()
        stream = torch.cuda.current_stream(Cd.device).cuda_stream
        with torch.cuda.device(Cd.device):
            plan.execute(Cd.data_ptr(), Cd.stride(0), Ad.data_ptr(), Ad.stride(0),
                         Bd.data_ptr(), Bd.stride(0), stream)
        st = plan.stats()
        self.last_stats = st
        self.pool.absorb_device(st)
        self.metrics.absorb_device(st, s.dtype.itemsize)
        return st

    def execute_host(self, algo, C, A, B, s, mode="pooled", flags=0, block_rows=0):
        """C <- C (+) A (x) B with C, A, B in HOST memory (CPU torch tensors, pinned for
        full copy/compute overlap, or numpy arrays): starmm_execute_host streams row
        blocks through the device.  C is updated in place."""
        import numpy as np
        ts = []
        for x in (C, A, B):
            if isinstance(x, np.ndarray):
                x = torch.from_numpy(x)
            if x.device.type != "cpu" or x.dtype != s.torch_dtype or x.dim() != 2:
                raise DimMismatch(f"host buffers must be 2-D CPU {s.torch_dtype} tensors")
            if x.shape[1] > 1 and x.stride(1) != 1:
                raise DimMismatch("row-major host buffers are required")
            ts.append(x)
        Ct, At, Bt = ts
        m, n = Ct.shape
        k = At.shape[1]
        if At.shape[0] != m or Bt.shape != (k, n):
            raise DimMismatch("A, B, C shapes do not compose")
        plan = self.plan(s, algo, mode, m, n, k, flags)
        plan.reset_stats()
        dev = torch.device("cuda", self.device)
        stream = torch.cuda.current_stream(dev).cuda_stream
        with torch.cuda.device(dev):
            plan.execute_host(Ct.data_ptr(), max(1, Ct.stride(0)), At.data_ptr(),
                              max(1, At.stride(0)), Bt.data_ptr(), max(1, Bt.stride(0)), stream,
                              block_rows)
        st = plan.stats()
        self.last_stats = st
        self.pool.absorb_device(st)
        self.metrics.absorb_device(st, s.dtype.itemsize)
        return st

    # -- temporaries (runtime.py:198-229) ------------------------------------
    def acquire_temp(self, dim, semiring, depth, mode="pooled", lazy=False, virgin=True):
        if mode == "pooled":
            words = (dim * dim * semiring.dtype.itemsize + 7) // 8
            token = self.pool.acquire(self.current_worker(), words)
            m = token.as_matrix(dim, semiring)
        elif mode == "raw":
            m = Matrix(torch.empty((dim, dim), dtype=semiring.torch_dtype,
                                   device=f"cuda:{self.device}"), semiring)
            self.metrics.raw_alloc_count += 1
            self.metrics.raw_alloc_elements += dim * dim
            token = None
        else:
            raise ValueError(f"unknown allocation mode {mode!r}")
        if virgin:
            m.ensure_table(min(self.cfg.base_dim, dim)).mark_virgin()
        if lazy:
            self.metrics.lazy_temp_acquires += 1
        return token, m

    def release_temp(self, token, depth=0, lazy=False):
        if token is not None:
            self.pool.release(token)

    def register_matrix(self, m):
        pass

    def trace_read(self, region):
        pass

    def trace_write(self, region):
        pass
