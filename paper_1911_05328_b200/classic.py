"""Classical semiring matrix multiplication schedules (reference classic.py:1-316).

Five schedules over the same eight-way quadrant recursion, differing only in
how they order tasks and where temporaries come from.  On the B200 each
schedule is a write-back protocol of one persistent tile kernel
(csrc/common.cuh); the recursion's top ``s`` levels
become k-slices of each output tile, the levels below run serially inside a
CTA (serial SAR = in place, serial CO2 phases = the in-CTA k loop):

* ``co2``  -- no concurrent k-halves: exclusive read-fold-write of C.
* ``co3``  -- k-slice 0 folds into C, slices 1.. store into workspace
  temporaries (virgin first touch), then merge_tasks folds them bottom-up.
* ``tar``  -- all k-slices concurrent; each CTA's accumulator is its worker's
  b x b block, merged with per-element atomic-madd.
* ``sar``  -- sibling k-halves race on a per-tile pair state; only a half that
  finds its sibling running buys a temporary from its worker's LIFO pool;
  every merge goes through the tile's exclusion slot.
* ``star`` -- TAR protocol for the top switch_depth(p) split levels, SAR below.

All entry points compute C <- C (+) A (x) B.
"""
from __future__ import annotations

import torch

from . import _lib
from .errors import ContractViolation, DimMismatch
from .matrix import Matrix

__all__ = [
    "co2", "co3", "tar_mm", "sar_mm", "star_mm",
    "atomic_accumulate", "switch_depth", "host_mm",
    "PAIR_EMPTY", "PAIR_FIRST_RUNNING", "PAIR_FIRST_DONE",
]

PAIR_EMPTY = "Empty"
PAIR_FIRST_RUNNING = "FirstRunning"
PAIR_FIRST_DONE = "FirstDone"


def switch_depth(p):
    """Hybrid switch depth: smallest k with 4**k >= p (classic.py:78-83)."""
    k = 0
    while 4 ** k < p:
        k += 1
    return k


def _region(x):
    return x.region() if isinstance(x, Matrix) else x


def atomic_accumulate(C, P, s, table=None, ex=None):
    """Concurrent-safe elementwise merge of P into C: C <- C (+) P (classic.py:268-284).

    Uses the semiring's hardware atomic-madd (red.add.f64 / red.add.u64 /
    red.min.s32, CAS loops for the float minima), so concurrent callers on
    overlapping tiles serialise per element in L2 -- the device analogue of
    the reference's per-tile exclusion slots."""
    C, P = _region(C), _region(P)
    if C.rows != P.rows or C.cols != P.cols:
        raise DimMismatch(f"accumulate shapes differ: {C.rows}x{C.cols} vs {P.rows}x{P.cols}")
    if table is not None:
        if table.tiles_r * table.tile != C.buffer.rows:
            raise ContractViolation("exclusion table does not match C's buffer")
        C.buffer.table = table
    tile = C.buffer.table.tile if C.buffer.table is not None else None
    if tile is not None:
        C.tile_range(tile)                     # AlignmentError unless b-aligned (ops.py:86)
    t = C.buffer.data
    with torch.cuda.device(t.device):
        _lib.check(_lib.lib().starmm_atomic_accumulate(
            s.sr_id, C.data_ptr(), C.row_stride, P.data_ptr(), P.row_stride, C.rows, C.cols,
            torch.cuda.current_stream(t.device).cuda_stream, 0), "atomic_accumulate")
    if C.buffer.table is not None:
        ti0, tj0, tr, tc = C.tile_range(C.buffer.table.tile)
        C.buffer.table.entry_counts[ti0:ti0 + tr, tj0:tj0 + tc] += 1
    if ex is not None:
        ex.metrics.count_serialization(max(1, (C.rows * C.cols) // max(1, (tile or 1) ** 2)))


def _run_public(algo, C, A, B, s, cfg, mode="pooled"):
    from .registry import run_algorithm
    from .runtime import Executor
    with Executor(cfg) as ex:
        run_algorithm(ex, algo, C, A, B, s, mode=mode)


def co2(C, A, B, s, cfg):
    """C <- C (+) A (x) B; quadrant recursion in two parallel steps per level."""
    _run_public("co2", C, A, B, s, cfg)


def co3(C, A, B, s, cfg, mode="pooled"):
    """Eight-way concurrent recursion with a per-level temporary, then merge."""
    _run_public("co3", C, A, B, s, cfg, mode=mode)


def tar_mm(C, A, B, s, cfg):
    """All eight sub-products concurrent; base cases merge through tile slots."""
    _run_public("tar", C, A, B, s, cfg)


def sar_mm(C, A, B, s, cfg):
    """Eight-way concurrent recursion with lazily allocated temporaries."""
    _run_public("sar", C, A, B, s, cfg)


def star_mm(C, A, B, s, cfg):
    """tar above the switch depth (ceil of half log2 p), sar below it."""
    _run_public("star", C, A, B, s, cfg)



def host_mm(algo, C, A, B, s, cfg, mode="pooled"):
    """C <- C (+) A (x) B for HOST-resident operands (the reference's entry points take
    host numpy matrices, classic.py:294-316).  C, A, B: 2-D CPU tensors (pinned memory
    overlaps the transfers with the tile kernels) or numpy arrays; C is updated in place.
    Same validation as run_algorithm (registry.py:28-42)."""
    from .registry import ALGORITHMS, CLASSICAL, _MODAL
    from .runtime import Executor
    if algo not in ALGORITHMS:
        raise KeyError(f"unknown algorithm {algo!r}; choose from {ALGORITHMS}")
    if algo not in CLASSICAL:
        raise ContractViolation(f"{algo}: only the classical schedules have a host path")
    if mode not in ("pooled", "raw"):
        raise ContractViolation(f"unknown mode {mode!r}")
    if mode == "raw" and algo not in _MODAL:
        raise ContractViolation(f"{algo} does not take an allocation mode")
    n = C.shape[0]
    if not (A.shape[0] == A.shape[1] == B.shape[0] == B.shape[1] == C.shape[1] == n):
        raise DimMismatch("A, B, C must be square with one common dimension")
    cfg.check_problem(n)
    with Executor(cfg) as ex:
        return ex.execute_host(algo, C, A, B, s, mode=mode)
