"""Fast (seven-product) matrix multiplication over rings (reference strassen.py:1-235).

Same entry points and semantics as the reference: every call OVERWRITES C with
A (x) B and needs an additive inverse (``int`` / ``float`` rings; the tropical
semirings raise NoAdditiveInverse, registry.py:41-42).  The recursion runs on the
host inside libstarmm_b200 (csrc/starmm_api.cu, "Strassen family"): operand sums
and the signed assembly are ring-combine kernels, leaves are the classical tile
kernels once the half size drops below max(base_dim, Config.strassen_leaf).

* ``strassen_parallel`` -- straightforward step: every operand sum and all seven
  products materialised (<= 17 half-size temporaries per level), then assembly.
* ``sar_strassen``      -- per product three LIFO-reused blocks (S, T, P); each
  finished product is merged, sign-aware, into the quadrants it feeds.
* ``star_strassen_1``   -- classical 8-way levels above switch_depth(workers),
  sar_strassen below.
* ``star_strassen_2``   -- straightforward levels above the switch, sar below.
"""
from __future__ import annotations

__all__ = ["strassen_parallel", "sar_strassen", "star_strassen_1", "star_strassen_2"]


def _run_public(algo, C, A, B, s, cfg, mode="pooled"):
    from .registry import run_algorithm
    from .runtime import Executor
    with Executor(cfg) as ex:
        run_algorithm(ex, algo, C, A, B, s, mode=mode)


def strassen_parallel(C, A, B, s, cfg, mode="pooled"):
    """C <- A (x) B by the straightforward seven-product parallelization."""
    _run_public("strassen", C, A, B, s, cfg, mode=mode)


def sar_strassen(C, A, B, s, cfg):
    """Seven-product recursion with three pooled scratch blocks per product."""
    _run_public("sar-strassen", C, A, B, s, cfg)


def star_strassen_1(C, A, B, s, cfg):
    """Classical eight-way levels above the switch depth, then sar_strassen."""
    _run_public("star-strassen-1", C, A, B, s, cfg)


def star_strassen_2(C, A, B, s, cfg):
    """Straightforward seven-way levels above the switch, then sar_strassen."""
    _run_public("star-strassen-2", C, A, B, s, cfg)
