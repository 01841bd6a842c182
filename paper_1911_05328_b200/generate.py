"""Counter-based input generation on the device.

``generate_panel`` fills rows [row0, row0+rows) x columns [col0, col0+cols) of a
conceptual matrix whose element (i, j) is a pure function of (seed, stream_id, i, j)
-- Philox4x32-10 on (j, i, stream_id, 0), keyed by the seed (csrc/generate.cuh,
``starmm_generate``).  A rank of a distributed run therefore generates exactly its own
A / B / C panels with no broadcast, the values do not depend on the panel cut, and the
CPU oracle regenerates any panel bit for bit to check sampled output tiles.

The reference's fixture generator (``random_matrix``, matrix.py:196-214, numpy) is
unchanged and remains what the parity tests use; this generator is for inputs that are
too large to build on the host and ship (BASELINE's full-size configs).
"""
from __future__ import annotations

import torch

from . import _lib
from .errors import ContractViolation

__all__ = ["DISTRIBUTIONS", "generate_panel"]

DISTRIBUTIONS = {"uniform_real": 0, "normal": 1, "uniform_int": 2, "graph": 3}
GEN_ZERO_DIAG = 0x1


def generate_panel(semiring, dist: str, rows: int, cols: int, row0: int = 0, col0: int = 0,
                   seed: int = 0, stream_id: int = 0, a: float = 0.0, b: float = 1.0,
                   p: float = 0.0, zero_diag: bool = False, out: torch.Tensor | None = None,
                   device=None) -> torch.Tensor:
    """A (rows x cols) panel of the generated matrix, on the GPU (stream-ordered).

    dist: "uniform_real" (a + (b-a) u), "normal" (a + b z), "uniform_int" (integers in
    [a, b]) or "graph" (edge with probability p carrying a uniform integer weight in
    [a, b], else the semiring's additive identity); zero_diag sets (i, i) to 0."""
    if dist not in DISTRIBUTIONS:
        raise ContractViolation(f"unknown distribution {dist!r}; choose from {sorted(DISTRIBUTIONS)}")
    if out is None:
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        out = torch.empty((rows, cols), dtype=semiring.torch_dtype, device=dev)
    if out.dtype != semiring.torch_dtype or out.dim() != 2 or tuple(out.shape) != (rows, cols) or \
            (cols > 1 and out.stride(1) != 1):
        raise ContractViolation("out must be a row-major (rows x cols) tensor of the semiring dtype")
    stream = torch.cuda.current_stream(out.device).cuda_stream
    with torch.cuda.device(out.device):
        _lib.check(_lib.lib().starmm_generate(
            semiring.sr_id, DISTRIBUTIONS[dist], out.data_ptr(), max(1, out.stride(0)), rows, cols,
            row0, col0, seed & 0xffffffffffffffff, stream_id & 0xffffffff, float(a), float(b), float(p),
            GEN_ZERO_DIAG if zero_diag else 0, stream), "starmm_generate")
    return out
