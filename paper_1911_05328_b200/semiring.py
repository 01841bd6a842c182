"""Element algebras the multiplication kernels are generic over.

Mirrors the reference's semiring module (semiring.py:63-152): same class,
same ids ("int", "float", "tropical"), same identities and ``add``/``mul``/
``sub`` elementwise operations.  ``matmul`` and ``fold_add`` -- the two
overridable hooks the schedules use (semiring.py:92-98) -- run on the B200
through the C ABI (``starmm_matmul`` / ``starmm_madd``) instead of numba.

This build adds two 32-bit ids (SURVEY.md key finding 1; BASELINE configs 3
and 5), which the reference has no counterpart for:
  "tropical_f32"  float32 (min,+), +inf identity
  "tropical_i32"  int32 (min,+), INT32_MAX plays +inf (absorbing for the
                  product, identity for the sum); finite sums saturate.

Operands may be CUDA torch tensors (the native representation) or numpy
arrays; numpy inputs are uploaded, and results come back as numpy, so code
written against the reference keeps working.
"""
from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .errors import DimMismatch, NoAdditiveInverse

__all__ = ["Semiring", "INT_RING", "FLOAT_RING", "TROPICAL", "TROPICAL_F32", "TROPICAL_I32",
           "get_semiring", "SEMIRINGS"]

I32_INF = int(np.iinfo(np.int32).max)


def _to_device(x, dtype: torch.dtype):
    """(tensor on cuda, was_numpy)."""
    if isinstance(x, torch.Tensor):
        if x.device.type != "cuda":
            return x.to(device="cuda", dtype=dtype), True
        if x.dtype != dtype:
            raise DimMismatch(f"tensor dtype {x.dtype} does not match semiring dtype {dtype}")
        return x, False
    return torch.from_numpy(np.ascontiguousarray(x)).to(device="cuda", dtype=dtype), True


def _row_major_ld(t: torch.Tensor) -> int:
    if t.dim() != 2:
        raise DimMismatch("matrices are two-dimensional")
    if t.shape[1] > 1 and t.stride(1) != 1:
        raise DimMismatch("row-major views with unit column stride are required")
    return max(int(t.stride(0)), int(t.shape[1]), 1)


def _stream(t: torch.Tensor) -> int:
    return torch.cuda.current_stream(t.device).cuda_stream


class Semiring:
    """Algebra descriptor (semiring.py:63-105) plus the C-ABI id of its kernels."""

    def __init__(self, sid, dtype, zero, one, add, mul, sub=None, sr_id=None, torch_dtype=None):
        self.id = sid
        self.dtype = np.dtype(dtype)
        self.zero = dtype(zero)
        self.one = dtype(one)
        self._add = add
        self._mul = mul
        self._sub = sub
        self.sr_id = sr_id
        self.torch_dtype = torch_dtype

    @property
    def has_sub(self):
        return self._sub is not None

    def add(self, a, b):
        return self._add(a, b)

    def mul(self, a, b):
        return self._mul(a, b)

    def sub(self, a, b):
        if self._sub is None:
            raise NoAdditiveInverse(f"semiring {self.id!r} has no additive inverse")
        return self._sub(a, b)

    def neg(self, a):
        """Map a to its additive inverse, i.e. (0 - 1) * a on a ring."""
        return self.sub(self.zero, a)

    def matmul(self, A, B):
        """Dense product from the additive identity: out = A (x) B (semiring.py:92-94).

        Runs ``starmm_matmul`` on the GPU.  Rectangular panels are accepted
        (the sampled-tile oracle protocol)."""
        At, a_np = _to_device(A, self.torch_dtype)
        Bt, b_np = _to_device(B, self.torch_dtype)
        m, k = At.shape
        k2, n = Bt.shape
        if k != k2:
            raise DimMismatch(f"inner dimensions differ: {m}x{k} vs {k2}x{n}")
        out = torch.empty((m, n), dtype=self.torch_dtype, device=At.device)
        with torch.cuda.device(At.device):
            _lib.check(_lib.lib().starmm_matmul(
                self.sr_id, out.data_ptr(), n, At.data_ptr(), _row_major_ld(At), Bt.data_ptr(),
                _row_major_ld(Bt), m, n, k, _stream(At), 0), "Semiring.matmul")
        return out.cpu().numpy() if (a_np and b_np) else out

    def fold_add(self, C, D):
        """C[i,j] <- C[i,j] (+) D[i,j], in place (semiring.py:96-98)."""
        if not isinstance(C, torch.Tensor):
            Ct = torch.from_numpy(np.ascontiguousarray(C)).cuda()
            self.fold_add(Ct, D)
            np.copyto(C, Ct.cpu().numpy())
            return
        Dt, _ = _to_device(D, self.torch_dtype)
        if tuple(C.shape) != tuple(Dt.shape):
            raise DimMismatch(f"fold shapes differ: {tuple(C.shape)} vs {tuple(Dt.shape)}")
        rows, cols = C.shape
        with torch.cuda.device(C.device):
            _lib.check(_lib.lib().starmm_madd(self.sr_id, C.data_ptr(), _row_major_ld(C),
                                              Dt.data_ptr(), _row_major_ld(Dt), rows, cols,
                                              _stream(C), 0), "Semiring.fold_add")

    def full(self, shape, device="cuda"):
        """Array filled with the additive identity (on the GPU)."""
        return torch.full(tuple(shape), self.zero.item(), dtype=self.torch_dtype, device=device)

    def __repr__(self):
        return f"Semiring({self.id!r})"


def _np_min(a, b):
    return np.minimum(a, b)


def _i32_trop_mul(a, b):
    """Saturating int32 (min,+) product with INT32_MAX as +inf."""
    a64 = np.asarray(a, dtype=np.int64)
    b64 = np.asarray(b, dtype=np.int64)
    s = np.clip(a64 + b64, np.iinfo(np.int32).min, I32_INF)
    s = np.where((a64 == I32_INF) | (b64 == I32_INF), I32_INF, s)
    return s.astype(np.int32)


INT_RING = Semiring("int", np.int64, 0, 1, add=np.add, mul=np.multiply, sub=np.subtract,
                    sr_id=_lib.SR_INT64, torch_dtype=torch.int64)

FLOAT_RING = Semiring("float", np.float64, 0.0, 1.0, add=np.add, mul=np.multiply,
                      sub=np.subtract, sr_id=_lib.SR_FP64, torch_dtype=torch.float64)

TROPICAL = Semiring("tropical", np.float64, np.inf, 0.0, add=_np_min, mul=np.add,
                    sr_id=_lib.SR_TROPICAL_F64, torch_dtype=torch.float64)

TROPICAL_F32 = Semiring("tropical_f32", np.float32, np.inf, 0.0, add=_np_min, mul=np.add,
                        sr_id=_lib.SR_TROPICAL_F32, torch_dtype=torch.float32)

TROPICAL_I32 = Semiring("tropical_i32", np.int32, I32_INF, 0, add=_np_min, mul=_i32_trop_mul,
                        sr_id=_lib.SR_TROPICAL_I32, torch_dtype=torch.int32)

SEMIRINGS = {s.id: s for s in (INT_RING, FLOAT_RING, TROPICAL, TROPICAL_F32, TROPICAL_I32)}


def get_semiring(sid):
    try:
        return SEMIRINGS[sid]
    except KeyError:
        raise KeyError(f"unknown semiring {sid!r}; choose from {sorted(SEMIRINGS)}") from None
