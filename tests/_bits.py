"""Bitwise comparison for parity tests: equal bit patterns element by element, so
+0.0 != -0.0; any NaN equals any NaN (numpy's NaN payloads are not part of the
reference's contract, its np.minimum only promises "NaN")."""
import numpy as np

_UINT = {1: np.uint8, 2: np.uint16, 4: np.uint32, 8: np.uint64}


def same_bits(a, b, equal_nan=True) -> bool:
    """Element-wise identical bits (+0.0 != -0.0; NaNs equal).  Arrays of different
    dtypes compare by value, plus the sign bit for floats."""
    a = np.ascontiguousarray(np.asarray(a))
    b = np.ascontiguousarray(np.asarray(b))
    if a.shape != b.shape:
        return False
    if a.dtype != b.dtype:
        if a.dtype.kind == "f" or b.dtype.kind == "f":
            af, bf = a.astype(np.float64), b.astype(np.float64)
            eq = (af == bf) & (np.signbit(af) == np.signbit(bf))
            return bool((eq | (np.isnan(af) & np.isnan(bf))).all())
        return bool(np.array_equal(a, b))
    u = _UINT[a.dtype.itemsize]
    eq = a.view(u) == b.view(u)
    if a.dtype.kind == "f":
        eq |= np.isnan(a) & np.isnan(b)
    return bool(eq.all())


def diff_count(a, b) -> int:
    a = np.ascontiguousarray(np.asarray(a))
    b = np.ascontiguousarray(np.asarray(b))
    u = _UINT[a.dtype.itemsize]
    ne = a.view(u) != b.view(u)
    if a.dtype.kind == "f":
        ne &= ~(np.isnan(a) & np.isnan(b))
    return int(ne.sum())
