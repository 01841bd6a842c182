"""Seeded input generators for the BASELINE.json configs (bench + tests + golden).

Convention (recorded in DESIGN.md §Inputs): one numpy PCG64 stream per config,
``rng = numpy.random.default_rng(seed)``, drawing A, then B, then C.  All inputs
are synthetic (BASELINE names no dataset).  ``n`` may be overridden to build a
same-distribution instance at a smaller size for tests.

  1 PR1  fp64 (+,x)     n=256   b=32  A,B ~ U[-1,1) (seed 0), C = 0; STAR
  2      int64 (+,x)    n=4096  b=64  A,B ~ U{-16..16} (seed 1), C = 0
  3      fp32 (min,+)   n=8192        A = B = Erdos-Renyi digraph, p=0.1, weights
                                      U{1..100}, diag 0, absent = +inf (seed 2, our
                                      choice: BASELINE states none); C = A
  4      fp64 (+,x)     n=16384       A,B ~ N(0,1) (seed 3), C ~ U[-1,1)
  5      int32 (min,+)  n=49152       W ~ U{1..10^6} dense, diag 0 (seed 4); A = B = W
                                      (our choice: BASELINE states only W); C = A
"""
from __future__ import annotations

import numpy as np

I32_INF = np.iinfo(np.int32).max

CONFIGS = {
    1: dict(name="pr1_fp64_star_n256", semiring="float", ref_semiring="float", n=256, b=32,
            dtype=np.float64, algo="star", seed=0, tol=1e-12),
    2: dict(name="int64_ring_n4096", semiring="int", ref_semiring="int", n=4096, b=64,
            dtype=np.int64, algo="star", seed=1, tol=0.0),
    3: dict(name="tropical_f32_er_n8192", semiring="tropical_f32", ref_semiring="tropical",
            n=8192, b=64, dtype=np.float32, algo="star", seed=2, tol=0.0),
    4: dict(name="fp64_ring_n16384", semiring="float", ref_semiring="float", n=16384, b=64,
            dtype=np.float64, algo="star", seed=3, tol=None),   # tol = 1e-10*sqrt(n)
    5: dict(name="tropical_i32_n49152", semiring="tropical_i32", ref_semiring="tropical",
            n=49152, b=64, dtype=np.int32, algo="star", seed=4, tol=0.0),
}


def tolerance(cid: int, n: int | None = None) -> float:
    cfg = CONFIGS[cid]
    if cfg["tol"] is not None:
        return cfg["tol"]
    return 1e-10 * float(np.sqrt(n or cfg["n"]))


def make_inputs(cid: int, n: int | None = None):
    """(A, B, C0) as host numpy arrays of the config dtype.  For configs 3 and 5
    A and B are the same array object (A = B = W)."""
    cfg = CONFIGS[cid]
    n = n or cfg["n"]
    rng = np.random.default_rng(cfg["seed"])
    if cid == 1:
        A = rng.uniform(-1, 1, (n, n))
        B = rng.uniform(-1, 1, (n, n))
        C = np.zeros((n, n))
    elif cid == 2:
        A = rng.integers(-16, 17, (n, n), dtype=np.int64)
        B = rng.integers(-16, 17, (n, n), dtype=np.int64)
        C = np.zeros((n, n), dtype=np.int64)
    elif cid == 3:
        edge = rng.random((n, n), dtype=np.float32) < 0.1
        W = rng.integers(1, 101, (n, n), dtype=np.int32).astype(np.float32)
        W[~edge] = np.inf
        np.fill_diagonal(W, 0.0)
        A = B = W
        C = W.copy()
    elif cid == 4:
        A = rng.standard_normal((n, n))
        B = rng.standard_normal((n, n))
        C = rng.uniform(-1, 1, (n, n))
    elif cid == 5:
        W = rng.integers(1, 10 ** 6 + 1, (n, n), dtype=np.int32)
        np.fill_diagonal(W, 0)
        A = B = W
        C = W.copy()
    else:
        raise KeyError(cid)
    return A, B, C


def sample_tiles(cid: int, count: int = 64, n: int | None = None, tile: int = 128):
    """Seeded random output-tile origins (any offset, not only tile-aligned)."""
    n = n or CONFIGS[cid]["n"]
    rng = np.random.default_rng(1000 + cid)
    t = min(tile, n)
    return [(int(rng.integers(0, n - t + 1)), int(rng.integers(0, n - t + 1)))
            for _ in range(count)]


def to_reference(cid: int, x: np.ndarray) -> np.ndarray:
    """Up-cast to the reference's 64-bit element type (exact for every config)."""
    cfg = CONFIGS[cid]
    if cfg["dtype"] == np.int32:          # int32 tropical -> float64 tropical
        y = x.astype(np.float64)
        y[x == I32_INF] = np.inf
        return y
    if cfg["dtype"] == np.float32:
        return x.astype(np.float64)
    return np.ascontiguousarray(x)


def from_reference(cid: int, y: np.ndarray) -> np.ndarray:
    cfg = CONFIGS[cid]
    if cfg["dtype"] == np.int32:
        x = np.where(np.isinf(y), float(I32_INF), y)
        return x.astype(np.int32)
    return y.astype(cfg["dtype"])


# ---- the device generator's spec of each config (csrc/generate.cuh) -------------------
# Same distributions as make_inputs, drawn from the counter-based device generator
# (Philox4x32-10 keyed by the config's seed; stream id 0 = A, 1 = B, 2 = C) so that any
# rank can generate its panels and the oracle can regenerate any sampled tile's panels.
# None: the matrix is a copy of another ("A" for C = A) or all zeros.
DEVICE_GEN = {
    1: {"A": dict(dist="uniform_real", stream_id=0, a=-1.0, b=1.0),
        "B": dict(dist="uniform_real", stream_id=1, a=-1.0, b=1.0), "C": "zeros"},
    2: {"A": dict(dist="uniform_int", stream_id=0, a=-16, b=16),
        "B": dict(dist="uniform_int", stream_id=1, a=-16, b=16), "C": "zeros"},
    3: {"A": dict(dist="graph", stream_id=0, a=1, b=100, p=0.1, zero_diag=True),
        "B": "A", "C": "A"},
    4: {"A": dict(dist="normal", stream_id=0, a=0.0, b=1.0),
        "B": dict(dist="normal", stream_id=1, a=0.0, b=1.0),
        "C": dict(dist="uniform_real", stream_id=2, a=-1.0, b=1.0)},
    5: {"A": dict(dist="uniform_int", stream_id=0, a=1, b=10 ** 6, zero_diag=True),
        "B": "A", "C": "A"},
}


def device_gen_spec(cid: int, which: str):
    """Resolve DEVICE_GEN[cid][which] to the generator kwargs (or "zeros")."""
    spec = DEVICE_GEN[cid][which]
    while isinstance(spec, str) and spec in ("A", "B", "C"):
        spec = DEVICE_GEN[cid][spec]
    if isinstance(spec, dict):
        return dict(spec, seed=CONFIGS[cid]["seed"])
    return spec
