"""Generate tests/golden/ from the REFERENCE implementation itself.

Run in the build container only (it needs /root/reference, which does not
exist on the GPU box):  python oracle/gen_golden.py

The reference package is imported from a private copy under /tmp with
NUMBA_CACHE_DIR redirected, so nothing is ever written into /root/reference.
Outputs (committed):
  tests/golden/ref_small.npz   -- every classical schedule x {int, float, tropical}
                                  at workers=1 on the reference's own fixture
                                  generator (matrix.py:196-214), n in {b..16b}
  tests/golden/ref_spec.json   -- the SPEC.md known answers, evaluated by the reference
  tests/golden/ref_pr1.npz     -- BASELINE config 1 (PR1): star_mm fp64 n=256 b=32,
                                  A,B ~ U[-1,1) seed 0, C=0, workers=1
  tests/golden/ref_signed_zero.npz -- tropical (float64) with +-0.0-heavy operands: every
                                  classical schedule at workers=1, naive_mm and madd, so the
                                  signed-zero tie rules (semiring.py:56-58 "if v < out",
                                  np.minimum's second-operand tie) are pinned bit for bit
  tests/golden/ref_tiles.json  -- sha256 of reference-computed 128x128 output tiles at
                                  the BASELINE configs' generators (bench/configs.py),
                                  for the larger configs (pins the sampled-tile oracle)
"""
from __future__ import annotations

import hashlib
import json
import os
import shutil
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
GOLDEN = os.path.join(REPO, "tests", "golden")


def import_reference():
    src = "/root/reference/pkg/src/starmm"
    tmp = tempfile.mkdtemp(prefix="starmm_ref_")
    shutil.copytree(src, os.path.join(tmp, "starmm"))
    os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join(tmp, "numba_cache"))
    sys.dont_write_bytecode = True
    sys.path.insert(0, tmp)
    import starmm  # noqa: E402
    return starmm


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def gen_small(ref):
    out = {}
    algos = [("co2", ref.co2), ("co3", ref.co3), ("tar", ref.tar_mm),
             ("sar", ref.sar_mm), ("star", ref.star_mm)]
    cases = [(2, 2), (2, 8), (4, 16), (8, 32), (32, 64)]
    for sid in ("int", "float", "tropical"):
        s = ref.get_semiring(sid)
        for b, n in cases:
            seed = 1000 * b + n
            A = ref.random_matrix(n, s, seed)
            B = ref.random_matrix(n, s, seed + 1)
            C0 = ref.random_matrix(n, s, seed + 2)
            key = f"{sid}_n{n}_b{b}"
            out[f"{key}_A"] = A.data
            out[f"{key}_B"] = B.data
            out[f"{key}_C0"] = C0.data
            out[f"{key}_naive"] = ref.naive_mm(A, B, s).data
            for name, fn in algos:
                C = ref.Matrix(C0.data.copy(), s)
                fn(C, A, B, s, ref.Config(base_dim=b, workers=1))
                out[f"{key}_{name}"] = C.data
    np.savez_compressed(os.path.join(GOLDEN, "ref_small.npz"), **out)
    print("ref_small.npz:", len(out), "arrays")


def gen_signed_zero(ref):
    out = {}
    s = ref.TROPICAL
    algos = [("co2", ref.co2), ("co3", ref.co3), ("tar", ref.tar_mm),
             ("sar", ref.sar_mm), ("star", ref.star_mm)]
    rng = np.random.default_rng(1911)
    vals = np.array([0.0, -0.0, 1.0, -1.0, 2.0, np.inf])
    prob = [0.3, 0.3, 0.1, 0.1, 0.1, 0.1]
    for b, n in [(1, 4), (2, 8), (4, 16), (8, 32), (16, 32), (32, 32)]:
        A = rng.choice(vals, (n, n), p=prob)
        B = rng.choice(vals, (n, n), p=prob)
        C0 = rng.choice(vals, (n, n), p=prob)
        key = f"n{n}_b{b}"
        out[f"{key}_A"], out[f"{key}_B"], out[f"{key}_C0"] = A, B, C0
        out[f"{key}_naive"] = ref.naive_mm(ref.Matrix(A, s), ref.Matrix(B, s), s).data
        for name, fn in algos:
            C = ref.Matrix(C0.copy(), s)
            fn(C, ref.Matrix(A, s), ref.Matrix(B, s), s, ref.Config(base_dim=b, workers=1))
            out[f"{key}_{name}"] = C.data
        C = ref.Matrix(C0.copy(), s)
        ref.madd(C, ref.Matrix(A, s), s)
        out[f"{key}_madd"] = C.data
    np.savez_compressed(os.path.join(GOLDEN, "ref_signed_zero.npz"), **out)
    print("ref_signed_zero.npz:", len(out), "arrays")


def gen_spec(ref):
    s_int, s_trop = ref.INT_RING, ref.TROPICAL
    res = {}
    M = lambda x, s: ref.Matrix(np.array(x, dtype=s.dtype), s)  # noqa: E731
    res["naive_1x1"] = ref.naive_mm(M([[2]], s_int), M([[3]], s_int), s_int).data.tolist()
    res["naive_2x2"] = ref.naive_mm(M([[1, 2], [3, 4]], s_int), M([[5, 6], [7, 8]], s_int),
                                    s_int).data.tolist()
    res["naive_trop_2x2"] = ref.naive_mm(M([[0, 1], [2, 3]], s_trop), M([[0, 4], [1, 0]], s_trop),
                                         s_trop).data.tolist()
    C = M([[5]], s_int)
    ref.base_kernel(C, M([[2]], s_int), M([[3]], s_int), s_int, ref.Config(base_dim=1))
    res["base_kernel_b1"] = C.data.tolist()
    C = M([[4]], s_trop)
    ref.base_kernel(C, M([[1]], s_trop), M([[2]], s_trop), s_trop, ref.Config(base_dim=1))
    res["base_kernel_trop_b1"] = C.data.tolist()
    C = M([[1, 2], [3, 4]], s_int)
    ref.madd(C, M([[10, 20], [30, 40]], s_int), s_int)
    res["madd_int"] = C.data.tolist()
    C = M([[1, 5]], s_trop)
    ref.madd(C, M([[3, 2]], s_trop), s_trop)
    res["madd_trop"] = C.data.tolist()
    res["switch_depth"] = {str(p): ref.switch_depth(p) for p in (1, 2, 3, 4, 5, 16, 17, 64, 65, 148, 256)}
    # int wrap mod 2**64 (semiring.py:5-9): 2**62 * 4 -> 0
    res["int_wrap"] = ref.naive_mm(M([[2 ** 62]], s_int), M([[4]], s_int), s_int).data.tolist()
    with open(os.path.join(GOLDEN, "ref_spec.json"), "w") as fh:
        json.dump(res, fh, indent=1, sort_keys=True)
    print("ref_spec.json:", res)


def gen_pr1(ref):
    sys.path.insert(0, REPO)
    from bench_configs import make_inputs  # noqa: E402
    A, B, C0 = make_inputs(1)
    s = ref.FLOAT_RING
    C = ref.Matrix(C0.copy(), s)
    ref.star_mm(C, ref.Matrix(A, s), ref.Matrix(B, s), s, ref.Config(base_dim=32, workers=1))
    np.savez_compressed(os.path.join(GOLDEN, "ref_pr1.npz"), star=C.data)
    print("ref_pr1.npz written")


def gen_tiles(ref):
    """sha256 of reference-computed output tiles for the larger configs.

    expected = fold_add(C0[tile], Semiring.matmul(A[rows,:], B[:,cols])) computed by
    the reference's own Semiring object on float64/int64 up-casts,
    then cast back to the config dtype (exact for every config's value range).
    """
    sys.path.insert(0, REPO)
    from bench_configs import CONFIGS, make_inputs, sample_tiles, to_reference  # noqa: E402
    res = {}
    for cid in (2, 3, 4, 5):
        cfg = CONFIGS[cid]
        A, B, C0 = make_inputs(cid)
        s = ref.get_semiring(cfg["ref_semiring"])
        tiles = sample_tiles(cid, count=4)
        entries = []
        for (i0, j0) in tiles:
            Ar = to_reference(cid, A[i0:i0 + 128, :])
            Bc = to_reference(cid, B[:, j0:j0 + 128])
            Ct = to_reference(cid, C0[i0:i0 + 128, j0:j0 + 128]).copy()
            s.fold_add(Ct, s.matmul(Ar, Bc))
            from bench_configs import from_reference  # noqa: E402
            entries.append({"i0": int(i0), "j0": int(j0), "sha256": sha(from_reference(cid, Ct))})
        res[str(cid)] = entries
        print("config", cid, "tiles", len(entries))
    with open(os.path.join(GOLDEN, "ref_tiles.json"), "w") as fh:
        json.dump(res, fh, indent=1)


if __name__ == "__main__":
    os.makedirs(GOLDEN, exist_ok=True)
    ref = import_reference()
    which = sys.argv[1:] or ["small", "spec", "pr1", "tiles", "signed_zero"]
    if "small" in which:
        gen_small(ref)
    if "spec" in which:
        gen_spec(ref)
    if "pr1" in which:
        gen_pr1(ref)
    if "tiles" in which:
        gen_tiles(ref)
    if "signed_zero" in which:
        gen_signed_zero(ref)
