"""CPU checks of the Ozaki-II design behind STARMM_F_FP64_EMU (csrc/ozaki.cuh,
DESIGN.md §5d), in exact Python integers: the moduli, the bit budget t(k), the
device's residue formulas, and the scale -> residues -> per-modulus products ->
CRT pipeline reproducing the exact integer product.  No GPU needed.
"""
import math
import random
from fractions import Fraction

import numpy as np

MODULI = [256, 255, 253, 251, 247, 241, 239, 233, 229, 227, 223, 217, 211, 199, 197, 193]
M = math.prod(MODULI)


def t_bits(k):   # starmm_api.cu: ozaki_bits
    lm = sum(math.log2(m) for m in MODULI)
    return min(62, int(math.floor((lm - math.log2(max(1, k)) - 2) / 2)))


def sym(r, m):   # symmetric int8 residue as stored in the planes
    r %= m
    return r - m if r > (m - 1) // 2 else r


def res_limbs(x, m):
    """oz_res_limbs: x = x2 2^42 + x1 2^21 + x0 with int32 arithmetic."""
    if m == 256:
        b = x & 0xff
        return b - 256 if b > 127 else b
    x0, x1, x2 = x & 0x1FFFFF, (x >> 21) & 0x1FFFFF, x >> 42
    c1, c2 = (1 << 21) % m, (1 << 42) % m
    off = m * ((1 << 30) // m + 1)
    s = x2 * c2 + x1 * c1 + x0 + off
    assert 0 <= s < 2 ** 32 and abs(x2 * c2 + x1 * c1 + x0) < 2 ** 30
    u = s % m
    return u - m if u > (m - 1) // 2 else u


def res_f64(x, m):
    """oz_res_f64: q = rint(x * (1/m)) in double, exact fma remainder, integer fold."""
    q = round(float(np.float64(x) * np.float64(1.0 / m)))
    r = int(x - m * q)
    assert abs(r) <= m + m // 2
    if r < -((m - 1) // 2):
        r += m
    if r > (m - 1) // 2:
        r -= m
    return r


def crt(residues):
    x = 0
    for r, m in zip(residues, MODULI):
        Mi = M // m
        x += (r % m) * Mi * pow(Mi, -1, m)
    x %= M
    return x - M if x > M // 2 else x


def test_moduli_pairwise_coprime_and_int8():
    for i, a in enumerate(MODULI):
        assert a <= 256
        for b in MODULI[i + 1:]:
            assert math.gcd(a, b) == 1
    assert 125 < math.log2(M) < 126


def test_bit_budget_covers_every_k():
    for k in list(range(1, 5000)) + [2 ** e for e in range(13, 17)] + [2 ** 17 - 1]:
        t = t_bits(k)
        assert t >= 53, k
        assert 2 * k * 2 ** (2 * t) < M, k
        assert k * 128 * 128 < 2 ** 31      # per-modulus int32 accumulators stay exact


def test_residue_formulas_match_exact_mod():
    rng = random.Random(7)
    xs = [rng.randrange(-2 ** 54, 2 ** 54) for _ in range(3000)]
    xs += [0, 1, -1, 2 ** 54, -2 ** 54, 2 ** 62 - 1, -2 ** 62]
    for x in xs:
        for i, m in enumerate(MODULI):
            want = sym(x, m)
            assert -128 <= want <= 127
            assert res_limbs(x, m) == want, (x, m)
            if abs(x) <= 2 ** 54 and i % 2 == 1:    # the FP64-pipe moduli
                assert res_f64(x, m) == want, (x, m)


def test_scale_residue_crt_pipeline_is_exact():
    rng = np.random.default_rng(3)
    m, k, n = 5, 40, 6
    A = rng.standard_normal((m, k)) * 2.0 ** rng.integers(-20, 20, (m, 1))
    B = rng.standard_normal((k, n))
    t = t_bits(k)
    sig = [t - math.frexp(float(np.max(np.abs(A[i]))))[1] for i in range(m)]
    tau = [t - math.frexp(float(np.max(np.abs(B[:, j]))))[1] for j in range(n)]
    Ai = [[int(round(math.ldexp(float(A[i, q]), sig[i]))) for q in range(k)] for i in range(m)]
    Bi = [[int(round(math.ldexp(float(B[q, j]), tau[j]))) for j in range(n)] for q in range(k)]
    assert max(abs(v) for r in Ai for v in r) <= 2 ** t
    for i in range(m):
        for j in range(n):
            exact = sum(Ai[i][q] * Bi[q][j] for q in range(k))
            # per modulus: int8 residues, int32 products, residue of the sum
            rho = []
            for mm in MODULI:
                acc = sum(sym(Ai[i][q], mm) * sym(Bi[q][j], mm) for q in range(k))
                assert abs(acc) < 2 ** 31
                rho.append(acc % mm)
            assert crt(rho) == exact
            # one rounding of the exact scaled integer, then the truncation bound
            got = math.ldexp(float(exact), -sig[i] - tau[j])
            true = Fraction(0)
            for q in range(k):
                true += Fraction(float(A[i, q])) * Fraction(float(B[q, j]))
            bound = 2.0 ** (1 - t) * k * float(np.max(np.abs(A[i]))) * float(np.max(np.abs(B[:, j])))
            assert abs(Fraction(got) - true) <= Fraction(bound) + Fraction(abs(got)) * Fraction(2) ** -52
