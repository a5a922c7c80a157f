"""Floating-point primitives (TEST INFRASTRUCTURE ONLY — see oracle/__init__.py).

PAPER.md §2.1 (lines 108-136): u = 2^-53 for binary64, ufp(α) = 2^⌊log2|α|⌋ (0 for α = 0),
fl(·) = round-to-nearest. §2.2 (lines 140-161): TwoSum (Knuth) and the pair arithmetic that omits
the lower part of the second double-word. All functions are elementwise over numpy float64 arrays;
numpy evaluates + - * / as single IEEE operations (no contraction), which the EFTs rely on.
"""
import numpy as np

U = 2.0 ** -53  # PAPER.md:123 "u = 2^{-53} for binary64"


def ufp(a):
    """unit in the first place: 2^⌊log2|a|⌋, 0 for a = 0 (exact, via frexp)."""
    a = np.asarray(a, dtype=np.float64)
    m, e = np.frexp(np.abs(a))  # |a| = m 2^e, m in [0.5, 1)
    return np.where(a == 0, 0.0, np.ldexp(1.0, e - 1))


def ceil_log2(v):
    """⌈log2 v⌉ for v > 0, exact (PAPER.md:172-182 use it in σ, τ). Reading R2: computed from the
    exponent field, never a log routine; ⌈log2 2^k⌉ = k. Returns int64; 0 where v == 0."""
    v = np.asarray(v, dtype=np.float64)
    m, e = np.frexp(v)
    c = np.where(m == 0.5, e - 1, e)
    return np.where(v == 0, 0, c).astype(np.int64)


def two_sum(a, b):
    """PAPER.md:143-153 TwoSum: x = fl(a+b), y = fl((a-(x-z)) + (b-z)), z = fl(x-a); a+b = x+y."""
    x = a + b
    z = x - a
    y = (a - (x - z)) + (b - z)
    return x, y


def fast_two_sum(a, b):
    """x = fl(a+b), y = b - (x - a); exact when |a| >= |b| (Dekker)."""
    x = a + b
    return x, b - (x - a)


_SPLITTER = 134217729.0  # 2^27 + 1


def _veltkamp(a):
    c = _SPLITTER * a
    hi = c - (c - a)
    return hi, a - hi


def two_prod(a, b):
    """x = fl(a*b), y = a*b - x exactly (Dekker's TwoProduct with Veltkamp splitting; no FMA needed,
    the error term is unique so this equals the FMA formulation)."""
    x = a * b
    ah, al = _veltkamp(a)
    bh, bl = _veltkamp(b)
    y = al * bl - (((x - ah * bh) - al * bh) - ah * bl)
    return x, y


def pair_add(a, bh, bl):
    """a + (b_h + b_l) ≈ c_h + c_l with [c_h, t] = TwoSum(a, b_h), c_l = fl(b_l + t)."""
    ch, t = two_sum(a, bh)
    return ch, bl + t


def dd_add(ah, al, bh, bl):
    """Accurate double-double addition (both lower parts kept)."""
    s, e = two_sum(ah, bh)
    t, f = two_sum(al, bl)
    e = e + t
    s, e = fast_two_sum(s, e)
    e = e + f
    return fast_two_sum(s, e)


def dd_mul_d(ah, al, b):
    """(ah + al) * b in double-double."""
    p, e = two_prod(ah, b)
    e = e + al * b
    return fast_two_sum(p, e)


def dd_div_dd(ah, al, bh, bl):
    """(ah + al) / (bh + bl) to double-double accuracy (one Newton correction)."""
    q1 = ah / bh
    ph, pl = dd_mul_d(bh, bl, q1)
    rh, rl = dd_add(ah, al, -ph, -pl)
    q2 = rh / bh
    return fast_two_sum(q1, q2)
