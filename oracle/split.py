"""Splitting (TEST INFRASTRUCTURE ONLY — see oracle/__init__.py).

Two things live here:

1. The paper's error-free splitting, literally (§2.3):
   v_i = max_j |a_ij|, w_j = max_i |x_ij|                                  (lines 166-169)
   σ_i = 0.75 · 2^⌈log2 v_i⌉ · 2^α,  τ_j = 0.75 · 2^⌈log2 w_j⌉ · 2^β       (eq. sigma / eq. tau, 170-183)
   a^(r) = fl(fl(σ + a) − σ), remainder fl(a − a^(r))                      (eq. a, 184-188)
   x^(s) = fl(fl(τ + x) − τ), remainder fl(x − x^(s))                      (eq. x, 189-193)
   and the choice of β / α: §3.3 eq. (proposed_beta) (lines 400-405) and the tuned §4.1 values
   (lines 458-463).

2. The build's INT8 digit reading of the slices (readings R4-R6): an FP64 slice with a
   limited significand is replaced by an integer p on a per-row/column fixed-point grid, written
   as k base-256 "excess-128" digits in [-128, 127]. Written here independently of the CUDA code,
   from the definitions in DESIGN.md.
"""
import numpy as np

from .fp import U, ceil_log2

# ----------------------------------------------------------------------------- paper §2.3


def sigma(v, alpha):
    """eq. (sigma): 0 if v = 0 else 0.75 · 2^⌈log2 v⌉ · 2^α."""
    v = np.asarray(v, dtype=np.float64)
    return np.where(v == 0, 0.0, 0.75 * np.ldexp(1.0, ceil_log2(v) + int(alpha)))


def tau(w, beta):
    """eq. (tau): 0 if w = 0 else 0.75 · 2^⌈log2 w⌉ · 2^β."""
    return sigma(w, beta)


def split_rows_paper(A, alpha, nA):
    """eq. (a), r = 1..nA-1, plus the final remainder A_(nA) (eq. mat_mul,
    PAPER.md:407-411: A = A^(1) + ... + A^(nA-1) + A_(nA)). Row-wise σ from the current remainder's
    row maxima (PAPER.md:166-169 recomputed per r). Returns a list of nA fp64 matrices."""
    rem = np.array(A, dtype=np.float64)
    out = []
    for _ in range(nA - 1):
        s = sigma(np.max(np.abs(rem), axis=1), alpha)[:, None]
        sl = (s + rem) - s
        out.append(sl)
        rem = rem - sl
    out.append(rem)
    return out


def split_cols_paper(X, beta, nX):
    """eq. (x), column-wise τ, s = 1..nX-1, plus the remainder."""
    rem = np.array(X, dtype=np.float64)
    out = []
    for _ in range(nX - 1):
        t = tau(np.max(np.abs(rem), axis=0), beta)[None, :]
        sl = (t + rem) - t
        out.append(sl)
        rem = rem - sl
    out.append(rem)
    return out


def x1_truncate(X, beta):
    """The proposed method's X̂ ← X̂^(1): eq. (x) with s = 1,
    x^(1)_ij = fl(fl(τ_j + x_ij) − τ_j). Returns (X1, w, c) with w_j the column maxima of |X̂| before
    truncation (reading R6 of DESIGN.md) and c_j = ⌈log2 w_j⌉."""
    X = np.asarray(X, dtype=np.float64)
    w = np.max(np.abs(X), axis=0)
    t = tau(w, beta)[None, :]
    X1 = (t + X) - t
    return X1, w, ceil_log2(w)


def sum_pow2_2c(c, w):
    """Σ_j 2^{2⌈log2 w_j⌉} over columns with w_j ≠ 0 (PAPER.md:380-383 eq. tau_ex, 403, 461).
    Reading R3b: summed in fp64 in ascending order of c_j (exact in every realistic case)."""
    cs = np.sort(np.asarray(c)[np.asarray(w) != 0])
    s = 0.0
    for ci in cs:
        s = s + float(np.ldexp(1.0, 2 * int(ci)))
    return s


def gap_min(lam):
    """min_{i≠j} |λ_j − λ_i|, as min over fl-differences of sorted λ̂."""
    ls = np.sort(np.asarray(lam, dtype=np.float64))
    if ls.size < 2:
        return np.inf
    return float(np.min(ls[1:] - ls[:-1]))


def _z_value(n_or_xi, delta, gap, maxlam, ssum):
    """(1/(0.75u)) · sqrt(c·δ·gap / (max|λ| · Σ)), evaluated in the order fixed by reading R3:
    t = ((c·δ)·gap) / (max|λ|·Σ);  Z = sqrt(t) / (0.75 u)."""
    t = ((float(n_or_xi) * float(delta)) * float(gap)) / (float(maxlam) * float(ssum))
    return np.sqrt(t) / (0.75 * U)


def gap_pos(lam):
    """Smallest POSITIVE neighbour gap of the sorted λ̂ (reading R13: with the cluster branch, equal
    estimates are allowed and the smallest nonzero gap sets β and the digit budgets); u·max|λ̂| when
    every gap is zero."""
    ls = np.sort(np.asarray(lam, dtype=np.float64))
    d = ls[1:] - ls[:-1]
    if np.any(d > 0):
        return float(np.min(d[d > 0]))
    return max(float(np.max(np.abs(ls))) * U, 1e-300)


def beta_dense(n, delta, lam, c, w, gap=None):
    """§4.1: β = ⌊log2((1/(0.75u)) · sqrt(nδ·gap / (max|λ̂| Σ_j 2^{2⌈log2 w_j⌉})))⌋.
    ⌊log2 Z⌋ is exact from the exponent of the fp64 Z. Returns the unclamped integer β."""
    Z = _z_value(n, delta, gap_min(lam) if gap is None else gap, np.max(np.abs(lam)), sum_pow2_2c(c, w))
    m, e = np.frexp(Z)
    return int(e) - 1


def beta_theoretical(xi, delta, lam, c, w, gap=None):
    """§3.3 eq. (proposed_beta): β = ⌈log2((1/(0.75u)) · sqrt(δξ·gap/(max|λ̂| Σ)))⌉."""
    Z = _z_value(xi, delta, gap_min(lam) if gap is None else gap, np.max(np.abs(lam)), sum_pow2_2c(c, w))
    m, e = np.frexp(Z)
    return int(e) - 1 if m == 0.5 else int(e)


def beta_sparse(n, k, delta, lam, c, w, gap=None):
    """§4.3, PAPER.md:585-591 (sparse A, k = the largest number of nonzeros in a row):
    γ = sqrt(δ·gap/max|λ̂|),  β = ⌊log2(γ·min(k, √n)/(0.75u) · sqrt(1/Σ_j 2^{2⌈log2 w_j⌉}))⌋.
    γ·min(k,√n)·sqrt(1/Σ) = sqrt(min(k², n)·δ·gap/(max|λ̂|·Σ)), so it is evaluated in the operation order of
    the §4.1 form (reading R3) with n replaced by min(k², n)."""
    m2 = min(int(k) * int(k), int(n))
    Z = _z_value(m2, delta, gap_min(lam) if gap is None else gap, np.max(np.abs(lam)), sum_pow2_2c(c, w))
    m, e = np.frexp(Z)
    return int(e) - 1


def alpha_sparse(k, beta):
    """§4.3: α = −(log2 u + β) + ⌈log2 k⌉ (reported only)."""
    return 53 - int(beta) + int(ceil_log2(float(k)))


def alpha_dense(n, beta):
    """§4.1: α = −(log2 u + β) + ⌈log2 √n⌉ = 53 − β + ⌈log2 √n⌉ (reported only)."""
    c = 0
    while 4 ** c < n:
        c += 1
    return 53 - int(beta) + c


def alpha_theoretical(n, beta):
    """eq. (proposed_beta): α = ⌈−log2 u + log2 n − β⌉ = 53 − β + ⌈log2 n⌉."""
    return 53 - int(beta) + int(ceil_log2(float(n)))


# ----------------------------------------------------------------------------- INT8 digit reading

def kx_for_beta(beta):
    """Digits needed for q = x^(1)/2^g, |q| ≤ 2^{53−β}: smallest k with 8(k−1)+6 ≥ 53−β (R5)."""
    need = 53 - int(beta)
    k = 1
    while 8 * (k - 1) + 6 < need:
        k += 1
    return k


def digit_scale(k):
    """S_k = 8(k−1)+6: a fixed-point integer |p| ≤ 2^{S_k} has k excess-128 digits (R5)."""
    return 8 * (k - 1) + 6


def excess_digits(p, k):
    """R5: integer p (object array of Python ints, or int64) -> k digits d_1..d_k in [-128, 127] with
    p = Σ_s d_s 256^{k−s}. With O = Σ_{s=2..k} 128·256^{k−s}, w = p + O: d_s = (w mod 256^{k−s+1}
    digit) − 128 for s ≥ 2 and d_1 = ⌊w / 256^{k−1}⌋. Returns int8 array of shape (k,) + p.shape."""
    p = np.asarray(p, dtype=object)
    O = sum(128 * 256 ** (k - s) for s in range(2, k + 1))
    w = p + O
    out = np.empty((k,) + p.shape, dtype=np.int64)
    for s in range(k - 1, 0, -1):
        out[s] = np.asarray(w % 256 - 128, dtype=np.int64)
        w = w // 256
    out[0] = np.asarray(w, dtype=np.int64)
    if out.size and (out.min() < -128 or out.max() > 127):
        raise ValueError("digit out of range: value too large for k digits")
    return out.astype(np.int8)


def digits_value(D):
    """Inverse of excess_digits: Σ_s d_s 256^{k−s} as Python ints (object array)."""
    D = np.asarray(D)
    k = D.shape[0]
    v = np.zeros(D.shape[1:], dtype=object)
    for s in range(k):
        v = v * 256 + D[s].astype(object)
    return v


def _rint_to_int(x):
    """exact conversion of integer-valued float64 (after np.rint, RNE) to Python ints."""
    r = np.rint(x)
    return np.vectorize(int, otypes=[object])(r) if r.size else np.zeros(r.shape, dtype=object)


def fixed_point_cols(M, k, Mlo=None):
    """R6: column-wise fixed point. e_j = ⌈log2 max_i |m_ij|⌉ (0 for a zero column), S = S_k,
    p_ij = RNE(m_ij · 2^{S−e_j})  [+ RNE(lo_ij · 2^{S−e_j}) for a double-double input].
    Returns (p as object ints, lsb exponent ℓ_j = e_j − S)."""
    M = np.asarray(M, dtype=np.float64)
    w = np.max(np.abs(M), axis=0) if M.shape[0] else np.zeros(M.shape[1])
    e = ceil_log2(w)
    S = digit_scale(k)
    sh = (S - e)[None, :]
    p = _rint_to_int(np.ldexp(M, sh))
    if Mlo is not None:
        p = p + _rint_to_int(np.ldexp(np.asarray(Mlo, dtype=np.float64), sh))
    return p, (e - S).astype(np.int64)


def split_digits_cols(M, k, Mlo=None):
    """Column-wise k-digit split (R5+R6): returns (D int8 (k, rows, cols), ℓ (cols,))."""
    p, ell = fixed_point_cols(M, k, Mlo)
    return excess_digits(p, k), ell


def split_digits_x1(X, beta):
    """R4+R5: X̂^(1) digits. q_ij = x^(1)_ij / 2^{g_j} with g_j = c_j + β − 53 (exact integer,
    |q| ≤ 2^{53−β}); k_X = kx_for_beta(β) digits; ℓ_j = g_j (c_j = 0 for a zero column, so
    g_j = β − 53 there and its digits are 0). Returns (D, g, X1, c)."""
    X1, w, c = x1_truncate(X, beta)
    g = (c + int(beta) - 53).astype(np.int64)
    q = np.ldexp(X1, (-g)[None, :])
    assert np.all(q == np.rint(q)), "x^(1)/2^g must be an integer"
    kx = kx_for_beta(beta)
    qi = _rint_to_int(q)
    return excess_digits(qi, kx), g, X1, c
