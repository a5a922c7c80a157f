"""Same-definition slice products and their recombination (TEST INFRASTRUCTURE ONLY).

PAPER.md §2.3 (lines 198-215): a product of two slices whose significands are short enough is exact
("A^(r) X^(s) = fl(A^(r) X^(s))", eq. alp_beta), and AX = Σ_r Σ_s A^(r) X^(s). §3.3 eq. (mat_mul)
(lines 412-421) keeps only X^(1), giving n_A products. In the build's INT8 reading every slice is a
digit plane and every slice product an exact integer matrix; the pair set kept is {(s,t): s+t ≤ L}
(reading R7). Here the planes are formed with float64 matrix products, which are EXACT because every
partial sum is an integer of magnitude < K·2^14·(pairs) < 2^53; recombination uses Python integers.
"""
import numpy as np

INT32_MAX = 2 ** 31 - 1


def max_pairs_per_group(K):
    """Largest number of digit pairs one int32 accumulator may hold exactly: K·npairs·2^14 ≤ 2^31−1
    (|digit| ≤ 128, so |product| ≤ 2^14). Reading R7b."""
    return max(1, INT32_MAX // (int(K) * 2 ** 14))


def plan_groups(kA, kB, L, K):
    """Reading R7: pairs (s,t), 1 ≤ s ≤ kA, 1 ≤ t ≤ kB, s+t ≤ L, grouped by diagonal d = s+t
    (ascending d, then ascending s); a diagonal with more pairs than max_pairs_per_group(K) is cut
    into consecutive chunks. Returns a list of (d, [(s,t), ...]) in output-plane order."""
    cap = max_pairs_per_group(K)
    groups = []
    for d in range(2, min(L, kA + kB) + 1):
        pairs = [(s, d - s) for s in range(1, kA + 1) if 1 <= d - s <= kB]
        for i in range(0, len(pairs), cap):
            groups.append((d, pairs[i:i + cap]))
    return groups


def slice_planes(DA, DB, groups):
    """Exact int planes C_g = Σ_{(s,t) in g} DA_sᵀ DB_t. DA: (kA, K, M), DB: (kB, K, N) int8, digits
    of the contraction-first operands (row index = contraction index). Returns int64 (G, M, N)."""
    K, M = DA.shape[1], DA.shape[2]
    N = DB.shape[2]
    out = np.zeros((len(groups), M, N), dtype=np.int64)
    for gi, (d, pairs) in enumerate(groups):
        acc = np.zeros((M, N))
        for (s, t) in pairs:
            acc += DA[s - 1].astype(np.float64).T @ DB[t - 1].astype(np.float64)
        assert np.all(np.abs(acc) <= INT32_MAX)
        out[gi] = acc.astype(np.int64)
    return out


def recombine_exact(planes, groups, L):
    """T'_ij = Σ_g 256^{L − d_g} C_g,ij as exact Python integers (object array)."""
    T = np.zeros(planes.shape[1:], dtype=object)
    for gi, (d, _) in enumerate(groups):
        T = T + planes[gi].astype(object) * (256 ** (L - d))
    return T


def to_dd(T, exp2):
    """Round exact integers T·2^exp2 to a correctly-rounded double-double (hi = RN(x), lo = RN(x−hi)).
    exp2 broadcasts against T (per-row / per-column exponents)."""
    T = np.asarray(T, dtype=object)
    hi = np.vectorize(float, otypes=[np.float64])(T) if T.size else np.zeros(T.shape)
    rest = T - np.vectorize(int, otypes=[object])(hi) if T.size else T
    lo = np.vectorize(float, otypes=[np.float64])(rest) if T.size else np.zeros(T.shape)
    return np.ldexp(hi, exp2), np.ldexp(lo, exp2)


def digit_product(DA, ellA, KA, DB, ellB, KB, L):
    """The whole same-definition product: value_ij = 2^{ℓA_i + ℓB_j} · 256^{KA+KB−L} · T'_ij
    (digit s of a K-digit split has weight 256^{K−s}·2^ℓ). Returns (hi, lo, planes, groups)."""
    kA, kB = DA.shape[0], DB.shape[0]
    groups = plan_groups(kA, kB, L, DA.shape[1])
    planes = slice_planes(DA, DB, groups)
    T = recombine_exact(planes, groups, L)
    e = np.asarray(ellA)[:, None] + np.asarray(ellB)[None, :] + 8 * (KA + KB - L)
    hi, lo = to_dd(T, e)
    return hi, lo, planes, groups


def accmul_fixed_k(A, B, k):
    """The prior work's two-sided accurate product with a FIXED number of slices (eq. mat3 -
    mat10; cost model PAPER.md:437-443: n_A = n_X = k slices and the ½k(k+1) slice products A^(s)X^(t) with
    s + t ≤ k + 1), in the build's INT8 digit reading (R5-R7): A split row-wise and B column-wise into k digits
    (fixed point per line, RNE), the pairs s + t ≤ k + 1 summed exactly, rounded once to double-double.
    Returns (hi, lo, npairs)."""
    from .split import split_digits_cols
    A = np.asarray(A, dtype=np.float64)
    B = np.asarray(B, dtype=np.float64)
    DA, eA = split_digits_cols(A.T, k)  # rows of A = columns of Aᵀ (contraction index first)
    DB, eB = split_digits_cols(B, k)
    hi, lo, _, groups = digit_product(DA, eA, k, DB, eB, k, k + 1)
    return hi, lo, sum(len(p) for _, p in groups)
