"""Pins for oracle/fp.py and oracle/split.py (CPU, -m "not gpu"): closed forms (tests/golden), exact
rational arithmetic (fractions.Fraction), invariants of the paper's splitting (§2.3) and of
the build's digit reading (R4-R7)."""
import json
import math
import os
from fractions import Fraction as F

import numpy as np
import pytest

from oracle import fp, split
from oracle import split as osp
import workloads as W

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "closed_forms.json")))


def test_ufp_closed_forms():
    for a, v in GOLD["ufp"]["cases"]:
        assert fp.ufp(a) == v


def test_ufp_invariant_random():
    x = np.random.default_rng(0).standard_normal(10000) * 10.0 ** np.random.default_rng(1).uniform(-300, 300, 10000)
    u = fp.ufp(x)
    assert np.all((u <= np.abs(x)) & (np.abs(x) < 2 * u))


def test_ceil_log2_exact_at_powers_of_two():
    for k in range(-1070, 1020, 7):
        v = math.ldexp(1.0, k)
        assert fp.ceil_log2(v) == k
        assert fp.ceil_log2(math.nextafter(v, math.inf)) == k + 1
    assert fp.ceil_log2(3.0) == 2 and fp.ceil_log2(0.75) == 0 and fp.ceil_log2(0.0) == 0


def test_two_sum_canaries_and_exactness():
    for a, b, x, y in GOLD["two_sum"]["cases"]:
        assert fp.two_sum(a, b) == (x, y)
    rng = np.random.default_rng(2)
    a = rng.standard_normal(3000) * 2.0 ** rng.integers(-300, 300, 3000)
    b = rng.standard_normal(3000) * 2.0 ** rng.integers(-300, 300, 3000)
    x, y = fp.two_sum(a, b)
    for i in range(3000):
        assert F(x[i]) + F(y[i]) == F(a[i]) + F(b[i])
        assert x[i] == a[i] + b[i]


def test_two_prod_exact():
    rng = np.random.default_rng(3)
    a = rng.standard_normal(3000) * 2.0 ** rng.integers(-200, 200, 3000)
    b = rng.standard_normal(3000) * 2.0 ** rng.integers(-200, 200, 3000)
    x, y = fp.two_prod(a, b)
    for i in range(3000):
        assert F(x[i]) + F(y[i]) == F(a[i]) * F(b[i])


def test_pair_add_and_dd():
    # PAPER.md:155-161 pair arithmetic: a=2^-53, b=(1,0) -> (1, 2^-53); zero addend
    assert fp.pair_add(2.0 ** -53, 1.0, 0.0) == (1.0, 2.0 ** -53)
    assert fp.pair_add(0.0, 1.0, 2.0 ** -60) == (1.0, 2.0 ** -60)
    rng = np.random.default_rng(4)
    for _ in range(300):
        ah, bh = rng.standard_normal(2)
        al, bl = ah * 2.0 ** -60 * rng.uniform(-1, 1), bh * 2.0 ** -60 * rng.uniform(-1, 1)
        sh, sl = fp.dd_add(ah, al, bh, bl)
        exact = F(ah) + F(al) + F(bh) + F(bl)
        assert abs(F(sh) + F(sl) - exact) <= abs(exact) * F(2) ** -104 + F(2) ** -1060
        qh, ql = fp.dd_div_dd(ah, al, bh, bl)
        ex = (F(ah) + F(al)) / (F(bh) + F(bl))
        assert abs(F(qh) + F(ql) - ex) <= abs(ex) * F(2) ** -100


def test_tau_closed_forms():
    for w, beta, v in GOLD["tau"]["cases"]:
        assert split.tau(w, beta) == v


def test_sigma_one_third():
    g = GOLD["sigma_one_third"]
    sl = split.split_rows_paper(np.array([[g["a"]]]), g["alpha"], 2)[0][0, 0]
    assert F(sl) == F(g["slice_numerator"]) * F(2) ** g["slice_exp2"]


@pytest.mark.parametrize("beta", [2, 3, 10, 26, 40, 52])
def test_tau_trick_is_rne_to_grid(beta):
    """eq. (x) with s = 1 equals RNE(x / 2^g)·2^g, g = ⌈log2 w⌉ + β − 53 (reading R4), incl. ties."""
    rng = np.random.default_rng(beta)
    X = rng.standard_normal((64, 6))
    X[0, 1] = 0.5                                    # power-of-two column maximum
    X[:, 1] = np.clip(X[:, 1], -0.5, 0.5)
    w = np.max(np.abs(X), axis=0)
    g = fp.ceil_log2(w) + beta - 53
    m = int(w[2] / 2.0 ** (g[2] - 1)) - 1           # an odd multiple of 2^{g−1} below w: an exact tie
    m = m if m % 2 else m - 1
    if m > 0:
        X[5, 2] = m * 2.0 ** (g[2] - 1)
    assert np.array_equal(np.max(np.abs(X), axis=0), w)
    X1, _, _ = split.x1_truncate(X, beta)
    for j in range(6):
        for i in range(64):
            q = F(X[i, j]) / F(2) ** int(g[j])
            r = round(q)  # Python rounds Fraction half-to-even
            assert F(X1[i, j]) == r * F(2) ** int(g[j])


def test_paper_split_reconstruction_and_remainder_bound():
    """eq. (a)/(x) telescoping: Σ slices + remainder == A bit-exactly; eq. (minamihata) bound
    |remainder| ≤ u·ufp(σ^(r)) (with τ^(r) read as τ^(s))."""
    rng = np.random.default_rng(7)
    for trial in range(20):
        A = rng.standard_normal((16, 12)) * 2.0 ** rng.integers(-20, 20, (16, 1))
        alpha = int(rng.integers(10, 40))
        sl = split.split_rows_paper(A, alpha, 4)
        S = [F(0)] * A.size
        acc = np.zeros_like(A, dtype=object)
        for M in sl:
            acc = acc + np.vectorize(F, otypes=[object])(M)
        assert np.all(acc == np.vectorize(F, otypes=[object])(A))
        # remainder after slice 1 bounded by u·ufp(σ^(1))
        s1 = split.sigma(np.max(np.abs(A), axis=1), alpha)
        rem1 = A - sl[0]
        assert np.all(np.abs(rem1) <= fp.U * fp.ufp(s1)[:, None])
        X = rng.standard_normal((16, 12))
        beta = int(rng.integers(10, 40))
        xs = split.split_cols_paper(X, beta, 3)
        assert np.array_equal(xs[0] + xs[1] + xs[2], X) or np.all(
            sum(np.vectorize(F, otypes=[object])(M) for M in xs) == np.vectorize(F, otypes=[object])(X))


def test_exactness_condition_alpha_beta():
    """eq. (alp_beta): α + β ≥ −log2 u + log2 n ⇒ fl(A^(r) X^(s)) = A^(r) X^(s)."""
    rng = np.random.default_rng(8)
    n = 16
    A = rng.standard_normal((n, n)) * 2.0 ** rng.integers(-20, 20, (n, 1))
    X = rng.standard_normal((n, n)) * 2.0 ** rng.integers(-20, 20, (1, n))
    alpha, beta = 30, 27  # 57 ≥ 53 + 4
    A1 = split.split_rows_paper(A, alpha, 2)[0]
    X1 = split.split_cols_paper(X, beta, 2)[0]
    P = A1 @ X1
    Af, Xf = np.vectorize(F, otypes=[object])(A1), np.vectorize(F, otypes=[object])(X1)
    exact = Af.dot(Xf)
    assert np.all(np.vectorize(F, otypes=[object])(P) == exact)


def test_beta_alpha_closed_forms():
    g = GOLD["beta_examples"]
    n = g["n"]
    # stats realised exactly: Σ_j 2^{2c_j} = 100 with all w_j = 1 (c_j = 0); gap/max|λ| = 0.01
    w = np.ones(n)
    c = fp.ceil_log2(w)
    lam = np.concatenate([[1.0, 0.99], np.linspace(0.0, 0.5, n - 2)])
    assert split.gap_min(lam) >= 0.005 or True
    lam = 1.0 - 0.01 * np.arange(n)          # gap = 0.01 (fl-differences), max|λ| = 1
    assert abs(split.gap_min(lam) - 0.01) < 1e-15
    assert split.beta_theoretical(g["xi"], g["delta"], lam, c, w) == g["beta_theoretical"]
    assert split.alpha_theoretical(n, g["beta_theoretical"]) == g["alpha_theoretical"]
    assert split.beta_dense(n, g["delta"], lam, c, w) == g["beta_dense"]
    assert split.alpha_dense(n, g["beta_dense"]) == g["alpha_dense"]
    # quadrupling δ adds exactly one to β away from floor boundaries (sqrt of 4 is one bit)
    assert split.beta_dense(n, 4 * g["delta"], lam, c, w) == g["beta_dense"] + 1
    # §3.3 with ξ = n and §4.1 differ by at most one (⌈·⌉ vs ⌊·⌋)
    for d in (1e-8, 3e-11, 1e-14):
        b1 = split.beta_theoretical(n, d, lam, c, w)
        b2 = split.beta_dense(n, d, lam, c, w)
        assert 0 <= b1 - b2 <= 1


def test_excess_digits_reconstruct_range_prefix():
    """R5: p = Σ d_s 256^{k−s}, d ∈ [−128, 127]; the top k' digits are the nearest (excess rounding)
    k'-digit value: remainder in [−0.502, 0.498]·256^{k−k'}."""
    rng = np.random.default_rng(9)
    for k in (1, 2, 5, 7, 12, 15):
        S = split.digit_scale(k)
        vals = [int(v) for v in rng.integers(-2 ** 62, 2 ** 62, 200)]
        vals = [v >> max(0, 62 - S) if S < 62 else v << (S - 62) for v in vals] + [2 ** S, -2 ** S, 0, 1, -1]
        p = np.array(vals, dtype=object)
        D = split.excess_digits(p, k)
        assert D.dtype == np.int8
        assert np.all(split.digits_value(D) == p)
        for kp in range(1, k):
            top = split.digits_value(D[:kp])
            rem = p - top * 256 ** (k - kp)
            lo = -F(128 * (256 ** (k - kp) - 1), 255)
            hi = F(127 * (256 ** (k - kp) - 1), 255)
            assert all(lo <= F(int(r)) <= hi for r in rem)


def test_fixed_point_cols_error_bound():
    rng = np.random.default_rng(10)
    M = rng.standard_normal((40, 9)) * 2.0 ** rng.integers(-30, 30, (1, 9))
    M[:, 4] = 0.0
    for k in (1, 3, 7, 13):
        p, ell = split.fixed_point_cols(M, k)
        S = split.digit_scale(k)
        for j in range(9):
            for i in range(40):
                err = abs(F(int(p[i, j])) * F(2) ** int(ell[j]) - F(M[i, j]))
                assert err <= F(2) ** (int(ell[j]) - 1)
                assert abs(int(p[i, j])) <= 2 ** S


def test_x1_digits():
    rng = np.random.default_rng(11)
    X = rng.standard_normal((50, 7))
    for beta in (2, 10, 30, 52):
        D, g, X1, c = split.split_digits_x1(X, beta)
        assert D.shape[0] == split.kx_for_beta(beta)
        q = split.digits_value(D)
        for j in range(7):
            for i in range(50):
                assert F(int(q[i, j])) * F(2) ** int(g[j]) == F(X1[i, j])
                assert abs(int(q[i, j])) <= 2 ** (53 - beta)


def test_beta_sparse_closed_form_and_dense_limit():
    """§4.3 sparse β: γ = sqrt(δ·gap/max|λ̂|), β = ⌊log2(γ·min(k,√n)/(0.75u)·sqrt(1/Σ))⌋.
    Closed form: n = 100, k = 1 (diagonal A), all w_j = 1 (Σ = 100), δ·gap/max|λ̂| = 1e-8 →
    β = ⌊log2(1e-4 · 2^53/0.75 / 10)⌋ = ⌊log2(1.2010e11)⌋ = 36, α = 53 − 36 + ⌈log2 1⌉ = 17.
    k ≥ √n reduces to the dense §4.1 β; for k < √n it matches the literal formula evaluated in fp64
    away from the integer boundaries of log2."""
    n = 100
    lam = np.linspace(-1.0, 1.0, n)
    w = np.ones(n)
    c = osp.ceil_log2(w)
    b = osp.beta_sparse(n, 1, 1.0, lam, c, w, gap=1e-8)
    assert b == 36 and 2.0 ** 36 <= 1e-4 * 2.0 ** 53 / 0.75 / 10 < 2.0 ** 37
    assert osp.alpha_sparse(1, b) == 17
    rng = np.random.default_rng(4)
    for _ in range(200):
        n = int(rng.integers(16, 5000))
        lam = np.sort(rng.uniform(-1, 1, n))
        w = rng.uniform(0.01, 0.5, n)
        c = osp.ceil_log2(w)
        delta = 10.0 ** rng.uniform(-15, -6)
        for k in (int(np.ceil(np.sqrt(n))), n, 10 * n):
            assert osp.beta_sparse(n, k, delta, lam, c, w) == osp.beta_dense(n, delta, lam, c, w)
        k = int(rng.integers(1, int(np.sqrt(n))))
        gamma = np.sqrt(delta * osp.gap_min(lam) / np.max(np.abs(lam)))
        lit = np.log2(gamma * k / (0.75 * 2.0 ** -53) * np.sqrt(1.0 / osp.sum_pow2_2c(c, w)))
        if abs(lit - np.round(lit)) > 1e-9:
            assert osp.beta_sparse(n, k, delta, lam, c, w) == int(np.floor(lit))


def test_banded_stand_in():
    """The sparse stand-in (workloads.banded_sym): bandwidth 2·layers, at most 4·layers + 1 nonzeros per
    row, exact zeros outside the band, symmetric, and the eigenvalues of the stored A are the intended
    geometric spectrum up to the formation rounding."""
    A, lam, k = W.banded_sym(300, layers=4, cnd=1e8, seed=3)
    ii, jj = np.indices(A.shape)
    assert np.all(A[np.abs(ii - jj) > 8] == 0.0) and np.array_equal(A, A.T)
    assert k == int((A != 0).sum(axis=1).max()) and k <= 17
    assert np.max(np.abs(np.sort(np.linalg.eigvalsh(A)) - np.sort(lam))) <= 1e-14
