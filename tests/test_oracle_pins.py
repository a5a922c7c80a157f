"""Pins for the oracle parts that round 1 left unpinned (CPU, -m "not gpu"):

 - refine.cluster_subsolve (the Rayleigh–Ritz sub-solve of reading R13, builder-defined: PAPER.md:333 and 730
   leave clusters open, PAPER.md:233-235 cite the Ogita–Aishima cluster refinement it restates) — against
   exactly known eigensystems: an exactly double eigenvalue and a dyadic near-double pair whose start mixes the
   pair by 30° (only a correct M, C = I + R/2, K = C·M·C and Z = C·Y recover it), and against __float128 Jacobi
   through the whole driver (orf.refine_to_tol) from an FP32 start of the c4 recipe;
 - split.gap_pos and split.gap_min — closed forms;
 - split.fixed_point_cols with a double-double input (reading R6: RNE(hi·2^{S−e}) + RNE(lo·2^{S−e})) — against
   exact rationals.
"""
from fractions import Fraction as F

import numpy as np
import pytest

import workloads as W
from oracle import _clib
from oracle import refine as orf
from oracle import split as osp

U = 2.0 ** -53


def _exact_A(A, X, lam):
    """A = X diag(λ) Xᵀ holds exactly in fp64 (integer check with the Householder scaling n/2 and 2^s)."""
    n = A.shape[0]
    s = 0
    while not np.all(np.ldexp(lam, s) == np.rint(np.ldexp(lam, s))):
        s += 1
    Hn = np.rint(X * n / 2).astype(object)
    m = np.rint(np.ldexp(lam, s)).astype(np.int64).astype(object)
    exact = (Hn * m[None, :]).dot(Hn.T)
    return all(F(int(exact[i, j])) == F(A[i, j]) * F(n // 2) ** 2 * F(2) ** s for i in range(n) for j in range(n))


def test_cluster_subsolve_exact_double_eigenvalue():
    """λ_10 = λ_11 exactly: the pair's Rayleigh quotients coincide to ~1e-18, so (10, 11) is an unresolved
    group; after ONE sweep (untruncated, so only the products' dd rounding remains) columns 10, 11 are an
    orthonormal basis of the exact eigenspace to 1e-15 and every other column equals the exact eigenvector
    to 1e-15 (a dropped C = I + R/2 leaves a 1e-11 orthogonality defect; a wrong Ẽ_{K,J}Z leaves the other
    columns' 1e-11 components). The start's other errors are 1e-11, so the quadratic term of the sweep,
    ~(1e-11·√n)²·‖A‖/gap (gap ≥ 2^-12), stays below 1e-16."""
    A, lam, X, X0 = W.householder_pair(split=0.0, noise=1e-11)
    assert _exact_A(A, X, lam)
    Xn, ln, info = orf.sweep(A, X0, lam, 1e-15, truncate=False)
    assert info["clusters"] == [[10, 11]]
    P = X[:, [10, 11]]
    XJ = Xn[:, [10, 11]]
    assert np.max(np.abs(XJ - P @ (P.T @ XJ))) <= 1e-15          # inside the exact eigenspace
    assert np.max(np.abs(XJ.T @ XJ - np.eye(2))) <= 1e-15          # orthonormal
    other = np.setdiff1d(np.arange(A.shape[0]), [10, 11])
    assert np.max(np.abs(Xn[:, other] - X[:, other])) <= 1e-15
    assert np.max(np.abs(ln[[10, 11]] - lam[10])) <= 1e-15


@pytest.mark.parametrize("angle", [np.pi / 6, 1.2])
def test_cluster_subsolve_recovers_rotated_pair(angle):
    """λ_11 = λ_10 + 2^-30 (dyadic: A stays exact) and X̂₀ mixes the two exact eigenvectors by `angle`: the
    first-order ẽ_ij = w_ij/(λ̂_j − λ̂_i) is O(1) > κ, the pair is a group, and the Rayleigh–Ritz sub-solve
    must undo the rotation — K's eigenvectors Y with y_kk ≥ 0 and Z = C·Y. One untruncated sweep: every
    column equals the exact eigenvector to 1e-15 (the start's other errors are 1e-13: the second-order term
    inside the pair, ~ε²‖A‖/2^-30, stays below 1e-16) and the pair's λ̂ are exact to 1e-15·‖A‖ (a sign error in
    M = W_JJ + (I − R_JJ)(D̂_J − μI) or in K's ordering swaps or mixes the pair)."""
    A, lam, X, X0 = W.householder_pair(split=2.0 ** -30, angle=angle, noise=1e-13)
    assert _exact_A(A, X, lam)
    Xn, ln, info = orf.sweep(A, X0, lam, 1e-15, truncate=False)
    assert [sorted(J) for J in info["clusters"]] == [[10, 11]]
    # beyond 45° the start's column 11 carries the smaller Rayleigh quotient: the group lists it first and it
    # receives the smaller Ritz value, so the columns are matched by ascending λ̂
    p = np.argsort(ln, kind="stable")
    Xn, ln = Xn[:, p], ln[p]
    s = np.sign(np.sum(Xn * X, axis=0))
    assert np.max(np.abs(Xn * s[None, :] - X)) <= 1e-15
    assert np.max(np.abs(ln - lam)) <= 1e-15
    # the start is far from X in the pair: the first-order correction alone could not have done this
    assert np.max(np.abs(X0[:, [10, 11]] - X[:, [10, 11]])) > 0.3


def test_driver_with_cluster_branch_vs_quad_jacobi():
    """The c4 recipe (cnd 1e14) at n = 24 from an FP32 eigensolver start, through the oracle's own driver
    (orf.refine_to_tol with the truncation and the cluster branch — not the reference's _reference_rr): the
    first sweep has unresolved groups (cluster_subsolve runs), and the driver reaches the __float128 Jacobi
    eigenvectors of the stored A within δ = 1e-14 (2-norm) and its eigenvalues within 1e-15·‖A‖."""
    A, _ = W.make_matrix(24, "geometric", 1e14, 1004)
    lam0, X0 = W.initial_eig(A, "fp32")
    wh, wl, Vh, Vl, sw = _clib.jacobi_q(A)
    assert sw > 0
    delta = 1e-14
    assert orf.sweep(A, X0, lam0, delta)[2]["clusters"], "the FP32 start must exercise the sub-solve"
    X, lam, hist = orf.refine_to_tol(A, X0, lam0, delta, max_sweeps=12, callback=lambda X, l: {})
    assert hist[-1]["stop"].startswith("converged"), hist
    fe = orf.forward_error(Vh, Vl, X, wh, lam)
    assert fe <= delta, (fe, hist)
    p, q = np.argsort(lam), np.argsort(wh)
    assert np.max(np.abs(lam[p] - (wh[q] + wl[q]))) <= 1e-15


def test_gap_pos_and_gap_min_closed_forms():
    assert osp.gap_pos([0.0, 2.0, 2.0, 5.0]) == 2.0
    assert osp.gap_min([0.0, 2.0, 2.0, 5.0]) == 0.0
    assert osp.gap_pos([3.0, 3.5, 3.5]) == 0.5
    assert osp.gap_pos([5.0, -1.0, 4.0, 4.0, -1.0]) == 1.0      # unsorted, with repeats
    assert osp.gap_min([5.0, -1.0, 4.25]) == 0.75
    assert osp.gap_pos([1.0, 1.0, 1.0]) == U                    # every gap zero: u·max|λ̂|
    assert osp.gap_pos([-4.0, -4.0]) == 4.0 * U
    assert osp.gap_pos([0.0, 0.0]) == 1e-300                    # zero spectrum: the floor
    assert osp.gap_min([7.0]) == np.inf
    # the fl-difference of neighbours: 1 + 2^-52 and 1 are one ulp apart
    assert osp.gap_pos([1.0 + 2.0 ** -52, 1.0, 1.0]) == 2.0 ** -52


def test_fixed_point_cols_double_double_vs_rationals():
    """R6 for a double-double column (Res = V − X̂D̂ in the sweep): p = RNE(hi·2^{S−e}) + RNE(lo·2^{S−e}) with
    e = ⌈log2 max|hi|⌉, so |p·2^ℓ − (hi + lo)| ≤ 2^ℓ (two roundings of half an LSB each), ℓ = e − S, and the
    digits reconstruct p exactly."""
    rng = np.random.default_rng(21)
    hi = rng.standard_normal((30, 6)) * 2.0 ** rng.integers(-40, 10, (1, 6))
    lo = hi * 2.0 ** -53 * rng.uniform(-1, 1, hi.shape)
    hi[:, 3] = 0.0
    lo[:, 3] = 0.0
    hi[0, 5] = 2.0 ** -7  # a power-of-two maximum: e = -7 exactly
    for k in (1, 4, 9, 15):
        p, ell = osp.fixed_point_cols(hi, k, lo)
        S = osp.digit_scale(k)
        for j in range(6):
            e = 0 if not np.any(hi[:, j]) else int(osp.ceil_log2(np.max(np.abs(hi[:, j]))))
            assert int(ell[j]) == e - S
            for i in range(30):
                err = abs(F(int(p[i, j])) * F(2) ** int(ell[j]) - (F(hi[i, j]) + F(lo[i, j])))
                assert err <= F(2) ** int(ell[j])
        D, ell2 = osp.split_digits_cols(hi, k, lo)
        assert np.array_equal(ell, ell2)
        q = osp.digits_value(D)
        assert all(int(q[i, j]) == int(p[i, j]) for i in range(30) for j in range(6))
