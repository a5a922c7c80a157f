"""Pins for oracle/products.py, oracle/_clib (ddmm.c) and oracle/refine.py (CPU, -m "not gpu"):
brute force in exact integers/rationals, __float128 Jacobi against closed forms, an exactly-known
eigensystem family, and the paper's qualitative claims (quadratic convergence, O(δ) forward error)."""
from fractions import Fraction as F

import numpy as np
import pytest

import workloads as W
from oracle import _clib
from oracle import products as opr
from oracle import refine as orf
from oracle import split as osp


def test_plan_groups_brute_force():
    for kA, kB, L, K in [(5, 3, 6, 100), (4, 4, 8, 50000), (15, 7, 13, 16384), (2, 6, 3, 1)]:
        gs = opr.plan_groups(kA, kB, L, K)
        flat = [p for _, ps in gs for p in ps]
        want = [(s, d - s) for d in range(2, min(L, kA + kB) + 1) for s in range(1, kA + 1) if 1 <= d - s <= kB]
        assert flat == want
        cap = opr.max_pairs_per_group(K)
        assert all(len(ps) <= cap and all(s + t == d for s, t in ps) for d, ps in gs)
        assert K * cap * 2 ** 14 <= 2 ** 31 - 1 or cap == 1


def test_slice_planes_vs_python_ints():
    rng = np.random.default_rng(1)
    DA = rng.integers(-128, 128, (3, 7, 5)).astype(np.int8)
    DB = rng.integers(-128, 128, (2, 7, 4)).astype(np.int8)
    gs = opr.plan_groups(3, 2, 5, 7)
    P = opr.slice_planes(DA, DB, gs)
    for gi, (d, ps) in enumerate(gs):
        for i in range(5):
            for j in range(4):
                v = sum(int(DA[s - 1, k, i]) * int(DB[t - 1, k, j]) for s, t in ps for k in range(7))
                assert P[gi, i, j] == v


def test_digit_product_all_pairs_is_exact_product_of_split_operands():
    """With every pair kept the recombined value is the exact product of the digit-represented
    operands, correctly rounded to double-double (vs Fractions)."""
    rng = np.random.default_rng(2)
    m, k, n = 6, 9, 5
    A = rng.standard_normal((m, k)) * 2.0 ** rng.integers(-10, 10, (m, 1))
    B = rng.standard_normal((k, n))
    kA, kB = 4, 3
    DA, eA = osp.split_digits_cols(A.T, kA)
    DB, eB = osp.split_digits_cols(B, kB)
    hi, lo, _, _ = opr.digit_product(DA, eA, kA, DB, eB, kB, kA + kB)
    a = osp.digits_value(DA)  # (k, m)
    b = osp.digits_value(DB)
    for i in range(m):
        for j in range(n):
            ex = sum(F(int(a[q, i])) * F(2) ** int(eA[i]) * F(int(b[q, j])) * F(2) ** int(eB[j]) for q in range(k))
            h = float(ex)
            assert hi[i, j] == h and lo[i, j] == float(ex - F(h))


def test_to_dd_correct_rounding():
    rng = np.random.default_rng(3)
    T = np.array([int(x) << int(s) for x, s in zip(rng.integers(-2 ** 62, 2 ** 62, 300), rng.integers(0, 60, 300))],
                 dtype=object)
    hi, lo = opr.to_dd(T, 0)
    for t, h, l_ in zip(T, hi, lo):
        assert h == float(t) and l_ == float(F(int(t)) - F(h))


def test_dd_gemm_vs_rationals():
    rng = np.random.default_rng(4)
    P = rng.standard_normal((5, 40)) * 2.0 ** rng.integers(-20, 20, (5, 1))
    Q = rng.standard_normal((3, 40))
    Ql = Q * 2.0 ** -55 * rng.uniform(-1, 1, Q.shape)
    Ch, Cl = _clib.dd_gemm_nt(P, Q, None, Ql)
    for i in range(5):
        for j in range(3):
            ex = sum(F(P[i, k]) * (F(Q[j, k]) + F(Ql[j, k])) for k in range(40))
            scale = sum(abs(F(P[i, k]) * F(Q[j, k])) for k in range(40))
            assert abs(F(Ch[i, j]) + F(Cl[i, j]) - ex) <= scale * F(2) ** -100


def test_jacobi_q_closed_forms():
    wh, wl, Vh, Vl, sw = _clib.jacobi_q(np.diag([3.0, 1.0, 2.0]))
    assert list(wh) == [1.0, 2.0, 3.0] and sw >= 0
    assert np.array_equal(np.abs(Vh), np.array([[0, 0, 1], [1, 0, 0], [0, 1, 0]], dtype=float))
    # 2x2 [[0,1],[1,0]]: λ = ∓1, x = (1, ∓1)/√2 (SPEC-style analytic case)
    wh, wl, Vh, Vl, _ = _clib.jacobi_q(np.array([[0.0, 1.0], [1.0, 0.0]]))
    assert abs(wh[0] + 1) < 1e-30 and abs(wh[1] - 1) < 1e-30
    x0, x1 = F(Vh[0, 0]) + F(Vl[0, 0]), F(Vh[1, 0]) + F(Vl[1, 0])
    assert abs(x0 * x0 - F(1, 2)) < F(1, 10 ** 30) and abs(x0 * x1 + F(1, 2)) < F(1, 10 ** 30)


def test_reference_eigvecs_vs_quad_jacobi():
    """The dd Ogita–Aishima reference (used for every forward error) agrees with __float128 Jacobi."""
    A, _ = W.make_matrix(24, "geometric", 1e8, 5)
    lam0, X0 = W.initial_eig(A)
    Xh, Xl, lh, ll, hist = orf.reference_eigvecs(A, X0, lam0)
    wh, wl, Vh, Vl, sw = _clib.jacobi_q(A)
    assert sw > 0
    assert np.max(np.abs((lh - wh) + (ll - wl))) < 1e-28
    s = np.sign(np.sum(Xh * Vh, axis=0))
    assert np.max(np.abs((Xh - Vh * s) + (Xl - Vl * s))) < 1e-24


def test_reference_cluster_branch_vs_quad_jacobi():
    """The reference's Rayleigh–Ritz branch (cluster_kappa): from an FP32 eigensolver start on the c4 recipe
    (cnd 1e14), where the first-order correction is not in its linear regime for the small eigenvalues, the
    dd iteration with the branch reaches the __float128 Jacobi eigensystem."""
    A, _ = W.make_matrix(24, "geometric", 1e14, 1004)
    lam0, X0 = W.initial_eig(A, "fp32")
    wh, wl, Vh, Vl, sw = _clib.jacobi_q(A)
    s0 = np.sign(np.sum(X0 * Vh, axis=0))
    assert np.max(np.abs(X0 - Vh * s0)) > 1e-3  # the start is far from the eigenvectors
    Xh, Xl, lh, ll, hist = orf.reference_eigvecs(A, X0, lam0, max_sweeps=30, cluster_kappa=2.0 ** -10)
    p, q = np.argsort(lh), np.argsort(wh)
    Xh, Xl, lh, ll, Vh, Vl, wh, wl = Xh[:, p], Xl[:, p], lh[p], ll[p], Vh[:, q], Vl[:, q], wh[q], wl[q]
    s = np.sign(np.sum(Xh * Vh, axis=0))
    assert np.max(np.abs((Xh - Vh * s) + (Xl - Vl * s))) < 1e-20, hist
    assert np.max(np.abs((lh - wh) + (ll - wl))) < 1e-28


def test_reference_cluster_branch_certified_c4_recipe():
    """Pin P8 for the c4 recipe (n = 128, cnd 1e14, eigenvalue gaps down to 3e-15) from the FP32 eigensolver
    start (BASELINE c4): the plain dd iteration diverges, the one with the Rayleigh–Ritz branch converges,
    and its residual certificate bounds every column's error by ‖A x_j − λ_j x_j‖/gap_j (Davis–Kahan)
    ≤ 1e-15 with ‖I − XᵀX‖ ≤ 1e-17."""
    A, _ = W.make_matrix(128, "geometric", 1e14, 1004)
    lam0, X0 = W.initial_eig(A, "fp32")
    with np.errstate(all="ignore"):
        _, _, _, _, plain = orf.reference_eigvecs(A, X0, lam0, max_sweeps=6)
    assert not (np.isfinite(plain[-1]) and plain[-1] < 1e-15), plain
    Xh, Xl, lh, ll, hist = orf.reference_eigvecs(A, X0, lam0, max_sweeps=30, cluster_kappa=2.0 ** -10)
    res, orth = orf.residual_certificate(A, Xh, Xl, lh, ll)
    order = np.argsort(lh)
    d = np.diff(lh[order])
    gap = np.empty_like(lh)
    gap[order] = np.minimum(np.r_[np.inf, d], np.r_[d, np.inf])
    assert np.max(res / gap) <= 1e-15, (np.max(res / gap), hist)
    assert orth <= 1e-17


def test_reference_on_exact_householder_family():
    """Pin P6: A = H diag(λ) H exactly representable, X = H exactly."""
    A, lam, X, H, lam_cols = W.householder_exact(6, lam_bits=12, seed=3)
    n = A.shape[0]
    # exactness of the stored A: integer check (n/2)^2 2^12 A = Hn diag(m) Hn with Hn = (n/2) H
    Hn = np.rint(H * n / 2).astype(np.int64)
    m = np.rint(lam_cols * 2 ** 12).astype(np.int64)
    assert np.array_equal(((Hn * m[None, :]) @ Hn).astype(np.float64), A * (n / 2) ** 2 * 2 ** 12)
    lam0, X0 = W.initial_eig(A)
    Xh, Xl, lh, ll, _ = orf.reference_eigvecs(A, X0, lam0)
    assert orf.forward_error(Xh, Xl, X) < 1e-25
    assert np.max(np.abs(lh - lam)) < 1e-28


def test_sweep_fixed_point_and_diag_rule():
    """Alg. 1 on an exact eigensystem: X̂ = I for diagonal A is a fixed point; ẽ_ii = r_i/2."""
    A = np.diag([1.0, 2.0, 3.0, 5.0])
    Xn, lam, info = orf.sweep(A, np.eye(4), np.array([1.0, 2, 3, 5]), 1e-12)
    assert np.array_equal(Xn, np.eye(4)) and np.array_equal(lam, [1.0, 2, 3, 5])
    A, lam0, X0, _ = W.make_config("c1")
    Xn, lam, info = orf.sweep(A, X0, lam0, 1e-12)
    assert np.array_equal(np.diag(info["E"]), (info["r"][0] + info["r"][1]) / 2)
    # ẽ_ij (λ_j − λ_i) reproduces w_ij (Alg. 1 line 5)
    E, Wm = info["E"], info["W"][0] + info["W"][1]
    dl = lam[None, :] - lam[:, None]
    off = ~np.eye(100, dtype=bool)
    assert np.max(np.abs(E[off] * dl[off] - Wm[off]) / np.abs(Wm[off])) < 1e-15


def test_sweep_2x2_rotation():
    """A = diag(1,2), X̂ = rotation by θ: one untruncated sweep leaves an O(θ²) error (Theorem 1)."""
    A, X = W.pivot_2x2(1e-4)
    Xn, lam, info = orf.sweep(A, X, np.array([1.0, 2.0]), 1e-15, truncate=False)
    err = np.max(np.abs(np.abs(Xn) - np.eye(2)))
    assert err < 1e-8
    # X = X̂(I + E) with X = I  =>  E ≈ X̂ᵀ − I: e_10 ≈ −θ, e_01 ≈ +θ
    assert abs(info["E"][1, 0] + 1e-4) < 1e-7 and abs(info["E"][0, 1] - 1e-4) < 1e-7


def test_quadratic_convergence_untruncated():
    """Theorem 1: ε_{k+1} = O(ε_k²) — regression slope ≥ 1.7."""
    A, _ = W.make_matrix(64, "geometric", 1e2, 9)  # gap_min ≈ 7.6e-4: ε ~ 1e-6 is inside Theorem 1's region
    lam0, X0 = W.initial_eig(A)
    Xh, Xl, lh, ll, _ = orf.reference_eigvecs(A, X0, lam0)
    rng = np.random.default_rng(0)
    X = X0 + rng.standard_normal(X0.shape) * 1e-7
    lam = lam0.copy()
    errs = [orf.forward_error(Xh, Xl, X)]
    for _ in range(2):
        X, lam, _ = orf.sweep(A, X, lam, 1e-15, truncate=False)
        errs.append(orf.forward_error(Xh, Xl, X))
    slope = np.log(errs[1]) / np.log(errs[0])
    assert slope >= 1.7 or errs[1] < 1e-13, errs


@pytest.mark.parametrize("delta", [1e-6, 1e-10, 1e-13])
def test_forward_error_targets_delta(delta):
    """‖X − X̂‖ = O(δ): within [δ/10³, 2δ] after the driver stops (c1 recipe)."""
    A, lam0, X0, _ = W.make_config("c1")
    Xh, Xl, lh, ll, _ = orf.reference_eigvecs(A, X0, lam0)
    X, lam, hist = orf.refine_to_tol(A, X0, lam0, delta)
    fe = orf.forward_error(Xh, Xl, X)
    assert delta / 1e3 <= fe <= 2 * delta or (fe <= 2 * delta and delta < 1e-12), (fe, hist)
    assert len(hist) <= 3


def test_sweep_columns_matches_sweep():
    A, lam0, X0, _ = W.make_config("c1")
    Xn, lam, info = orf.sweep(A, X0, lam0, 1e-12)
    J = np.array([0, 7, 50, 99])
    XJ, lamJ, beta = orf.sweep_columns(A, X0, lam0, 1e-12, J)
    assert beta == info["beta"]
    assert np.max(np.abs(XJ - Xn[:, J])) < 1e-15
    assert np.max(np.abs(lamJ - lam[J])) < 1e-15


def test_form_R_and_W_vanish_on_exact_eigensystem():
    """Pin of the oracle's R = I − X̂ᵀX̂ and W (form_R): on the Householder family A = H diag(λ) H with
    X̂ = H EXACTLY, untruncated, both are exactly zero and every λ̂ is exact."""
    A, lam, X, H, lam_cols = W.householder_exact(6, lam_bits=12, seed=5)
    Xn, lamn, info = orf.sweep(A, X, lam, 1e-12, truncate=False, form_R=True)
    assert np.all(info["R"] == 0.0) and info["normR_fro"] == 0.0
    assert info["normW_fro"] == 0.0
    assert np.array_equal(lamn, lam) and np.array_equal(Xn, X)


def test_driver_stop_rules(monkeypatch):
    """Reading R12 (the paper gives no iteration rule): the oracle driver's decisions on scripted sweeps and
    certificates — a sweep is certified when its estimate × CERT_SAFETY ≤ δ; a non-contracting estimate
    (> CONTRACT × the previous one, or with a next quadratic part est³/est_prev² ≤ δ/8) above δ escalates θ by
    the power of 4 that brings the floor below δ/2,
    at most max_escalations times, then "stagnation"; sweeps with unresolved groups are neither certified nor
    compared."""
    n = 8
    script = []

    last = [1.0]

    def fake_sweep(A, X, lam, delta, theta, **kw):
        clusters, est = script.pop(0)
        # ν = ‖X_k − X_{k−1}‖_F is the size of the error the sweep removed: the previous sweep's error
        info = dict(beta=20, alpha=40, normE_fro=0.0, clusters=clusters, net_update=last[0], E=est)
        last[0] = est if est > 0 else 1.0
        return X, lam, info

    monkeypatch.setattr(orf, "sweep", fake_sweep)
    monkeypatch.setattr(orf, "certificate", lambda E, lam, delta=None: dict(est=E))
    A, X0, lam0 = np.eye(n), np.eye(n), np.arange(n, dtype=float)
    d = 1e-12
    script[:] = [([], 1e-6), ([], 0.8 * d), ([], 0.1 * d)]
    _, _, h = orf.refine_to_tol(A, X0, lam0, d)
    assert len(h) == 2 and h[-1]["stop"] == "converged" and h[-1]["cert"] == 0.8 * d
    # still contracting with a quadratic part above δ/8 (1e-6³/1e-3² = 1e-12): no escalation
    script[:] = [([], 1e-3), ([], 1e-6), ([], 0.5 * d)]
    _, _, h = orf.refine_to_tol(A, X0, lam0, d)
    assert [r["theta"] for r in h] == [4.0, 4.0, 4.0] and h[-1]["stop"] == "converged"
    # 0.9δ · 1.15 > δ after a fast contraction (0.9δ³/1e-6² ≪ δ/8): the rest is the floor, θ × 4
    script[:] = [([], 1e-6), ([], 0.9 * d), ([], 0.5 * d)]
    _, _, h = orf.refine_to_tol(A, X0, lam0, d)
    assert [r["theta"] for r in h] == [4.0, 4.0, 16.0] and h[-1]["stop"] == "converged"
    # floor at 2.5δ: θ × 4^⌈log4(2·2.5·1.15)⌉ = ×16, then certified
    script[:] = [([], 1e-3), ([], 1e-6), ([], 2.5 * d), ([], 0.2 * d)]
    _, _, h = orf.refine_to_tol(A, X0, lam0, d)
    assert [r["theta"] for r in h] == [4.0, 4.0, 4.0, 64.0] and h[-1]["stop"] == "converged"
    # a floor that does not move: one escalation allowed, then stagnation
    script[:] = [([], 1e-3), ([], 1e-6), ([], 2.9 * d), ([], 2.8 * d), ([], 2.7 * d)]
    _, _, h = orf.refine_to_tol(A, X0, lam0, d, max_escalations=1)
    assert [r["theta"] for r in h] == [4.0, 4.0, 4.0, 64.0, 64.0] and h[-1]["stop"] == "stagnation"
    # the first certified sweep has no previous estimate: ν (the error it removed, here 1e-6) stands in — 5δ with a
    # quadratic part (5δ)³/1e-6² ≪ δ/8 is the floor, θ × 4^⌈log4(2·5·1.15)⌉ = ×16 at once, no sweep wasted on it
    last[0] = 1e-6
    script[:] = [([], 5 * d), ([], 0.3 * d)]
    _, _, h = orf.refine_to_tol(A, X0, lam0, d)
    assert [r["theta"] for r in h] == [4.0, 64.0] and h[-1]["stop"] == "converged"
    # ... but not when the sweep removed so little that its own quadratic part may still matter: (5δ)³/(20δ)² > δ/8
    last[0] = 20 * d
    script[:] = [([], 5 * d), ([], 0.3 * d)]
    _, _, h = orf.refine_to_tol(A, X0, lam0, d)
    assert [r["theta"] for r in h] == [4.0, 4.0] and h[-1]["stop"] == "converged"
    # ... nor when θ cannot grow (untruncated mode, or no escalation left): the next sweep decides
    last[0] = 1e-6
    script[:] = [([], 5 * d), ([], 0.3 * d)]
    _, _, h = orf.refine_to_tol(A, X0, lam0, d, truncate=False)
    assert [r["theta"] for r in h] == [4.0, 4.0] and h[-1]["stop"] == "converged"
    last[0] = 1e-6
    script[:] = [([], 5 * d), ([], 0.3 * d)]
    _, _, h = orf.refine_to_tol(A, X0, lam0, d, max_escalations=0)
    assert [r["theta"] for r in h] == [4.0, 4.0] and h[-1]["stop"] == "converged"
    # cluster sweeps are neither certified nor compared: a tiny estimate during them does not stop
    script[:] = [([[0, 1]], 0.0), ([[0, 1]], 0.0), ([], 1e-3), ([], 1e-7), ([], 0.1 * d)]
    _, _, h = orf.refine_to_tol(A, X0, lam0, d)
    assert len(h) == 5 and h[-1]["stop"] == "converged" and "cert" not in h[0]


def test_certificate_equals_forward_error_exact_family():
    """The certificate against an EXACT forward error: A = H diag(λ) H with X = H exactly, the start
    X + N(0, 1e-7²) — one sweep (untruncated and truncated at δ = 1e-12): the estimate's second-order term
    ‖Q∘H‖₂ equals ‖X̂_new − X‖₂ to 2 % (a wrong sign in c_kj = (λ̂_k − λ̂_j)ẽ_kj, a transposed Q or a dropped
    1/(λ̂_j − λ̂_i) changes it by orders of magnitude)."""
    A, lam, X, H, lam_cols = W.householder_exact(6, lam_bits=12, seed=3)
    X0 = X + 1e-7 * np.random.default_rng(1).standard_normal(X.shape)
    for trunc in (False, True):
        Xn, ln, info = orf.sweep(A, X0, lam, 1e-12, truncate=trunc)
        fe = float(np.linalg.norm(Xn - X, 2))
        c = orf.certificate(info["E"], ln)
        assert abs(c["est_q"] - fe) <= 0.02 * fe, (trunc, c, fe)
        assert c["est"] >= c["est_q"] and c["frob"] >= c["est_q"]


def test_certificate_tracks_forward_error_c4p_recipe():
    """The c4' recipe at n = 256 (cnd 1e10, FP64 start, δ = 1e-12): after each of 3 truncated sweeps the
    certificate agrees with the forward error against the reference eigenvectors to 5 % + 2u, and the
    driver's certified result is within δ."""
    A, lam0, X0, cfg = W.make_config("c4p", n=256)
    Xh, Xl, lh, ll, _ = orf.reference_eigvecs(A, X0, lam0)
    X, lam = X0, lam0
    for _ in range(3):
        X, lam, info = orf.sweep(A, X, lam, cfg["delta"])
        fe = orf.forward_error(Xh, Xl, X, lh, lam)
        c = orf.certificate(info["E"], lam)
        assert abs(c["est"] - fe) <= 0.05 * fe + 2 * 2.0 ** -53 + c["quad"], (c, fe)
    X, lam, hist = orf.refine_to_tol(A, X0, lam0, cfg["delta"])
    assert hist[-1]["stop"] == "converged"
    assert orf.forward_error(Xh, Xl, X, lh, lam) <= cfg["delta"]


@pytest.mark.parametrize("m", [3, 6])
def test_second_order_defect_vs_exact_correction(m):
    """R12's defect formula against the EXACT correction: A = H diag(λ) H with X = H exactly, the
    start X̂ = X(I + F₀) with a generic (non-skew) F₀ of size 1e-4, one untruncated sweep (X̂^(1) = X̂). The
    exact E solves X = X̂(I + E), so E − Ẽ is known to ~1e-16; second_order_defect(Ẽ) must equal −(E − Ẽ) up to
    third-order terms (≤ 1 % in Frobenius norm; measured 5e-4). At n = 8 (gaps ~ spread, so the unamplified
    terms matter) dropping the Ẽ² term, the diagonal ½‖ẽ_j‖² or transposing Q miss by ≥ 10 %."""
    A, lam, X, H, lam_cols = W.householder_exact(m, lam_bits=12, seed=5)
    n = A.shape[0]
    F0 = 1e-4 * np.random.default_rng(2).standard_normal((n, n))
    X0 = X @ (np.eye(n) + F0)
    Xn, ln, info = orf.sweep(A, X0, lam, 1e-12, truncate=False)
    assert not info["clusters"]
    Et = info["E"]
    E = np.linalg.solve(X0, X) - np.eye(n)
    true = E - Et
    D = orf.second_order_defect(Et, ln)
    rel = np.linalg.norm(D + true) / np.linalg.norm(true)
    assert rel <= 0.01, rel
    if m == 3:
        C = (ln[:, None] - ln[None, :]) * Et
        dl = ln[None, :] - ln[:, None]
        off = ~np.eye(n, dtype=bool)
        Qh = np.where(off, (Et.T @ C) / np.where(off, dl, 1.0), 0.0)
        for bad in (Qh, Qh - Et @ Et, Qh.T - Et @ Et - np.diag(0.5 * np.sum(Et * Et, axis=0))):
            assert np.linalg.norm(bad + true) / np.linalg.norm(true) >= 0.1
    # and its 2-norm is the forward error of the returned X̂ (X̂_new − X = X̂(Ẽ − E)) up to the same terms
    fe = float(np.linalg.norm(Xn - X, 2))
    c = orf.certificate(Et, ln)
    assert abs(c["est_q"] - fe) <= 0.03 * fe + 4 * 2.0 ** -53, (c, fe)


def test_accmul_fixed_k_vs_rationals():
    """§8(f) rank 1: the prior work's ½k(k+1)-product scheme pinned against exact
    rationals: (a) ½k(k+1) pairs; (b) hi + lo is the correctly rounded exact sum of the kept digit-pair
    products (Fractions from the digit values); (c) the error against the exact AB falls by ≥ 2^7 per extra
    slice and is within the bound Σ_i |a_i| |b_j| (2^{1−S_k}) + the dropped-pair tail."""
    from fractions import Fraction
    from oracle import split as osp
    rng = np.random.default_rng(4)
    A = rng.standard_normal((5, 7)) * np.exp(rng.uniform(-20, 20, (5, 1)))
    B = rng.standard_normal((7, 4))
    exact = [[sum(Fraction(A[i, l]) * Fraction(B[l, j]) for l in range(7)) for j in range(4)] for i in range(5)]
    errs = []
    for k in (2, 3, 4, 5):
        hi, lo, npairs = opr.accmul_fixed_k(A, B, k)
        assert npairs == k * (k + 1) // 2
        DA, eA = osp.split_digits_cols(A.T, k)
        DB, eB = osp.split_digits_cols(B, k)
        for i in range(5):
            for j in range(4):
                s = Fraction(0)
                for a in range(1, k + 1):
                    for b in range(1, k + 2 - a):
                        da = sum(int(DA[a - 1, l, i]) * int(DB[b - 1, l, j]) for l in range(7))
                        s += Fraction(da) * Fraction(2) ** int(eA[i] + eB[j] + 8 * (k - a) + 8 * (k - b))
                h = float(s)
                assert hi[i, j] == h and lo[i, j] == float(s - Fraction(h))
        e = max(abs(Fraction(hi[i, j]) + Fraction(lo[i, j]) - exact[i][j]) / (sum(abs(Fraction(A[i, l]) * Fraction(B[l, j]))
                                                                                  for l in range(7)))
                for i in range(5) for j in range(4))
        errs.append(float(e))
        assert e <= 2.0 ** (-(8 * (k - 1) + 6) + 2) * (k + 2)  # both splits' rounding + the dropped diagonal
    for a, b in zip(errs, errs[1:]):
        assert b <= a / 2 ** 7


@pytest.mark.parametrize("kind,start,delta", [("geometric", "fp64", 1e-13), ("clustered", "fp64", 1e-12),
                                              ("clustered", "fp32", 1e-12)])
def test_driver_reaches_target_on_exactly_known_eigenvectors(kind, start, delta):
    """W.hadamard_exact (A = Q B Q exactly representable, B integer 2 x 2 blocks: eigenpairs in closed form, pinned
    in integers / rationals by tests/test_abi_workloads.py): the oracle driver from an LAPACK start returns
    "converged" with ‖X − X̂‖₂ ≤ δ against the closed-form X (no computed reference involved; the closed form is
    good to ≈ 2u), its certificate within a factor 2 of that forward error + 4u, and λ̂ within 4u‖A‖."""
    A, lam, X = W.hadamard_exact(7, kind, seed=21)  # n = 128; "clustered": 2 clusters of 8, relative gaps ≥ 0.24·2^-37
    lam0, X0 = W.initial_eig(A, start)
    Xr, lr, hist = orf.refine_to_tol(A, X0, lam0, delta)
    assert hist[-1].get("stop") == "converged", hist
    p = np.argsort(lr, kind="stable")
    Xr, lr = Xr[:, p], lr[p]
    sg = np.sign(np.sum(Xr * X, axis=0))
    fe = float(np.linalg.norm(Xr * sg[None, :] - X, 2))
    assert fe <= delta, (fe, hist)
    # the certificate: not below the exact forward error (up to the closed form's own ≈ 2u), within 3x + 8u of it
    assert hist[-1]["cert"] >= fe / 1.15 - 2.0 ** -51 and hist[-1]["cert"] <= 3 * fe + 2.0 ** -50, (fe, hist[-1])
    assert np.max(np.abs(lr - lam)) <= 4 * 2.0 ** -53 * np.max(np.abs(lam))


def test_driver_soundness_scan_exact_family():
    """"converged" ⇒ ‖X − X̂‖₂ ≤ δ (+ the closed form's own ≈ 4u) over a grid of the exactly-known family (n = 64:
    geometric / clustered spectra, FP64 / FP32 starts, δ from 1e-8 to 1e-15, several seeds); every case must also
    converge within the driver's sweep limit."""
    for kind in ("geometric", "clustered"):
        for start in ("fp64", "fp32"):
            for delta in (1e-8, 1e-12, 1e-15):
                for seed in (31, 32):
                    A, lam, X = W.hadamard_exact(6, kind, seed=seed)
                    lam0, X0 = W.initial_eig(A, start)
                    Xr, lr, hist = orf.refine_to_tol(A, X0, lam0, delta)
                    assert hist[-1].get("stop") == "converged", (kind, start, delta, seed, hist)
                    p = np.argsort(lr, kind="stable")
                    sg = np.sign(np.sum(Xr[:, p] * X, axis=0))
                    fe = float(np.linalg.norm(Xr[:, p] * sg[None, :] - X, 2))
                    assert fe <= delta + 4 * 2.0 ** -53, (kind, start, delta, seed, fe, hist[-1])
