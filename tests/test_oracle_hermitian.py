"""Pins of the Hermitian oracle (oracle/hermitian.py, reading R18) against things other
than itself:
 - real input: A real symmetric, X̂ real ⇒ the Hermitian sweep is the real oracle sweep (itself pinned), bit for
   bit, and the imaginary parts stay exactly zero;
 - the exactly known complex Householder family A = H diag(λ) H (H = I − (2/n)vvᴴ, v ∈ {±1, ±i}ⁿ): the start
   H + complex noise converges to the exact eigenvectors within δ and the Rayleigh quotients to the exact λ;
 - a random Hermitian matrix against __float128 Jacobi of its real symmetric embedding [[Ar, −Ai], [Ai, Ar]]
   (eigenvalues in pairs; [Re x; Im x] must lie in the pair's eigenspace) — an independent algorithm;
 - the complex product helper against the definition written with numpy complex arithmetic on exactly
   representable integers;
 - quadratic convergence (Theorem 1) in the complex case."""
from fractions import Fraction as F

import numpy as np

import workloads as W
from oracle import _clib
from oracle import hermitian as oh
from oracle import refine as orf


def test_cmul_dd_exact_integers():
    rng = np.random.default_rng(5)
    Pr, Pi = rng.integers(-2 ** 20, 2 ** 20, (7, 9)).astype(float), rng.integers(-2 ** 20, 2 ** 20, (7, 9)).astype(float)
    Qr, Qi = rng.integers(-2 ** 20, 2 ** 20, (9, 5)).astype(float), rng.integers(-2 ** 20, 2 ** 20, (9, 5)).astype(float)
    Rh, Rl, Ih, Il = oh.cmul_dd(Pr, Pi, Qr, Qi)
    P = Pr.astype(np.int64) + 1j * 0
    ex_r = Pr.astype(object) @ Qr.astype(object) - Pi.astype(object) @ Qi.astype(object)
    ex_i = Pr.astype(object) @ Qi.astype(object) + Pi.astype(object) @ Qr.astype(object)
    assert P.shape == (7, 9)
    for a in range(7):
        for b in range(5):
            assert F(Rh[a, b]) + F(Rl[a, b]) == ex_r[a, b]
            assert F(Ih[a, b]) + F(Il[a, b]) == ex_i[a, b]


def test_real_input_is_the_real_sweep():
    A, lam0, X0, cfg = W.make_config("c1")
    Z = np.zeros_like(A)
    Xr, Xi, lam, info = oh.sweep_herm(A, Z, X0, np.zeros_like(X0), lam0, 1e-15)
    Xo, lo, io = orf.sweep(A, X0, lam0, 1e-15, cluster_mode=0)
    assert info["beta"] == io["beta"]
    assert np.array_equal(Xr, Xo) and np.array_equal(lam, lo)
    assert not np.any(Xi)


def _exact_herm(Ar, Ai, Xr, Xi, lam):
    """A = X diag(λ) Xᴴ holds exactly (integers after scaling by 2^s)."""
    n = Ar.shape[0]
    s = 2 ** 40
    to = lambda M: np.array([[int(F(x) * s) for x in row] for row in M], dtype=object)  # noqa: E731
    for M in (Ar, Ai, Xr, Xi):
        assert all(float(F(int(F(x) * s), s)) == x for x in M.ravel())
    Xr_, Xi_ = to(Xr), to(Xi)
    L = np.array([int(F(x) * s) for x in lam], dtype=object)
    # (X diag λ Xᴴ)_ij = Σ_k x_ik λ_k conj(x_jk), scaled by s³
    Br = (Xr_ * L[None, :]) @ Xr_.T + (Xi_ * L[None, :]) @ Xi_.T
    Bi = (Xi_ * L[None, :]) @ Xr_.T - (Xr_ * L[None, :]) @ Xi_.T
    return np.all(Br == to(Ar) * s * s) and np.all(Bi == to(Ai) * s * s)


def test_householder_family_converges_to_exact_eigenvectors():
    Ar, Ai, lam, Xr, Xi = W.householder_exact_herm(5)
    assert _exact_herm(Ar, Ai, Xr, Xi, lam)
    rng = np.random.default_rng(9)
    X0r = Xr + 1e-9 * rng.standard_normal(Xr.shape)
    X0i = Xi + 1e-9 * rng.standard_normal(Xi.shape)
    delta = 1e-15
    l0 = np.sum(X0r * ((Ar @ X0r) - Ai @ X0i) + X0i * ((Ar @ X0i) + Ai @ X0r), axis=0) / np.sum(X0r ** 2 + X0i ** 2,
                                                                                             axis=0)
    Yr, Yi, ly, hist = oh.refine_herm(Ar, Ai, X0r, X0i, l0, delta, sweeps=3)
    fe = oh.forward_error_herm(Xr, Xi, Yr, Yi, lam, ly)
    assert fe <= delta, (fe, [h["net_update"] for h in hist])
    assert np.max(np.abs(np.sort(ly) - lam)) <= 1e-16
    # the first sweep contracts the 1e-9 start quadratically (Theorem 1): ~ (1e-9·√n)²·‖A‖/gap
    fe1 = oh.forward_error_herm(Xr, Xi, *oh.refine_herm(Ar, Ai, X0r, X0i, l0, delta, sweeps=1)[:2], lam,
                                oh.refine_herm(Ar, Ai, X0r, X0i, l0, delta, sweeps=1)[2])
    assert fe1 < 1e-12


def test_random_hermitian_vs_quad_jacobi_of_the_embedding():
    n = 10
    Ar, Ai, _ = W.make_hermitian(n, "geometric", 1e6, seed=31)
    lam0, X0r, X0i = W.initial_eig_herm(Ar, Ai, "fp32")
    delta = 1e-15
    Xr, Xi, lam, hist = oh.refine_herm(Ar, Ai, X0r, X0i, lam0, delta, sweeps=4)
    M = np.block([[Ar, -Ai], [Ai, Ar]])
    wh, wl, Vh, Vl, sw = _clib.jacobi_q(M)
    assert sw > 0
    p = np.argsort(wh)
    wh, Vh = wh[p], Vh[:, p]
    assert np.max(np.abs(wh[0::2] - wh[1::2])) <= 1e-15          # the embedding doubles every eigenvalue
    q = np.argsort(lam)
    for k, j in enumerate(q):
        P = Vh[:, 2 * k:2 * k + 2]                                   # the pair's eigenspace (orthonormal)
        y = np.concatenate([Xr[:, j], Xi[:, j]])
        assert np.linalg.norm(y - P @ (P.T @ y)) <= delta, (k, np.linalg.norm(y - P @ (P.T @ y)))
        assert abs(lam[j] - wh[2 * k]) <= 1e-15
    # the unit-norm property of the refined columns
    assert np.max(np.abs(np.sum(Xr ** 2 + Xi ** 2, axis=0) - 1.0)) <= 1e-15


def test_quadratic_convergence_complex():
    """Theorem 1: ‖E_{k+1}‖ = O(‖E_k‖²) — with δ far below the errors the truncation keeps all
    bits that matter, and successive net updates square until fp64 rounding."""
    n = 24
    Ar, Ai, _ = W.make_hermitian(n, "geometric", 1e4, seed=33)
    lam0, X0r, X0i = W.initial_eig_herm(Ar, Ai, "fp32")
    _, _, _, hist = oh.refine_herm(Ar, Ai, X0r, X0i, lam0, 1e-30, sweeps=3)
    nu = [h["net_update"] for h in hist]
    assert nu[1] <= 50 * nu[0] ** 2 * np.sqrt(n) and nu[1] < nu[0] / 1e3, nu
