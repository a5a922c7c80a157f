"""GPU tests of ozr_syev — the hand-written dense symmetric eigensolver of the large-group Rayleigh–Ritz
sub-solve (R13; Householder tridiagonalisation, Cuppen divide and conquer with Gu–Eisenstat
eigenvectors, blocked back-transformation; include/ozr.h).

Pinned against (a) the oracle's __float128 cyclic Jacobi (oracle/ddmm.c) for m ≤ 48: eigenvalues to
1e-14·‖K‖ and eigenvector columns up to sign to u‖K‖/gap; (b) at any size, the properties a backward-stable
eigensolver has: ‖KY − YΘ‖_F ≤ c·u·√m·‖K‖_F, ‖YᵀY − I‖_max ≤ c·u·√m·log m, θ ascending, and the exactly known
spectrum of the Householder family A = H diag(λ) H to c·u·‖K‖. Sizes span one leaf (≤ 32), several
merge levels, the INT8 product path (dimension ≥ 1024), ragged tails, and spectra with heavy deflation (repeated
and graded eigenvalues, a diagonal matrix)."""
import numpy as np
import pytest
import torch

import paper_2602_19090_b200 as ozr
import workloads as W
from oracle import _clib

pytestmark = pytest.mark.gpu

U = 2.0 ** -53


def _run(ctx, K):
    Kd = ozr.colmajor(torch.from_numpy(np.asfortranarray(K)).cuda())
    th, Y = ozr.ozr_syev(ctx, Kd)
    return th.cpu().numpy(), Y.cpu().numpy()


def _check_props(K, th, Y, c=64.0):
    """Backward stability: ‖KY − YΘ‖_F ≤ c·u·√m·‖K‖_F (the usual p(m) = √m growth), orthogonality to c·u·√m·log m."""
    m = K.shape[0]
    nK = np.linalg.norm(K)
    res = np.linalg.norm(K @ Y - Y * th[None, :])
    orth = np.max(np.abs(Y.T @ Y - np.eye(m)))
    assert np.all(np.diff(th) >= 0), "not ascending"
    assert res <= c * U * max(nK, 1e-300) * np.sqrt(m), (res, nK)
    assert orth <= c * U * np.sqrt(m) * (np.log2(m + 1) + 1), orth
    return res, orth


def _random_sym(m, seed, scale=1.0):
    G = np.random.default_rng(seed).standard_normal((m, m)) * scale
    return (G + G.T) * 0.5


@pytest.mark.parametrize("m", [1, 2, 3, 17, 32, 33, 48])
def test_syev_vs_quad_jacobi(ctx, m):
    K = _random_sym(m, 100 + m)
    th, Y = _run(ctx, K)
    wh, wl, Vh, Vl, _ = _clib.jacobi_q(K)
    nK = np.linalg.norm(K, 2)
    assert np.max(np.abs(th - (wh + wl))) <= 1e-14 * nK
    gaps = np.array([np.min(np.abs(np.delete(wh, j) - wh[j])) if m > 1 else np.inf for j in range(m)])
    for j in range(m):
        v = Vh[:, j] + Vl[:, j]
        err = min(np.linalg.norm(Y[:, j] - v), np.linalg.norm(Y[:, j] + v))
        assert err <= 64 * U * nK / gaps[j] + 1e-15, (j, err, gaps[j])
    _check_props(K, th, Y)


@pytest.mark.parametrize("m", [64, 100, 257, 700, 1031, 2100])
def test_syev_random_properties(ctx, m):
    K = _random_sym(m, 7 + m)
    th, Y = _run(ctx, K)
    _check_props(K, th, Y)
    ref = np.linalg.eigvalsh(K)
    assert np.max(np.abs(th - ref)) <= 64 * U * np.linalg.norm(K, 2) * np.sqrt(m)


@pytest.mark.parametrize("m", [128, 1100])
def test_syev_graded_group_spectrum(ctx, m):
    """The shape of BASELINE c4's first large group: eigenvalues graded over 12 decades (1e-14 .. 1e-2) plus a
    dense 1e-8 perturbation (the FP32 start's coupling) — heavy deflation at every merge level."""
    rng = np.random.default_rng(m)
    Q = W.haar(m, rng)
    lam = np.geomspace(1e-14, 1e-2, m)
    K = (Q * lam[None, :]) @ Q.T
    K = (K + K.T) * 0.5 + 1e-8 * _random_sym(m, 3)
    th, Y = _run(ctx, K)
    _check_props(K, th, Y)
    ref = np.linalg.eigvalsh(K)
    assert np.max(np.abs(th - ref)) <= 64 * U * np.linalg.norm(K, 2) * np.sqrt(m)


@pytest.mark.parametrize("mexp", [6, 8])
def test_syev_householder_exact_spectrum(ctx, mexp):
    """A = H diag(λ) H is exact in fp64 with exactly known eigenvalues λ, including a doubled one."""
    A, lam, X, H, lam_cols = W.householder_exact(mexp, lam_bits=12, seed=2)
    th, Y = _run(ctx, A)
    assert np.max(np.abs(th - lam)) <= 32 * U * np.sqrt(A.shape[0])
    _check_props(A, th, Y)


@pytest.mark.parametrize("m", [40, 300])
def test_syev_repeated_and_diagonal(ctx, m):
    """Exactly repeated eigenvalues (every merge deflates by rotation) and a diagonal matrix (ρ = 0)."""
    d = np.repeat(np.arange(m // 4, dtype=np.float64), 4)[:m]
    Q = W.haar(m, np.random.default_rng(5))
    K = (Q * d[None, :]) @ Q.T
    K = (K + K.T) * 0.5
    th, Y = _run(ctx, K)
    _check_props(K, th, Y)
    assert np.max(np.abs(th - np.sort(d))) <= 64 * U * m
    D = np.diag(np.random.default_rng(6).permutation(m).astype(np.float64))
    th, Y = _run(ctx, D)
    assert np.array_equal(th, np.arange(m, dtype=np.float64))
    _check_props(D, th, Y)


@pytest.mark.parametrize("m,cl", [(3, "1"), (33, "1"), (64, "1"), (100, "1"), (257, "1"), (257, "0"), (640, "1"),
                                  (700, "1"), (700, "0"), (1000, "1")])
def test_stage_tridiagonalisation(ctx, m, cl, monkeypatch):
    """Stage (1) alone: the reflectors H_c = I − τ_c v_c v_cᵀ it returns satisfy Q_Hᵀ K Q_H = tridiag(d, e) with
    Q_H = H_0⋯H_{m−2} (LAPACK dsytrd's lower convention), to c·u·‖K‖. cl = "1": trailing matrices of up to ~640
    columns run in one thread-block cluster (k_trd_cluster; m = 700 and 1000 hand over from the panel kernel,
    m ≤ 640 runs there entirely); "0": the panel kernel throughout (OZR_TRD_CLUSTER=0)."""
    monkeypatch.setenv("OZR_TRD_CLUSTER", cl)
    K = _random_sym(m, 11 + m)
    Kd = ozr.colmajor(torch.from_numpy(np.asfortranarray(K)).cuda())
    d, e, tau, R = (t.cpu().numpy() for t in ozr.ozr_syev_tridiag(ctx, Kd))
    T = K.copy()
    for c in range(m - 1):  # T ← H_c T H_c, in order (O(m²) per reflector)
        v = np.zeros(m)
        v[c + 1] = 1.0
        v[c + 2:] = R[c + 2:, c]
        T -= tau[c] * np.outer(v, v @ T)
        T -= tau[c] * np.outer(T @ v, v)
    Tref = np.diag(d) + np.diag(e[:m - 1], -1) + np.diag(e[:m - 1], 1)
    assert np.max(np.abs(T - Tref)) <= 64 * U * np.linalg.norm(K) * np.sqrt(m), np.max(np.abs(T - Tref))


@pytest.mark.parametrize("m", [300, 640, 739])
def test_syev_cluster_tridiagonalisation_properties(ctx, m, monkeypatch):
    """The whole eigensolver with and without the cluster-resident tail of the tridiagonalisation: both meet the
    backward-stability bounds, and the eigenvalues agree to c·u·‖K‖."""
    K = _random_sym(m, 5 + m)
    out = []
    for cl in ("1", "0"):
        monkeypatch.setenv("OZR_TRD_CLUSTER", cl)
        th, Y = _run(ctx, K)
        _check_props(K, th, Y)
        out.append(th)
    assert np.max(np.abs(out[0] - out[1])) <= 64 * U * np.linalg.norm(K)


@pytest.mark.parametrize("m", [33, 64, 100, 700])
def test_stage_divide_and_conquer(ctx, m):
    """Stage (2) alone on a random tridiagonal: eigenvalues against LAPACK's tridiagonal solver (scipy), residual
    and orthogonality of the Gu–Eisenstat eigenvectors."""
    from scipy.linalg import eigh_tridiagonal
    rng = np.random.default_rng(m)
    d = rng.standard_normal(m)
    e = rng.standard_normal(m)
    e[m - 1] = 0.0
    th, Y = ozr.ozr_syev_tridiag_eig(ctx, torch.from_numpy(d).cuda(), torch.from_numpy(e).cuda())
    th, Y = th.cpu().numpy(), Y.cpu().numpy()
    T = np.diag(d) + np.diag(e[:m - 1], -1) + np.diag(e[:m - 1], 1)
    ref = eigh_tridiagonal(d, e[:m - 1], eigvals_only=True)
    assert np.max(np.abs(th - ref)) <= 64 * U * np.linalg.norm(T, 2) * np.sqrt(m)
    _check_props(T, th, Y)
