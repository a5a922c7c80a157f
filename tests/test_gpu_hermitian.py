"""GPU parity of the Hermitian extension (ozr_refine_step_herm, reading R18) against the
Hermitian oracle (oracle/hermitian.py, pinned in tests/test_oracle_hermitian.py):
 - one sweep with tightened budgets (θ_V = θ_W = θ_U = 1e-15/δ): X̂ (both parts) and λ̂ within 1e-13 of the
   oracle's exact-product sweep, β identical — at sizes spanning several 256-column tiles and a ragged tail;
 - one sweep with the default budgets: within δ/4 of the oracle (the budgets' design accuracy, R8);
 - the exactly known complex Householder family (n = 256): from a 1e-6 start, three GPU sweeps reach the exact
   eigenvectors within δ = 1e-14 and the exact eigenvalues;
 - an FP32 (complex64 zheevd) start of a random Hermitian recipe converges to the oracle's result;
 - equal estimates are OZR_ERR_DEGENERATE (the paper's Algorithm 1 assumes distinct eigenvalues)."""
import numpy as np
import pytest

import workloads as W
from gpu_util import to_dev, to_np, vec_dev
from oracle import hermitian as oh

pytestmark = pytest.mark.gpu


def _gpu(ctx, Ar, Ai, Xr, Xi, lam, delta, **kw):
    import paper_2602_19090_b200 as ozr
    Xrd, Xid, ld = to_dev(Xr), to_dev(Xi), vec_dev(lam)
    rep = ozr.ozr_refine_step_herm(ctx, to_dev(Ar), to_dev(Ai), Xrd, Xid, ld, ozr.default_params(delta=delta, **kw))
    return to_np(Xrd), to_np(Xid), to_np(ld), rep


CASES = [(100, 1e8, "fp64", 1e-15), (300, 1e10, "fp64", 1e-12), (517, 1e6, "fp32", 1e-12)]


@pytest.mark.parametrize("n,cnd,start,delta", CASES)
def test_sweep_matches_oracle_tight_budgets(ctx, n, cnd, start, delta):
    Ar, Ai, _ = W.make_hermitian(n, "geometric", cnd, seed=n)
    lam0, Xr, Xi = W.initial_eig_herm(Ar, Ai, start)
    th = min(1.0 / 16, 1e-15 / delta)
    Xg_r, Xg_i, lg, rep = _gpu(ctx, Ar, Ai, Xr, Xi, lam0, delta, theta_V=th, theta_W=th, theta_U=th)
    Xo_r, Xo_i, lo, info = oh.sweep_herm(Ar, Ai, Xr, Xi, lam0, delta)
    assert rep["beta"] == info["beta"]
    assert np.max(np.abs(Xg_r - Xo_r)) <= 1e-13 and np.max(np.abs(Xg_i - Xo_i)) <= 1e-13
    assert np.max(np.abs(lg - lo)) <= 1e-13 * np.max(np.abs(lo))
    assert rep["pairs_V"] > 0 and rep["pairs_W"] > 0 and rep["pairs_U"] > 0


@pytest.mark.parametrize("n,cnd,start,delta", CASES)
def test_sweep_default_budgets_within_delta(ctx, n, cnd, start, delta):
    Ar, Ai, _ = W.make_hermitian(n, "geometric", cnd, seed=n)
    lam0, Xr, Xi = W.initial_eig_herm(Ar, Ai, start)
    Xg_r, Xg_i, lg, rep = _gpu(ctx, Ar, Ai, Xr, Xi, lam0, delta)
    Xo_r, Xo_i, lo, info = oh.sweep_herm(Ar, Ai, Xr, Xi, lam0, delta)
    assert np.max(np.abs(Xg_r - Xo_r)) <= delta / 4 and np.max(np.abs(Xg_i - Xo_i)) <= delta / 4


def test_householder_family_exact_eigenvectors(ctx):
    """From a 1e-6 start the truncated iteration reaches its floor after two sweeps. With the default θ = 4 that
    floor is O(δ) (the oracle's own forward error, 8.4e-14 = 8.4δ here — the paper promises O(δ), cf.
    the real c3 spectrum in DESIGN.md R11): the GPU's error equals the oracle's; with θ = 64 (β two bits lower)
    both stay ≤ δ."""
    Ar, Ai, lam, Xr, Xi = W.householder_exact_herm(8)  # n = 256
    A = Ar + 1j * Ai
    assert np.max(np.abs(A @ (Xr + 1j * Xi) - (Xr + 1j * Xi) * lam[None, :])) == 0.0
    rng = np.random.default_rng(2)
    X0r = Xr + 1e-6 * rng.standard_normal(Xr.shape)
    X0i = Xi + 1e-6 * rng.standard_normal(Xi.shape)
    lam0 = lam + 1e-9 * rng.standard_normal(lam.shape)
    delta = 1e-14
    for theta in (4.0, 64.0):
        Yr, Yi, ly = X0r, X0i, lam0
        Or, Oi, lo = X0r, X0i, lam0
        for _ in range(3):
            Yr, Yi, ly, rep = _gpu(ctx, Ar, Ai, Yr, Yi, ly, delta, theta=theta)
            Or, Oi, lo, _ = oh.sweep_herm(Ar, Ai, Or, Oi, lo, delta, theta=theta)
        fe = oh.forward_error_herm(Xr, Xi, Yr, Yi, lam, ly)
        fo = oh.forward_error_herm(Xr, Xi, Or, Oi, lam, lo)
        assert abs(fe - fo) <= 0.1 * fo + delta / 10, (theta, fe, fo)
        if theta == 64.0:
            assert fe <= delta, fe
        assert np.max(np.abs(np.sort(ly) - lam)) <= 1e-15


def test_fp32_start_converges_like_the_oracle(ctx):
    n, delta = 192, 1e-13
    Ar, Ai, _ = W.make_hermitian(n, "geometric", 1e5, seed=77)
    lam0, Xr, Xi = W.initial_eig_herm(Ar, Ai, "fp32")
    # reference: the oracle iterated far below δ (its own accuracy pinned against __float128 Jacobi of the
    # real embedding in tests/test_oracle_hermitian.py)
    Rr, Ri, lr, _ = oh.refine_herm(Ar, Ai, Xr, Xi, lam0, 1e-18, sweeps=5)
    Yr, Yi, ly = Xr, Xi, lam0
    for _ in range(4):
        Yr, Yi, ly, rep = _gpu(ctx, Ar, Ai, Yr, Yi, ly, delta)
    assert oh.forward_error_herm(Rr, Ri, Yr, Yi, lr, ly) <= delta


def test_equal_estimates_are_degenerate(ctx):
    import paper_2602_19090_b200 as ozr
    Ar, Ai, _ = W.make_hermitian(64, "geometric", 1e4, seed=5)
    lam0, Xr, Xi = W.initial_eig_herm(Ar, Ai, "fp64")
    lam0[3] = lam0[4]
    with pytest.raises(ozr.OzrError) as e:
        _gpu(ctx, Ar, Ai, Xr, Xi, lam0, 1e-12)
    assert e.value.status == 4
