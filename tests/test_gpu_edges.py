"""Edge cases of the refinement boundary (include/ozr.h): the smallest and ragged sizes (n = 2, 3, 5,
257 — ragged against the 128/256 tiles, the 4-row digit packing and the 16-byte TMA alignment, which
switch the recombination to its register path), non-finite input, a zero column, a δ at the limit,
and the argument checks of the partitioned entry point. Results against the oracle where defined."""
import numpy as np
import pytest

from gpu_util import parity_sweep, to_dev, to_np, vec_dev
import workloads as W

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n", [2, 3, 5, 37, 257])
def test_small_and_ragged_sizes_match_oracle(ctx, n):
    rng = np.random.default_rng(n)
    lam_true = np.sort(rng.uniform(0.1, 1.0, n))
    Q, R = np.linalg.qr(rng.standard_normal((n, n)))
    Q = Q * np.sign(np.diag(R))[None, :]
    A = (Q * lam_true[None, :]) @ Q.T
    A = (A + A.T) / 2
    lam0, X0 = W.initial_eig(A, "fp64")
    Xg, lg, rep, Xo, lo, info, groups = parity_sweep(ctx, A, X0, lam0, 1e-12)
    assert rep["beta"] == info["beta"]
    assert np.max(np.abs(Xg - Xo)) <= 1e-13
    assert np.max(np.abs(lg - lo)) <= 1e-13


def test_nonfinite_and_degenerate_inputs(ctx):
    import paper_2602_19090_b200 as ozr
    A, lam0, X0, cfg = W.make_config("c1")
    Xbad = X0.copy()
    Xbad[3, 7] = np.nan
    with pytest.raises(ozr.OzrError) as e:
        ozr.ozr_refine_step(ctx, to_dev(A), to_dev(Xbad), vec_dev(lam0), ozr.default_params(delta=1e-12))
    assert e.value.status == 2                      # OZR_ERR_NONFINITE
    Abad = A.copy()
    Abad[5, 5] = np.inf
    with pytest.raises(ozr.OzrError) as e:
        ozr.ozr_refine_step(ctx, to_dev(Abad), to_dev(X0), vec_dev(lam0), ozr.default_params(delta=1e-12))
    assert e.value.status == 2
    Xz = X0.copy()
    Xz[:, 4] = 0.0                                  # a zero column: r_j = 1 (Alg. 1 line 2 divides by 1 − r_j)
    with pytest.raises(ozr.OzrError) as e:
        ozr.ozr_refine_step(ctx, to_dev(A), to_dev(Xz), vec_dev(lam0), ozr.default_params(delta=1e-12))
    assert e.value.status == 4                      # OZR_ERR_DEGENERATE
    lam_bad = lam0.copy()
    lam_bad[0] = np.inf
    with pytest.raises(ozr.OzrError) as e:
        ozr.ozr_refine_step(ctx, to_dev(A), to_dev(X0), vec_dev(lam_bad), ozr.default_params(delta=1e-12))
    assert e.value.status == 2


def test_delta_limits(ctx):
    """δ just above u runs (the budgets saturate at the 15-digit A split and β at its lower clamp); δ ≤ u
    is OZR_ERR_RANGE (tested in test_gpu_refine); a δ so loose that β hits its upper clamp still
    returns a sweep matching the oracle."""
    import paper_2602_19090_b200 as ozr
    A, lam0, X0, cfg = W.make_config("c1")
    rep = ozr.ozr_refine_step(ctx, to_dev(A), to_dev(X0), vec_dev(lam0), ozr.default_params(delta=2.0 ** -52))
    assert rep["beta"] >= 2 and rep["kA"] <= 15
    # exact-product parity needs product budgets tightened below the bar (as in test_gpu_refine) ...
    th = 1e-15 / 1e-1
    Xg, lg, rep, Xo, lo, info, groups = parity_sweep(ctx, A, X0, lam0, 1e-1, theta_V=th, theta_W=th, theta_U=th)
    assert rep["beta"] == info["beta"] and rep["beta_raw"] == info["beta_raw"]
    assert np.max(np.abs(Xg - Xo)) <= 1e-13
    # ... while the default budgets stay within δ/4 of the exact-product sweep (R8)
    Xg, lg, rep, Xo, lo, info, groups = parity_sweep(ctx, A, X0, lam0, 1e-1)
    assert np.max(np.abs(Xg - Xo)) <= 1e-1 / 4


def test_partitioned_argument_checks(ctx):
    import paper_2602_19090_b200 as ozr
    comms = ozr.ozr_comm_create_host_group(3)
    A, lam0, X0, cfg = W.make_config("c1")          # n = 100 is not a multiple of 3 ranks
    with pytest.raises(ozr.OzrError) as e:
        ozr.ozr_refine_step_dist(ctx, comms[0], to_dev(A), to_dev(X0), vec_dev(lam0), ozr.default_params(delta=1e-12))
    assert e.value.status == 1                      # OZR_ERR_ARG
    for c in comms:
        c.close()
