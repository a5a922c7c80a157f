"""GPU parity of the refinement sweep (Algorithm 1, one-sided product §3.3, β §4.1)
against the oracle sweep, and the forward error of ozr_refine_to_tol against the oracle's reference
eigenvectors. Bars (BASELINE.json north star): X̂ and D̂ within 1e-13 (D̂ relative to ‖A‖), the
same β as the oracle, forward error at or below the prescribed target."""
import numpy as np
import pytest

from gpu_util import parity_sweep, to_dev, to_np, vec_dev
from oracle import refine as orf
import workloads as W

pytestmark = pytest.mark.gpu


def _gpu_sweep(ctx, A, X, lam, delta, **kw):
    import paper_2602_19090_b200 as ozr
    Xd, ld = to_dev(X), vec_dev(lam)
    rep = ozr.ozr_refine_step(ctx, to_dev(A), Xd, ld, ozr.default_params(delta=delta, **kw))
    return to_np(Xd), to_np(ld), rep


CASES = [("c1", 100, 1e-15, "fp64"), ("c1", 100, 1e-10, "fp64"), ("c1", 100, 1e-6, "fp64"),
         ("c2", 256, 1e-14, "fp64"), ("c2", 1024, 1e-14, "fp64"), ("c3", 512, 1e-12, "fp64")]


def _case(cfg, n, start):
    c = dict(W.CONFIGS[cfg])
    A, _ = W.make_matrix(n, c["kind"], c["cnd"], c["seed"])
    lam0, X0 = W.initial_eig(A, start)
    return A, lam0, X0


@pytest.mark.parametrize("cfg,n,delta,start", CASES)
def test_sweep_matches_oracle(ctx, cfg, n, delta, start):
    """North-star bar: |ΔX̂| ≤ 1e-13 and |ΔD̂| ≤ 1e-13·‖A‖ against the exact-product oracle sweep. The
    product budgets are tightened (θ·δ ≤ 1e-15) so the digit truncations sit below the bar for any δ."""
    A, lam0, X0 = _case(cfg, n, start)
    th = min(1.0 / 16, 1e-15 / delta)
    Xg, lg, rep, Xo, lo, info, groups = parity_sweep(ctx, A, X0, lam0, delta, theta_V=th, theta_W=th, theta_U=th)
    assert rep["beta"] == info["beta"]
    assert rep["n_clusters"] == len(groups)
    # group columns come out of an fp64 (GPU) vs __float128 (oracle) eigensolver of the sub-problem K:
    # they agree to ~u·‖K‖/gap_K (info["cluster_cond"]); every other column to the north-star 1e-13
    cond = info.get("cluster_cond", 0.0) if groups else 0.0
    mmax = max([len(J) for J in groups], default=1)
    tol = 1e-13 + 10 * np.sqrt(mmax) * 2.0 ** -53 * cond
    dX = np.max(np.abs(Xg - Xo))
    dl = np.max(np.abs(lg - lo)) / np.max(np.abs(lam0))
    assert dX <= tol, (dX, tol)
    assert dl <= tol, (dl, tol)


@pytest.mark.parametrize("cfg,n,delta,start", CASES)
def test_sweep_default_budgets_within_delta(ctx, cfg, n, delta, start):
    """With the default budgets (θ = 1/16 of δ'·gap / δ', R8) the sweep stays within δ/4 of
    the exact-product sweep: the digit truncation is a deliberate, bounded part of the method."""
    A, lam0, X0 = _case(cfg, n, start)
    Xg, lg, rep, Xo, lo, info, groups = parity_sweep(ctx, A, X0, lam0, delta)
    assert rep["beta"] == info["beta"]
    assert np.max(np.abs(Xg - Xo)) <= delta / 4


def test_refine_to_tol_c1_forward_error(ctx):
    """BASELINE c1 (n = 100, cnd 1e8, FP64 start): status OK ⇒ ‖X − X̂‖₂ ≤ δ against the reference, one or two
    sweeps ("one or two iterations")."""
    import paper_2602_19090_b200 as ozr
    A, lam0, X0, cfg = W.make_config("c1")
    Xh, Xl, lh, ll, _ = orf.reference_eigvecs(A, X0, lam0)
    for delta in (1e-8, 1e-12, 1e-15):
        Xd, ld = to_dev(X0), vec_dev(lam0)
        st, hist = ozr.ozr_refine_to_tol(ctx, to_dev(A), Xd, ld, ozr.default_params(delta=delta))
        fe = orf.forward_error(Xh, Xl, to_np(Xd))
        assert st == 0, hist
        assert fe <= delta, (delta, fe, hist)
        assert hist[-1]["cert"] * 1.15 <= delta and len(hist) <= 2


def test_refine_step_errors(ctx):
    import paper_2602_19090_b200 as ozr
    A = np.diag([1.0, 2.0, 3.0, 4.0])
    X = np.eye(4)
    with pytest.raises(ozr.OzrError) as e:   # δ ≤ u
        _gpu_sweep(ctx, A, X, np.array([1.0, 2, 3, 4]), 1e-17)
    assert e.value.status == 3
    with pytest.raises(ozr.OzrError) as e:   # equal eigenvalue estimates, cluster branch off
        _gpu_sweep(ctx, A, X, np.array([1.0, 1.0, 3, 4]), 1e-10, cluster_mode=0)
    assert e.value.status == 4 and "λ̂_0 = λ̂_1" in str(e.value)  # the error names the offending pair


@pytest.mark.parametrize("cfg,n,start", [("c2", 512, "fp64"), ("c3", 1024, "fp64")])
def test_form_R_matches_oracle(ctx, cfg, n, start):
    """form_R = 1: R = I − X̂^(1)ᵀX̂^(1) by INT8 slice products (the R/S form's first product)
    against the oracle's double-double product, and the reported ‖R‖_F, ‖W‖_F and OA threshold ω."""
    import paper_2602_19090_b200 as ozr
    A, lam0, X0 = _case(cfg, n, start)
    delta = 1e-12
    th = 1e-16 / delta
    p = ozr.default_params(delta=delta, form_R=1, theta_V=th, theta_W=th, theta_U=th)
    Xd, ld = to_dev(X0), vec_dev(lam0)
    rep = ozr.ozr_refine_step(ctx, to_dev(A), Xd, ld, p)
    Rg = to_np(ozr.ozr_last_R(ctx, n))
    Xo, lo, info = orf.sweep(A, X0, lam0, delta, theta=p.theta, form_R=True)
    assert rep["beta"] == info["beta"] and rep["pairs_G"] > 0
    assert np.max(np.abs(Rg - info["R"])) <= 1e-16
    assert abs(rep["normR_fro"] - info["normR_fro"]) <= 1e-6 * info["normR_fro"]
    assert abs(rep["normW_fro"] - info["normW_fro"]) <= 1e-6 * info["normW_fro"] + 1e-30
    assert rep["omega_oa"] == pytest.approx(2 * (rep["normW_fro"] + 2 * np.max(np.abs(lam0)) * rep["normR_fro"]))


@pytest.mark.parametrize("cfg,start", [("c4p", "fp64"), ("c2", "fp32")])
def test_column_bands_bit_identical(ctx, cfg, start, monkeypatch):
    """The column-band pipeline of the slice products (ozr_api.cu run_banded, OZR_BANDS=k: band b's
    recombination on the side stream next to band b + 1's GEMM, register path; the last band TMA-staged)
    computes every column with the same arithmetic as the single launch: X̂, λ̂ and the report agree bit for
    bit, including a sweep with unresolved groups (FP32 start)."""
    A, lam0, X0 = _case(cfg, 4096, start)
    X1, l1, r1 = _gpu_sweep(ctx, A, X0, lam0, 1e-12)
    monkeypatch.setenv("OZR_BANDS", "4")
    X4, l4, r4 = _gpu_sweep(ctx, A, X0, lam0, 1e-12)
    assert np.array_equal(X1, X4) and np.array_equal(l1, l4)
    for k in ("beta", "kX", "kA", "kR", "kE", "L_V", "L_W", "L_U", "n_clusters", "max_cluster"):
        assert r1[k] == r4[k], k
    assert r4["launches"] > r1["launches"]


CERT_CASES = [("c4p", 2048, 1e-12), ("c3", 1024, 1e-12), ("c5", 1024, 1e-15), ("c1", 100, 1e-15),
              ("c2", 1024, 1e-14)]


@pytest.mark.parametrize("cfg,n,delta", CERT_CASES)
def test_certificate_matches_oracle_and_forward_error(ctx, cfg, n, delta):
    """R12: the library's a-posteriori estimate (bf16 tensor-core Q = ẼᵀC, power iteration; params.certify = 2)
    after the second sweep of an FP64 start, against (a) the oracle's certificate of its own exact-product sweep
    on the same input (3 %) and (b) the forward error of the GPU's X̂ against the reference eigenvectors (the
    estimate may not fall below it by more than 10 %: the digit budgets' error is part of what it certifies)."""
    import paper_2602_19090_b200 as ozr
    c = dict(W.CONFIGS[cfg])
    A, _ = W.make_matrix(n, c["kind"], c["cnd"], c["seed"])
    lam0, X0 = W.initial_eig(A, "fp64")
    X1, l1, _ = orf.sweep(A, X0, lam0, delta)
    Xg, lg, rep = _gpu_sweep(ctx, A, X1, l1, delta, certify=2)
    Xo, lo, info = orf.sweep(A, X1, l1, delta)
    co = orf.certificate(info["E"], lo, delta=delta)
    assert rep["n_clusters"] == 0 and rep["cert"] > 0
    assert abs(rep["cert"] - co["est"]) <= 0.03 * co["est"], (rep["cert"], co)
    Xh, Xl, lh, ll, _ = orf.reference_eigvecs(A, X0, lam0)
    fe = orf.forward_error(Xh, Xl, Xg, lh, lg)
    assert rep["cert"] >= 0.9 * fe, (rep["cert"], fe, co)
