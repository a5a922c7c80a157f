"""The Hermitian extension of Algorithm 1 ("the proposed method can be extended in a straightforward
manner to Hermitian matrices") — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The paper gives the extension in one sentence; reading R18 fixes it as Algorithm 1
with every transpose read as the conjugate transpose and every product complex:
  line 1  V = A·X̂^(1)                         (complex product, exact to double-double)
  line 2  r_j = 1 − x̂_jᴴx̂_j                    (real)
  line 3  λ̂_j = Re(x̂_jᴴv_j)/(1 − r_j)          (real: A is Hermitian)
  line 4  W = X̂ᴴ(V − X̂D̂)
  line 5  ẽ_ij = w_ij/(λ̂_j − λ̂_i) (i ≠ j),  ẽ_jj = r_j/2  (real: the phase of x̂_j is left where the start put it,
          the imaginary part of w_jj/… being the first-order phase drift, which the refinement does not correct)
  line 6  X̂ ← accsum(X̂^(1), X̂^(1)Ẽ)           (real and imaginary parts separately)
and the truncation X̂ → X̂^(1) of §3.1 (eq. x with s = 1) applied to the real and imaginary
parts with the column's one τ_j = 0.75·2^⌈log2 w_j⌉·2^β, w_j = max_i max(|Re x̂_ij|, |Im x̂_ij|); β from §4.1
 with n the complex dimension. Every complex product is written as the definition
Re(PQ) = [Re P, −Im P]·[Re Q; Im Q], Im(PQ) = [Im P, Re P]·[Re Q; Im Q] — one double-double triple loop
(oracle/ddmm.c) over the 2k-long contraction each."""
import numpy as np

from . import _clib
from .fp import ceil_log2, dd_add, dd_div_dd, fast_two_sum, two_prod, two_sum
from .refine import BETA_MAX, BETA_MIN, THETA_DEFAULT, choose_beta, col_dot_dd
from .split import tau


def cmul_dd(Pr, Pi, Qr, Qi, Qr_lo=None, Qi_lo=None):
    """P·Q for complex P (m x k, real/imag fp64) and Q (k x n, optionally double-double parts), in double-double:
    Re = [Pr, −Pi]·[Qr; Qi], Im = [Pi, Pr]·[Qr; Qi]. Returns (Re_hi, Re_lo, Im_hi, Im_lo)."""
    Q = np.ascontiguousarray(np.vstack([Qr, Qi]).T)
    Ql = None
    if Qr_lo is not None or Qi_lo is not None:
        zr = np.zeros_like(Qr) if Qr_lo is None else Qr_lo
        zi = np.zeros_like(Qi) if Qi_lo is None else Qi_lo
        Ql = np.ascontiguousarray(np.vstack([zr, zi]).T)
    Rh, Rl = _clib.dd_gemm_nt(np.hstack([Pr, -Pi]), Q, None, Ql)
    Ih, Il = _clib.dd_gemm_nt(np.hstack([Pi, Pr]), Q, None, Ql)
    return Rh, Rl, Ih, Il


def x1_truncate_herm(Xr, Xi, beta):
    """X̂ → X̂^(1) (eq. x, s = 1) on both parts with the column's τ_j from w_j = max_i max(|Re|, |Im|).
    Returns (X1r, X1i, w)."""
    w = np.maximum(np.max(np.abs(Xr), axis=0), np.max(np.abs(Xi), axis=0))
    t = tau(w, beta)[None, :]
    return (t + Xr) - t, (t + Xi) - t, w


def sweep_herm(Ar, Ai, Xr, Xi, lam_prev, delta, theta=THETA_DEFAULT):
    """One sweep of the Hermitian Algorithm 1 (reading R18). A = Ar + i·Ai Hermitian (Ar symmetric, Ai
    antisymmetric), X̂ = Xr + i·Xi, λ̂_prev real (ascending or not). Returns (Xr_new, Xi_new, λ̂, info)."""
    Ar, Ai = np.asarray(Ar, dtype=np.float64), np.asarray(Ai, dtype=np.float64)
    Xr, Xi = np.asarray(Xr, dtype=np.float64), np.asarray(Xi, dtype=np.float64)
    n = Ar.shape[0]
    w = np.maximum(np.max(np.abs(Xr), axis=0), np.max(np.abs(Xi), axis=0))
    c = ceil_log2(w)
    beta_raw, _ = choose_beta(n, delta / theta, lam_prev, c, w, cluster_mode=0)
    beta = int(min(max(beta_raw, BETA_MIN), BETA_MAX))
    X1r, X1i, _ = x1_truncate_herm(Xr, Xi, beta)
    # line 1: V = A X̂^(1)
    Vrh, Vrl, Vih, Vil = cmul_dd(Ar, Ai, X1r, X1i)
    # line 2: r_j = 1 − x̂_jᴴx̂_j = 1 − Σ (Re² + Im²)
    s1h, s1l = col_dot_dd(X1r, X1r)
    s2h, s2l = col_dot_dd(X1i, X1i)
    sh, sl = dd_add(s1h, s1l, s2h, s2l)
    rh, rl = dd_add(np.ones(n), np.zeros(n), -sh, -sl)
    if np.any(rh >= 1.0):
        raise ValueError("degenerate column: r_j >= 1")
    # line 3: λ̂_j = Re(x̂_jᴴv_j)/(1 − r_j)
    t1h, t1l = col_dot_dd(X1r, Vrh, Vrl)
    t2h, t2l = col_dot_dd(X1i, Vih, Vil)
    th, tl = dd_add(t1h, t1l, t2h, t2l)
    lh, ll = dd_div_dd(th, tl, sh, sl)
    lam = lh + ll
    # line 4: W = X̂ᴴ(V − X̂D̂)
    prh, prl = two_prod(X1r, lam[None, :])
    pih, pil = two_prod(X1i, lam[None, :])
    Rrh, Rrl = dd_add(Vrh, Vrl, -prh, -prl)
    Rih, Ril = dd_add(Vih, Vil, -pih, -pil)
    Wrh, Wrl, Wih, Wil = cmul_dd(np.ascontiguousarray(X1r.T), -np.ascontiguousarray(X1i.T), Rrh, Rih, Rrl, Ril)
    # line 5: ẽ_ij = w_ij/(λ̂_j − λ̂_i), ẽ_jj = r_j/2
    dl = lam[None, :] - lam[:, None]
    off = ~np.eye(n, dtype=bool)
    if np.any(dl[off] == 0):
        raise ValueError("equal λ̂ (PAPER.md:333 assumes distinct eigenvalues)")
    dls = np.where(off, dl, 1.0)
    Er = np.where(off, Wrh / dls, 0.0)
    Ei = np.where(off, Wih / dls, 0.0)
    Er[np.arange(n), np.arange(n)] = (rh + rl) / 2
    # line 6: X̂ ← accsum(X̂^(1), X̂^(1)Ẽ)
    Urh, Url, Uih, Uil = cmul_dd(X1r, X1i, Er, Ei)
    s, e = two_sum(X1r, Urh)
    Xrn = fast_two_sum(s, e + Url)[0]
    s, e = two_sum(X1i, Uih)
    Xin = fast_two_sum(s, e + Uil)[0]
    info = {"beta": beta, "beta_raw": int(beta_raw), "X1": (X1r, X1i), "E": (Er, Ei), "r": (rh, rl),
            "W": (Wrh, Wih), "normE_fro": float(np.sqrt(np.sum(Er * Er + Ei * Ei))),
            "net_update": float(np.sqrt(np.sum((Xrn - Xr) ** 2 + (Xin - Xi) ** 2)))}
    return Xrn, Xin, lam, info


def forward_error_herm(Xr_ref, Xi_ref, Xr, Xi, lam_ref=None, lam=None):
    """‖X − X̂‖₂ (PAPER.md:48-50, 2-norm PAPER.md:121) for complex eigenvector matrices: columns matched by
    ascending λ, each reference column multiplied by the unit phase of x_refᴴx̂ (the complex analogue of the
    sign alignment), exact 2-norm by SVD."""
    Xref = np.asarray(Xr_ref) + 1j * np.asarray(Xi_ref)
    X = np.asarray(Xr) + 1j * np.asarray(Xi)
    if lam_ref is not None and lam is not None:
        Xref = Xref[:, np.argsort(lam_ref, kind="stable")]
        X = X[:, np.argsort(lam, kind="stable")]
    p = np.sum(np.conj(Xref) * X, axis=0)
    ph = np.where(np.abs(p) > 0, p / np.where(np.abs(p) > 0, np.abs(p), 1.0), 1.0)
    return float(np.linalg.norm(Xref * ph[None, :] - X, 2))


def refine_herm(Ar, Ai, Xr, Xi, lam, delta, sweeps, theta=THETA_DEFAULT):
    """`sweeps` sweeps of sweep_herm (the paper's experiments use fixed iteration counts)."""
    hist = []
    for _ in range(sweeps):
        Xr, Xi, lam, info = sweep_herm(Ar, Ai, Xr, Xi, lam, delta, theta)
        hist.append(info)
    return Xr, Xi, lam, hist
