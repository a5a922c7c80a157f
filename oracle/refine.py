"""Algorithm 1 with the one-sided product, its driver, reference eigenvectors and the forward error
(TEST INFRASTRUCTURE ONLY — see oracle/__init__.py).

The sweep follows PAPER.md Algorithm 1 (lines 261-278) line by line, with
  * X̂ replaced by its leading slice X̂^(1) (§3.1, eq. E' line 331: X' = X̂^(1)(I+Ẽ)),
  * β from §4.1 (lines 458-463) or §3.3 eq. (proposed_beta) (lines 400-405),
  * accmul(A, X̂^(1)) = A·X̂^(1) EXACTLY (the quantity eq. mat_mul, computes with
    n_A error-free slice products), here as a naive double-double triple loop (ddmm.c),
  * accsum (line 275, "for example, Section 2.2") = the double-double sum rounded once to fp64.
The other products of the sweep (W = X̂ᵀ(V − X̂D̂), X̂Ẽ) are also formed in double-double, so this is
Algorithm 1 evaluated with products accurate to ~2^-100: the GPU path differs from it only by its
documented digit budgets.
"""
import numpy as np

from . import _clib
from .fp import U, ceil_log2, dd_add, dd_div_dd, fast_two_sum, two_prod, two_sum
from .split import (alpha_dense, alpha_sparse, alpha_theoretical, beta_dense, beta_sparse, beta_theoretical, gap_min, gap_pos, sum_pow2_2c,
                    x1_truncate)

BETA_MIN, BETA_MAX = 2, 52  # reading R4: τ + x stays in τ's binade iff β ≥ 2; ≥ 1 bit kept iff β ≤ 52
THETA_DEFAULT = 4.0  # reading R11: δ' = δ/θ so that the O(δ) result lands at or below δ


def col_dot_dd(X, Yh, Yl=None):
    """s_j = Σ_i x_ij (yh_ij + yl_ij) in double-double, summed in row order i = 0..n-1."""
    n, m = X.shape
    sh = np.zeros(m)
    sl = np.zeros(m)
    for i in range(n):
        p, e = two_prod(X[i], Yh[i])
        if Yl is not None:
            e = e + X[i] * Yl[i]
        sh, sl = dd_add(sh, sl, p, e)
    return sh, sl


def choose_beta(n, delta_p, lam_prev, c, w, beta_mode="dense", xi=None, cluster_mode=1, row_nnz=None):
    """β for this sweep from the PREVIOUS sweep's λ̂ (reading R9; the paper computes λ̂ only after V).
    With the cluster branch, equal estimates are tolerated and the smallest positive gap is used (R13).
    beta_mode: "dense" (§4.1), "theoretical" (§3.3, ξ), "sparse" (§4.3, k = row_nnz)."""
    gap = gap_min(lam_prev)
    if cluster_mode and not gap > 0:
        gap = gap_pos(lam_prev)
    if beta_mode == "dense":
        b = beta_dense(n, delta_p, lam_prev, c, w, gap)
        a = alpha_dense(n, min(max(b, BETA_MIN), BETA_MAX))
    elif beta_mode == "sparse":
        k = row_nnz if row_nnz and row_nnz < n else n
        b = beta_sparse(n, k, delta_p, lam_prev, c, w, gap)
        a = alpha_sparse(k, min(max(b, BETA_MIN), BETA_MAX))
    else:
        b = beta_theoretical(xi if xi else n, delta_p, lam_prev, c, w, gap)
        a = alpha_theoretical(n, min(max(b, BETA_MIN), BETA_MAX))
    return b, a


KAPPA_DEFAULT = 2.0 ** -10


def unresolved_groups(E, lam, kappa=KAPPA_DEFAULT):
    """Reading R13 (builder-defined; PAPER.md:333 and 730 leave clusters open): the first-order
    correction ẽ_ij = w_ij / (λ̂_j − λ̂_i) of Algorithm 1 line 5 linearises (I + E)^{-1}
    and is only trustworthy while |ẽ_ij| ≪ 1. Pairs (i, j), i ≠ j, with λ̂_i = λ̂_j or |ẽ_ij| > κ are
    "unresolved"; the groups are the connected components of that graph with ≥ 2 members, each listed
    in ascending (λ̂, index) order, the groups ordered by their first member. E: n x n with the
    first-order values off the diagonal (0 where λ̂_i = λ̂_j)."""
    n = E.shape[0]
    parent = list(range(n))

    def find(a):
        while parent[a] != a:
            parent[a] = parent[parent[a]]
            a = parent[a]
        return a

    dl = lam[None, :] - lam[:, None]
    mask = (np.abs(E) > kappa) | (dl == 0)
    np.fill_diagonal(mask, False)
    for i, j in zip(*np.nonzero(mask)):
        a, b = find(int(i)), find(int(j))
        if a != b:
            parent[max(a, b)] = min(a, b)
    groups = {}
    for i in range(n):
        groups.setdefault(find(i), []).append(i)
    out = []
    for g in groups.values():
        if len(g) >= 2:
            out.append(sorted(g, key=lambda k: (lam[k], k)))
    out.sort(key=lambda J: J[0])
    return out


def cluster_subsolve(E, lam, J, X1, Wh, Wl, rh, rl):
    """Rayleigh–Ritz in span(X̂^(1)_J) for one unresolved group J (reading R13; the construction follows
    the cited Ogita–Aishima cluster refinement, restated here). Pinned by
    tests/test_oracle_pins.py: exact double / dyadic near-double eigenvalues of the Householder family (the
    eigenspace, the undone 30° and 69° rotations) and, through refine_to_tol, __float128 Jacobi.
    With G = X̂ᵀX̂ = I − R and S = X̂ᵀAX̂ = W + (I − R)D̂ (Alg. 1 line 4):
      μ = mean λ̂_J,  M = S_JJ − μ G_JJ = W_JJ + (I − R_JJ)(D̂_J − μI),  K₀ = (M + Mᵀ)/2,
      C = I + R_JJ/2  (= G_JJ^{-1/2} to first order),  K = C K₀ C = Y Θ Yᵀ  (Θ ascending),
      Z = C Y:  Ẽ_JJ ← Z − I,  Ẽ_{i,J} ← Ẽ_{i,J} Z for i ∉ J,  λ̂_J ← μ + Θ.
    Y's column k is signed so that y_kk ≥ 0 (the largest-|y| entry positive if y_kk = 0).
    R_JJ: r_jj = r_j exact; r_ij = −x̂_iᵀx̂_j (i ≠ j) in double-double. Modifies E and lam in place."""
    J = np.asarray(J)
    m = len(J)
    XJ = np.ascontiguousarray(X1[:, J].T)
    Gh, Gl = _clib.dd_gemm_nt(XJ, XJ)
    R = -(Gh + Gl)
    R[np.arange(m), np.arange(m)] = rh[J] + rl[J]
    mu = 0.0
    for j in J:
        mu = mu + lam[j]
    mu = mu / m
    WJ = Wh[np.ix_(J, J)] + Wl[np.ix_(J, J)]
    M = WJ + (np.eye(m) - R) * (lam[J] - mu)[None, :]
    K0 = (M + M.T) * 0.5
    C = np.eye(m) + R * 0.5
    K = C @ K0 @ C
    K = (K + K.T) * 0.5
    th, tl, Yh, Yl, _ = _clib.jacobi_q(K)
    Y = Yh + Yl
    for k in range(m):
        piv = Y[k, k] if Y[k, k] != 0 else Y[np.argmax(np.abs(Y[:, k])), k]
        if piv < 0:
            Y[:, k] = -Y[:, k]
    Z = C @ Y
    notJ = np.setdiff1d(np.arange(E.shape[0]), J)
    E[np.ix_(notJ, J)] = E[np.ix_(notJ, J)] @ Z
    E[np.ix_(J, J)] = Z - np.eye(m)
    lam[J] = mu + (th + tl)
    # conditioning of the sub-solve: ‖K‖ / min eigenvalue gap of K (an fp64 eigensolver's eigenvectors
    # are accurate to ~u·this; the tests derive their tolerance for clustered sweeps from it)
    gK = np.min(np.diff(th)) if m > 1 else np.inf
    return float(np.max(np.abs(th)) / gK) if gK > 0 else np.inf


def sweep(A, X, lam_prev, delta, theta=THETA_DEFAULT, beta=None, beta_mode="dense", xi=None, truncate=True,
          cluster_mode=1, kappa=KAPPA_DEFAULT, max_cluster=None, groups=None, form_R=False, row_nnz=None):
    """One iteration of Algorithm 1. Returns (X_new fp64, λ̂ fp64, info dict).

    cluster_mode 0: the paper's Algorithm 1 (distinct eigenvalues assumed); equal
    λ̂ raise. cluster_mode 1: unresolved groups get a Rayleigh–Ritz sub-solve (cluster_subsolve,
    DESIGN.md reading R13; not in the paper — pinned against exact eigensystems, tests/test_oracle_pins.py).
    groups: use these unresolved groups instead of finding them (parity runs: a pair whose |ẽ_ij| sits
    at κ may be classified differently by the GPU's digit-budget W; the tests check that is the only
    difference, then evaluate the same groups)."""
    A = np.asarray(A, dtype=np.float64)
    X = np.asarray(X, dtype=np.float64)
    n = A.shape[0]
    info = {}
    w = np.max(np.abs(X), axis=0)
    c = ceil_log2(w)
    if beta is None:
        beta, alpha = choose_beta(n, delta / theta, lam_prev, c, w, beta_mode, xi, cluster_mode, row_nnz)
    else:
        alpha = alpha_dense(n, beta)
    info["beta_raw"] = int(beta)
    beta = int(min(max(beta, BETA_MIN), BETA_MAX))
    info["beta"], info["alpha"] = beta, int(alpha)
    # X̂ <- X̂^(1): eq. (x), s = 1
    X1 = x1_truncate(X, beta)[0] if truncate else X.copy()
    # line 1: V = accmul(A, X̂)  — exact product (A symmetric: V = A X̂^(1))
    Vh, Vl = _clib.dd_gemm_nt(A, np.ascontiguousarray(X1.T))
    # line 2: r_i = 1 − x̂_iᵀ x̂_i
    sh, sl = col_dot_dd(X1, X1)
    rh, rl = dd_add(np.ones(n), np.zeros(n), -sh, -sl)
    if np.any(rh >= 1.0):
        raise ValueError("degenerate column: r_i >= 1")
    # line 3: λ̂_i = x̂_iᵀ v̂_i / (1 − r_i)   (1 − r_i = x̂_iᵀx̂_i)
    th, tl = col_dot_dd(X1, Vh, Vl)
    lh, ll = dd_div_dd(th, tl, sh, sl)
    lam = lh + ll
    # line 4: W = X̂ᵀ (V − X̂ D̂)
    ph, pl = two_prod(X1, lam[None, :])
    Rh, Rl = dd_add(Vh, Vl, -ph, -pl)
    Wh, Wl = _clib.dd_gemm_nt(np.ascontiguousarray(X1.T), np.ascontiguousarray(Rh.T), None,
                              np.ascontiguousarray(Rl.T))
    W = Wh + Wl
    if form_R:
        # R = I − X̂ᵀX̂ (the R/S form): off the diagonal −x̂_iᵀx̂_j in dd, on it the r_i of
        # line 2; and ‖W‖_F (for the OA-2018 threshold diagnostic, reading R13)
        X1T = np.ascontiguousarray(X1.T)
        Gh, Gl = _clib.dd_gemm_nt(X1T, X1T)
        R = -(Gh + Gl)
        R[np.arange(n), np.arange(n)] = rh + rl
        info["R"] = R
        info["normW_fro"] = float(np.sqrt(np.sum(Wh * Wh)))
        info["normR_fro"] = float(np.sqrt(np.sum(R * R)))
    # line 5: ẽ_ij = w_ij / (λ̃_j − λ̃_i), i ≠ j;  ẽ_ii = r_i / 2
    dl = lam[None, :] - lam[:, None]
    off = ~np.eye(n, dtype=bool)
    if cluster_mode == 0 and np.any(dl[off] == 0):
        raise ValueError("clustered eigenvalues: equal λ̂ (PAPER.md:333 assumes none)")
    with np.errstate(divide="ignore", invalid="ignore"):
        E = np.where(off & (dl != 0), Wh / np.where(dl != 0, dl, 1.0), 0.0)
    E[np.arange(n), np.arange(n)] = (rh + rl) / 2
    info["clusters"] = []
    info["E_first_order"] = E.copy() if cluster_mode else None
    info["lam_rq"] = lam.copy()
    if cluster_mode:
        comps = unresolved_groups(E, lam, kappa) if groups is None else [list(J) for J in groups]
        if max_cluster and any(len(J) > max_cluster for J in comps):
            raise ValueError("cluster larger than max_cluster")
        conds = []
        for J in comps:
            conds.append(cluster_subsolve(E, lam, J, X1, Wh, Wl, rh, rl))
        info["clusters"] = comps
        info["cluster_cond"] = max(conds, default=0.0)
    # line 6: X̂ <- accsum(X̂, X̂Ẽ)  on X̂^(1) (eq. E')
    Uh, Ul = _clib.dd_gemm_nt(X1, np.ascontiguousarray(E.T))
    s, e = two_sum(X1, Uh)
    Xn, _ = fast_two_sum(s, e + Ul)
    info["normE_fro"] = float(np.sqrt(np.sum(E * E)))
    info["net_update"] = float(np.sqrt(np.sum((Xn - X) ** 2)))
    info["gap_min"] = gap_min(lam_prev)
    info["X1"] = X1
    info["V"] = (Vh, Vl)
    info["W"] = (Wh, Wl)
    info["r"] = (rh, rl)
    info["E"] = E
    return Xn, lam, info


CERT_SAFETY = 1.15  # power-iteration / bf16-GEMM slack of the library's estimate (reading R12)
CONTRACT = 1.0 / 8  # a certified sweep whose estimate fell by less than this factor sits at the truncation floor


def second_order_defect(E, lam):
    """−(E − Ẽ) to second order in Ẽ (reading R12), E the exact correction X = X̂^(1)(I + E).
    Derivation (the paper gives only the order, Theorem 1): with H = (I + E)^{-1} = I + η,
    G = X̂ᵀX̂ = HᵀH and S = X̂ᵀAX̂ = HᵀΛH exactly, so Alg. 1's W = S − G·D̂ (line 4) is
        w_ij = Σ_k h_ki (λ_k − λ̂_j) h_kj = (λ_i − λ_j) η_ij + Σ_k η_ki (λ_k − λ_j) η_kj + O(η³)   (i ≠ j),
    and r_jj = 1 − g_jj = −2η_jj − ‖η_j‖². Line 5's ẽ_ij = w_ij/(λ̂_j − λ̂_i), ẽ_jj = r_jj/2 against the exact
    e = −η + η² + O(η³), with η = −Ẽ + O(Ẽ²), leave
        (E − Ẽ)_ij = (Ẽ²)_ij − q_ij/(λ̂_j − λ̂_i)   (i ≠ j),   (E − Ẽ)_jj = (Ẽ²)_jj + ½‖ẽ_j‖²,
    Q = ẼᵀC, c_kj = (λ̂_k − λ̂_j) ẽ_kj. Returns D = −(E − Ẽ) (the sign the library's kernel produces)."""
    E = np.asarray(E, dtype=np.float64)
    lam = np.asarray(lam, dtype=np.float64)
    n = E.shape[0]
    C = (lam[:, None] - lam[None, :]) * E
    Q = E.T @ C
    E2 = E @ E
    dl = lam[None, :] - lam[:, None]
    off = ~np.eye(n, dtype=bool)
    if np.any(dl[off] == 0):
        return None
    D = np.where(off, Q / np.where(off, dl, 1.0), 0.0) - E2
    D[np.diag_indices(n)] -= 0.5 * np.sum(E * E, axis=0)
    return D


def certificate(E, lam, n_power=None, delta=None):
    """A-posteriori forward error of the sweep that produced Ẽ (reading R12; the paper gives no iteration rule,
    PAPER.md:536-540, and its error model eq. assume2/gamma, predicts the error only on
    average over the columns). The sweep returns X̂_new = X̂^(1)(I + Ẽ) while the exact eigenvectors are
    X = X̂^(1)(I + E), so X − X̂_new = X̂^(1)(E − Ẽ): Ẽ's second-order defect
    (second_order_defect()) in the 2-norm of PAPER.md:121, plus X̂_new's rounding to fp64 (a noise-like matrix
    of entries ≤ u|x_ij|: 2-norm ≈ 2u), an allowance ‖Ẽ‖_F·‖D‖_F for the third-order terms, and the defect from
    the fp64 rounding of the λ̂ in Ẽ's denominators, ≤ 2u·‖(λ̂_i ẽ_ij/(λ̂_j − λ̂_i))_{i≠j}‖_F (pinned by the
    exactly-known clustered family, where it is the whole error). Returns
        est = sqrt(‖D‖₂² + (2u)²) + ‖Ẽ‖_F‖D‖_F + 2u‖(λ̂_i ẽ_ij/(λ̂_j − λ̂_i))‖_F
    and the parts (quad = the last two terms). ‖·‖₂ exactly (LAPACK) for n ≤ 2048, else `n_power` (default 60) power iterations. With δ
    given, the library's shortcut is mirrored: when even the lower bound max_j ‖D_{:,j}‖ + quad exceeds
    16δ (no decision of the driver can then tell the value from its Frobenius upper bound), or the Frobenius
    upper bound already certifies, ‖D‖_F stands in for ‖D‖₂."""
    E = np.asarray(E, dtype=np.float64)
    lam = np.asarray(lam, dtype=np.float64)
    D = second_order_defect(E, lam)
    if D is None:
        return dict(est=np.inf, est_q=np.inf, quad=np.inf, frob=np.inf)
    n = E.shape[0]
    frob = float(np.linalg.norm(D))
    # the λ̂ the sweep divided by are Rayleigh quotients ROUNDED to fp64: with ε_i = λ̂_i − λ_i, |ε_i| ≤ u|λ̂_i|, the
    # first-order part of w_ij is −(λ̂_j − λ̂_i)η_ij − ε_i η_ij − ε_j η_ji, which leaves the defect
    # (ε_i ẽ_ij + ε_j ẽ_ji)/(λ̂_j − λ̂_i) in Ẽ — first order in Ẽ, and u|λ̂|/gap is not small in a tight cluster
    off = ~np.eye(n, dtype=bool)
    dl = np.where(off, lam[None, :] - lam[:, None], 1.0)
    rlam = 2 * U * float(np.sqrt(np.sum(np.where(off, lam[:, None] * E / dl, 0.0) ** 2)))
    quad = float(np.sqrt(np.sum(E * E))) * frob + rlam
    if delta is not None:
        upper = float(np.sqrt(frob * frob + (2 * U) ** 2)) + quad
        lower = float(np.max(np.sqrt(np.sum(D * D, axis=0)))) + quad
        if upper * CERT_SAFETY <= delta or lower > 16 * delta:
            return dict(est=upper, est_q=frob, quad=quad, frob=frob)
    if n <= 2048 and n_power is None:
        s = float(np.linalg.norm(D, 2))
    else:
        v = np.random.default_rng(0).standard_normal(n)
        v /= np.linalg.norm(v)
        s = 0.0
        for _ in range(n_power or 60):
            y = D.T @ (D @ v)
            s = float(np.sqrt(np.linalg.norm(y)))
            v = y / np.linalg.norm(y)
    est = float(np.sqrt(s * s + (2 * U) ** 2)) + quad
    return dict(est=est, est_q=s, quad=quad, frob=frob)


def refine_to_tol(A, X0, lam0, delta, theta=THETA_DEFAULT, max_sweeps=6, beta_mode="dense", xi=None, callback=None,
                  cluster_mode=1, kappa=KAPPA_DEFAULT, max_escalations=2, truncate=True, row_nnz=None):
    """Driver (reading R12; the paper iterates a fixed number of times). After every sweep
    without unresolved groups the sweep's own Ẽ certifies the returned X̂ (certificate(): the second-order
    defect of Ẽ, in the 2-norm of PAPER.md:121): stop with "converged" when est·CERT_SAFETY ≤ δ. An uncertified
    sweep whose estimate did not fall below CONTRACT × the previous one — or fell so fast that the next sweep's
    quadratic part, est³/est_prev² at the observed rate, is below δ/8 while est ≤ 16δ (est_prev: the previous
    estimate, or ν = ‖X_k − X_{k−1}‖_F when the previous sweep had none) — sits at the truncation floor (the
    quadratic error of the deliberately truncated X̂^(1)): θ grows by the power of 4 that
    brings the floor (∝ 1/θ: β falls by ½ log2 θ, the error is quadratic in 2^-β) below δ/2 — at most
    `max_escalations` times, then "stagnation". Sweeps with unresolved groups (a Rayleigh–Ritz rotation, R13) are never certified or
    compared. The paper's ξ = n prediction ν²·max|λ̂|/(n·gap) (eq. assume2 / gamma) and ν = ‖X_k − X_{k−1}‖_F
    are recorded, not used."""
    X, lam = np.asarray(X0, dtype=np.float64), np.asarray(lam0, dtype=np.float64)
    n = X.shape[0]
    hist = []
    est_prev = None
    for k in range(max_sweeps):
        Xn, lamn, info = sweep(A, X, lam, delta, theta, beta_mode=beta_mode, xi=xi, cluster_mode=cluster_mode,
                               kappa=kappa, truncate=truncate, row_nnz=row_nnz)
        nu = info["net_update"]
        ls = np.sort(lamn)
        d = np.diff(ls)
        gpos = np.min(d[d > 0]) if np.any(d > 0) else max(np.max(np.abs(lamn)) * U, 1e-300)
        pred = nu * nu * np.max(np.abs(lamn)) / (n * gpos)
        rec = dict(sweep=k + 1, beta=info["beta"], alpha=info["alpha"], net_update=nu, predicted=pred,
                   normE_fro=info["normE_fro"], theta=theta, clusters=len(info["clusters"]))
        X, lam = Xn, lamn
        hist.append(rec)
        if info["clusters"]:
            est_prev = None
            if callback:
                rec.update(callback(X, lam))
            continue
        cert = certificate(info["E"], lam, delta=delta)
        rec["cert"] = cert["est"]
        if callback:
            rec.update(callback(X, lam))
        if cert["est"] * CERT_SAFETY <= delta:
            rec["stop"] = "converged"
            break
        # at the floor: not contracting, or contracting so fast that the next sweep's quadratic part
        # (est³/est_prev² from the observed rate) is below δ/8, i.e. what remains is the truncation floor
        # (floors are O(δ) by the choice of β, so only an estimate within 16δ is read that way)
        # the first certified sweep after a start, a cluster sweep or an escalation has no previous estimate: there
        # ν = ‖X_k − X_{k−1}‖_F, the size of the error this sweep removed, stands in for it in the second test
        # (only while θ can still grow: without an escalation to spend, a floor read off ν would stop a run that
        # the next sweep may well finish)
        prev = est_prev if est_prev is not None else (nu if nu > 0 and truncate and max_escalations > 0 else None)
        floor = (est_prev is not None and cert["est"] > CONTRACT * est_prev) or \
                (prev is not None and cert["est"] <= 16 * delta and cert["est"] ** 3 / prev ** 2 <= delta / 8)
        if floor:
            if truncate and max_escalations > 0:
                max_escalations -= 1
                m = max(1, int(np.ceil(np.log(2.0 * cert["est"] * CERT_SAFETY / delta) / np.log(4.0))))
                theta = theta * 4.0 ** m
                est_prev = None
                continue
            rec["stop"] = "stagnation"
            break
        est_prev = cert["est"]
    return X, lam, hist


# ----------------------------------------------------------------------------- reference solution

def _reference_rr(E, lh, ll, J, Sh, Sl, Gh, Gl, R):
    """Rayleigh–Ritz of one unresolved group J inside reference_eigvecs ("use the cluster
    branch when [the first-order correction fails]"; the construction of reading R13 on the dd products of
    the R/S form): μ = mean λ̃_J, M = S_JJ − μG_JJ (dd, rounded once), K = C·(M + Mᵀ)/2·C with
    C = I + R_JJ/2, K = YΘYᵀ by LAPACK (numpy.linalg.eigh; its u‖K‖/gap_K error is removed by the dd
    sweeps that follow), Z = CY: Ẽ_JJ ← Z − I, Ẽ_{i,J} ← Ẽ_{i,J}Z (i ∉ J), λ̃_J ← μ + Θ."""
    J = np.asarray(J)
    m = len(J)
    mu = float(np.mean(lh[J]))
    ix = np.ix_(J, J)
    ph, pl = two_prod(Gh[ix], mu)
    M = (Sh[ix] - ph) + (Sl[ix] - pl - Gl[ix] * mu)
    C = np.eye(m) + 0.5 * R[ix]
    K = C @ ((M + M.T) * 0.5) @ C
    th, Y = np.linalg.eigh((K + K.T) * 0.5)
    for k in range(m):
        piv = Y[k, k] if Y[k, k] != 0 else Y[np.argmax(np.abs(Y[:, k])), k]
        if piv < 0:
            Y[:, k] = -Y[:, k]
    Z = C @ Y
    notJ = np.setdiff1d(np.arange(E.shape[0]), J)
    E[np.ix_(notJ, J)] = E[np.ix_(notJ, J)] @ Z
    E[ix] = Z - np.eye(m)
    lh[J] = mu + th
    ll[J] = 0.0


def reference_eigvecs(A, X0, lam0, tol=1e-27, max_sweeps=10, cluster_kappa=None, X0_lo=None):
    """Reference eigenvectors of the STORED A (PAPER.md:62 uses a pseudo-quadruple reference): the
    Ogita–Aishima iteration (the R/S form ẽ_ij = (s_ij + λ̃_j r_ij)/(λ̃_j − λ̃_i))
    with X̂ kept in double-double and every product in double-double, untruncated, from an LAPACK
    start, until ‖Ẽ‖_F ≤ tol. cluster_kappa (None: off): groups of pairs with |ẽ_ij| > cluster_kappa
    (unresolved_groups) get a Rayleigh–Ritz step (_reference_rr) — needed where the LAPACK start is not in
    the linear regime (BASELINE c4: cnd 1e14, gaps below u‖A‖). Returns (Xh, Xl, λh, λl, history).
    Certified separately by residual_certificate() and pinned against __float128 Jacobi (n ≤ 32) and
    exact families."""
    A = np.asarray(A, dtype=np.float64)
    n = A.shape[0]
    Xh = np.array(X0, dtype=np.float64)  # X0_lo: resume from a double-double state of an earlier call
    Xl = np.zeros((n, n)) if X0_lo is None else np.array(X0_lo, dtype=np.float64)
    hist = []
    lh = ll = None
    for k in range(max_sweeps):
        XhT, XlT = np.ascontiguousarray(Xh.T), np.ascontiguousarray(Xl.T)
        Vh, Vl = _clib.dd_gemm_nt(A, XhT, None, XlT)               # V = A X
        Gh, Gl = _clib.dd_gemm_nt(XhT, XhT, XlT, XlT)             # G = XᵀX
        VT_h, VT_l = np.ascontiguousarray(Vh.T), np.ascontiguousarray(Vl.T)
        Sh, Sl = _clib.dd_gemm_nt(XhT, VT_h, XlT, VT_l)           # S = XᵀA X
        dh, dl_ = np.diag(Gh).copy(), np.diag(Gl).copy()
        th, tl = np.diag(Sh).copy(), np.diag(Sl).copy()
        lh, ll = dd_div_dd(th, tl, dh, dl_)                        # Rayleigh quotients
        Rh, Rl = dd_add(np.eye(n), np.zeros((n, n)), -Gh, -Gl)    # R = I − XᵀX
        lam = lh + ll
        R = Rh + Rl
        # s_ij + λ̃_j r_ij in dd, then divided in fp64 (Ẽ needs only relative accuracy ~ ‖Ẽ‖)
        ph, pl = two_prod(Rh, lh[None, :])
        Nh, Nl = dd_add(Sh, Sl, ph, pl + Rl * lh[None, :] + Rh * ll[None, :])
        dlam = (lh[None, :] - lh[:, None]) + (ll[None, :] - ll[:, None])
        off = ~np.eye(n, dtype=bool)
        E = np.where(off, (Nh + Nl) / np.where(off, dlam, 1.0), 0.0)
        E[np.arange(n), np.arange(n)] = np.diag(R) / 2
        if cluster_kappa is not None:
            for J in unresolved_groups(E, lh, cluster_kappa):
                _reference_rr(E, lh, ll, J, Sh, Sl, Gh, Gl, R)
        Uh, Ul = _clib.dd_gemm_nt(Xh, np.ascontiguousarray(E.T), Xl, None)  # U = X Ẽ
        Xh, Xl = dd_add(Xh, Xl, Uh, Ul)
        nE = float(np.sqrt(np.sum(E * E)))
        hist.append(nE)
        if nE <= tol or (len(hist) >= 3 and nE > hist[-2] / 4 and nE < 1e-15):
            break
    return Xh, Xl, lh, ll, hist


def residual_certificate(A, Xh, Xl, lh, ll):
    """Pin P8: per-column residual ‖A x_j − λ_j x_j‖₂ in double-double and the
    orthogonality defect; with the eigenvalue gaps these bound the reference's own forward error
    (Davis–Kahan sin θ ≤ ‖r_j‖ / gap_j). Returns (res_norms, ortho_max)."""
    n = A.shape[0]
    XhT, XlT = np.ascontiguousarray(Xh.T), np.ascontiguousarray(Xl.T)
    Vh, Vl = _clib.dd_gemm_nt(A, XhT, None, XlT)
    ph, pl = two_prod(Xh, lh[None, :])
    pl = pl + Xl * lh[None, :] + Xh * ll[None, :]
    Rh, Rl = dd_add(Vh, Vl, -ph, -pl)
    res = np.sqrt(np.sum((Rh + Rl) ** 2, axis=0))
    Gh, Gl = _clib.dd_gemm_nt(XhT, XhT, XlT, XlT)
    Dh, Dl = dd_add(Gh, Gl, -np.eye(n), np.zeros((n, n)))
    return res, float(np.max(np.abs(Dh + Dl)))


def forward_error(Xh_ref, Xl_ref, X, lam_ref=None, lam=None, power_iters=None):
    """‖X − X̂‖₂ (PAPER.md:48-50, 2-norm per PAPER.md:121). Columns are matched by ascending λ (when
    λ's are given) and signs by sign(x_refᵀ x̂). For n ≤ 2048 the exact 2-norm (SVD); beyond, a
    power iteration of `power_iters` (default 40) steps on DᵀD."""
    X = np.asarray(X, dtype=np.float64)
    if lam_ref is not None and lam is not None:
        pr, px = np.argsort(lam_ref, kind="stable"), np.argsort(lam, kind="stable")
        Xh_ref, Xl_ref, X = Xh_ref[:, pr], Xl_ref[:, pr], X[:, px]
    sgn = np.sign(np.sum(Xh_ref * X, axis=0))
    sgn[sgn == 0] = 1.0
    D = (Xh_ref * sgn[None, :] - X) + Xl_ref * sgn[None, :]
    n = D.shape[0]
    if power_iters is None and n <= 2048:
        return float(np.linalg.norm(D, 2))
    v = np.random.default_rng(0).standard_normal(n)
    v /= np.linalg.norm(v)
    s = 0.0
    for _ in range(power_iters or 40):
        y = D.T @ (D @ v)
        s = np.linalg.norm(y)
        v = y / s
    return float(np.sqrt(s))


def sweep_columns(A, X, lam_prev, delta, J, theta=THETA_DEFAULT, beta=None, lam_rows=None):
    """Algorithm 1 restricted to the output columns J (bench.py's bounded CPU sample; identical formulas
    to sweep(), only the products' column sets shrink): V_J = A X̂^(1)_J, λ̂_J, Res_J,
    W_{:,J} = X̂^(1)ᵀ Res_J, Ẽ_{:,J} (needs λ̂ of all columns: `lam_rows` for i ∉ J — the full sweep's
    Rayleigh quotients when given, else λ_prev), U_J = X̂^(1) Ẽ_{:,J}. Returns (X_new[:, J], λ̂_J, β)."""
    A = np.asarray(A, dtype=np.float64)
    X = np.asarray(X, dtype=np.float64)
    n = A.shape[0]
    J = np.asarray(J)
    w = np.max(np.abs(X), axis=0)
    c = ceil_log2(w)
    if beta is None:
        beta, _ = choose_beta(n, delta / theta, lam_prev, c, w)
    beta = int(min(max(beta, BETA_MIN), BETA_MAX))
    X1 = x1_truncate(X, beta)[0]
    X1J = X1[:, J]
    Vh, Vl = _clib.dd_gemm_nt(A, np.ascontiguousarray(X1J.T))
    sh, sl = col_dot_dd(X1J, X1J)
    rh, rl = dd_add(np.ones(len(J)), np.zeros(len(J)), -sh, -sl)
    th, tl = col_dot_dd(X1J, Vh, Vl)
    lh, ll = dd_div_dd(th, tl, sh, sl)
    lamJ = lh + ll
    ph, pl = two_prod(X1J, lamJ[None, :])
    Rh, Rl = dd_add(Vh, Vl, -ph, -pl)
    Wh, Wl = _clib.dd_gemm_nt(np.ascontiguousarray(X1.T), np.ascontiguousarray(Rh.T), None,
                              np.ascontiguousarray(Rl.T))
    lam = np.array(lam_prev if lam_rows is None else lam_rows, dtype=np.float64)
    lam[J] = lamJ
    dl = lamJ[None, :] - lam[:, None]
    E = np.where(dl != 0, (Wh + Wl) / np.where(dl != 0, dl, 1.0), 0.0)
    E[J, np.arange(len(J))] = (rh + rl) / 2
    Uh, Ul = _clib.dd_gemm_nt(X1, np.ascontiguousarray(E.T))
    s, e = two_sum(X1J, Uh)
    return fast_two_sum(s, e + Ul)[0], lamJ, beta


def sweep_block(A, X, lam_prev, delta, col0, nl, allgather, theta=THETA_DEFAULT):
    """Algorithm 1 (cluster branch off) for the column block J = [col0, col0 + nl) of one
    rank of the block-column partition: X̂^(1) from the full X̂ (column-local truncation,
    β from the all-gathered column maxima — here the full X̂ is at hand), V_J = A X̂^(1)_J, λ̂_J, then
    `allgather(λ̂_J)` → λ̂ (n), W_{:,J} = X̂^(1)ᵀ(V_J − X̂^(1)_J D̂_J), Ẽ_{:,J}, X̂_new,J. The same per-element
    arithmetic as sweep(), so the concatenated blocks equal the full sweep bit for bit.
    Returns (X_new[:, J], λ̂ (n))."""
    A = np.asarray(A, dtype=np.float64)
    X = np.asarray(X, dtype=np.float64)
    n = A.shape[0]
    J = np.arange(col0, col0 + nl)
    w = np.max(np.abs(X), axis=0)
    beta, _ = choose_beta(n, delta / theta, lam_prev, ceil_log2(w), w, cluster_mode=0)
    beta = int(min(max(beta, BETA_MIN), BETA_MAX))
    X1 = x1_truncate(X, beta)[0]
    X1J = X1[:, J]
    Vh, Vl = _clib.dd_gemm_nt(A, np.ascontiguousarray(X1J.T))
    sh, sl = col_dot_dd(X1J, X1J)
    rh, rl = dd_add(np.ones(nl), np.zeros(nl), -sh, -sl)
    th, tl = col_dot_dd(X1J, Vh, Vl)
    lh, ll = dd_div_dd(th, tl, sh, sl)
    lam = allgather(lh + ll)
    ph, pl = two_prod(X1J, lam[J][None, :])
    Rh, Rl = dd_add(Vh, Vl, -ph, -pl)
    Wh, Wl = _clib.dd_gemm_nt(np.ascontiguousarray(X1.T), np.ascontiguousarray(Rh.T), None,
                              np.ascontiguousarray(Rl.T))
    dl = lam[J][None, :] - lam[:, None]
    E = np.where(dl != 0, Wh / np.where(dl != 0, dl, 1.0), 0.0)
    E[J, np.arange(nl)] = (rh + rl) / 2
    Uh, Ul = _clib.dd_gemm_nt(X1, np.ascontiguousarray(E.T))
    s, e = two_sum(X1J, Uh)
    return fast_two_sum(s, e + Ul)[0], lam
