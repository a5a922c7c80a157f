"""workloads — seeded synthetic inputs shared by the tests, the bench and the oracle.

Holds NONE of the method's arithmetic (no splitting, no products beyond forming the test matrix,
no refinement): it only builds A = Q·diag(λ)·Qᵀ like the paper's test matrices and the initial
approximation X̂₀ from an LAPACK eigensolver, exactly as BASELINE.json's configs describe them.

PAPER.md:447 `gallery('randsvd',n,-cnd,3,n-1,n-1,1)`: mode 3 = geometric singular values
σ_i = cnd^{-(i-1)/(n-1)}, negative cnd = symmetric positive definite, full bandwidth. MATLAB's PRNG
stream cannot be reproduced, so Q is a Haar orthogonal matrix from numpy's PCG64 (QR of a seeded
N(0,1) matrix, columns multiplied by sign(diag R)); A is formed in fp64 and symmetrised as
(A + Aᵀ)/2. The reference solution is always the eigensystem of the STORED A.
"""
import numpy as np

# BASELINE.json configs (c1..c5): n, spectrum, start precision, target δ
CONFIGS = {
    "c1": dict(n=100, kind="geometric", cnd=1e8, start="fp64", delta=1e-15, seed=1001),
    "c2": dict(n=1024, kind="geometric", cnd=1e12, start="fp32", delta=1e-14, seed=1002),
    "c3": dict(n=4096, kind="clustered", cnd=None, start="fp64", delta=1e-12, seed=1003),
    "c4": dict(n=8192, kind="geometric", cnd=1e14, start="fp32", delta=1e-10, seed=1004),
    "c5": dict(n=16384, kind="geometric", cnd=1e10, start="fp64", delta=1e-15, seed=1005),
    # c4': the paper's own Fig. 4(h-j) setting at n = 8192 (cnd 1e10, FP64 eig start, δ = 1e-12)
    "c4p": dict(n=8192, kind="geometric", cnd=1e10, start="fp64", delta=1e-12, seed=1014),
}


def haar(n, rng):
    """Haar orthogonal Q: QR of N(0,1)^{n×n}, columns times sign(diag R)."""
    G = rng.standard_normal((n, n))
    Q, R = np.linalg.qr(G)
    return Q * np.sign(np.diag(R))[None, :]


def geometric_spectrum(n, cnd):
    """λ_i = cnd^{-(i-1)/(n-1)}, i = 1..n (randsvd mode 3): λ_max = 1, λ_min = 1/cnd."""
    i = np.arange(n, dtype=np.float64)
    return cnd ** (-i / max(n - 1, 1))


def clustered_spectrum(n, rng, nclusters=None, csize=8, sep=1e-10):
    """BASELINE.json c3: λ uniform in [−1, 1] with `nclusters` clusters of `csize` eigenvalues
    separated by `sep`: n − nclusters·csize singletons plus nclusters anchors c drawn U[−1, 1], each
    anchor expanded to {c + m·sep, m = 0..csize−1}. nclusters defaults to 64 at n = 4096 (the
    config) and n/64 at other sizes (so 1/8 of the spectrum is clustered at every n)."""
    if nclusters is None:
        nclusters = max(1, n // 64)
    nsingle = n - nclusters * csize
    draws = rng.uniform(-1.0, 1.0, nsingle + nclusters)
    anchors = draws[:nclusters]
    lam = list(draws[nclusters:])
    for c in anchors:
        lam.extend(c + sep * np.arange(csize))
    return np.sort(np.array(lam))


def make_matrix(n, kind="geometric", cnd=1e10, seed=0):
    """A = fl(Q diag(λ) Qᵀ), symmetrised. Returns (A, λ_design)."""
    rng = np.random.default_rng(seed)
    if kind == "geometric":
        lam = geometric_spectrum(n, cnd)
    elif kind == "clustered":
        lam = clustered_spectrum(n, rng)
    else:
        raise ValueError(kind)
    Q = haar(n, rng)
    A = (Q * lam[None, :]) @ Q.T
    A = (A + A.T) * 0.5
    return np.ascontiguousarray(A), lam


def sign_fix(X):
    """Make the largest-|entry| of every column positive (lowest index on ties)."""
    idx = np.argmax(np.abs(X), axis=0)
    s = np.sign(X[idx, np.arange(X.shape[1])])
    s[s == 0] = 1.0
    return X * s[None, :]


def initial_eig(A, start="fp64"):
    """X̂₀, λ̂₀ from LAPACK (numpy.linalg.eigh = syevd): in fp64, or in fp32 on fl32(A) and cast
    back (BASELINE.json c2/c4 'mixed-precision start'). Ascending λ, sign-fixed columns."""
    if start == "fp64":
        lam, X = np.linalg.eigh(A)
    elif start == "fp32":
        lam, X = np.linalg.eigh(A.astype(np.float32))
        lam, X = lam.astype(np.float64), X.astype(np.float64)
    else:
        raise ValueError(start)
    return lam, np.ascontiguousarray(sign_fix(X))


def make_config(name, n=None):
    """(A, λ̂₀, X̂₀, cfg) for a named BASELINE config (optionally at a smaller n, same recipe)."""
    cfg = dict(CONFIGS[name])
    if n is not None:
        cfg["n"] = n
    A, _ = make_matrix(cfg["n"], cfg["kind"], cfg["cnd"], cfg["seed"])
    lam0, X0 = initial_eig(A, cfg["start"])
    return A, lam0, X0, cfg


def make_config_torch(name, device, n=None, seed_offset=0):
    """Same recipe as make_config, built on the GPU with torch (fp64 QR / GEMM / syevd via cuSOLVER)
    so that n = 8192..16384 inputs take seconds. Returns column-major CUDA tensors
    (A, λ̂₀, X̂₀) and cfg. The N(0,1) matrix comes from numpy's PCG64 with the config seed."""
    import torch
    cfg = dict(CONFIGS[name])
    if n is not None:
        cfg["n"] = n
    n = cfg["n"]
    rng = np.random.default_rng(cfg["seed"] + seed_offset)
    if cfg["kind"] == "geometric":
        lam = geometric_spectrum(n, cfg["cnd"])
        G = rng.standard_normal((n, n))
    else:
        lam = clustered_spectrum(n, rng)
        G = rng.standard_normal((n, n))
    Gt = torch.from_numpy(G).to(device)
    del G
    Q, R = torch.linalg.qr(Gt)
    del Gt
    Q = Q * torch.sign(torch.diagonal(R))[None, :]
    del R
    lt = torch.from_numpy(lam).to(device)
    A = (Q * lt[None, :]) @ Q.T
    del Q
    A = (A + A.T) * 0.5
    if cfg["start"] == "fp64":
        lam0, X0 = torch.linalg.eigh(A)
    else:
        lam0, X0 = torch.linalg.eigh(A.float())
        lam0, X0 = lam0.double(), X0.double()
    idx = torch.argmax(X0.abs(), dim=0)
    s = torch.sign(X0[idx, torch.arange(n, device=device)])
    s[s == 0] = 1.0
    X0 = X0 * s[None, :]
    colmajor = lambda t: t.t().contiguous().t()  # noqa: E731
    return colmajor(A), lam0.contiguous(), colmajor(X0), cfg


def banded_sym(n, layers=4, cnd=1e8, seed=0):
    """Sparse stand-in for the paper's ELSES matrices (the collection is not in the
    container): A = Q·diag(λ)·Qᵀ with geometric λ and Q a product of `layers` layers of disjoint 2x2 Givens
    rotations with seeded angles — odd layers on the pairs (0,1), (2,3), …, even layers on (1,2), (3,4), … —
    so Q has bandwidth `layers` and A bandwidth 2·layers: at most k = 4·layers + 1 nonzeros per row. A is
    formed in fp64, entries outside the band are exact zeros, symmetrised as (A + Aᵀ)/2.
    Returns (A, λ, k) with k the realised largest number of nonzeros in a row."""
    rng = np.random.default_rng(seed)
    lam = geometric_spectrum(n, cnd)
    Q = np.eye(n)
    for l in range(layers):
        i0 = l % 2
        for i in range(i0, n - 1, 2):
            t = rng.uniform(0.0, 2.0 * np.pi)
            c, s = np.cos(t), np.sin(t)
            qi, qj = Q[:, i].copy(), Q[:, i + 1].copy()
            Q[:, i], Q[:, i + 1] = c * qi - s * qj, s * qi + c * qj
    A = (Q * lam[None, :]) @ Q.T
    bw = 2 * layers
    ii, jj = np.indices((n, n))
    A[np.abs(ii - jj) > bw] = 0.0
    A = (A + A.T) * 0.5
    return A, lam, int((A != 0).sum(axis=1).max())


def householder_exact(m, lam_bits=12, seed=0):
    """Pin family: n = 2^m, v ∈ {±1}^n, H = I − (2/n) v vᵀ (exactly orthogonal,
    symmetric, dyadic). λ_k = distinct dyadic numbers with `lam_bits`-bit numerators in (0, 1].
    A = H diag(λ) H is then exactly representable for moderate n and lam_bits, and its exact
    eigenvectors are the columns of H. Returns (A, λ ascending, X exact (columns of H, sign-fixed,
    ordered by λ))."""
    n = 2 ** m
    rng = np.random.default_rng(seed)
    v = rng.choice([-1.0, 1.0], size=n)
    H = np.eye(n) - (2.0 / n) * np.outer(v, v)
    nums = rng.choice(np.arange(1, 2 ** lam_bits), size=n, replace=False)
    lam = np.sort(nums.astype(np.float64) / 2 ** lam_bits)
    order = rng.permutation(n)
    lam_cols = np.empty(n)
    lam_cols[order] = lam  # column order[k] of H carries λ_k
    A = (H * lam_cols[None, :]) @ H
    X = H[:, order]
    return A, lam, sign_fix(X), H, lam_cols


def pivot_2x2(theta):
    """A = diag(1, 2) and X̂ = rotation by θ (SPEC-style closed form)."""
    A = np.diag([1.0, 2.0])
    c, s = np.cos(theta), np.sin(theta)
    X = np.array([[c, -s], [s, c]])
    return A, X


def householder_pair(m=6, pair=(10, 11), split=0.0, angle=0.0, noise=1e-9, lam_bits=12, seed=3):
    """Householder-exact family with a designed pair: λ_b = λ_a + `split` (split = 0: an exactly
    double eigenvalue; a dyadic split keeps A exact), A = X diag(λ) Xᵀ with the exact eigenvectors X
    (columns of H). The start X̂₀ rotates the pair's two exact eigenvectors by `angle` (radians) and adds
    seeded N(0, noise²) entries. Returns (A, λ, X exact, X̂₀)."""
    A0, lam, X, H, lam_cols = householder_exact(m, lam_bits=lam_bits, seed=seed)
    a, b = pair
    lam = lam.copy()
    lam[b] = lam[a] + split
    A = (X * lam[None, :]) @ X.T
    X0 = X.copy()
    c, s = np.cos(angle), np.sin(angle)
    X0[:, a], X0[:, b] = c * X[:, a] - s * X[:, b], s * X[:, a] + c * X[:, b]
    X0 = X0 + noise * np.random.default_rng(seed + 4).standard_normal(X.shape)
    return A, lam, X, X0


# ---------------------------------------------------------------- Hermitian extension (reading R18)
def haar_unitary(n, rng):
    """Haar unitary Q: QR of a complex N(0,1) matrix (real and imaginary parts N(0, ½)), columns times the
    phase of diag R."""
    G = (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))) / np.sqrt(2.0)
    Q, R = np.linalg.qr(G)
    d = np.diag(R)
    return Q * (d / np.abs(d))[None, :]


def make_hermitian(n, kind="geometric", cnd=1e10, seed=0):
    """A = Q diag(λ) Qᴴ with Haar unitary Q and the same spectra as make_matrix, Hermitian-symmetrised as
    (A + Aᴴ)/2. Returns (Ar, Ai, λ_design) — real and imaginary parts as separate fp64 arrays (Ar symmetric,
    Ai antisymmetric with a zero diagonal)."""
    rng = np.random.default_rng(seed)
    if kind == "geometric":
        lam = geometric_spectrum(n, cnd)
    elif kind == "clustered":
        lam = clustered_spectrum(n, rng)
    else:
        raise ValueError(kind)
    Q = haar_unitary(n, rng)
    A = (Q * lam[None, :]) @ Q.conj().T
    A = (A + A.conj().T) * 0.5
    return np.ascontiguousarray(A.real), np.ascontiguousarray(A.imag), lam


def phase_fix(X):
    """Multiply every column by the unit phase that makes its largest-modulus entry (lowest index on ties) real
    and positive (the complex analogue of sign_fix)."""
    idx = np.argmax(np.abs(X), axis=0)
    p = X[idx, np.arange(X.shape[1])]
    ph = np.where(np.abs(p) > 0, np.conj(p) / np.where(np.abs(p) > 0, np.abs(p), 1.0), 1.0)
    return X * ph[None, :]


def initial_eig_herm(Ar, Ai, start="fp64"):
    """X̂₀, λ̂₀ of the Hermitian A from LAPACK (numpy.linalg.eigh = zheevd) in complex128, or in complex64 on
    fl32(A) and cast back. Ascending λ, phase-fixed columns. Returns (λ̂₀, Xr, Xi)."""
    A = np.asarray(Ar) + 1j * np.asarray(Ai)
    if start == "fp64":
        lam, X = np.linalg.eigh(A)
    elif start == "fp32":
        lam, X = np.linalg.eigh(A.astype(np.complex64))
        lam, X = lam.astype(np.float64), X.astype(np.complex128)
    else:
        raise ValueError(start)
    X = phase_fix(X)
    return lam, np.ascontiguousarray(X.real), np.ascontiguousarray(X.imag)


def householder_exact_herm(m, lam_bits=12, seed=0):
    """Exactly known Hermitian family (the complex analogue of householder_exact): n = 2^m, v ∈ {±1, ±i}^n,
    H = I − (2/n) v vᴴ (exactly unitary and Hermitian; every real and imaginary part is 0, ±2/n or 1 ± 2/n),
    distinct dyadic λ with `lam_bits`-bit numerators, A = H diag(λ) H — exactly representable for moderate n and
    lam_bits (checked by the caller). Returns (Ar, Ai, λ ascending, Xr, Xi exact (columns of H ordered by λ))."""
    n = 2 ** m
    rng = np.random.default_rng(seed)
    v = rng.choice(np.array([1.0, -1.0, 1j, -1j]), size=n)
    H = np.eye(n, dtype=np.complex128) - (2.0 / n) * np.outer(v, v.conj())
    nums = rng.choice(np.arange(1, 2 ** lam_bits), size=n, replace=False)
    lam = np.sort(nums.astype(np.float64) / 2 ** lam_bits)
    order = rng.permutation(n)
    lam_cols = np.empty(n)
    lam_cols[order] = lam
    A = (H * lam_cols[None, :]) @ H
    X = H[:, order]
    return np.ascontiguousarray(A.real), np.ascontiguousarray(A.imag), lam, np.ascontiguousarray(X.real), \
        np.ascontiguousarray(X.imag)


# ---------------------------------------------------------------- exactly known eigenvectors at full size
def _fwht_rows(M):
    """In-place-style fast Walsh–Hadamard transform along axis 0 (Sylvester ordering), integer arithmetic."""
    n = M.shape[0]
    h = 1
    while h < n:
        M = M.reshape(n // (2 * h), 2, h, -1)
        M = np.concatenate((M[:, 0:1] + M[:, 1:2], M[:, 0:1] - M[:, 1:2]), axis=1).reshape(n, -1)
        h *= 2
    return M


def hadamard_exact(m, kind="geometric", cnd=1e4, seed=0, lam_bits=None, pairs=True):
    """Full-size family with eigenpairs known in CLOSED FORM (no reference computation needed): n = 2^m, H the
    Sylvester Hadamard matrix, s ∈ {±1}^n seeded, Q = H diag(s) H / n (symmetric, exactly orthogonal: Q Qᵀ =
    H S (H H/n) S H/n = I; its entries are integers / n, q_ij = ŝ(i ⊕ j)/n with ŝ the Walsh transform of s), μ
    distinct INTEGERS below 2^lam_bits (default 53 − 2m − 2, so every numerator below stays under 2^53).
    pairs = False: A = Q diag(μ) Q — eigenvalues exactly μ, eigenvectors exactly the columns of Q (dyadic entries
    of a few bits: a refinement in fp64 lands ON them, forward error exactly 0).
    pairs = True (default): A = Q B Q with B the direct sum of n/2 integer blocks [[a, b], [b, c]] on seeded column
    pairs of Q, (a, c) consecutive designed μ and b = ±max(1, (c − a)//2): eigenvalues (a + c)/2 ± h,
    h = sqrt(((c − a)/2)² + b²), eigenvectors cos φ·q_1 + sin φ·q_2 and −sin φ·q_1 + cos φ·q_2 with
    (cos φ, sin φ) ∝ (b, (c − a)/2 + h)·sign — irrational, evaluated in closed form in extended precision and
    rounded once to fp64 (error ≤ u per entry and per eigenvalue: the reference is good to ≈ 2u in the 2-norm).
    Either way n² A = N B Nᵀ (N = n Q) has integer entries below 2^53: A is formed in int64 (four Walsh transforms,
    no rounding anywhere) and is exactly representable in fp64; A and λ are returned scaled by 2^-lam_bits (exact),
    so ‖A‖₂ ≤ 1.
    kind = "geometric": μ_i = round(2^lam_bits · cnd^{-(i-1)/(n-1)}) (cnd small enough that they stay distinct);
    kind = "clustered": n/64 clusters of 8 integers separated by 1 (relative separation 2^-lam_bits of ‖A‖₂; with
    pairs the cluster's eigenvalues are a + ½ ± √5/2: separations of 0.24 and 2 units) among otherwise
    16-separated integers of both signs (the BASELINE c3 structure with the tightest separation that keeps A
    exact). Returns (A, λ ascending, X (sign-fixed, columns in λ order))."""
    n = 2 ** m
    if lam_bits is None:
        lam_bits = 53 - 2 * m - 2
    rng = np.random.default_rng(seed)
    s = rng.choice(np.array([-1, 1], dtype=np.int64), size=n)
    if kind == "geometric":
        lam = np.rint(2.0 ** lam_bits * cnd ** (-np.arange(n) / max(n - 1, 1))).astype(np.int64)
    elif kind == "clustered":
        ncl = max(n // 64, 1)
        slots = 2 ** (lam_bits - 3)  # centres are multiples of 16 in (−2^lam_bits, 2^lam_bits)
        nc = n - 7 * ncl
        centres = (rng.choice(slots - 2, size=nc, replace=False).astype(np.int64) - (slots - 2) // 2) * 16
        lam = np.concatenate([centres[ncl:]] + [centres[c] + np.arange(8, dtype=np.int64) for c in range(ncl)])
    else:
        raise ValueError(kind)
    lam = np.sort(lam)
    assert lam.shape == (n,) and np.all(np.diff(lam) > 0) and np.max(np.abs(lam)) <= 2 ** lam_bits, "μ not distinct"
    # numerators of Q: N = H S H (|N_ij| ≤ n); column perm[k] of Q carries the k-th designed value
    N = _fwht_rows(_fwht_rows(np.eye(n, dtype=np.int64)) * s[:, None])
    perm = rng.permutation(n)
    B = np.zeros((n, n), dtype=np.int64)
    B[perm, perm] = lam
    if pairs:
        a, c = lam[0::2], lam[1::2]
        b = np.maximum(1, (c - a) // 2) * rng.choice(np.array([-1, 1], dtype=np.int64), size=n // 2)
        B[perm[0::2], perm[1::2]] = b
        B[perm[1::2], perm[0::2]] = b
    # n² A = N B Nᵀ = H S (H B H) S H, every intermediate an exact int64 (bounded by n^1.5 ‖B‖₂ entrywise)
    T = _fwht_rows(B)                            # H B
    T = _fwht_rows(np.ascontiguousarray(T.T))    # H B H (symmetric)
    T = T * s[:, None] * s[None, :]              # S H B H S
    T = _fwht_rows(T)
    T = _fwht_rows(np.ascontiguousarray(T.T))    # H S H B H S H
    assert np.max(np.abs(T)) < 2 ** 53
    sc = 2.0 ** -lam_bits                        # power-of-two scaling to ‖A‖₂ ≤ 1 (exact)
    A = T.astype(np.float64) / float(n) ** 2 * sc  # exact: |numerator| < 2^53, n² a power of two
    Q = N[:, perm].astype(np.float64) / float(n)
    if not pairs:
        return A, lam.astype(np.float64) * sc, sign_fix(Q)
    LD = np.longdouble
    d = (c - a).astype(LD) / 2
    bb = b.astype(LD)
    h = np.sqrt(d * d + bb * bb)
    mid = (a + c).astype(LD) / 2
    nrm = np.sqrt(bb * bb + (d + h) * (d + h))
    cphi, sphi = bb / nrm, (d + h) / nrm         # (cos φ, sin φ): eigenvector of the block for mid + h; d + h > 0
    Q1, Q2 = Q[:, 0::2].astype(LD), Q[:, 1::2].astype(LD)
    X = np.empty((n, n))
    ev = np.empty(n, dtype=LD)
    X[:, 1::2] = (Q1 * cphi[None, :] + Q2 * sphi[None, :]).astype(np.float64)   # mid + h
    X[:, 0::2] = (Q1 * sphi[None, :] - Q2 * cphi[None, :]).astype(np.float64)   # mid − h
    ev[1::2], ev[0::2] = mid + h, mid - h
    o = np.argsort(ev, kind="stable")
    ev = ev[o]
    assert np.all(np.diff(ev) > LD(0.1)), "eigenvalues of the pair blocks not separated"
    return A, (ev * LD(sc)).astype(np.float64), sign_fix(X[:, o])
