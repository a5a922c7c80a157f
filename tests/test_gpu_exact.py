"""Forward error at BASELINE sizes against EXACTLY known eigenvectors (north star: "forward error ‖X − X̂‖₂ … at or
below the prescribed target"; PAPER.md:48-50, 2-norm per PAPER.md:121).

W.hadamard_exact builds A = Q diag(λ) Q with Q = H S H / n and integer λ entirely in int64: A is exactly
representable in fp64, its eigenvalues are exactly λ and its eigenvectors exactly the columns of Q (pinned in Python
integers by tests/test_abi_workloads.py; the oracle driver is pinned on the same family at n = 128 by
tests/test_oracle_products_refine.py). So the forward error of the library's result needs no computed reference at
any n: D = X̂·diag(±1) − Q is formed entrywise and ‖D‖₂ measured (σ_max through eigvalsh(DᵀD) with torch on the
GPU — measurement only, a library routine outside the product path).

The start X̂₀ is an LAPACK-type eigensolver's output (torch.linalg.eigh on the device, fp64, or fp32 on fl32(A)),
as in BASELINE.json's recipes. ozr_refine_to_tol must return OZR_OK ⇒ forward error ≤ δ, its certificate must not
under-estimate the exact forward error by more than the safety factor, and λ̂ must match the exact integers."""
import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

U = 2.0 ** -53

# m (n = 2^m), spectrum, start, δ — c3's structure and size (clusters of 8, relative separation 2^-28 — the tightest
# that keeps A exact), an FP32 start whose lower spectrum is unresolved (large groups → the dense sub-solve), and the
# headline size n = 8192 from an FP64 start (c4') and from an FP32 start at c4's δ = 1e-10 (c4's structure: the lower
# spectrum is unresolved in FP32, thousands of columns in one group)
CASES = [(12, "clustered", "fp64", 1e-12), (11, "geometric", "fp32", 1e-12), (13, "geometric", "fp64", 1e-12),
         (13, "geometric", "fp32", 1e-10)]


def _start(A, start):
    import torch
    Ad = torch.from_numpy(A).cuda()
    if start == "fp32":
        lam, X = torch.linalg.eigh(Ad.float())
        lam, X = lam.double(), X.double()
    else:
        lam, X = torch.linalg.eigh(Ad)
    return Ad, lam.contiguous(), X


def _norm2(D):
    import torch
    return float(torch.sqrt(torch.linalg.eigvalsh(D.T @ D)[-1].clamp_min(0.0)))


@pytest.mark.parametrize("m,kind,start,delta", CASES)
def test_refine_to_tol_forward_error_against_exact_eigenvectors(ctx, m, kind, start, delta):
    import torch

    import paper_2602_19090_b200 as ozr
    import workloads as W
    A, lam, X = W.hadamard_exact(m, kind, seed=100 + m)
    n = 2 ** m
    Ad, l0, X0 = _start(A, start)
    Xe = torch.from_numpy(X).cuda()
    sg0 = torch.sign(torch.sum(X0 * Xe, dim=0))
    fe0 = _norm2(X0 * sg0[None, :] - Xe)       # the start's own forward error (it must be the library that fixes it)
    Xd = ozr.colmajor(X0.clone())
    ld = l0.clone()
    st, hist = ozr.ozr_refine_to_tol(ctx, ozr.colmajor(Ad), Xd, ld, ozr.default_params(delta=delta))
    assert st == 0, hist
    p = torch.argsort(ld, stable=True)
    Xr, lr = Xd[:, p], ld[p]
    sg = torch.sign(torch.sum(Xr * Xe, dim=0))
    assert bool(torch.all(sg != 0))
    fe = _norm2(Xr * sg[None, :] - Xe)
    assert fe0 > 10 * delta, (fe0, delta)       # the case is not trivial
    assert fe <= delta, (fe, fe0, hist)
    # the certificate that stopped the driver does not under-estimate the exact forward error (×1.15 safety)
    assert hist[-1]["cert"] * 1.15 >= fe - 4 * U, (fe, hist[-1])
    # λ̂ against the exact eigenvalues, relative to ‖A‖ (north star: ≤ 1e-13‖A‖)
    dl = float(torch.max(torch.abs(lr - torch.from_numpy(lam).cuda())))
    assert dl <= 1e-13 * float(np.max(np.abs(lam))), dl
    # orthogonality of the returned basis
    G = Xr.T @ Xr
    assert float(torch.max(torch.abs(G - torch.eye(n, device=G.device, dtype=G.dtype)))) <= max(4 * delta, 1e-13)
    print(f"exact-eigenvector check n={n} {kind} {start}: start fe {fe0:.2e} -> {fe:.2e} (delta {delta:g}, "
          f"cert {hist[-1]['cert']:.2e}, {len(hist)} sweeps, max|dlam| {dl:.1e})")


def test_refine_to_tol_soundness_scan_exact_family(ctx):
    """OZR_OK ⇒ ‖X − X̂‖₂ ≤ δ (+ the closed form's own ≈ 4u) over a grid of the exactly-known family at n = 256
    (geometric / clustered spectra, FP64 / FP32 starts, δ from 1e-8 to 1e-14, two seeds), every case converging; the
    stopping certificate never below the exact forward error by more than its safety factor."""
    import torch

    import paper_2602_19090_b200 as ozr
    import workloads as W
    worst = 0.0
    for kind in ("geometric", "clustered"):
        for start in ("fp64", "fp32"):
            for delta in (1e-8, 1e-12, 1e-14):
                for seed in (41, 42):
                    A, lam, X = W.hadamard_exact(8, kind, seed=seed)
                    Ad, l0, X0 = _start(A, start)
                    Xe = torch.from_numpy(X).cuda()
                    Xd, ld = ozr.colmajor(X0.clone()), l0.clone()
                    st, hist = ozr.ozr_refine_to_tol(ctx, ozr.colmajor(Ad), Xd, ld, ozr.default_params(delta=delta))
                    assert st == 0, (kind, start, delta, seed, hist)
                    p = torch.argsort(ld, stable=True)
                    Xr = Xd[:, p]
                    sg = torch.sign(torch.sum(Xr * Xe, dim=0))
                    fe = float(torch.linalg.matrix_norm(Xr * sg[None, :] - Xe, ord=2))
                    assert fe <= delta + 4 * U, (kind, start, delta, seed, fe, hist[-1])
                    assert hist[-1]["cert"] * 1.15 >= fe - 4 * U, (kind, start, delta, seed, fe, hist[-1])
                    worst = max(worst, fe / delta)
    print(f"exact-family scan: worst forward error / delta = {worst:.3f}")
