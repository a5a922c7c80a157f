"""§8(f) rank 1: the prior work's two-sided fixed-slice refinement (PAPER.md:217-227 eq. mat3-mat10, cost model
PAPER.md:437-443: n_A = n_X = k slices, the ½k(k+1) slice products s + t ≤ k + 1, X̂ untruncated) as a digit
plan of the same kernels (ozr_params.fixed_k).
 - the product: ozr_gemm(kA = kB = k, L = k + 1) bit-exact against the oracle's accmul_fixed_k (itself pinned
   against rationals in tests/test_oracle_products_refine.py);
 - the refinement: ozr_refine_to_tol with fixed_k reaches δ against the oracle reference, with every product at
   the plan's pair count; the proposed method reaches the same δ with fewer pair-GEMMs."""
import numpy as np
import pytest
import torch

import paper_2602_19090_b200 as ozr
import workloads as W
from gpu_util import to_dev, to_np, vec_dev
from oracle import products as opr
from oracle import refine as orf

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("k", [2, 3, 4, 6, 8])
def test_fixed_k_product_bit_exact(ctx, k):
    rng = np.random.default_rng(k)
    A = rng.standard_normal((300, 260)) * np.exp(rng.uniform(-8, 8, (300, 1)))
    B = rng.standard_normal((260, 130))
    hi, lo, npairs = opr.accmul_fixed_k(A, B, k)
    Ch, Cl, _ = ozr.ozr_gemm(ctx, to_dev(A), to_dev(B), k, k, k + 1)
    assert np.array_equal(to_np(Ch), hi) and np.array_equal(to_np(Cl), lo)
    assert npairs == k * (k + 1) // 2


def test_fixed_k_refinement_reaches_delta(ctx):
    A, lam0, X0, cfg = W.make_config("c4p", n=512)
    delta = cfg["delta"]
    Xh, Xl, lh, ll, _ = orf.reference_eigvecs(A, X0, lam0)
    res = {}
    for name, kw in (("proposed", {}), ("fixed_k=12", {"fixed_k": 12})):
        Xd, ld = to_dev(X0), vec_dev(lam0)
        st, hist = ozr.ozr_refine_to_tol(ctx, to_dev(A), Xd, ld, ozr.default_params(delta=delta, max_sweeps=8, **kw))
        fe = orf.forward_error(Xh, Xl, to_np(Xd), lh, to_np(ld))
        assert st == 0 and fe <= delta, (name, st, fe, hist)
        res[name] = sum(h["pairs_V"] + h["pairs_W"] + h["pairs_U"] for h in hist)
        if kw:
            for h in hist:  # X̂ untruncated (7 digits), A and the other operands ≥ 12 digits: pairs s + t ≤ 13
                assert h["L_V"] == h["L_W"] == h["L_U"] == 13
    assert res["proposed"] < res["fixed_k=12"], res
