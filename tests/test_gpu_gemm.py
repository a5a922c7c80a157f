"""GPU parity: ozr_gemm (tcgen05 INT8 slice products + exact recombination) vs the oracle.
 - the int32 group planes are bit-exact vs the oracle's exact float64 digit products;
 - the double-double result is bit-exact vs the oracle's exact recombination (single-chunk plans)
   and within 2^-104 relative otherwise;
 - the product is within the dropped-digit bound of the exact product A·B (dd triple loop)."""
import numpy as np
import pytest

from gpu_util import to_dev, to_np
from oracle import _clib
from oracle import products as opr
from oracle import split as osp

pytestmark = pytest.mark.gpu


def _oracle_product(A, B, kA, kB, L):
    DA, eA = osp.split_digits_cols(A.T, kA)       # row-wise split of A = column-wise of Aᵀ (contraction first)
    DB, eB = osp.split_digits_cols(B, kB)
    return opr.digit_product(DA, eA, kA, DB, eB, kB, L)


@pytest.mark.parametrize("m,n,k,kA,kB,L", [
    (128, 256, 128, 1, 1, 0),       # one tile, one pair
    (200, 300, 1000, 4, 3, 0),      # ragged in every dimension, all pairs
    (333, 129, 777, 7, 5, 8),       # triangle pair budget
    (1024, 1024, 1024, 6, 6, 7),    # many tiles
    (32, 48, 50000, 3, 3, 0),       # pair cap: K·pairs·2^14 < 2^31 splits diagonals
])
def test_gemm_planes_and_dd_bit_exact(ctx, m, n, k, kA, kB, L):
    import paper_2602_19090_b200 as ozr
    rng = np.random.default_rng(m + n + k)
    A = rng.standard_normal((m, k)) * np.exp(rng.uniform(-5, 5, (m, 1)))
    B = rng.standard_normal((k, n)) * np.exp(rng.uniform(-5, 5, (1, n)))
    Ch, Cl, planes = ozr.ozr_gemm(ctx, to_dev(A), to_dev(B), kA, kB, L, want_planes=True)
    Lr = L if L > 0 else kA + kB
    hi, lo, P, groups = _oracle_product(A, B, kA, kB, Lr)
    plan = ozr.ozr_gemm_plan(k, kA, kB, L)
    assert plan == [(d, len(p)) for d, p in groups]
    got = to_np(planes).transpose(0, 2, 1)
    assert np.array_equal(got, P)
    assert np.array_equal(to_np(Ch), hi)
    rel = np.abs((to_np(Cl) - lo)) <= np.abs(hi) * 2.0 ** -104
    assert np.all(rel | (to_np(Cl) == lo))


def test_gemm_accuracy_vs_exact_product(ctx):
    import paper_2602_19090_b200 as ozr
    rng = np.random.default_rng(5)
    m = n = k = 512
    A = rng.standard_normal((m, k))
    B = rng.standard_normal((k, n))
    Eh, El = _clib.dd_gemm_nt(A, np.ascontiguousarray(B.T))
    for kk in (3, 7, 13):
        Ch, Cl, _ = ozr.ozr_gemm(ctx, to_dev(A), to_dev(B), kk, kk)
        err = np.max(np.abs((to_np(Ch) - Eh) + (to_np(Cl) - El)))
        # digits of a k-digit split resolve 8k-2 bits below the line maximum (R6): RN error ≤ 2^{e-S-1}
        bound = k * 2 * 2.0 ** (np.ceil(np.log2(np.abs(A).max())) - (8 * kk - 2)) * np.abs(B).max() * 2
        assert err <= bound, (kk, err, bound)
    assert err < 1e-25  # 13 digits: far beyond fp64


def test_gemm_fp64_only_output_and_args(ctx):
    import paper_2602_19090_b200 as ozr
    A = np.eye(16)
    Ch, Cl, _ = ozr.ozr_gemm(ctx, to_dev(A), to_dev(A), 2, 2, want_lo=False)
    assert Cl is None and np.array_equal(to_np(Ch), np.eye(16))
    with pytest.raises(ozr.OzrError) as e:
        ozr.ozr_gemm(ctx, to_dev(A), to_dev(A), 0, 2)
    assert e.value.status == 3
