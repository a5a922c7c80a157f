"""GPU parity: ozr_split (CUDA) vs the oracle's same-definition splitting — bit-exact digits,
exponents and X̂^(1) (§2.3 eq. tau/x, R4-R6)."""
import numpy as np
import pytest

from gpu_util import to_dev, to_np
from oracle import split as osp
import workloads as W

pytestmark = pytest.mark.gpu


def _eigvec_like(n, m, seed):
    rng = np.random.default_rng(seed)
    Q = W.haar(n, rng)[:, :m]
    return Q + rng.standard_normal((n, m)) * 1e-9


@pytest.mark.parametrize("n,m,beta", [(100, 100, 15), (300, 257, 10), (1024, 64, 2), (129, 33, 30), (64, 5, 52)])
def test_x1_split_bit_exact(ctx, n, m, beta):
    import paper_2602_19090_b200 as ozr
    X = _eigvec_like(n, m, seed=n + beta)
    X[:, 0] *= 2.0 ** -40          # tiny column
    if m > 2:
        X[:, 2] = 0.0              # zero column
        X[3, 1] = 0.5               # power-of-two column max
        X[:, 1] = np.clip(X[:, 1], -0.5, 0.5)
    dig, g, k, X1 = ozr.ozr_split(ctx, to_dev(X), beta, ozr.OZR_COLWISE, ozr.OZR_SPLIT_X1, want_x1=True)
    D_o, g_o, X1_o, _ = osp.split_digits_x1(X, beta)
    assert k == osp.kx_for_beta(beta)
    assert np.array_equal(to_np(X1), X1_o)
    assert np.array_equal(to_np(g), g_o.astype(np.int32))
    dg = to_np(dig)[:, :, :n]
    assert np.array_equal(dg, D_o.transpose(0, 2, 1))


@pytest.mark.parametrize("rows,cols,k", [(100, 100, 15), (257, 130, 1), (1000, 77, 7), (64, 64, 12)])
def test_fixed_split_cols_bit_exact(ctx, rows, cols, k):
    import paper_2602_19090_b200 as ozr
    rng = np.random.default_rng(rows * k)
    M = rng.standard_normal((rows, cols)) * np.exp(rng.uniform(-30, 5, (1, cols)))
    M[:, 3] = 0.0
    M[5, 4] = 2.0 ** 7  # exact power of two as column max
    dig, ell, kk, _ = ozr.ozr_split(ctx, to_dev(M), k)
    D_o, ell_o = osp.split_digits_cols(M, k)
    assert kk == k
    assert np.array_equal(to_np(ell), ell_o.astype(np.int32))
    assert np.array_equal(to_np(dig)[:, :, :rows], D_o.transpose(0, 2, 1))


def test_fixed_split_dd_bit_exact(ctx):
    import paper_2602_19090_b200 as ozr
    rng = np.random.default_rng(7)
    rows, cols, k = 300, 40, 13
    Mh = rng.standard_normal((rows, cols)) * 1e-9
    Ml = Mh * 2.0 ** -53 * rng.uniform(-1, 1, (rows, cols))
    Mh2 = Mh + Ml
    Ml2 = (Mh - Mh2) + Ml  # normalised double-double
    dig, ell, _, _ = ozr.ozr_split(ctx, to_dev(Mh2), k, M_lo=to_dev(Ml2))
    D_o, ell_o = osp.split_digits_cols(Mh2, k, Ml2)
    assert np.array_equal(to_np(ell), ell_o.astype(np.int32))
    assert np.array_equal(to_np(dig)[:, :, :rows], D_o.transpose(0, 2, 1))


def test_rowwise_split_bit_exact(ctx):
    import paper_2602_19090_b200 as ozr
    rng = np.random.default_rng(11)
    M = rng.standard_normal((150, 333)) * np.exp(rng.uniform(-10, 10, (150, 1)))
    dig, ell, _, _ = ozr.ozr_split(ctx, to_dev(M), 9, ozr.OZR_ROWWISE)
    D_o, ell_o = osp.split_digits_cols(M.T, 9)
    assert np.array_equal(to_np(ell), ell_o.astype(np.int32))
    assert np.array_equal(to_np(dig)[:, :, :333], D_o.transpose(0, 2, 1))


def test_split_errors(ctx):
    import paper_2602_19090_b200 as ozr
    M = np.ones((32, 8))
    M[3, 3] = np.nan
    with pytest.raises(ozr.OzrError) as e:
        ozr.ozr_split(ctx, to_dev(M), 4)
    assert e.value.status == 2
    with pytest.raises(ozr.OzrError) as e:
        ozr.ozr_split(ctx, to_dev(np.ones((8, 8))), 16)
    assert e.value.status == 3
    with pytest.raises(ozr.OzrError) as e:
        ozr.ozr_split(ctx, to_dev(np.ones((8, 8))), 1, ozr.OZR_COLWISE, ozr.OZR_SPLIT_X1)
    assert e.value.status == 3
