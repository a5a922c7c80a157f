"""Memory safety without compute-sanitizer (closed on this pool): with OZR_GUARD=1 every workspace buffer of the
context carries a 4 KB guard band of a fixed pattern behind its end, and every ABI call that ran kernels checks
all of them afterwards (OZR_ERR_CUDA "guard band … overwritten" otherwise). These calls exercise every kernel
family at ragged sizes (not multiples of the 256-column tile, the 64-row tiles or 16-byte lines): the splits,
the CTA-pair tcgen05 slice GEMM, the recombinations, the certificate's bf16 GEMMs and Lanczos, the cluster
branch's Jacobi CTAs and cooperative Jacobi, the dense sub-solve with the hand-written eigensolver, and the
Hermitian sweep."""
import os

import numpy as np
import pytest

import workloads as W
from gpu_util import to_dev, vec_dev

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gctx():
    import paper_2602_19090_b200 as ozr
    old = os.environ.get("OZR_GUARD")
    os.environ["OZR_GUARD"] = "1"
    try:
        c = ozr.Context(0)
    finally:
        if old is None:
            del os.environ["OZR_GUARD"]
        else:
            os.environ["OZR_GUARD"] = old
    yield c
    c.close()


def test_guard_refine_and_certificate(gctx):
    import paper_2602_19090_b200 as ozr
    A, lam0, X0, cfg = W.make_config("c4p", n=300)
    st, hist = ozr.ozr_refine_to_tol(gctx, to_dev(A), to_dev(X0), vec_dev(lam0), ozr.default_params(delta=1e-12))
    assert st == 0 and hist[-1]["cert"] > 0


@pytest.mark.parametrize("dense", [2, 1 << 20])
def test_guard_cluster_paths(gctx, dense):
    import paper_2602_19090_b200 as ozr
    A, _ = W.make_matrix(333, "geometric", 1e12, 1002)
    lam0, X0 = W.initial_eig(A, "fp32")
    rep = ozr.ozr_refine_step(gctx, to_dev(A), to_dev(X0), vec_dev(lam0),
                              ozr.default_params(delta=1e-14, dense_cluster=dense))
    assert rep["n_clusters"] > 0


def test_guard_gemm_split_syev(gctx):
    import torch

    import paper_2602_19090_b200 as ozr
    rng = np.random.default_rng(3)
    ozr.ozr_gemm(gctx, to_dev(rng.standard_normal((301, 261))), to_dev(rng.standard_normal((261, 131))), 7, 5, 9)
    G = rng.standard_normal((301, 301))
    ozr.ozr_syev(gctx, to_dev((G + G.T) / 2))
    torch.cuda.synchronize()


def test_guard_hermitian(gctx):
    import paper_2602_19090_b200 as ozr
    Ar, Ai, _ = W.make_hermitian(157, "geometric", 1e6, seed=8)
    lam0, Xr, Xi = W.initial_eig_herm(Ar, Ai, "fp64")
    ozr.ozr_refine_step_herm(gctx, to_dev(Ar), to_dev(Ai), to_dev(Xr), to_dev(Xi), vec_dev(lam0),
                             ozr.default_params(delta=1e-12))
