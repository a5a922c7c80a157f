"""Forward error / δ after ozr_refine_to_tol for product-budget factors θ_V = θ_W = θ_U (GPU) against
the oracle reference (dev experiment for DESIGN.md R8)."""
import sys; sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import numpy as np, workloads as W
from gpu_util import to_dev, to_np, vec_dev
import paper_2602_19090_b200 as ozr
from oracle import refine as orf
ctx = ozr.Context(0)
cases = [('c1', 100, 'fp64', 1e-15), ('c2', 512, 'fp32', 1e-14), ('c2', 1024, 'fp64', 1e-14),
         ('c3', 512, 'fp32', 1e-12), ('c4p', 1024, 'fp64', 1e-12), ('c4p', 2048, 'fp64', 1e-12),
         ('c4p', 1024, 'fp64', 1e-8)]
for cfg, n, start, delta in cases:
    c = W.CONFIGS[cfg]
    A, _ = W.make_matrix(n, c['kind'], c['cnd'], c['seed'])
    lam0, X0 = W.initial_eig(A, start)
    lr, Xr = W.initial_eig(A, 'fp64')
    Xh, Xl, lh, ll, _ = orf.reference_eigvecs(A, Xr, lr)
    out = []
    for th in (1 / 16, 1 / 8, 1 / 4, 1 / 2):
        Xd, ld = to_dev(X0), vec_dev(lam0)
        st, hist = ozr.ozr_refine_to_tol(ctx, to_dev(A), Xd, ld,
                                         ozr.default_params(delta=delta, max_sweeps=12, theta_V=th, theta_W=th, theta_U=th))
        fe = orf.forward_error(Xh, Xl, to_np(Xd), lh, to_np(ld))
        pairs = sum(h['pairs_V'] + h['pairs_W'] + h['pairs_U'] for h in hist)
        out.append((th, st, len(hist), pairs, round(fe / delta, 3)))
    print(cfg, n, start, delta, out, flush=True)
