"""§8(f) rank 2: the paper's two β rules (§4.1 tuned ⌊·⌋ with nδ — default — vs §3.3 eq. proposed_beta
⌈·⌉ with ξ) and the θ of δ' = δ/θ: sweeps, device time to the stop rule and final forward error / δ
against the oracle reference, on the GPU (dev study for DESIGN.md)."""
import sys, time
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import numpy as np, torch, workloads as W
from gpu_util import to_dev, to_np, vec_dev
import paper_2602_19090_b200 as ozr
from oracle import refine as orf
ctx = ozr.Context(0)
cases = [('c1', 100, 'fp64', 1e-15), ('c2', 1024, 'fp64', 1e-14), ('c3', 1024, 'fp64', 1e-12),
         ('c4p', 2048, 'fp64', 1e-12), ('c4p', 2048, 'fp64', 1e-8)]
for cfg, n, start, delta in cases:
    c = W.CONFIGS[cfg]
    A, _ = W.make_matrix(n, c['kind'], c['cnd'], c['seed'])
    lam0, X0 = W.initial_eig(A, start)
    lr, Xr = W.initial_eig(A, 'fp64')
    Xh, Xl, lh, ll, _ = orf.reference_eigvecs(A, Xr, lr)
    Ad = to_dev(A)
    rows = []
    for bm, xi, th in [(0, 0, 1.0), (0, 0, 4.0), (1, 1, 1.0), (1, 0, 1.0), (1, 0, 4.0)]:
        Xd, ld = to_dev(X0), vec_dev(lam0)
        p = ozr.default_params(delta=delta, beta_mode=bm, xi=float(xi), theta=th, max_sweeps=10)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        st, hist = ozr.ozr_refine_to_tol(ctx, Ad, Xd, ld, p)
        torch.cuda.synchronize()
        ms = (time.perf_counter() - t0) * 1e3
        fe = orf.forward_error(Xh, Xl, to_np(Xd), lh, to_np(ld))
        rows.append(dict(beta_mode=bm, xi=xi if bm else n, theta=th, status=st, sweeps=len(hist),
                         betas=[h['beta'] for h in hist], ms=round(ms, 2), fe_over_delta=round(fe / delta, 3)))
    print(cfg, n, delta)
    for r in rows:
        print('   ', r, flush=True)
