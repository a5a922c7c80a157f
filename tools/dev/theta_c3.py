"""θ needed for ‖X − X̂‖ ≤ δ on the clustered c3 spectrum (64 clusters of 8 at 1e-10 for n = 4096, n/64 at
smaller n): final forward error / δ vs θ (dev study for DESIGN.md R11)."""
import sys, time
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import numpy as np, torch, workloads as W
from gpu_util import to_dev, to_np, vec_dev
import paper_2602_19090_b200 as ozr
from oracle import refine as orf
ctx = ozr.Context(0)
for n in [int(a) for a in sys.argv[1:]] or [1024, 2048]:
    c = W.CONFIGS['c3']
    A, _ = W.make_matrix(n, c['kind'], c['cnd'], c['seed'])
    lam0, X0 = W.initial_eig(A, 'fp64')
    t = time.time()
    Xh, Xl, lh, ll, hh = orf.reference_eigvecs(A, X0, lam0)
    print('ref', n, round(time.time() - t, 1), 's', hh[-2:], flush=True)
    Ad = to_dev(A)
    for th in (4.0, 8.0, 16.0, 32.0, 64.0):
        Xd, ld = to_dev(X0), vec_dev(lam0)
        st, hist = ozr.ozr_refine_to_tol(ctx, Ad, Xd, ld, ozr.default_params(delta=1e-12, theta=th, max_sweeps=10))
        fe = orf.forward_error(Xh, Xl, to_np(Xd), lh, to_np(ld))
        print('  n', n, 'theta', th, 'status', st, 'sweeps', len(hist), 'beta', hist[0]['beta'],
              'pairs', sum(h['pairs_V'] + h['pairs_W'] + h['pairs_U'] for h in hist), 'fe/delta', round(fe / 1e-12, 3),
              flush=True)
