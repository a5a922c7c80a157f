"""§8(f) rank 1: the prior work's two-sided fixed-slice refinement (both A and X̂
split into the same number of slices, every product of the ½k(k+1) leading slice pairs, X̂ untruncated)
expressed as a digit plan — truncate = 0 and the pair budget s + t ≤ k + 1 forced on all three products —
against the proposed method (X̂ → X̂^(1) by §4.1's β, accuracy-driven budgets). Per case: sweeps, pair-GEMMs,
device time to the stop rule and the final forward error / δ against the oracle reference."""
import sys
import time

sys.path.insert(0, '/root/repo')
sys.path.insert(0, '/root/repo/tests')
import torch

import paper_2602_19090_b200 as ozr
import workloads as W
from gpu_util import to_dev, to_np, vec_dev
from oracle import refine as orf

ctx = ozr.Context(0)
for cfg, n, delta in [('c4p', 2048, 1e-12), ('c4p', 2048, 1e-8), ('c2', 1024, 1e-14)]:
    c = W.CONFIGS[cfg]
    A, _ = W.make_matrix(n, c['kind'], c['cnd'], c['seed'])
    lam0, X0 = W.initial_eig(A, 'fp64')
    Xh, Xl, lh, ll, _ = orf.reference_eigvecs(A, X0, lam0)
    Ad = to_dev(A)
    print(cfg, n, delta, flush=True)
    plans = [('proposed', {})] + [(f'fixed k={k}', dict(truncate=0, L_V=k + 1, L_W=k + 1, L_U=k + 1))
                                  for k in (4, 6, 8, 10, 12, 14)]
    for name, kw in plans:
        Xd, ld = to_dev(X0), vec_dev(lam0)
        p = ozr.default_params(delta=delta, max_sweeps=8, **kw)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        st, hist = ozr.ozr_refine_to_tol(ctx, Ad, Xd, ld, p)
        torch.cuda.synchronize()
        ms = (time.perf_counter() - t0) * 1e3
        fe = orf.forward_error(Xh, Xl, to_np(Xd), lh, to_np(ld))
        pairs = sum(h['pairs_V'] + h['pairs_W'] + h['pairs_U'] for h in hist)
        print(f'   {name:12s} status {st} sweeps {len(hist)} pair-GEMMs {pairs:4d} ms {ms:8.2f} '
              f'fe/delta {fe / delta:.3g}', flush=True)
