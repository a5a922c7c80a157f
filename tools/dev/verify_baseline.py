"""Oracle-verified status and forward error of ozr_refine_to_tol on a BASELINE recipe at its stated size.

The problem is built with the GPU recipe (workloads.make_config_torch), refined by the library with DEFAULT
parameters (device time of the whole call, A split included), and its forward error ‖X − X̂‖₂ (and that of every
intermediate sweep, ozr_refine_step one sweep at a time) is measured against the oracle's double-double
reference eigenvectors of the stored A (oracle/refine.reference_eigvecs from an FP64 LAPACK start, with its
Rayleigh–Ritz branch for pairs outside the linear regime), whose own error is bounded by its sampled residual
certificate ‖A x_j − λ_j x_j‖/gap_j. Usage: python tools/dev/verify_baseline.py <config> [n] > out.json"""
import json
import sys
import time

sys.path.insert(0, "/root/repo")
import numpy as np
import torch

import paper_2602_19090_b200 as ozr
import workloads as W
from oracle import _clib
from oracle import refine as orf
from oracle.fp import dd_add, two_prod

name = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else None
dev = torch.device("cuda", 0)
A, lam0, X0, cfg = W.make_config_torch(name, dev, n=n)
n = cfg["n"]
delta = cfg["delta"]
ctx = ozr.Context(0)
out = {"config": name, "n": n, "delta": delta, "workload": cfg}
# the library's stop rule, timed (second run: the first grows the workspace)
for rep_ in range(2):
    X = ozr.colmajor(X0.clone())
    lam = lam0.clone()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    st, hist = ozr.ozr_refine_to_tol(ctx, A, X, lam, ozr.default_params(delta=delta))
    e1.record()
    torch.cuda.synchronize()
out["refine_to_tol"] = {"status": int(st), "sweeps": len(hist), "ms": e0.elapsed_time(e1),
                        "cert": [h["cert"] for h in hist], "theta": [h["theta"] for h in hist],
                        "max_cluster": [h["max_cluster"] for h in hist]}
X_final, lam_final = X.cpu().numpy(), lam.cpu().numpy()
# every sweep of the same iteration (ozr_refine_step, the driver's θ schedule replayed)
Xs = ozr.colmajor(X0.clone())
ls = lam0.clone()
sweep_X = []
for h in hist:
    ozr.ozr_refine_step(ctx, A, Xs, ls, ozr.default_params(delta=delta, theta=h["theta"]))
    sweep_X.append((Xs.cpu().numpy(), ls.cpu().numpy()))
An = A.cpu().numpy()
X0n = X0.cpu().numpy()
lam0n = lam0.cpu().numpy()
ctx.close()
del A, X0, X, Xs
torch.cuda.empty_cache()
t0 = time.time()
w, V = np.linalg.eigh(An)  # FP64 LAPACK start of the reference (the reference is a property of A alone)
Xh, Xl, lh, ll, rh = orf.reference_eigvecs(An, V, w, tol=1e-24, max_sweeps=8, cluster_kappa=2.0 ** -10)
out["reference"] = {"seconds": time.time() - t0, "normE_per_iteration": rh, "threads": _clib.num_threads()}
J = np.unique(np.linspace(0, n - 1, 16).astype(np.int64))
XJh, XJl = np.ascontiguousarray(Xh[:, J]), np.ascontiguousarray(Xl[:, J])
Vh, Vl = _clib.dd_gemm_nt(An, np.ascontiguousarray(XJh.T), None, np.ascontiguousarray(XJl.T))
ph, pl = two_prod(XJh, lh[J][None, :])
pl = pl + XJl * lh[J][None, :] + XJh * ll[J][None, :]
Rh, Rl = dd_add(Vh, Vl, -ph, -pl)
res = np.sqrt(np.sum((Rh + Rl) ** 2, axis=0))
gaps = np.array([np.min(np.abs(np.delete(lh, j) - lh[j])) for j in J])
out["reference_certificate"] = {"columns": J.tolist(), "sin_theta_bound_max": float(np.max(res / gaps))}
PI = None if n <= 2048 else 300  # exact 2-norm (SVD) up to 2048, else 300 power iterations on DᵀD
out["forward_error_start"] = orf.forward_error(Xh, Xl, X0n, lh, lam0n, power_iters=PI)
out["forward_error_per_sweep"] = [orf.forward_error(Xh, Xl, Xk, lh, lk, power_iters=PI) for Xk, lk in sweep_X]
fe = orf.forward_error(Xh, Xl, X_final, lh, lam_final, power_iters=PI)
out["forward_error_returned"] = fe
out["fe_over_delta"] = fe / delta
out["ok_implies_within_delta"] = bool(st != 0 or fe <= delta)
print(json.dumps(out))
