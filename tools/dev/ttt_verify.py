"""Time-to-target at n = 8192 verified against the ORACLE (SURVEY §8(d) "first hit"): the c4' problem
(n = 8192, cnd 1e10, FP64 eigensolver start, δ = 1e-12) is refined on the GPU with 1, 2, 3 sweeps (each
run from X̂₀, device time of the whole ozr_refine_to_tol call, A split included), and the forward error
‖X − X̂_k‖₂ of each result is measured against the oracle's reference eigenvectors of the stored A (dd
Ogita–Aishima iteration from the LAPACK start, oracle/refine.reference_eigvecs, on the host cores), with the
reference's own residual certificate (‖A x_j − λ_j x_j‖/gap_j in dd) on sampled columns.
Runs ~1 h of host time at n = 8192. Usage: python tools/dev/ttt_verify.py [n]"""
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

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
dev = torch.device("cuda", 0)
A, lam0, X0, cfg = W.make_config_torch("c4p", dev, n=n)
delta = cfg["delta"]
ctx = ozr.Context(0)
out = {"config": "c4p", "n": n, "delta": delta, "runs": []}
Xk = {}
for k in (1, 2, 3):
    for rep_ in range(2):  # the second run is timed (the first warms the context's workspace)
        X = ozr.colmajor(X0.clone())
        lam = lam0.clone()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        st, hist = ozr.ozr_refine_to_tol(ctx, A, X, lam, ozr.default_params(delta=delta, max_sweeps=k))
        e1.record()
        torch.cuda.synchronize()
    Xk[k] = (X.cpu().numpy(), lam.cpu().numpy())
    out["runs"].append({"sweeps": k, "ms": e0.elapsed_time(e1), "status": int(st),
                        "net_update": [h["net_update"] for h in hist]})
# the library's own stop
X = ozr.colmajor(X0.clone())
lam = lam0.clone()
st, hist = ozr.ozr_refine_to_tol(ctx, A, X, lam, ozr.default_params(delta=delta))
out["self_certified_sweeps"] = len(hist)
An, X0n, l0n = A.cpu().numpy(), X0.cpu().numpy(), lam0.cpu().numpy()
ctx.close()
del A, X0, X
torch.cuda.empty_cache()

t0 = time.time()
Xh, Xl, lh, ll, refhist = orf.reference_eigvecs(An, X0n, l0n, tol=1e-20, max_sweeps=4)
out["reference"] = {"seconds": time.time() - t0, "normE_per_iteration": refhist, "threads": _clib.num_threads()}
# certificate on sampled columns: sin θ_j ≤ ‖A x_j − λ_j x_j‖ / gap_j (Davis–Kahan), residual in dd
J = np.array([0, 1, 2, n // 2, n - 2, n - 1])
XJh, XJl = np.ascontiguousarray(Xh[:, J]), np.ascontiguousarray(Xl[:, J])
Vh, Vl = _clib.dd_gemm_nt(An, np.ascontiguousarray(XJh.T), None, np.ascontiguousarray(XJl.T))
ph, pl = two_prod(XJh, lh[J][None, :])
pl = pl + XJl * lh[J][None, :] + XJh * ll[J][None, :]
Rh, Rl = dd_add(Vh, Vl, -ph, -pl)
res = np.sqrt(np.sum((Rh + Rl) ** 2, axis=0))
ls = np.sort(lh)
gaps = np.array([np.min(np.abs(np.delete(lh, j) - lh[j])) for j in J])
out["reference_certificate"] = {"columns": J.tolist(), "residual": res.tolist(), "sin_theta_bound": (res / gaps).tolist()}
for r in out["runs"]:
    Xr, lr = Xk[r["sweeps"]]
    r["forward_error"] = orf.forward_error(Xh, Xl, Xr, lh, lr)
    r["fe_over_delta"] = r["forward_error"] / delta
out["forward_error_start"] = orf.forward_error(Xh, Xl, X0n, lh, l0n)
hit = [r for r in out["runs"] if r["forward_error"] <= delta]
out["first_hit"] = {"sweeps": hit[0]["sweeps"], "ms": hit[0]["ms"]} if hit else None
print(json.dumps(out))
