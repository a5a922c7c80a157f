"""Oracle-verified status and forward error of ozr_refine_to_tol on a BASELINE recipe at its stated size.

Phase 2 (GPU box) of tools/dev/verify_prep.py: the problem phase 1 stored (A, X̂₀, λ̂₀) is loaded and checked
against the hashes phase 1 recorded; it is refined by the library with DEFAULT
parameters (device time of the whole call, A split included), and its forward error ‖X − X̂‖₂ (and that of
every intermediate sweep, ozr_refine_step one sweep at a time with the driver's θ schedule) is measured against
the oracle's double-double reference eigenvectors of the stored A that phase 1 computed on the CPU (its own
error bounded by its sampled residual certificate ‖A x_j − λ_j x_j‖/gap_j, in meta.json).
Usage: python tools/dev/verify_baseline.py <ref_dir> > out.json"""
import hashlib
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np
import torch

import paper_2602_19090_b200 as ozr
import workloads as W
from oracle import refine as orf

ref_dir = sys.argv[1]
with open(os.path.join(ref_dir, "meta.json")) as f:
    meta = json.load(f)
name, n = meta["config"], meta["n"]
cfg = dict(W.CONFIGS[name])
cfg["n"] = n
An, X0n, lam0n = (np.load(os.path.join(ref_dir, f)) for f in ("A.npy", "X0.npy", "lam0.npy"))
sha = lambda a: hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()  # noqa: E731
assert sha(An) == meta["sha_A"] and sha(X0n) == meta["sha_X0"] and sha(lam0n) == meta["sha_lam0"], \
    "the rebuilt problem differs from the one the reference was computed for"
delta = cfg["delta"]
out = {"config": name, "n": n, "delta": delta, "workload": cfg, "hashes_match": True,
       "reference": meta["reference"], "reference_certificate": meta["reference_certificate"]}
dev = torch.device("cuda", 0)
col = lambda a: ozr.colmajor(torch.from_numpy(np.asfortranarray(a)).to(dev))  # noqa: E731
A, X0, lam0 = col(An), col(X0n), torch.from_numpy(lam0n.copy()).to(dev)
ctx = ozr.Context(0)
for rep_ in range(2):  # the second run is timed (the first grows the workspace)
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
                        "beta": [h["beta"] for h in hist], "pairs": [h["pairs_V"] + h["pairs_W"] + h["pairs_U"] for h in hist],
                        "max_cluster": [h["max_cluster"] for h in hist]}
X_final, lam_final = X.cpu().numpy(), lam.cpu().numpy()
Xs = ozr.colmajor(X0.clone())
ls = lam0.clone()
sweep_X = []
for h in hist:
    ozr.ozr_refine_step(ctx, A, Xs, ls, ozr.default_params(delta=delta, theta=h["theta"]))
    sweep_X.append((Xs.cpu().numpy(), ls.cpu().numpy()))
ctx.close()
Xh = np.load(os.path.join(ref_dir, "Xh.npy"))
Xl = np.load(os.path.join(ref_dir, "Xl.npy")).astype(np.float64)
lh = np.load(os.path.join(ref_dir, "lh.npy"))
PI = None if n <= 2048 else 300  # exact 2-norm (SVD) up to 2048, else 300 power iterations on DᵀD
out["forward_error_start"] = orf.forward_error(Xh, Xl, X0n, lh, lam0n, power_iters=PI)
out["forward_error_per_sweep"] = [orf.forward_error(Xh, Xl, Xk, lh, lk, power_iters=PI) for Xk, lk in sweep_X]
fe = orf.forward_error(Xh, Xl, X_final, lh, lam_final, power_iters=PI)
out["forward_error_returned"] = fe
out["fe_over_delta"] = fe / delta
out["ok_implies_within_delta"] = bool(st != 0 or fe <= delta)
print(json.dumps(out))
