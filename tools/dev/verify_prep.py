"""Phase 1 of the oracle verification at BASELINE sizes (CPU, no GPU): build a BASELINE recipe with the
numpy recipe (workloads.make_config), compute the oracle's double-double reference eigenvectors of the stored A
(oracle/refine.reference_eigvecs from an FP64 LAPACK start, Rayleigh–Ritz branch on) and its sampled residual
certificate, and store them under scratch/verify/<config>_<n>/ with the sha256 of A and X̂₀ so that phase 2
(tools/dev/verify_baseline.py --ref DIR, on the GPU box) can rebuild the same A and X̂₀ from the seed, check the
hashes, and measure the library's forward error against this reference.
Usage: python tools/dev/verify_prep.py <config> <n>"""
import hashlib
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np

import workloads as W
from oracle import _clib
from oracle import refine as orf
from oracle.fp import dd_add, two_prod

name, n = sys.argv[1], int(sys.argv[2])
out_dir = os.path.join(ROOT, "scratch", "verify", f"{name}_{n}")
os.makedirs(out_dir, exist_ok=True)
A, lam0, X0, cfg = W.make_config(name, n=n)
meta = {"config": name, "n": n, "workload": cfg,
        "sha_A": hashlib.sha256(np.ascontiguousarray(A).tobytes()).hexdigest(),
        "sha_X0": hashlib.sha256(np.ascontiguousarray(X0).tobytes()).hexdigest(),
        "sha_lam0": hashlib.sha256(np.ascontiguousarray(lam0).tobytes()).hexdigest()}
t0 = time.time()
w, V = np.linalg.eigh(A)  # FP64 LAPACK start of the reference (the reference is a property of A alone)
Xh, Xl, lh, ll, hist = orf.reference_eigvecs(A, V, w, tol=1e-24, max_sweeps=8, cluster_kappa=2.0 ** -10)
meta["reference"] = {"seconds": time.time() - t0, "normE_per_iteration": hist, "threads": _clib.num_threads()}
J = np.unique(np.linspace(0, n - 1, 32).astype(np.int64))
XJh, XJl = np.ascontiguousarray(Xh[:, J]), np.ascontiguousarray(Xl[:, J])
Vh, Vl = _clib.dd_gemm_nt(A, np.ascontiguousarray(XJh.T), None, np.ascontiguousarray(XJl.T))
ph, pl = two_prod(XJh, lh[J][None, :])
pl = pl + XJl * lh[J][None, :] + XJh * ll[J][None, :]
Rh, Rl = dd_add(Vh, Vl, -ph, -pl)
res = np.sqrt(np.sum((Rh + Rl) ** 2, axis=0))
gaps = np.array([np.min(np.abs(np.delete(lh, j) - lh[j])) for j in J])
meta["reference_certificate"] = {"columns": J.tolist(), "residual_max": float(np.max(res)),
                                 "sin_theta_bound_max": float(np.max(res / gaps))}
# the problem itself travels with the reference: numpy's LAPACK results depend on the thread count, so the GPU
# box cannot rebuild A and X̂₀ bit for bit from the seed
np.save(os.path.join(out_dir, "A.npy"), A)
np.save(os.path.join(out_dir, "X0.npy"), X0)
np.save(os.path.join(out_dir, "lam0.npy"), lam0)
np.save(os.path.join(out_dir, "Xh.npy"), Xh)
np.save(os.path.join(out_dir, "Xl.npy"), Xl.astype(np.float32))  # |Xl| ≤ u|Xh|: fp32 keeps it to 1e-23
np.save(os.path.join(out_dir, "lh.npy"), lh)
with open(os.path.join(out_dir, "meta.json"), "w") as f:
    json.dump(meta, f, indent=1)
print(json.dumps(meta))
