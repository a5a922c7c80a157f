"""BASELINE c4 at full size (n = 8192, geometric cnd 1e14, FP32-eigensolver start, gate 1e-10): ozr_refine_to_tol
with the cluster branch (large groups through the dense sub-solve), per-sweep history, device time, and
backward-error properties of the result (fp64 torch products; validation only, not the product path):
max_j ‖A x_j − λ_j x_j‖ and ‖I − XᵀX‖_max. Usage: python tools/dev/c4_full.py [config] [n] [max_sweeps]"""
import json
import sys
import time

sys.path.insert(0, "/root/repo")
import torch

import paper_2602_19090_b200 as ozr
import workloads as W

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
n = int(sys.argv[2]) if len(sys.argv) > 2 else None
maxs = int(sys.argv[3]) if len(sys.argv) > 3 else 10
dev = torch.device("cuda", 0)
A, lam0, X0, cfg = W.make_config_torch(name, dev, n=n)
n = cfg["n"]
ctx = ozr.Context(0)
X = ozr.colmajor(X0.clone())
lam = lam0.clone()
torch.cuda.synchronize()
t0 = time.perf_counter()
st, hist = ozr.ozr_refine_to_tol(ctx, A, X, lam, ozr.default_params(delta=cfg["delta"], max_sweeps=maxs))
torch.cuda.synchronize()
wall = time.perf_counter() - t0
R = A @ X - X * lam[None, :]
res = torch.linalg.vector_norm(R, dim=0)
orth = (X.T @ X - torch.eye(n, dtype=torch.float64, device=dev)).abs().max()
out = {"config": name, "n": n, "delta": cfg["delta"], "status": int(st), "error": ozr.lib().ozr_last_error(ctx.h).decode() if st else "",
       "wall_s": wall, "sweeps": [{k: h[k] for k in ("theta", "beta", "kA", "kR", "kE", "pairs_V", "pairs_W", "pairs_U",
                                                    "n_clusters", "max_cluster", "net_update", "predicted_error",
                                                    "normE_fro", "cert", "ms_total", "ms_gemm")} for h in hist],
       "max_residual": float(res.max()), "orth_max": float(orth)}
print(json.dumps(out))
