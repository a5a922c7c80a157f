"""Large-group threshold study: ozr_refine_to_tol on BASELINE c4 (n = 8192) and c2 (n = 1024) with the dense
sub-solve taking groups of >= `dense_cluster` columns (smaller groups: one Jacobi CTA each). Prints time to target
(second call, device-synchronised wall clock), sweeps, status, per-sweep ms and the residual / orthogonality of the
result (validation only). Usage: python tools/dev/dense_thr.py [thresholds...]"""
import json
import sys
import time

sys.path.insert(0, "/root/repo")
import torch

import paper_2602_19090_b200 as ozr
import workloads as W

thr = [int(x) for x in sys.argv[1:]] or [192, 128, 96, 64, 32]
dev = torch.device("cuda", 0)
ctx = ozr.Context(0)
for name in ("c2", "c4"):
    A, lam0, X0, cfg = W.make_config_torch(name, dev)
    n = cfg["n"]
    for t in thr:
        p = ozr.default_params(delta=cfg["delta"], dense_cluster=t)
        for rep in range(2):
            X = ozr.colmajor(X0.clone())
            lam = lam0.clone()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            st, hist = ozr.ozr_refine_to_tol(ctx, A, X, lam, p)
            torch.cuda.synchronize()
            wall = time.perf_counter() - t0
        R = A @ X - X * lam[None, :]
        res = float(torch.linalg.vector_norm(R, dim=0).max())
        orth = float((X.T @ X - torch.eye(n, dtype=torch.float64, device=dev)).abs().max())
        print(json.dumps({"config": name, "dense_cluster": t, "status": int(st), "wall_ms": 1e3 * wall,
                          "sweeps": len(hist), "ms": [round(h["ms_total"], 2) for h in hist],
                          "groups": [(h["n_clusters"], h["max_cluster"]) for h in hist],
                          "max_residual": res, "orth_max": orth}), flush=True)
