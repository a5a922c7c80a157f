"""Diagnostics of the a-posteriori certificate (R12): per sweep of ozr_refine_step from X̂₀, the report's
cert / cert_q / cert_frob / normE_fro, the device time, and (torch, fp64 SVD on the GPU) the 2-norm of the
update ‖X̂_k − X̂_{k−1}‖₂. Also times torch.linalg.eigh (cuSOLVER syevd) at the cluster sizes seen in c2/c4.
Usage: python tools/dev/cert_diag.py [config] [n] [sweeps]"""
import json
import sys
import time

sys.path.insert(0, "/root/repo")
import torch

import paper_2602_19090_b200 as ozr
import workloads as W

name = sys.argv[1] if len(sys.argv) > 1 else "c4p"
n = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2] != "0" else None
sweeps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
dev = torch.device("cuda", 0)
A, lam0, X0, cfg = W.make_config_torch(name, dev, n=n)
delta = cfg["delta"]
ctx = ozr.Context(0)
X = ozr.colmajor(X0.clone())
lam = lam0.clone()
rows = []
for k in range(sweeps):
    Xp = X.clone()
    rep = ozr.ozr_refine_step(ctx, A, X, lam, ozr.default_params(delta=delta, certify=2))
    d2 = float(torch.linalg.matrix_norm(X - Xp, ord=2))
    rows.append({k_: rep[k_] for k_ in ("beta", "theta", "cert", "cert_q", "cert_frob", "cert_iters", "normE_fro",
                                        "net_update", "ms_total", "ms_gemm", "n_clusters", "max_cluster")})
    rows[-1]["update_2norm_svd"] = d2
    print(json.dumps(rows[-1]), flush=True)
X = ozr.colmajor(X0.clone())
lam = lam0.clone()
torch.cuda.synchronize()
t0 = time.time()
st, hist = ozr.ozr_refine_to_tol(ctx, A, X, lam, ozr.default_params(delta=delta))
torch.cuda.synchronize()
print(json.dumps({"refine_to_tol": {"status": int(st), "sweeps": len(hist), "wall_ms": 1e3 * (time.time() - t0),
                                    "cert": [h["cert"] for h in hist], "theta": [h["theta"] for h in hist],
                                    "ms": [h["ms_total"] for h in hist]}}), flush=True)
ctx.close()
del A, X0, X, Xp
torch.cuda.empty_cache()
if "--eigh" in sys.argv:
    for m in (739, 2734, 6628):
        K = torch.randn(m, m, dtype=torch.float64, device=dev)
        K = K + K.T
        for r in range(2):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            torch.linalg.eigh(K)
            e1.record()
            torch.cuda.synchronize()
        print(json.dumps({"eigh_m": m, "ms": e0.elapsed_time(e1)}), flush=True)
