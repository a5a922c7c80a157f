"""Time ozr_syev (OZR_TRACE=1 prints the stage split) on graded group-like matrices of several sizes, and
compare with torch.linalg.eigh (cuSOLVER) on the same matrix: residual and orthogonality."""
import sys
import time
sys.path.insert(0, "/root/repo")
import numpy as np
import torch
import paper_2602_19090_b200 as ozr
ctx = ozr.Context(0)
for m in [int(x) for x in sys.argv[1:]] or [739, 2734, 6628]:
    g = torch.Generator(device="cuda").manual_seed(m)
    Q, _ = torch.linalg.qr(torch.randn(m, m, dtype=torch.float64, device="cuda", generator=g))
    lam = torch.logspace(-14, -2, m, dtype=torch.float64, device="cuda")
    K = (Q * lam) @ Q.T
    N = torch.randn(m, m, dtype=torch.float64, device="cuda", generator=g)
    K = (K + K.T) * 0.5 + 1e-8 * (N + N.T) * 0.5
    K = ozr.colmajor(K.contiguous())
    for rep in range(2):
        torch.cuda.synchronize()
        t0 = time.time()
        th, Y = ozr.ozr_syev(ctx, K)
        torch.cuda.synchronize()
        t1 = time.time()
    res = float(torch.linalg.matrix_norm(K @ Y - Y * th) / torch.linalg.matrix_norm(K))
    orth = float((Y.T @ Y - torch.eye(m, dtype=torch.float64, device="cuda")).abs().max())
    torch.cuda.synchronize()
    t2 = time.time()
    w, V = torch.linalg.eigh(K)
    torch.cuda.synchronize()
    t3 = time.time()
    resl = float(torch.linalg.matrix_norm(K @ V - V * w) / torch.linalg.matrix_norm(K))
    orthl = float((V.T @ V - torch.eye(m, dtype=torch.float64, device="cuda")).abs().max())
    print(f"m={m} ozr_syev {1e3*(t1-t0):.1f} ms res {res:.2e} orth {orth:.2e} | eigh {1e3*(t3-t2):.1f} ms res {resl:.2e} "
          f"orth {orthl:.2e} | max|dtheta| {float((th - w).abs().max()):.2e}", flush=True)
