"""Small sweeps for compute-sanitizer (memcheck / racecheck / synccheck): the CTA-pair tcgen05 slice GEMM, the
recombination / split kernels, the certificate's bf16 GEMMs, the whole-GPU cooperative Jacobi (a c2 FP32-start
group of ≥ 192 columns with the dense path disabled), the hand-written dense eigensolver (ozr_syev and the
default dense sub-solve). Usage: compute-sanitizer --tool memcheck python tools/dev/sanitize_sweep.py"""
import sys

sys.path.insert(0, "/root/repo")
import numpy as np
import torch

import paper_2602_19090_b200 as ozr
import workloads as W

ctx = ozr.Context(0)


def dev(M):
    return ozr.colmajor(torch.from_numpy(np.asfortranarray(M)).cuda())


# (1) c4' recipe, n = 256: V/W/U slice GEMMs, recombinations, splits, certificate
A, lam0, X0, cfg = W.make_config("c4p", n=256)
X, lam = dev(X0), torch.from_numpy(lam0.copy()).cuda()
st, hist = ozr.ozr_refine_to_tol(ctx, dev(A), X, lam, ozr.default_params(delta=1e-12, max_sweeps=3))
print("c4p n=256:", st, [h["cert"] for h in hist], flush=True)
# (2) c2 recipe, FP32 start, n = 512: unresolved groups; the large one on the cooperative Jacobi
A, _ = W.make_matrix(512, "geometric", 1e12, 1002)
lam0, X0 = W.initial_eig(A, "fp32")
X, lam = dev(X0), torch.from_numpy(lam0.copy()).cuda()
rep = ozr.ozr_refine_step(ctx, dev(A), X, lam, ozr.default_params(delta=1e-14, dense_cluster=1 << 20))
print("c2 n=512 coop Jacobi: groups", rep["n_clusters"], "max", rep["max_cluster"], flush=True)
# (3) the same with the default dense sub-solve (hand-written eigensolver, INT8 products)
X, lam = dev(X0), torch.from_numpy(lam0.copy()).cuda()
rep = ozr.ozr_refine_step(ctx, dev(A), X, lam, ozr.default_params(delta=1e-14))
print("c2 n=512 dense: groups", rep["n_clusters"], "max", rep["max_cluster"], flush=True)
# (4) ozr_syev on a graded 300 x 300 (several merge levels, deflation) and ozr_gemm
rng = np.random.default_rng(1)
G = rng.standard_normal((300, 300))
K = (G + G.T) / 2
th, Y = ozr.ozr_syev(ctx, dev(K))
C, Cl, _ = ozr.ozr_gemm(ctx, dev(rng.standard_normal((200, 300))), dev(rng.standard_normal((300, 130))), 7, 7)
torch.cuda.synchronize()
print("syev / gemm ok", float(th[0]), float(C[0, 0]), flush=True)
ctx.close()
