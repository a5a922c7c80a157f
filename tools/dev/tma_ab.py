"""A/B of the recombination kernels' TMA and register paths (OZR_NO_TMA bit mask, read once per process):
one c4p sweep at n = 4096, X̂ and λ̂ written to a .npy pair for comparison across processes.
Usage: OZR_NO_TMA=<mask> python tools/dev/tma_ab.py out_prefix [config] [start]"""
import sys

sys.path.insert(0, "/root/repo")
import numpy as np
import torch

import paper_2602_19090_b200 as ozr
import workloads as W

out = sys.argv[1]
cfg = sys.argv[2] if len(sys.argv) > 2 else "c4p"
A, _ = W.make_matrix(4096, W.CONFIGS[cfg]["kind"], W.CONFIGS[cfg]["cnd"], W.CONFIGS[cfg]["seed"])
lam0, X0 = W.initial_eig(A, sys.argv[3] if len(sys.argv) > 3 else "fp64")
ctx = ozr.Context(0)
dev = lambda M: ozr.colmajor(torch.from_numpy(np.asfortranarray(M)).cuda())  # noqa: E731
X, lam = dev(X0), torch.from_numpy(lam0.copy()).cuda()
rep = ozr.ozr_refine_step(ctx, dev(A), X, lam, ozr.default_params(delta=1e-12))
np.save(out + "_X.npy", X.cpu().numpy())
np.save(out + "_l.npy", lam.cpu().numpy())
print({k: rep[k] for k in ("L_V", "L_W", "L_U", "planes_V", "planes_W", "planes_U")})
