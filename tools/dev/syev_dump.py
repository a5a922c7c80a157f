"""Debug: run ozr_syev_tridiag_eig with OZR_SYEV_DUMP set (per-level inputs of the D&C) for a random tridiagonal."""
import os
import sys
sys.path.insert(0, "/root/repo")
import numpy as np
import torch
import paper_2602_19090_b200 as ozr
m = int(sys.argv[1])
rng = np.random.default_rng(m)
d = rng.standard_normal(m)
e = rng.standard_normal(m)
e[m - 1] = 0.0
ctx = ozr.Context(0)
th, Y = ozr.ozr_syev_tridiag_eig(ctx, torch.from_numpy(d).cuda(), torch.from_numpy(e).cuda())
np.save(os.environ["OZR_SYEV_DUMP"] + "_out.npy", np.concatenate([th.cpu().numpy()[None, :], Y.cpu().numpy()]))
