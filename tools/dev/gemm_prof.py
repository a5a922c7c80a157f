"""ozr_gemm at n = 8192 with the full-fp64 plan (8 + 8 digits, s + t <= 9) and the sweep's V plan, for launch lists
(ncu --metrics gpu__time_duration.sum) of the per-product path. Usage: python tools/dev/gemm_prof.py"""
import sys

sys.path.insert(0, "/root/repo")
import torch

import paper_2602_19090_b200 as ozr
import workloads as W

dev = torch.device("cuda", 0)
A, lam0, X0, cfg = W.make_config_torch("c4p", dev)
ctx = ozr.Context(0)
for kA, kB, L in ((8, 8, 9), (12, 5, 13)):
    for _ in range(2):
        ozr.ozr_gemm(ctx, A, X0, kA, kB, L)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        ozr.ozr_gemm(ctx, A, X0, kA, kB, L)
    e1.record()
    torch.cuda.synchronize()
    print(kA, kB, L, "ms", e0.elapsed_time(e1) / 3)
