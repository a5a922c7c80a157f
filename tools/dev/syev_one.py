"""One ozr_syev call on a graded m x m group-like matrix (for ncu captures)."""
import sys
sys.path.insert(0, "/root/repo")
import torch
import paper_2602_19090_b200 as ozr
m = int(sys.argv[1]) if len(sys.argv) > 1 else 6628
g = torch.Generator(device="cuda").manual_seed(m)
Q, _ = torch.linalg.qr(torch.randn(m, m, dtype=torch.float64, device="cuda", generator=g))
lam = torch.logspace(-14, -2, m, dtype=torch.float64, device="cuda")
K = ozr.colmajor(((Q * lam) @ Q.T).contiguous())
ctx = ozr.Context(0)
th, Y = ozr.ozr_syev(ctx, K)
torch.cuda.synchronize()
print("ok", float(th[0]), float(th[-1]))
