"""Backward errors of the eigensolver's stages on a graded group-like matrix (diagnostics)."""
import sys
sys.path.insert(0, "/root/repo")
import numpy as np
import torch
import paper_2602_19090_b200 as ozr
m = int(sys.argv[1]) if len(sys.argv) > 1 else 739
rng = np.random.default_rng(m)
G = rng.standard_normal((m, m))
Q, _ = np.linalg.qr(G)
lam = np.geomspace(1e-14, 1e-2, m)
K = (Q * lam) @ Q.T
N = rng.standard_normal((m, m))
K = (K + K.T) * 0.5 + 1e-8 * (N + N.T) * 0.5
ctx = ozr.Context(0)
Kd = ozr.colmajor(torch.from_numpy(np.asfortranarray(K)).cuda())
d, e, tau, R = (t.cpu().numpy() for t in ozr.ozr_syev_tridiag(ctx, Kd))
QH = np.eye(m)
for c in range(m - 2, -1, -1):
    v = np.zeros(m); v[c + 1] = 1.0; v[c + 2:] = R[c + 2:, c]
    QH[c + 1:, :] -= tau[c] * np.outer(v[c + 1:], v[c + 1:] @ QH[c + 1:, :])
T = np.diag(d) + np.diag(e[:m - 1], -1) + np.diag(e[:m - 1], 1)
nK = np.linalg.norm(K)
print("tridiag: ||QᵀKQ − T||/||K|| = %.2e  ||QᵀQ − I|| = %.2e" % (np.linalg.norm(QH.T @ K @ QH - T) / nK,
      np.max(np.abs(QH.T @ QH - np.eye(m)))))
th, Y = ozr.ozr_syev_tridiag_eig(ctx, torch.from_numpy(d).cuda(), torch.from_numpy(e).cuda())
th, Y = th.cpu().numpy(), Y.cpu().numpy()
print("d&c: ||TY − YΘ||/||T|| = %.2e  orth %.2e" % (np.linalg.norm(T @ Y - Y * th) / np.linalg.norm(T),
      np.max(np.abs(Y.T @ Y - np.eye(m)))))
w, V = np.linalg.eigh(T)
print("lapack on T: %.2e" % (np.linalg.norm(T @ V - V * w) / np.linalg.norm(T)))
Yf = QH @ Y
print("tridiag Q · d&c Y (numpy): ||KY − YΘ||/||K|| = %.2e" % (np.linalg.norm(K @ Yf - Yf * th) / nK))
th2, Y2 = ozr.ozr_syev(ctx, Kd)
th2, Y2 = th2.cpu().numpy(), Y2.cpu().numpy()
print("full: %.2e ; back-transform vs numpy: %.2e" % (np.linalg.norm(K @ Y2 - Y2 * th2) / nK, np.max(np.abs(Y2 - Yf))))
w, V = np.linalg.eigh(K)
print("lapack on K: %.2e" % (np.linalg.norm(K @ V - V * w) / nK))
