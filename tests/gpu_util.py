"""Helpers for the -m gpu parity tests: numpy <-> column-major CUDA tensors."""
import numpy as np


def to_dev(M):
    import torch
    from paper_2602_19090_b200 import colmajor
    return colmajor(torch.from_numpy(np.ascontiguousarray(M, dtype=np.float64)).cuda())


def to_np(T):
    return T.detach().cpu().numpy()


def vec_dev(v):
    import torch
    return torch.from_numpy(np.ascontiguousarray(v, dtype=np.float64)).cuda()


def _components(n, pairs):
    parent = list(range(n))

    def find(a):
        while parent[a] != a:
            parent[a] = parent[parent[a]]
            a = parent[a]
        return a

    for i, j in pairs:
        a, b = find(int(i)), find(int(j))
        if a != b:
            parent[max(a, b)] = min(a, b)
    return [find(i) for i in range(n)]


def check_groups_within_band(info, groups, kappa):
    """The GPU's unresolved groups may differ from the oracle's only through pairs whose first-order
    |ẽ_ij| lies within a factor 2 of κ (the GPU's W carries its digit budget): every pair with
    |ẽ_ij| > 2κ (or equal λ̂) lies inside one GPU group, and every GPU group is connected through
    pairs with |ẽ_ij| > κ/2."""
    E = info["E_first_order"]
    lam = info["lam_rq"]
    n = E.shape[0]
    dl = lam[None, :] - lam[:, None]
    sure = (np.abs(E) > 2 * kappa) | (dl == 0)
    np.fill_diagonal(sure, False)
    where = {}
    for g, J in enumerate(groups):
        for j in J:
            where[j] = g
    for i, j in zip(*np.nonzero(sure)):
        assert where.get(int(i), -1) == where.get(int(j), -2), ("sure pair split", int(i), int(j))
    poss = np.abs(E) > kappa / 2
    np.fill_diagonal(poss, False)
    root = _components(n, list(zip(*np.nonzero(poss | sure))))
    for J in groups:
        assert len({root[j] for j in J}) == 1, ("GPU group not connected by possible pairs", J)


def parity_sweep(ctx, A, X0, lam0, delta, **params):
    """One GPU sweep (ozr_refine_step) and the oracle sweep on the same input with the same parameters.
    The oracle evaluates the GPU's unresolved groups when its own differ only inside the κ band.
    Returns (X_gpu, λ_gpu, report, X_oracle, λ_oracle, oracle info, groups)."""
    import paper_2602_19090_b200 as ozr
    from oracle import refine as orf
    p = ozr.default_params(delta=delta, **params)
    Xd, ld = to_dev(X0), vec_dev(lam0)
    rep = ozr.ozr_refine_step(ctx, to_dev(A), Xd, ld, p)
    groups = ozr.ozr_last_clusters(ctx) if p.cluster_mode else []
    kw = dict(theta=p.theta, truncate=bool(p.truncate), cluster_mode=p.cluster_mode, kappa=p.kappa)
    Xo, lo, info = orf.sweep(A, X0, lam0, delta, **kw)
    if p.cluster_mode and info["clusters"] != groups:
        check_groups_within_band(info, groups, p.kappa)
        Xo, lo, info = orf.sweep(A, X0, lam0, delta, groups=groups, **kw)
    return to_np(Xd), to_np(ld), rep, Xo, lo, info, groups
