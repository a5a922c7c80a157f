#!/usr/bin/env python
"""One ozr_refine_to_tol run on the exactly-known family (workloads.hadamard_exact) at any size, with the forward
error against the closed-form eigenvectors measured after the run (and, with --per-sweep, after every sweep through
ozr_refine_step's own driver loop being replayed with max_sweeps = 1, 2, ...). Prints one JSON line.
usage: python tools/dev/exact_verify.py M KIND START DELTA [CND] [--per-sweep]   (n = 2^M)"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2602_19090_b200 as ozr  # noqa: E402
import workloads as W  # noqa: E402


def norm2(D):
    return float(torch.sqrt(torch.linalg.eigvalsh(D.T @ D)[-1].clamp_min(0.0)))


def main():
    m, kind, start, delta = int(sys.argv[1]), sys.argv[2], sys.argv[3], float(sys.argv[4])
    cnd = float(sys.argv[5]) if len(sys.argv) > 5 and not sys.argv[5].startswith("--") else 1e4
    t0 = time.time()
    A, lam, X = W.hadamard_exact(m, kind, cnd=cnd, seed=100 + m)
    t_gen = time.time() - t0
    n = 2 ** m
    Ad = torch.from_numpy(A).cuda()
    del A
    if start == "fp32":
        l0, X0 = torch.linalg.eigh(Ad.float())
        l0, X0 = l0.double(), X0.double()
    else:
        l0, X0 = torch.linalg.eigh(Ad)
    Xe = torch.from_numpy(X).cuda()
    del X

    def fe_of(Xd, ld):
        p = torch.argsort(ld, stable=True)
        Xr = Xd[:, p]
        sg = torch.sign(torch.sum(Xr * Xe, dim=0))
        Xr = Xr * sg[None, :]
        Xr -= Xe
        return norm2(Xr), float(torch.max(torch.abs(ld[p] - torch.from_numpy(lam).cuda())))

    fe0, _ = fe_of(X0, l0)
    ctx = ozr.Context(0)
    Ac = ozr.colmajor(Ad)
    out = dict(n=n, kind=kind, start=start, delta=delta, cnd=cnd, gen_s=round(t_gen, 1), fe_start=fe0, runs=[])
    for rep in range(2):  # the second call is the timed one (the first allocates workspaces)
        Xd, ld = ozr.colmajor(X0.clone()), l0.contiguous().clone()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        st, hist = ozr.ozr_refine_to_tol(ctx, Ac, Xd, ld, ozr.default_params(delta=delta))
        e1.record()
        torch.cuda.synchronize()
        fe, dl = fe_of(Xd, ld)
        out["runs"].append(dict(status=st, sweeps=len(hist), ms=e0.elapsed_time(e1), forward_error=fe,
                                fe_over_delta=fe / delta, max_dlam=dl, cert=[h.get("cert") for h in hist],
                                clusters=[h.get("max_cluster", h.get("clusters")) for h in hist]))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
