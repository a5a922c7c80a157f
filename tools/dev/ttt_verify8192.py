"""Oracle-verified time to target at n = 8192 (c4'), in two gpurun calls of < 1 h each that share the box's
/tmp (the second call must follow the first within 5 minutes to land on the same box):
  phase 1: the problem on the GPU recipe (workloads.make_config_torch), ozr_refine_to_tol with 1, 2, 3 sweeps
           and with the stop rule (device time of each whole call, A split included), then the first two
           iterations of the oracle's dd reference from the LAPACK start (oracle/refine.reference_eigvecs);
  phase 2: the remaining reference iterations (resumed from the dd state), its sampled residual
           certificate, and the forward error ‖X − X̂‖₂ of every GPU result against it.
Usage: python tools/dev/ttt_verify8192.py phase1|phase2"""
import json
import os
import sys
import time

sys.path.insert(0, "/root/repo")
import numpy as np

D = "/tmp/ozr_ttt8192/"
phase = sys.argv[1]
if phase == "phase1":
    import torch

    import paper_2602_19090_b200 as ozr
    import workloads as W
    os.makedirs(D, exist_ok=True)
    dev = torch.device("cuda", 0)
    A, lam0, X0, cfg = W.make_config_torch("c4p", dev)
    delta = cfg["delta"]
    ctx = ozr.Context(0)
    runs = []
    for k in (1, 2, 3, 0):
        for rep_ in range(2):  # the second run is timed
            X = ozr.colmajor(X0.clone())
            lam = lam0.clone()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            p = ozr.default_params(delta=delta, max_sweeps=k) if k else ozr.default_params(delta=delta)
            st, hist = ozr.ozr_refine_to_tol(ctx, A, X, lam, p)
            e1.record()
            torch.cuda.synchronize()
        np.save(D + f"X_{k}.npy", X.cpu().numpy())
        np.save(D + f"lam_{k}.npy", lam.cpu().numpy())
        runs.append({"max_sweeps": k or "stop rule", "sweeps": len(hist), "status": int(st), "ms": e0.elapsed_time(e1),
                     "net_update": [h["net_update"] for h in hist], "update_2norm": [h["update_2norm"] for h in hist]})
    An, X0n, l0n = A.cpu().numpy(), X0.cpu().numpy(), lam0.cpu().numpy()
    np.save(D + "A.npy", An)
    np.save(D + "X0.npy", X0n)
    np.save(D + "lam0.npy", l0n)
    ctx.close()
    json.dump({"delta": delta, "runs": runs}, open(D + "runs.json", "w"))
    from oracle import refine as orf
    t0 = time.time()
    Xh, Xl, lh, ll, hist = orf.reference_eigvecs(An, X0n, l0n, tol=0.0, max_sweeps=2)
    np.save(D + "Xh.npy", Xh)
    np.save(D + "Xl.npy", Xl)
    json.dump({"seconds": time.time() - t0, "normE": hist}, open(D + "ref1.json", "w"))
    print(json.dumps({"phase": 1, "runs": runs, "ref_seconds": time.time() - t0, "normE": hist}))
else:
    from oracle import _clib
    from oracle import refine as orf
    from oracle.fp import dd_add, two_prod
    An, X0n, l0n = np.load(D + "A.npy"), np.load(D + "X0.npy"), np.load(D + "lam0.npy")
    r1 = json.load(open(D + "ref1.json"))
    meta = json.load(open(D + "runs.json"))
    t0 = time.time()
    Xh, Xl, lh, ll, hist = orf.reference_eigvecs(An, np.load(D + "Xh.npy"), l0n, tol=1e-20, max_sweeps=3,
                                                 X0_lo=np.load(D + "Xl.npy"))
    n = An.shape[0]
    J = np.array([0, 1, 2, n // 2, n - 2, n - 1])
    XJh, XJl = np.ascontiguousarray(Xh[:, J]), np.ascontiguousarray(Xl[:, J])
    Vh, Vl = _clib.dd_gemm_nt(An, np.ascontiguousarray(XJh.T), None, np.ascontiguousarray(XJl.T))
    ph, pl = two_prod(XJh, lh[J][None, :])
    pl = pl + XJl * lh[J][None, :] + XJh * ll[J][None, :]
    Rh, Rl = dd_add(Vh, Vl, -ph, -pl)
    res = np.sqrt(np.sum((Rh + Rl) ** 2, axis=0))
    gaps = np.array([np.min(np.abs(np.delete(lh, j) - lh[j])) for j in J])
    delta = meta["delta"]
    for r in meta["runs"]:
        k = r["max_sweeps"] if r["max_sweeps"] != "stop rule" else 0
        fe = orf.forward_error(Xh, Xl, np.load(D + f"X_{k}.npy"), lh, np.load(D + f"lam_{k}.npy"))
        r["forward_error"] = fe
        r["fe_over_delta"] = fe / delta
    hits = [r for r in meta["runs"] if r["max_sweeps"] != "stop rule" and r["forward_error"] <= delta]
    out = {"config": "c4p", "n": n, "delta": delta, "runs": meta["runs"],
           "forward_error_start": orf.forward_error(Xh, Xl, X0n, lh, l0n),
           "first_hit": {"sweeps": hits[0]["sweeps"], "ms": hits[0]["ms"]} if hits else None,
           "reference": {"normE_per_iteration": r1["normE"] + hist, "seconds": r1["seconds"] + time.time() - t0,
                         "threads": _clib.num_threads()},
           "reference_certificate": {"columns": J.tolist(), "residual": res.tolist(),
                                     "sin_theta_bound": (res / gaps).tolist()}}
    print(json.dumps(out))
