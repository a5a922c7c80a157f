"""Thin ctypes binding of libozr (include/ozr.h). Argument marshalling only: every step of the method
runs in the CUDA kernels of libozr.so. There is no fallback — if the library or a GPU is missing,
the calls raise.

Matrices are torch CUDA tensors in COLUMN-MAJOR layout: a (rows x cols) tensor with stride (1, ld),
ld ≥ rows (e.g. ``colmajor(t)``). Vectors are contiguous CUDA tensors.
"""
import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libozr.so")

OZR_COLWISE, OZR_ROWWISE = 0, 1
OZR_SPLIT_FIXED, OZR_SPLIT_X1 = 0, 1
STATUS = {0: "OZR_OK", 1: "OZR_ERR_ARG", 2: "OZR_ERR_NONFINITE", 3: "OZR_ERR_RANGE", 4: "OZR_ERR_DEGENERATE",
          5: "OZR_ERR_NOT_CONVERGED", 6: "OZR_ERR_CUDA", 7: "OZR_ERR_COMM", 8: "OZR_ERR_NOMEM"}
EXPORTS = ["ozr_version", "ozr_create", "ozr_destroy", "ozr_last_error", "ozr_split", "ozr_gemm", "ozr_gemm_plan",
           "ozr_params_default", "ozr_refine_step", "ozr_refine_to_tol", "ozr_last_clusters", "ozr_syev", "ozr_syev_tridiag", "ozr_syev_tridiag_eig", "ozr_comm_nccl_id",
           "ozr_comm_create_nccl", "ozr_comm_create_host_group", "ozr_comm_destroy", "ozr_comm_size", "ozr_comm_rank",
           "ozr_refine_step_dist", "ozr_refine_to_tol_dist", "ozr_last_R", "ozr_refine_step_herm"]


class OzrError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class Params(ctypes.Structure):
    _fields_ = [("delta", ctypes.c_double), ("theta", ctypes.c_double), ("beta_mode", ctypes.c_int),
                ("xi", ctypes.c_double), ("beta_override", ctypes.c_int), ("truncate", ctypes.c_int),
                ("max_sweeps", ctypes.c_int), ("kA_split", ctypes.c_int), ("theta_V", ctypes.c_double),
                ("theta_W", ctypes.c_double), ("theta_U", ctypes.c_double), ("L_V", ctypes.c_int),
                ("L_W", ctypes.c_int), ("L_U", ctypes.c_int), ("cluster_mode", ctypes.c_int),
                ("tile_budgets", ctypes.c_int), ("kappa", ctypes.c_double), ("max_cluster", ctypes.c_int),
                ("form_R", ctypes.c_int), ("dense_cluster", ctypes.c_int),
                ("row_nnz", ctypes.c_int), ("max_escalations", ctypes.c_int), ("certify", ctypes.c_int),
                ("fixed_k", ctypes.c_int)]


class StepReport(ctypes.Structure):
    _fields_ = ([(f, ctypes.c_int) for f in ["sweep", "beta", "beta_raw", "alpha", "kX", "kA", "kR", "kE", "L_V",
                                              "L_W", "L_U", "pairs_V", "pairs_W", "pairs_U", "n_clusters", "max_cluster",
                                              "launches", "exchanges"]] +
                [(f, ctypes.c_double) for f in ["gap_min", "max_abs_lambda", "normE_fro", "net_update",
                                                 "predicted_error", "ms_total", "ms_gemm", "int8_ops"]] +
                [("pairs_G", ctypes.c_int)] +
                [(f, ctypes.c_double) for f in ["normR_fro", "normW_fro", "omega_oa", "theta", "cert", "cert_q", "cert_frob"]] +
                [("cert_iters", ctypes.c_int)] +
                [(f, ctypes.c_double) for f in ["planes_V", "planes_W", "planes_U"]])

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


_lib = None


def lib():
    """Load libozr.so (built in-tree by __graft_entry__.build()); raise if it is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(_SO):
            raise OSError(f"libozr.so not built ({_SO}); run __graft_entry__.build()")
        L = ctypes.CDLL(_SO)
        vp, i64, i32, dbl = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
        ip = ctypes.POINTER(ctypes.c_int)
        L.ozr_version.restype = ctypes.c_char_p
        L.ozr_create.argtypes = [ctypes.POINTER(vp), i32, vp, i64]
        L.ozr_create.restype = i32
        L.ozr_destroy.argtypes = [vp]
        L.ozr_destroy.restype = None
        L.ozr_last_error.argtypes = [vp]
        L.ozr_last_error.restype = ctypes.c_char_p
        L.ozr_split.argtypes = [vp, vp, vp, i64, i64, i64, i32, i32, i32, vp, i64, i64, vp, vp, i64, ip]
        L.ozr_split.restype = i32
        L.ozr_gemm.argtypes = [vp, i64, i64, i64, vp, i64, vp, i64, i32, i32, i32, vp, vp, i64, vp, i64, ip]
        L.ozr_gemm.restype = i32
        L.ozr_gemm_plan.argtypes = [i64, i32, i32, i32, ip, ip, ip, i32]
        L.ozr_gemm_plan.restype = i32
        L.ozr_params_default.argtypes = [ctypes.POINTER(Params)]
        L.ozr_params_default.restype = None
        L.ozr_refine_step.argtypes = [vp, vp, i64, i64, vp, i64, vp, ctypes.POINTER(Params),
                                      ctypes.POINTER(StepReport)]
        L.ozr_refine_step.restype = i32
        L.ozr_refine_step_herm.argtypes = [vp, vp, vp, i64, i64, vp, vp, i64, vp, ctypes.POINTER(Params),
                                           ctypes.POINTER(StepReport)]
        L.ozr_refine_step_herm.restype = i32
        L.ozr_refine_to_tol.argtypes = [vp, vp, i64, i64, vp, i64, vp, ctypes.POINTER(Params),
                                        ctypes.POINTER(StepReport), i32, ip]
        L.ozr_refine_to_tol.restype = i32
        L.ozr_last_clusters.argtypes = [vp, ip, i32, ip, i32, ip]
        L.ozr_last_clusters.restype = i32
        L.ozr_syev.argtypes = [vp, i64, vp, i64, vp, vp, i64]
        L.ozr_syev.restype = i32
        L.ozr_syev_tridiag.argtypes = [vp, i64, vp, i64, vp, vp, vp]
        L.ozr_syev_tridiag.restype = i32
        L.ozr_syev_tridiag_eig.argtypes = [vp, i64, vp, vp, vp, vp, i64]
        L.ozr_syev_tridiag_eig.restype = i32
        L.ozr_comm_nccl_id.argtypes = [vp]
        L.ozr_comm_nccl_id.restype = i32
        L.ozr_comm_create_nccl.argtypes = [ctypes.POINTER(vp), vp, i32, i32, i32]
        L.ozr_comm_create_nccl.restype = i32
        L.ozr_comm_create_host_group.argtypes = [ctypes.POINTER(vp), i32]
        L.ozr_comm_create_host_group.restype = i32
        L.ozr_comm_destroy.argtypes = [vp]
        L.ozr_comm_destroy.restype = None
        L.ozr_comm_size.argtypes = [vp]
        L.ozr_comm_size.restype = i32
        L.ozr_comm_rank.argtypes = [vp]
        L.ozr_comm_rank.restype = i32
        L.ozr_refine_step_dist.argtypes = [vp, vp, vp, i64, i64, vp, i64, vp, ctypes.POINTER(Params),
                                           ctypes.POINTER(StepReport)]
        L.ozr_refine_step_dist.restype = i32
        L.ozr_refine_to_tol_dist.argtypes = [vp, vp, vp, i64, i64, vp, i64, vp, ctypes.POINTER(Params),
                                             ctypes.POINTER(StepReport), i32, ip]
        L.ozr_refine_to_tol_dist.restype = i32
        L.ozr_last_R.argtypes = [vp, vp, i64]
        L.ozr_last_R.restype = i32
        _lib = L
    return _lib


def colmajor(t):
    """Column-major copy of a 2-D tensor (stride (1, rows))."""
    return t.t().contiguous().t()


def empty_colmajor(rows, cols, dtype, device):
    """An uninitialised column-major rows x cols tensor (no copy kernel)."""
    return torch.empty((cols, rows), dtype=dtype, device=device).t()


def _ld(t):
    if t.dim() != 2 or t.stride(0) != 1 or t.stride(1) < t.shape[0]:
        raise ValueError("expected a column-major 2-D tensor (stride (1, ld), ld >= rows)")
    return t.stride(1)


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)


def default_params(**kw):
    p = Params()
    lib().ozr_params_default(ctypes.byref(p))
    for k, v in kw.items():
        if not hasattr(p, k):
            raise KeyError(k)
        setattr(p, k, v)
    return p


class Context:
    """An ozr context on one CUDA device, issuing work on `stream` (default: torch's current stream)."""

    def __init__(self, device=0, stream=None):
        if not torch.cuda.is_available():
            raise RuntimeError("ozr needs a CUDA device (no CPU fallback)")
        self.device = device
        self.stream = stream if stream is not None else torch.cuda.current_stream(device)
        h = ctypes.c_void_p()
        st = lib().ozr_create(ctypes.byref(h), device, ctypes.c_void_p(self.stream.cuda_stream), 0)
        if st != 0:
            raise OzrError(st, "ozr_create failed")
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            lib().ozr_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def check(self, st):
        if st != 0:
            raise OzrError(st, lib().ozr_last_error(self.h).decode())
        return st


def ozr_version():
    return lib().ozr_version().decode()


def ozr_split(ctx, M, k_or_beta, axis=OZR_COLWISE, mode=OZR_SPLIT_FIXED, M_lo=None, want_x1=False):
    """Returns (digits [k, lines, ldd] int8, lsb_exp int32[lines], k, X1 or None)."""
    rows, cols = M.shape
    lines, length = (cols, rows) if axis == OZR_COLWISE else (rows, cols)
    ldd = (length + 15) // 16 * 16
    kmax = 7 if mode == OZR_SPLIT_X1 else k_or_beta
    dig = torch.empty((kmax, lines, ldd), dtype=torch.int8, device=M.device)
    ell = torch.empty(lines, dtype=torch.int32, device=M.device)
    x1 = empty_colmajor(rows, cols, torch.float64, M.device) if want_x1 else None
    kout = ctypes.c_int(0)
    ctx.check(lib().ozr_split(ctx.h, _ptr(M), _ptr(M_lo), rows, cols, _ld(M), axis, mode, k_or_beta, _ptr(dig), ldd,
                              lines * ldd, _ptr(ell), _ptr(x1), _ld(x1) if x1 is not None else 0,
                              ctypes.byref(kout)))
    return dig[:kout.value], ell, kout.value, x1


def ozr_gemm_plan(k, kA, kB, L=0, max_groups=256):
    ng = ctypes.c_int(0)
    gd = (ctypes.c_int * max_groups)()
    gp = (ctypes.c_int * max_groups)()
    st = lib().ozr_gemm_plan(k, kA, kB, L, ctypes.byref(ng), gd, gp, max_groups)
    if st != 0:
        raise OzrError(st, "ozr_gemm_plan")
    return [(gd[i], gp[i]) for i in range(ng.value)]


def ozr_gemm(ctx, A, B, kA, kB, L=0, want_lo=True, want_planes=False):
    """C = A·B (column-major). Returns (C_hi, C_lo or None, planes [G, n, m] or None)."""
    m, k = A.shape
    k2, n = B.shape
    if k != k2:
        raise ValueError("inner dimensions differ")
    dev = A.device
    Ch = empty_colmajor(m, n, torch.float64, dev)
    Cl = empty_colmajor(m, n, torch.float64, dev) if want_lo else None
    planes = None
    if want_planes:
        G = len(ozr_gemm_plan(k, kA, kB, L))
        planes = torch.empty((G, n, m), dtype=torch.int32, device=dev)
    ng = ctypes.c_int(0)
    ctx.check(lib().ozr_gemm(ctx.h, m, n, k, _ptr(A), _ld(A), _ptr(B), _ld(B), kA, kB, L, _ptr(Ch), _ptr(Cl), m,
                             _ptr(planes), m * n, ctypes.byref(ng)))
    return Ch, Cl, planes


def ozr_refine_step(ctx, A, X, lam, params):
    """One sweep in place on X (column-major n x n) and lam (n). Returns the report dict."""
    n = A.shape[0]
    rep = StepReport()
    ctx.check(lib().ozr_refine_step(ctx.h, _ptr(A), n, _ld(A), _ptr(X), _ld(X), _ptr(lam), ctypes.byref(params),
                                    ctypes.byref(rep)))
    return rep.as_dict()


def ozr_refine_step_herm(ctx, Ar, Ai, Xr, Xi, lam, params):
    """One Hermitian sweep in place on Xr, Xi (column-major n x n, real and imaginary parts) and
    lam (n). Ar, Ai: the Hermitian A's parts (column-major). Returns the report dict."""
    n = Ar.shape[0]
    if _ld(Ai) != _ld(Ar) or _ld(Xi) != _ld(Xr):
        raise ValueError("the real and imaginary parts must share a leading dimension")
    rep = StepReport()
    ctx.check(lib().ozr_refine_step_herm(ctx.h, _ptr(Ar), _ptr(Ai), n, _ld(Ar), _ptr(Xr), _ptr(Xi), _ld(Xr),
                                         _ptr(lam), ctypes.byref(params), ctypes.byref(rep)))
    return rep.as_dict()


def ozr_refine_to_tol(ctx, A, X, lam, params, raise_on_nonconvergence=False):
    """Sweeps until the stop rule; returns (status, [report dicts])."""
    n = A.shape[0]
    H = (StepReport * 64)()
    done = ctypes.c_int(0)
    st = lib().ozr_refine_to_tol(ctx.h, _ptr(A), n, _ld(A), _ptr(X), _ld(X), _ptr(lam), ctypes.byref(params), H, 64,
                                 ctypes.byref(done))
    if st != 0 and (st != 5 or raise_on_nonconvergence):
        ctx.check(st)
    return st, [H[i].as_dict() for i in range(done.value)]


def ozr_syev(ctx, K):
    """θ (ascending), Y with K = Y diag(θ) Yᵀ for a symmetric column-major device matrix K (lower triangle read)."""
    m = K.shape[0]
    th = torch.empty(m, dtype=torch.float64, device=K.device)
    Y = empty_colmajor(m, m, torch.float64, K.device)
    ctx.check(lib().ozr_syev(ctx.h, m, _ptr(K), _ld(K), _ptr(th), _ptr(Y), m))
    return th, Y


def ozr_syev_tridiag(ctx, K):
    """Stage 1 alone: (d, e, τ, R) with R = K's copy holding the Householder vectors below its sub-diagonal."""
    m = K.shape[0]
    R = colmajor(K.clone())
    d, e, tau = (torch.zeros(m, dtype=torch.float64, device=K.device) for _ in range(3))
    ctx.check(lib().ozr_syev_tridiag(ctx.h, m, _ptr(R), m, _ptr(d), _ptr(e), _ptr(tau)))
    return d, e, tau, R


def ozr_syev_tridiag_eig(ctx, d, e):
    """Stage 2 alone: θ ascending and Y for the symmetric tridiagonal (d, e)."""
    m = d.shape[0]
    th = torch.empty(m, dtype=torch.float64, device=d.device)
    Y = empty_colmajor(m, m, torch.float64, d.device)
    ctx.check(lib().ozr_syev_tridiag_eig(ctx.h, m, _ptr(d), _ptr(e), _ptr(th), _ptr(Y), m))
    return th, Y


def ozr_last_clusters(ctx, max_members=1 << 20, max_groups=1 << 16):
    """The unresolved groups of the context's last sweep: a list of lists of global column indices."""
    mem = (ctypes.c_int * max_members)()
    off = (ctypes.c_int * (max_groups + 1))()
    ng = ctypes.c_int(0)
    ctx.check(lib().ozr_last_clusters(ctx.h, mem, max_members, off, max_groups, ctypes.byref(ng)))
    return [list(mem[off[g]:off[g + 1]]) for g in range(ng.value)]


# ------------------------------------------------------------------------------------------ multi-GPU
class Comm:
    """A communicator of the block-column partition (include/ozr.h "Multi-GPU")."""

    def __init__(self, handle):
        self.h = handle

    @property
    def size(self):
        return lib().ozr_comm_size(self.h)

    @property
    def rank(self):
        return lib().ozr_comm_rank(self.h)

    def close(self):
        if getattr(self, "h", None):
            lib().ozr_comm_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def ozr_comm_nccl_id():
    buf = ctypes.create_string_buffer(128)
    st = lib().ozr_comm_nccl_id(buf)
    if st != 0:
        raise OzrError(st, "ozr_comm_nccl_id (is libnccl.so.2 loadable?)")
    return bytes(buf.raw)


def ozr_comm_create_nccl(uid, nranks, rank, device):
    if len(uid) != 128:
        raise ValueError("NCCL unique id is 128 bytes")
    h = ctypes.c_void_p()
    st = lib().ozr_comm_create_nccl(ctypes.byref(h), ctypes.create_string_buffer(uid, 128), nranks, rank, device)
    if st != 0:
        raise OzrError(st, "ozr_comm_create_nccl")
    return Comm(h)


def ozr_comm_create_host_group(nranks):
    """`nranks` communicators for ranks that are threads of this process (single-GPU protocol harness)."""
    hs = (ctypes.c_void_p * nranks)()
    st = lib().ozr_comm_create_host_group(hs, nranks)
    if st != 0:
        raise OzrError(st, "ozr_comm_create_host_group")
    return [Comm(ctypes.c_void_p(hs[r])) for r in range(nranks)]


def _comm_h(comm):
    return comm.h if comm is not None else ctypes.c_void_p(0)


def ozr_refine_step_dist(ctx, comm, A, X, lam, params):
    """One sweep on this rank's column block of X (full n x n column-major array; columns
    [rank·n/P, (rank+1)·n/P) are read and written); lam (n) replicated. Returns the report dict."""
    n = A.shape[0]
    rep = StepReport()
    ctx.check(lib().ozr_refine_step_dist(ctx.h, _comm_h(comm), _ptr(A), n, _ld(A), _ptr(X), _ld(X), _ptr(lam),
                                         ctypes.byref(params), ctypes.byref(rep)))
    return rep.as_dict()


def ozr_refine_to_tol_dist(ctx, comm, A, X, lam, params, raise_on_nonconvergence=False):
    n = A.shape[0]
    H = (StepReport * 64)()
    done = ctypes.c_int(0)
    st = lib().ozr_refine_to_tol_dist(ctx.h, _comm_h(comm), _ptr(A), n, _ld(A), _ptr(X), _ld(X), _ptr(lam),
                                      ctypes.byref(params), H, 64, ctypes.byref(done))
    if st != 0 and (st != 5 or raise_on_nonconvergence):
        ctx.check(st)
    return st, [H[i].as_dict() for i in range(done.value)]


def ozr_last_R(ctx, n, n_local=None):
    """R = I − X̂^(1)ᵀX̂^(1) of the last sweep run with form_R=1 (this rank's columns), column-major."""
    R = empty_colmajor(n, n_local or n, torch.float64, torch.device("cuda", ctx.device))
    ctx.check(lib().ozr_last_R(ctx.h, _ptr(R), n))
    return R
