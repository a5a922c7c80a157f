"""ctypes loader for oracle/ddmm.c (TEST INFRASTRUCTURE ONLY — see oracle/__init__.py).

The shared object is built in-tree by ``__graft_entry__.build()`` (or lazily here, with gcc, the
first time it is needed). Compiled with -ffp-contract=off so TwoSum / TwoProd run as written.
"""
import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ddmm.c")
_SO = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force=False):
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-fPIC", "-shared", "-fopenmp", "-ffp-contract=off", "-fno-fast-math",
               "-o", _SO, _SRC, "-lquadmath", "-lm"]
        subprocess.check_call(cmd)
    return _SO


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        dp = ctypes.POINTER(ctypes.c_double)
        L.oracle_dd_gemm_nt.argtypes = [ctypes.c_int64] * 3 + [dp] * 6
        L.oracle_dd_gemm_nt.restype = None
        L.oracle_jacobi_q.argtypes = [ctypes.c_int, dp, dp, ctypes.c_double, dp, dp, dp, dp]
        L.oracle_jacobi_q.restype = ctypes.c_int
        L.oracle_num_threads.argtypes = []
        L.oracle_num_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def _p(a):
    if a is None:
        return ctypes.POINTER(ctypes.c_double)()
    assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def dd_gemm_nt(P, Q, Pl=None, Ql=None):
    """C = (P + Pl) @ (Q + Ql).T in double-double (naive triple loop). P: m x K, Q: n x K."""
    P = np.ascontiguousarray(P, dtype=np.float64)
    Q = np.ascontiguousarray(Q, dtype=np.float64)
    Pl = None if Pl is None else np.ascontiguousarray(Pl, dtype=np.float64)
    Ql = None if Ql is None else np.ascontiguousarray(Ql, dtype=np.float64)
    m, K = P.shape
    n, K2 = Q.shape
    assert K == K2
    Ch = np.empty((m, n))
    Cl = np.empty((m, n))
    lib().oracle_dd_gemm_nt(m, n, K, _p(P), _p(Pl), _p(Q), _p(Ql), _p(Ch), _p(Cl))
    return Ch, Cl


def jacobi_q(Ah, Al=None, tol=1e-32):
    """__float128 cyclic Jacobi: returns (w_hi, w_lo, V_hi, V_lo, sweeps), ascending, sign-fixed."""
    Ah = np.ascontiguousarray(Ah, dtype=np.float64)
    Al = None if Al is None else np.ascontiguousarray(Al, dtype=np.float64)
    n = Ah.shape[0]
    wh, wl = np.empty(n), np.empty(n)
    Vh, Vl = np.empty((n, n)), np.empty((n, n))
    sw = lib().oracle_jacobi_q(n, _p(Ah), _p(Al), tol, _p(wh), _p(wl), _p(Vh), _p(Vl))
    return wh, wl, Vh, Vl, sw


def num_threads():
    return int(lib().oracle_num_threads())
