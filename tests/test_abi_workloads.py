"""CPU checks (-m "not gpu"): libozr.so builds, loads without a GPU and exports every symbol that
include/ozr.h declares; host-only planning agrees with the oracle's plan; the product path refuses to
run without a GPU (no CPU fallback); the seeded workloads have the paper's structure."""
import ctypes
import json
import os
import re
import subprocess
import sys

import numpy as np
import pytest

import workloads as W
from oracle import products as opr

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def libozr():
    from paper_2602_19090_b200 import build
    build.build()
    import paper_2602_19090_b200 as ozr
    return ozr.lib()


def test_header_symbols_exported(libozr):
    hdr = open(os.path.join(ROOT, "include", "ozr.h")).read()
    declared = set(re.findall(r"\b(ozr_[a-z_0-9]+)\s*\(", hdr))
    assert {"ozr_split", "ozr_gemm", "ozr_refine_step", "ozr_refine_to_tol"} <= declared
    out = subprocess.check_output(["nm", "-D", "--defined-only", os.path.join(ROOT, "paper_2602_19090_b200",
                                                                              "libozr.so")]).decode()
    exported = set(re.findall(r"\bT (ozr_[a-z_0-9]+)", out))
    assert declared <= exported, declared - exported
    for s in declared:
        assert hasattr(libozr, s)


def test_no_torch_types_in_abi():
    hdr = open(os.path.join(ROOT, "include", "ozr.h")).read()
    assert not re.search(r"\btorch\b|at::|Tensor|c10", hdr)


def test_version_and_plan_on_cpu(libozr):
    import paper_2602_19090_b200 as ozr
    assert "sm_100a" in ozr.ozr_version()
    for K, kA, kB, L in [(1024, 12, 6, 13), (16384, 15, 7, 16), (50000, 3, 3, 0), (100, 4, 4, 5)]:
        plan = ozr.ozr_gemm_plan(K, kA, kB, L)
        want = [(d, len(p)) for d, p in opr.plan_groups(kA, kB, L if L > 0 else kA + kB, K)]
        assert plan == want


def test_params_default(libozr):
    import paper_2602_19090_b200 as ozr
    p = ozr.default_params()
    assert p.kA_split == 15 and p.truncate == 1 and p.beta_mode == 0 and abs(p.theta_V - 1 / 16) < 1e-18
    # the ctypes mirror of ozr_params matches the C layout up to its last field
    assert p.theta == 4.0 and p.cluster_mode == 1 and p.max_cluster == 16384 and p.form_R == 0
    assert p.dense_cluster == 64 and p.row_nnz == 0 and p.max_escalations == 2

def test_ctypes_structs_match_header(tmp_path):
    """The binding's ctypes mirrors of ozr_params / ozr_step_report have the C header's size and field
    offsets (compiled with gcc against include/ozr.h)."""
    import paper_2602_19090_b200 as ozr
    fields_p = [f for f, _ in ozr.Params._fields_]
    fields_r = [f for f, _ in ozr.StepReport._fields_]
    src = ["#include <stddef.h>", "#include <stdio.h>", '#include "ozr.h"', "int main(void) {",
           '  printf("%zu %zu\\n", sizeof(ozr_params), sizeof(ozr_step_report));']
    src += [f'  printf("%zu\\n", offsetof(ozr_params, {f}));' for f in fields_p]
    src += [f'  printf("%zu\\n", offsetof(ozr_step_report, {f}));' for f in fields_r]
    src += ["  return 0;", "}"]
    c = tmp_path / "layout.c"
    c.write_text("\n".join(src) + "\n")
    exe = tmp_path / "layout"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), "-o", str(exe), str(c)])
    vals = subprocess.check_output([str(exe)]).decode().split()
    assert int(vals[0]) == ctypes.sizeof(ozr.Params) and int(vals[1]) == ctypes.sizeof(ozr.StepReport)
    offs = [int(v) for v in vals[2:]]
    assert offs[:len(fields_p)] == [getattr(ozr.Params, f).offset for f in fields_p]
    assert offs[len(fields_p):] == [getattr(ozr.StepReport, f).offset for f in fields_r]


def test_no_cpu_fallback(libozr):
    """Without a CUDA device the product path fails loudly (status OZR_ERR_CUDA / RuntimeError)."""
    import torch

    import paper_2602_19090_b200 as ozr
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    h = ctypes.c_void_p()
    st = libozr.ozr_create(ctypes.byref(h), 0, None, 0)
    assert st == 6
    with pytest.raises(RuntimeError):
        ozr.Context(0)


def test_product_package_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2602_19090_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dp, f)).read()
                assert "oracle" not in re.sub(r"#.*|//.*", "", txt).replace("no oracle", ""), f


def test_workload_spectra_and_symmetry():
    A, lam = W.make_matrix(200, "geometric", 1e8, 1)
    assert np.array_equal(A, A.T)
    assert lam[0] == 1.0 and abs(lam[-1] - 1e-8) < 1e-22
    assert np.allclose(np.sort(np.linalg.eigvalsh(A))[::-1], lam, rtol=0, atol=1e-14)
    A2, _ = W.make_matrix(200, "geometric", 1e8, 1)
    assert np.array_equal(A, A2)  # seeded, deterministic
    lam3 = W.clustered_spectrum(4096, np.random.default_rng(1003))
    d = np.diff(lam3)
    assert lam3.size == 4096 and np.sum(np.abs(d - 1e-10) < 1e-15) >= 64 * 7
    assert np.all((lam3 >= -1) & (lam3 <= 1 + 1e-9))


def test_initial_eig_sign_and_precision():
    A, _ = W.make_matrix(128, "geometric", 1e6, 4)
    l64, X64 = W.initial_eig(A, "fp64")
    l32, X32 = W.initial_eig(A, "fp32")
    assert np.all(np.diff(l64) >= 0)
    idx = np.argmax(np.abs(X64), axis=0)
    assert np.all(X64[idx, np.arange(128)] > 0)
    assert np.max(np.abs(X32.astype(np.float32).astype(np.float64) - X32)) == 0  # an fp32 start


def test_householder_exact_eigensystem():
    A, lam, X, H, lc = W.householder_exact(5, lam_bits=10, seed=2)
    assert np.array_equal(A @ X, X * lam[None, :]) or np.max(np.abs(A @ X - X * lam[None, :])) < 1e-15


def test_bench_reference_arm_cpu():
    out = subprocess.check_output([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--n",
                                   "128", "--steps", "1", "--warmup", "0", "--ref-cols", "4"], cwd=ROOT)
    line = json.loads(out.decode().strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["value"] > 0 and line["e2e"]["h2d_bytes_per_step"] == 0
    assert line["cpu_baseline"]["kind"] == "oracle"


@pytest.mark.parametrize("kind", ["geometric", "clustered"])
def test_hadamard_exact_eigensystem_in_integers(kind):
    """W.hadamard_exact(pairs=False): A Q = Q Λ and QᵀQ = I hold EXACTLY — checked in Python integers on the
    numerators (n·Q, n²·2^b·A, 2^b·λ are integers), not in floating point."""
    m = 6
    n, b = 2 ** m, 53 - 2 * m - 2
    A, lam, X = W.hadamard_exact(m, kind, seed=11, pairs=False)
    NA = (A * float(n) ** 2 * 2.0 ** b)
    NL = lam * 2.0 ** b
    assert np.all(X * n == np.rint(X * n)) and np.all(NA == np.rint(NA)) and np.all(NL == np.rint(NL))
    NA = np.vectorize(int, otypes=[object])(NA)
    NL = np.vectorize(int, otypes=[object])(NL)
    NQ = np.vectorize(int, otypes=[object])(X * n)
    assert np.all(NQ.T.dot(NQ) == n * n * np.eye(n, dtype=object).astype(object))
    assert np.all(NA.dot(NQ) == n * n * (NQ * NL[None, :]))      # (n² 2^b A)(n Q) = n² (n Q)(2^b Λ)
    assert np.all(np.diff(lam) > 0) and np.all(NA == NA.T)
    if kind == "clustered":
        assert np.sum(np.diff(NL) == 1) == 7 * max(n // 64, 1)    # the designed clusters: gaps of one unit


@pytest.mark.parametrize("kind", ["geometric", "clustered"])
def test_hadamard_exact_pairs_closed_form_in_rationals(kind):
    """W.hadamard_exact (pairs: 2 x 2 integer blocks, irrational eigenvectors in closed form): A is the SAME kind of
    exact integer matrix (n²·2^b·A integer), and the returned fp64 (λ, X) satisfy A x − λ x and XᵀX − I to a few u
    when evaluated EXACTLY in rationals (so the bound is on the closed form's single rounding, not on the check's
    arithmetic). A wrong sign or a swapped (cos φ, sin φ) leaves a residual of the size of the coupling b."""
    from fractions import Fraction as Fr
    m = 5
    n, b = 2 ** m, 53 - 2 * m - 2
    A, lam, X = W.hadamard_exact(m, kind, seed=12)
    NA = A * float(n) ** 2 * 2.0 ** b
    assert np.all(NA == np.rint(NA)) and np.array_equal(A, A.T) and np.all(np.diff(lam) > 0)
    fr = np.vectorize(Fr, otypes=[object])
    Af, Xf, lf = fr(A), fr(X), fr(lam)
    R = Af.dot(Xf) - Xf * lf[None, :]
    G = Xf.T.dot(Xf) - np.eye(n, dtype=object)
    u = Fr(1, 2 ** 53)
    nrmA = max(abs(v) for v in lf)
    assert max(abs(v) for v in R.ravel()) <= 8 * u * nrmA
    assert max(abs(v) for v in G.ravel()) <= 8 * u
    # not the trivial family: the eigenvectors are not the dyadic columns of Q
    assert np.any(X * n != np.rint(X * n))
