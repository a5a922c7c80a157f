/* ozr.h — C ABI of libozr: forward-error-oriented Ogita–Aishima eigenvector refinement with an
 * INT8 Ozaki-scheme accurate product, native to NVIDIA B200 (sm_100a).
 *
 * Method: Terao & Ozaki, arXiv 2602.19090 (reference text: PAPER.md). Citations are PAPER.md lines.
 *   Problem: symmetric A, approximate eigenvectors X̂ (and D̂); return a
 *             refined X̂ with ‖X − X̂‖₂ ≈ δ and the Rayleigh-quotient eigenvalues D̂.
 *   Sweep     (Algorithm 1) with the one-sided accurate product (§3.1/§3.3,
 *             PAPER.md:308-317, 400-421) and the tuned β of §4.1.
 *   Splitting (§2.3, eq. sigma/tau/a/x) realised as INT8 digit planes
 *             (readings R4-R7).
 *
 * Conventions (all entry points):
 *   - Matrix pointers are DEVICE pointers to column-major storage with the given leading dimension
 *     (in elements). Vectors (lambda, exponents) are device pointers unless marked "host".
 *   - The caller owns every buffer passed in; the library owns only the workspace inside the context
 *     (allocated lazily and grown on demand, freed by ozr_destroy).
 *   - Work is issued on the context's stream. ozr_split and ozr_gemm are stream-ordered and do not
 *     synchronise; ozr_refine_step / ozr_refine_to_tol synchronise a few times per sweep to read
 *     scalars that choose digit budgets, and return with all work complete.
 *   - Errors never cross the ABI as exceptions: every call returns an ozr_status; the text of the last
 *     error is available from ozr_last_error(ctx). On error, outputs are unspecified and inputs are
 *     untouched, except OZR_ERR_NOT_CONVERGED (see ozr_refine_to_tol).
 *   - Results are deterministic (fixed reduction orders, integer accumulation, no FP atomics).
 *   - A context is not thread-safe; use one per host thread and device.
 */
#ifndef OZR_H_
#define OZR_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ozr_ctx_s* ozr_ctx;

typedef enum {
  OZR_OK = 0,
  OZR_ERR_ARG = 1,           /* bad argument: null pointer, bad size/stride/leading dimension, bad mode */
  OZR_ERR_NONFINITE = 2,     /* NaN or Inf in an input matrix */
  OZR_ERR_RANGE = 3,         /* δ ≤ u, digit count out of range, or an exponent/int range limit exceeded */
  OZR_ERR_DEGENERATE = 4,    /* r_j ≥ 1 (zero column), or equal eigenvalue estimates with the cluster
                                branch disabled (PAPER.md:333 assumes distinct eigenvalues) */
  OZR_ERR_NOT_CONVERGED = 5, /* stagnation / divergence; X and lambda hold the last accepted sweep */
  OZR_ERR_CUDA = 6,          /* CUDA runtime error (message in ozr_last_error) */
  OZR_ERR_COMM = 7,          /* collective (NCCL / host group) failure, or NCCL not loadable */
  OZR_ERR_NOMEM = 8          /* device allocation failed */
} ozr_status;

/* Library version string (static storage). */
const char* ozr_version(void);

/* Create a context on CUDA device `device`, issuing work on `stream` (a cudaStream_t; NULL = the
 * legacy default stream). n_max is a sizing hint for the workspace (0 = grow on demand). */
ozr_status ozr_create(ozr_ctx* out, int device, void* stream, int64_t n_max);
void ozr_destroy(ozr_ctx ctx);
const char* ozr_last_error(ozr_ctx ctx);

/* ------------------------------------------------------------------------------------------------
 * ozr_split — error-free splitting into INT8 digit planes (§2.3, eq. tau/x lines 176-193).
 *
 * mode OZR_SPLIT_FIXED (k = k_or_beta, 1..15): per-line exponent e = ⌈log2 max|m|⌉ (0 for a zero
 *   line), LSB exponent ℓ = e − (8(k−1)+6), integer p = RNE(m·2^−ℓ) [+ RNE(m_lo·2^−ℓ) when M_lo is
 *   given: the double-double M + M_lo], written as k "excess-128" base-256 digits d_1..d_k in
 *   [−128, 127], p = Σ d_s 256^{k−s} (R5/R6).
 * mode OZR_SPLIT_X1 (β = k_or_beta, 2..52): the proposed method's truncation X̂ → X̂^(1),
 *   x^(1) = fl(fl(τ_j + x) − τ_j), τ_j = 0.75·2^{⌈log2 w_j⌉}·2^β (eq. tau/x with s = 1); the digits
 *   are those of q = x^(1)/2^{g_j}, g_j = ⌈log2 w_j⌉ + β − 53, with k = k_X(β) = smallest k such that
 *   8(k−1)+6 ≥ 53−β, and ℓ_j = g_j. COLWISE only. If x1_out is non-null it receives X̂^(1) (fp64).
 *
 * axis OZR_COLWISE: one exponent per column of M (rows x cols); digit plane p holds element (i,j) at
 *   digits[p*plane_stride + j*ldd + i] (ldd ≥ rows).
 * axis OZR_ROWWISE: one exponent per row; plane p holds element (i,j) at digits[p*plane_stride +
 *   i*ldd + j] (ldd ≥ cols) — the digits of Mᵀ column-wise (FIXED mode only).
 * ldd and plane_stride are in bytes and must be multiples of 16 (TMA requirement).
 * lsb_exp (device, int32[cols or rows]) receives ℓ. k_out (host, nullable) receives k.
 * Errors: OZR_ERR_ARG, OZR_ERR_RANGE (k or β out of range), OZR_ERR_NONFINITE (checked).
 * ------------------------------------------------------------------------------------------------ */
enum { OZR_COLWISE = 0, OZR_ROWWISE = 1 };
enum { OZR_SPLIT_FIXED = 0, OZR_SPLIT_X1 = 1 };
ozr_status ozr_split(ozr_ctx ctx, const double* M, const double* M_lo, int64_t rows, int64_t cols, int64_t ldm,
                     int axis, int mode, int k_or_beta, int8_t* digits, int64_t ldd, int64_t plane_stride,
                     int32_t* lsb_exp, double* x1_out, int64_t ldx1, int* k_out);

/* ------------------------------------------------------------------------------------------------
 * ozr_gemm — accurate product C = A·B by the Ozaki scheme (§2.3) with INT8
 * digits: A (m x k) split ROWWISE into kA digits, B (k x n) COLWISE into kB digits, keep digit pairs
 * with s + t ≤ L (L = 0: all kA·kB pairs), each group of pairs of one diagonal d = s+t accumulated
 * exactly in int32 on the tcgen05 tensor cores (K·pairs·2^14 < 2^31), then recombined exactly and
 * rounded once to double-double: C_hi = RN(c), C_lo = RN(c − C_hi) for the exact value c of the kept
 * pairs when it fits one int128 Horner chunk (otherwise a deterministic chunked sum, error < 2^-104|c|).
 * C_lo may be NULL (fp64 result C_hi only). planes (nullable, device): the int32 group planes,
 * element (i,j) of group g at planes[g*plane_stride + j*m + i] (plane_stride in elements ≥ m*n).
 * ngroups_out (host, nullable). Errors: OZR_ERR_ARG, OZR_ERR_RANGE (kA/kB not in 1..15, k ≥ 2^31/2^14).
 * ------------------------------------------------------------------------------------------------ */
ozr_status ozr_gemm(ozr_ctx ctx, int64_t m, int64_t n, int64_t k, const double* A, int64_t lda, const double* B,
                    int64_t ldb, int kA, int kB, int L, double* C_hi, double* C_lo, int64_t ldc, int32_t* planes,
                    int64_t plane_stride, int* ngroups_out);

/* Host-only: the group plan ozr_gemm uses for contraction length k (pairs (s,t), 1≤s≤kA, 1≤t≤kB,
 * s+t ≤ L, by ascending diagonal then s, diagonals cut into chunks of ≤ ⌊(2^31−1)/(k·2^14)⌋ pairs).
 * group_diag / group_npairs receive up to max_groups entries. */
ozr_status ozr_gemm_plan(int64_t k, int kA, int kB, int L, int* ngroups, int* group_diag, int* group_npairs,
                         int max_groups);

/* ------------------------------------------------------------------------------------------------
 * Refinement (Algorithm 1, one-sided product §3.3, β of §4.1 by default).
 * ------------------------------------------------------------------------------------------------ */
typedef struct {
  double delta;      /* prescribed forward error δ (> u)                                     */
  double theta;      /* β and the budgets are chosen for δ' = δ/θ (R11; default 4) */
  int beta_mode;     /* 0: §4.1 tuned β (⌊·⌋, nδ) [default]; 1: §3.3 eq. proposed_beta (⌈·⌉, ξ);
                        2: §4.3 sparse β (γ·min(k, √n), k = row_nnz)              */
  double xi;         /* ξ for beta_mode 1 (0 → n)                                            */
  int beta_override; /* > 0: use this β instead of the formula                               */
  int truncate;      /* 1: X̂ → X̂^(1) (the proposed method) [default]; 0: keep all of X̂        */
  int max_sweeps;    /* ozr_refine_to_tol: sweep limit (default 6)                            */
  int kA_split;      /* digits of the one-time A split (default 15)                          */
  double theta_V, theta_W, theta_U; /* accuracy targets of the three products as fractions of δ'·gap (V, W)
                                       and δ' (X̂Ẽ) (R8; defaults 1/16, 1/16, 1/16)  */
  int L_V, L_W, L_U; /* > 0: force the pair budgets (s+t ≤ L) instead of the planner          */
  int cluster_mode;  /* 0: the paper's Algorithm 1 — equal λ̂ are an error;
                        1: unresolved groups (|ẽ_ij| > κ or λ̂_i = λ̂_j) get a Rayleigh–Ritz sub-solve
                           in span(X̂^(1)_J) (R13) [default]                          */
  int tile_budgets;  /* 1: per-256-column pair budgets from the local gaps gap_j (R8b) [default]  */
  double kappa;      /* cluster_mode 1: linearisation threshold κ on |ẽ_ij| (default 2^-10)     */
  int max_cluster;   /* cluster_mode 1: largest group solved (default 16384; larger → OZR_ERR_RANGE) */
  int form_R;        /* 1: also form R = I − X̂^(1)ᵀX̂^(1) by INT8 slice products (to θ_W·δ' absolute; the
                        R/S form's first product, PAPER.md:241-250 — Algorithm 1's W-form needs only its
                        diagonal, which is always exact); reports ‖R‖_F and the OA threshold ω, and
                        ozr_last_R returns R. Default 0 */
  int dense_cluster; /* cluster_mode 1: groups of at least this many columns are solved by a dense symmetric
                        eigensolver (ozr_syev: Householder tridiagonalisation, divide and conquer, back-
                        transformation, all in libozr's kernels) instead of the parallel Jacobi; same K,
                        same conventions (R13).
                        Default 64 (smaller groups: one Jacobi CTA each, all groups in one launch) */
  int row_nnz;       /* k = maximum number of nonzeros in a row of A (beta_mode 2; also the contraction
                        length of the V-product's dropped-pair bound, R8). 0 → n (dense)            */
  int max_escalations; /* ozr_refine_to_tol: when the certified error stalls above δ at the truncated iteration's
                          floor (R12), continue with θ × 4^m (β m bits lower, m from the estimate) at most
                          this many times before OZR_ERR_NOT_CONVERGED. Default 2 */
  int certify;       /* the a-posteriori forward-error certificate (R12, report.cert): 0 never — ozr_refine_to_tol
                        then runs max_sweeps sweeps (the paper's fixed iteration count) and
                        returns OZR_ERR_NOT_CONVERGED with X, λ from the last sweep; 1 after every sweep of
                        ozr_refine_to_tol without unresolved groups [default]; 2 also in ozr_refine_step  */
  int fixed_k;       /* > 0: the prior work's two-sided fixed-slice plan instead of the proposed method
                        (PAPER.md:217-227 eq. mat3-mat10, cost model PAPER.md:437-443): X̂ is not truncated
                        and every product keeps the ½k(k+1) leading digit pairs s + t ≤ k + 1 (truncate = 0,
                        L_V = L_W = L_U = k + 1, Res and Ẽ' split into exactly k digits; the products of
                        ozr_gemm(kA = kB = k, L = k + 1)).
                        Default 0 (the proposed method)                                              */
} ozr_params;

void ozr_params_default(ozr_params* p);

typedef struct {
  int sweep;
  int beta, beta_raw, alpha;        /* β used (clamped to [2,52]), formula β, reported α (§4.1)       */
  int kX, kA, kR, kE;               /* digit counts of X̂^(1), A (prefix used), Res, Ẽ'               */
  int L_V, L_W, L_U;                /* pair budgets                                                    */
  int pairs_V, pairs_W, pairs_U;    /* INT8 slice products (each an n x n_local x n INT8 GEMM)         */
  int n_clusters;                   /* unresolved groups given the Rayleigh–Ritz sub-solve (R13)       */
  int max_cluster;                  /* size of the largest such group                                  */
  int launches;                     /* CUDA kernels this sweep launched                                */
  int exchanges;                    /* collectives this rank issued (0 on one GPU)                     */
  double gap_min, max_abs_lambda;   /* from the λ̂ that chose β                                         */
  double normE_fro;                 /* ‖Ẽ‖_F                                                          */
  double net_update;                /* ν = ‖X̂_new − X̂_old‖_F                                          */
  double predicted_error;           /* ν² max|λ̂| / (n gap) (eq. assume2 with ξ = n), information       */
  double ms_total, ms_gemm;         /* device time of the sweep and of its slice-product kernels       */
  double int8_ops;                  /* 2·m·n·k·pairs summed over the sweep's slice products            */
  int pairs_G;                      /* form_R: pairs of the X̂ᵀX̂ slice product                          */
  double normR_fro, normW_fro;      /* form_R: ‖R‖_F, ‖W‖_F                                            */
  double omega_oa;                  /* form_R: ω = 2(‖W‖_F + 2·max|λ̂|·‖R‖_F), the Frobenius form of the
                                       OA-2018 cluster threshold 2(‖S − D̃‖ + ‖A‖‖R‖) (diagnostic, R13) */
  double theta;                     /* the θ this sweep used (params.theta, × 16 per escalation)       */
  double cert;                      /* a-posteriori estimate of ‖X − X̂_new‖₂ (R12): sqrt(‖D‖₂² + (2u)²)
                                       + ‖Ẽ‖_F‖D‖_F + 2u‖(λ̂_i ẽ_ij/(λ̂_j − λ̂_i))_{i≠j}‖_F (the last term: the
                                       fp64 rounding of the λ̂ in Ẽ's denominators) with Ẽ's second-order
                                       defect D = −(E − Ẽ):
                                       D_ij = q_ij/(λ̂_j − λ̂_i) − (Ẽ²)_ij (i ≠ j), D_jj = −(Ẽ²)_jj − ½‖ẽ_j‖²,
                                       Q = ẼᵀC, c_kj = (λ̂_k − λ̂_j)ẽ_kj; −1 when not evaluated
                                       (params.certify, or unresolved groups)                           */
  double cert_q;                    /* its ‖D‖₂ (Golub–Kahan–Lanczos; ‖D‖_F when that already decides)   */
  double cert_frob;                 /* ‖D‖_F                                                            */
  int cert_iters;                   /* Lanczos steps of the certificate                                 */
  double planes_V, planes_W, planes_U; /* int32 group planes recombined per element, averaged over the
                                          columns (per-tile budgets): 4 × this = the plane bytes per element
                                          the recombination kernels read                                   */
} ozr_step_report;

/* One sweep on columns [0, n): A (n x n, symmetric — only its columns are read), X (n x n, in/out:
 * X̂ → X̂^(1)(I + Ẽ) rounded to fp64), lambda (device, n, in: λ̂ of the previous sweep / the initial
 * eigensolver, used for β and the digit budgets; out: the new Rayleigh quotients). report: host.
 * Errors: OZR_ERR_ARG, OZR_ERR_RANGE (δ ≤ u), OZR_ERR_DEGENERATE, OZR_ERR_CUDA, OZR_ERR_NOMEM. */
ozr_status ozr_refine_step(ozr_ctx ctx, const double* A, int64_t n, int64_t lda, double* X, int64_t ldx,
                           double* lambda, const ozr_params* params, ozr_step_report* report);

/* ozr_refine_step_herm — the Hermitian extension ("the proposed method can be extended in a
 * straightforward manner to Hermitian matrices"; reading R18): one sweep of Algorithm 1
 * with conjugate transposes — V = A·X̂^(1), r_j = 1 − x̂_jᴴx̂_j, λ̂_j = Re(x̂_jᴴv_j)/(1 − r_j),
 * W = X̂ᴴ(V − X̂D̂), ẽ_ij = w_ij/(λ̂_j − λ̂_i), ẽ_jj = r_j/2, X̂ ← RN(X̂^(1) + X̂^(1)Ẽ) — with the truncation
 * X̂ → X̂^(1) of §3.1 on both parts (one τ_j per column from max_i max(|Re x̂_ij|, |Im x̂_ij|)) and β of §4.1.
 * Planar complex storage, column-major, device pointers: A = Ar + i·Ai (n x n, Hermitian: Ar symmetric, Ai
 * antisymmetric; lda ≥ n), X = Xr + i·Xi (n x n, in/out, ldx ≥ n), lambda (n, in: previous estimates, out: the
 * new Rayleigh quotients). Each complex product is one real INT8 slice product of the real-stacked operands
 * (2n-long contractions), budgets from the accuracy each product needs (R8, per product); params: delta, theta,
 * theta_V/W/U, beta_mode/xi, beta_override, L_V/L_W/L_U (cluster_mode, certify, fixed_k and tile budgets do
 * not apply: equal estimates are OZR_ERR_DEGENERATE). report: host, nullable (cert = −1).
 * Errors: OZR_ERR_ARG, OZR_ERR_RANGE, OZR_ERR_DEGENERATE, OZR_ERR_NONFINITE, OZR_ERR_CUDA, OZR_ERR_NOMEM. */
ozr_status ozr_refine_step_herm(ozr_ctx ctx, const double* Ar, const double* Ai, int64_t n, int64_t lda, double* Xr,
                                double* Xi, int64_t ldx, double* lambda, const ozr_params* params,
                                ozr_step_report* report);

/* The R = I − X̂^(1)ᵀX̂^(1) of the context's last sweep run with params.form_R = 1: this rank's columns
 * (n x n_local, column-major) copied to R (device, ldr ≥ n). OZR_ERR_ARG if none was formed. */
ozr_status ozr_last_R(ozr_ctx ctx, double* R, int64_t ldr);

/* Host: the unresolved groups of the context's last sweep (cluster_mode 1). members receives the global
 * column indices of every group, concatenated, each group in ascending (λ̂, index) order; offsets[g] is
 * the start of group g (offsets has ngroups + 1 entries). Returns OZR_ERR_RANGE if a buffer is too small
 * (*ngroups / offsets still tell the sizes needed when offsets has room). */
ozr_status ozr_last_clusters(ozr_ctx ctx, int* members, int max_members, int* offsets, int max_groups, int* ngroups);

/* Repeat sweeps until the returned X̂ is certified (R12; the paper iterates a fixed number of times,
 * PAPER.md:536-540): after every sweep without unresolved groups, the a-posteriori estimate report.cert of
 * ‖X − X̂‖₂ (the 2-norm of PAPER.md:121) is formed from the sweep's own Ẽ — the second-order defect of Alg. 1's
 * correction, two bf16 tensor-core products (Q = ẼᵀC, Ẽ²) and Golub–Kahan–Lanczos — and the call returns OZR_OK with
 * that X̂ once cert·1.15 ≤ δ. An estimate that stalls above δ (the truncated iteration's floor, quadratic in
 * 2^-β: it fell by less than 8x, or the next sweep's quadratic part cert³/prev² is below δ/8 while
 * cert ≤ 16δ — prev the previous estimate, or net_update when the previous sweep had none and an escalation is
 * left) escalates θ ← θ·4^m up to max_escalations times, then OZR_ERR_NOT_CONVERGED, as does
 * reaching max_sweeps — X / lambda then hold the last completed sweep. Sweeps with unresolved groups (cluster
 * sub-solves rotate columns) are neither certified nor compared. history (host, nullable) receives up to
 * max_hist reports; sweeps_done (host, nullable). */
ozr_status ozr_refine_to_tol(ozr_ctx ctx, const double* A, int64_t n, int64_t lda, double* X, int64_t ldx,
                             double* lambda, const ozr_params* params, ozr_step_report* history, int max_hist,
                             int* sweeps_done);

/* ------------------------------------------------------------------------------------------------
 * Multi-GPU: block-column partition of X̂. Rank r of P owns the columns
 * [r·n/P, (r+1)·n/P) of X̂ (n % P == 0; a P-rank result equals the 1-GPU result bit for bit when n/P
 * is a multiple of 256). A (n x n) and λ̂ (n) are replicated. Per sweep the ranks all-gather the digit
 * planes of X̂^(1) and the column exponents g (the left operand of W = X̂ᵀRes and of X̂Ẽ), the column
 * maxima w, λ̂ and a few scalars, plus — only when an unresolved group spans ranks — its W_JJ and
 * Ẽ_{:,J} blocks. The paper itself is single-node dense (§4); the partition is the build's.
 *
 * Communicators:
 *   ozr_comm_nccl_id        rank 0: a 128-byte NCCL unique id to broadcast to the other ranks
 *   ozr_comm_create_nccl    every rank, CUDA device `device` (NCCL is dlopen'ed: libnccl.so.2)
 *   ozr_comm_create_host_group  `nranks` communicators (out[0..nranks-1]) for ranks that are host
 *                           threads of ONE process sharing memory (device→host→device exchange):
 *                           the harness that runs the multi-rank protocol on a single GPU
 * Errors: OZR_ERR_ARG, OZR_ERR_COMM (message in *_last_error is not available: no context; the
 * status says what failed).
 * ------------------------------------------------------------------------------------------------ */
/* ------------------------------------------------------------------------------------------------
 * ozr_syev — the dense symmetric eigensolver of the Rayleigh–Ritz sub-solve of large unresolved groups
 * (reading R13; the paper leaves clusters open, and cites the Ogita–Aishima
 * cluster refinement, whose sub-problem is a small dense symmetric eigenproblem):
 * K = Y diag(θ) Yᵀ by Householder tridiagonalisation, Cuppen divide and conquer with Gu–Eisenstat
 * eigenvectors, and the blocked back-transformation, all in libozr's own kernels (products with a
 * dimension ≥ 1024 on the INT8 slice GEMM at FP64 accuracy).
 * K: device, m x m column-major (ldk ≥ m), symmetric; only its lower triangle is read; K is preserved.
 * theta: device, m, ascending. Y: device, m x m (ldy ≥ m), orthonormal columns (sign not normalised).
 * Workspace ~5m² doubles inside the context. Errors: OZR_ERR_ARG, OZR_ERR_NONFINITE (not checked: NaN
 * propagates), OZR_ERR_CUDA (no convergence of a leaf iteration), OZR_ERR_NOMEM.
 * ------------------------------------------------------------------------------------------------ */
ozr_status ozr_syev(ozr_ctx ctx, int64_t m, const double* K, int64_t ldk, double* theta, double* Y, int64_t ldy);
/* Its two stages alone (stage checks): ozr_syev_tridiag overwrites K (device, m x m, ldk = m, lower triangle read)
 * with the Householder vectors v_c below its sub-diagonal (v_{c+1} = 1 implied; H_c = I − τ_c v_c v_cᵀ,
 * H_0⋯H_{m−2} K H_{m−2}⋯H_0 = T) and writes T's diagonal d (m), sub-diagonal e (m − 1 used) and τ (m − 1 used);
 * ozr_syev_tridiag_eig returns θ ascending and the eigenvectors Y (m x m, ldy = m) of the tridiagonal (d, e). */
ozr_status ozr_syev_tridiag(ozr_ctx ctx, int64_t m, double* K, int64_t ldk, double* d, double* e, double* tau);
ozr_status ozr_syev_tridiag_eig(ozr_ctx ctx, int64_t m, const double* d, const double* e, double* theta, double* Y,
                                int64_t ldy);

typedef struct ozr_comm_s* ozr_comm;
ozr_status ozr_comm_nccl_id(void* id128);
ozr_status ozr_comm_create_nccl(ozr_comm* out, const void* id128, int nranks, int rank, int device);
ozr_status ozr_comm_create_host_group(ozr_comm* out, int nranks);
void ozr_comm_destroy(ozr_comm comm);
int ozr_comm_size(ozr_comm comm);
int ozr_comm_rank(ozr_comm comm);

/* ozr_refine_step / ozr_refine_to_tol on this rank's column block. X is the full n x n column-major
 * array (ldx ≥ n) of which only columns [col0, col0 + n/P), col0 = rank·n/P, are read and written;
 * lambda (n, replicated) is in/out on every rank; reports are identical on every rank. comm = NULL is
 * the single-GPU call. Every rank must make the same calls with the same parameters. */
ozr_status ozr_refine_step_dist(ozr_ctx ctx, ozr_comm comm, const double* A, int64_t n, int64_t lda, double* X,
                                int64_t ldx, double* lambda, const ozr_params* params, ozr_step_report* report);
ozr_status ozr_refine_to_tol_dist(ozr_ctx ctx, ozr_comm comm, const double* A, int64_t n, int64_t lda, double* X,
                                  int64_t ldx, double* lambda, const ozr_params* params, ozr_step_report* history,
                                  int max_hist, int* sweeps_done);

#ifdef __cplusplus
}
#endif
#endif /* OZR_H_ */
