// cluster.cu — the clustered-eigenvalue branch of the Ẽ correction (reading R13; the paper
// assumes distinct eigenvalues, and leaves clusters open).
//
// Unresolved groups J (connected components of the pairs with |ẽ_ij| > κ or λ̂_i = λ̂_j, found on the
// host from the edge list k_recombine_E emits) get a Rayleigh–Ritz sub-solve in span(X̂^(1)_J), restated
// from the Ogita–Aishima cluster refinement cited at PAPER.md:233-235:
//   G_JJ = X̂_JᵀX̂_J (exact, from the integer digits), R_JJ = I − G_JJ (diagonal: the exact r_j),
//   M = W_JJ + (I − R_JJ)(D̂_J − μI)      (= S_JJ − μG_JJ since S = W + (I − R)D̂, Alg. 1 line 4)
//   K = C·(M + Mᵀ)/2·C,  C = I + R_JJ/2   (C ≈ G_JJ^{-1/2})
//   K = YΘYᵀ (cyclic parallel Jacobi, Θ ascending, y_kk ≥ 0),  Z = C·Y
//   Ẽ_JJ ← Z − I,  Ẽ_{i,J} ← Ẽ_{i,J}·Z (i ∉ J),  λ̂_J ← μ + Θ.
// All on Ẽ' = diag(2^g)Ẽ, the scaled matrix the X̂Ẽ product consumes (rows scale, Z acts on columns).
//
//   k_cluster_build   (group, 16x16 tile of (a,b)): exact g_ab from the digits (int128), w_ab from the
//                     W slice-product planes, M_ab and R_ab into the group's workspace
//   k_cluster_jacobi  one CTA per group: K, Jacobi, sort, sign, Z = C·Y, λ̂_J
//   k_cluster_gather  T = Ẽ'[:, J] (compact copy, the apply reads old values)
//   k_cluster_apply   Ẽ'[:, J] ← T·Z off the group rows, (Z − I)·2^{g_i} on them
//   k_cluster_colstats column maxima exponents and ‖ẽ_j‖² of the rewritten columns
#include <cooperative_groups.h>
#include <cstdint>
#include <cuda_runtime.h>

#include "ddmath.cuh"
#include "kernels.h"
#include "ozr_internal.h"

#include <algorithm>

namespace ozr {

namespace cg = cooperative_groups;

namespace {

// Horner recombination of one element of a slice-product (same contract as kernels.cu; kept local so
// the cluster kernels do not depend on that translation unit's internals).
__device__ __forceinline__ dd recomb_one(const int32_t* __restrict__ planes, long long pstride, long long off,
                                         const RecombPlan& rp, int e, int Lj) {
  dd acc{0.0, 0.0};
  bool first = true;
  for (int c = 0; c < rp.nchunks; ++c) {
    i128 T = 0;
    int dprev = rp.diag[rp.chunk_first[c]];
    for (int g = rp.chunk_first[c]; g < rp.chunk_first[c + 1]; ++g) {
      const int d = rp.diag[g];
      const int32_t cv = (d <= Lj) ? planes[g * pstride + off] : 0;
      T = static_cast<i128>(static_cast<u128>(T) << (8 * (d - dprev))) + static_cast<i128>(cv);
      dprev = d;
    }
    dd v = i128_to_dd(T);
    const int sc = 8 * (rp.L - dprev) + e;
    v.hi = ldexp_fast(v.hi, sc);
    v.lo = ldexp_fast(v.lo, sc);
    acc = first ? v : dd_add(acc, v);
    first = false;
  }
  return acc;
}

// q = Σ_s d_s 256^{k−s} from the k digit planes of column `col`, row `row`.
__device__ __forceinline__ long long digits_q(const int8_t* __restrict__ dig, long long ldd, long long pstride, int kx,
                                              int col, int row) {
  long long q = 0;
  const int8_t* p = dig + static_cast<long long>(col) * ldd + row;
  for (int s = 0; s < kx; ++s) q = q * 256 + static_cast<long long>(p[s * pstride]);
  return q;
}

constexpr int TB = 16;   // (a,b) tile edge of k_cluster_build
constexpr int KC = 64;   // rows per staged chunk

// Exact partial Gram sums Σ_{k in split} q_ki q_kj (int128 as two u64) of one 16 x 16 tile of (a,b) over
// one row split: grid (tile, split); partials[(tile·nsplit + split)·256 + thread] (lo, hi).
__global__ void __launch_bounds__(TB* TB)
    k_cluster_dot(const int4* __restrict__ tiles, const int* __restrict__ goff, const int* __restrict__ mem,
                  const int8_t* __restrict__ xdig, long long ldd, long long pstride, int kx, int rows, int nsplit,
                  unsigned long long* __restrict__ part) {
  __shared__ long long qa[KC][TB + 1];
  __shared__ long long qb[KC][TB + 1];
  const int4 t = tiles[blockIdx.x];  // (group, a0, b0, m)
  const int grp = t.x, a0 = t.y, b0 = t.z, m = t.w;
  const int tx = threadIdx.x % TB, ty = threadIdx.x / TB;
  const int* J = mem + goff[grp];
  const int span = ((rows + nsplit - 1) / nsplit + KC - 1) / KC * KC;
  const int r0 = blockIdx.y * span, r1 = min(rows, r0 + span);
  // exact Σ_k q_ki q_kj in int128 (|q| < 2^52, rows < 2^16)
  unsigned long long lo = 0;
  long long hi = 0;
  for (int k0 = r0; k0 < r1; k0 += KC) {
    for (int e = threadIdx.x; e < KC * TB; e += TB * TB) {
      const int kk = e % KC, c = e / KC;  // consecutive threads: consecutive rows of one column
      const int k = k0 + kk;
      qa[kk][c] = (k < r1 && a0 + c < m) ? digits_q(xdig, ldd, pstride, kx, J[a0 + c], k) : 0;
      qb[kk][c] = (k < r1 && b0 + c < m) ? digits_q(xdig, ldd, pstride, kx, J[b0 + c], k) : 0;
    }
    __syncthreads();
#pragma unroll 8
    for (int kk = 0; kk < KC; ++kk) {
      const long long x = qa[kk][ty], y = qb[kk][tx];
      const unsigned long long pl = static_cast<unsigned long long>(x) * static_cast<unsigned long long>(y);
      const long long ph = __mul64hi(x, y);
      const unsigned long long s = lo + pl;
      hi += ph + (s < lo ? 1 : 0);
      lo = s;
    }
    __syncthreads();
  }
  unsigned long long* o = part + ((static_cast<long long>(blockIdx.x) * nsplit + blockIdx.y) * (TB * TB) + threadIdx.x) * 2;
  o[0] = lo;
  o[1] = static_cast<unsigned long long>(hi);
}

__global__ void __launch_bounds__(TB* TB)
    k_cluster_build(const int4* __restrict__ tiles, const int* __restrict__ goff, const int* __restrict__ gsq,
                    const int* __restrict__ mem, const double* __restrict__ mu, int nsplit,
                    const unsigned long long* __restrict__ part, int rows, const int32_t* __restrict__ gexp,
                    const double* __restrict__ r_hi, const double* __restrict__ r_lo, const int32_t* __restrict__ wplanes,
                    long long wpstride, const __grid_constant__ RecombPlan rpW, const int32_t* __restrict__ ellR,
                    int scale8, const double* __restrict__ lam, double* __restrict__ Mbuf, double* __restrict__ Rbuf,
                    int col0, int ncols, int ntiles_dot, const double* __restrict__ Gbuf) {
  const int4 t = tiles[blockIdx.x];  // (group, a0, b0, m)
  const int grp = t.x, a0 = t.y, b0 = t.z, m = t.w;
  const int tx = threadIdx.x % TB, ty = threadIdx.x / TB;
  const int a = a0 + ty, b = b0 + tx;
  const int* J = mem + goff[grp];
  const bool from_digits = static_cast<int>(blockIdx.x) < ntiles_dot;
  unsigned long long lo = 0;
  long long hi = 0;
  if (from_digits)
    for (int q = 0; q < nsplit; ++q) {  // fixed order (exact anyway)
      const unsigned long long* p = part + ((static_cast<long long>(blockIdx.x) * nsplit + q) * (TB * TB) + threadIdx.x) * 2;
      const unsigned long long s = lo + p[0];
      hi += static_cast<long long>(p[1]) + (s < lo ? 1 : 0);
      lo = s;
    }
  if (a >= m || b >= m) return;
  const int i = J[a], j = J[b];
  double g;
  if (from_digits) {
    const i128 SQ = static_cast<i128>((static_cast<u128>(static_cast<unsigned long long>(hi)) << 64) | lo);
    const dd gdd = i128_to_dd(SQ);
    g = ldexp_fast(gdd.hi, gexp[i] + gexp[j]);
  } else {  // RN of the same exact integer, scaled by the same power of two (tensor-core Gram)
    g = Gbuf[static_cast<long long>(gsq[grp]) + static_cast<long long>(b) * m + a];
  }
  const double r = (a == b) ? (r_hi[i] + r_lo[i]) : -g;
  const long long o = static_cast<long long>(gsq[grp]) + static_cast<long long>(b) * m + a;
  Rbuf[o] = r;  // every rank (from the all-gathered digits)
  const int jl = j - col0;
  if (jl < 0 || jl >= ncols) {  // column owned by another rank: its M entries arrive by the all-reduce
    Mbuf[o] = 0.0;
    return;
  }
  // w_ij from the W = X̂ᵀRes slice-product planes (row i: ℓ = g_i, local column jl: ℓ = ℓ_Res,jl + scale)
  const int Lj = rpW.tile_budgets ? rpW.tileL[jl / 256] : rpW.L;
  const dd w = recomb_one(wplanes, wpstride, static_cast<long long>(jl) * rows + i, rpW, gexp[i] + ellR[jl] + scale8, Lj);
  const double mug = mu[grp];
  Mbuf[o] = (w.hi + w.lo) + ((a == b ? 1.0 : 0.0) - r) * (lam[j] - mug);
}

constexpr int JT = 512;        // threads of a Jacobi CTA
constexpr int kCoopMin = 192;  // groups at least this large use the whole-GPU cooperative kernel

// Execution policies of the Jacobi core: one CTA per group, or the whole (cooperative) grid on one group.
struct CtaExec {
  __device__ int tid() const { return threadIdx.x; }
  __device__ int nth() const { return blockDim.x; }
  __device__ void sync() const { __syncthreads(); }
  __device__ int any(int v, int* /*flag*/) const { return __syncthreads_or(v); }
};
struct GridExec {
  __device__ int tid() const { return blockIdx.x * blockDim.x + threadIdx.x; }
  __device__ int nth() const { return gridDim.x * blockDim.x; }
  __device__ void sync() const { cg::this_grid().sync(); }
  __device__ int any(int v, int* flag) const {  // flag: a fresh zeroed global int per call
    if (v) atomicOr(flag, 1);
    cg::this_grid().sync();
    return *reinterpret_cast<volatile int*>(flag);
  }
};

// tournament (round-robin) schedule: round r pairs position k with position mm−1−k; position 0 is fixed
__device__ __forceinline__ void rr_pair(int k, int r, int mm, int& p, int& q) {
  auto pos = [&](int x) { return x == 0 ? 0 : 1 + ((x - 1 + r) % (mm - 1)); };
  p = pos(k);
  q = pos(mm - 1 - k);
  if (p > q) {
    const int t = p;
    p = q;
    q = t;
  }
}

// Rayleigh–Ritz sub-solve of one group (see the header): K = C·(M+Mᵀ)/2·C, cyclic parallel Jacobi
// (tournament ordering, the K update of a round applied as independent 2x2 blocks J_aᵀ K_ab J_b),
// eigenvalues ascending (ties by index), y_kk ≥ 0, Z = C·Y, λ̂_J = μ + Θ. Deterministic: every phase is
// element-parallel with fixed arithmetic per element; the only reduction is an exact max.
// scratch: cs[np], sn[np], th[m], sg[m], perm[m], flags[>= 48], amax (1 u64).
template <class X>
__device__ void jacobi_group(const X& ex, int m, const double* __restrict__ M, const double* __restrict__ R,
                             double* __restrict__ K, double* __restrict__ V, double* __restrict__ Z, double* cs,
                             double* sn, double* th, double* sg, int* perm, int* flags, unsigned long long* amax, double mu,
                             const int* __restrict__ J, double* __restrict__ lam, int* sweeps_out) {
  const int tid = ex.tid(), nth = ex.nth();
  const long long m2 = static_cast<long long>(m) * m;
  const int mm = m + (m & 1), np = mm / 2;
  for (long long e = tid; e < m2; e += nth) {  // V ← K0 = (M + Mᵀ)/2
    const int a = static_cast<int>(e % m), b = static_cast<int>(e / m);
    V[e] = 0.5 * (M[e] + M[static_cast<long long>(a) * m + b]);
  }
  ex.sync();
  for (long long e = tid; e < m2; e += nth) {  // K ← C·K0, C = I + R/2
    const int a = static_cast<int>(e % m), b = static_cast<int>(e / m);
    double s = V[e];
    for (int l = 0; l < m; ++l) s = fma(0.5 * R[static_cast<long long>(l) * m + a], V[static_cast<long long>(b) * m + l], s);
    K[e] = s;
  }
  ex.sync();
  for (long long e = tid; e < m2; e += nth) {  // V ← K·C
    const int a = static_cast<int>(e % m), b = static_cast<int>(e / m);
    double s = K[e];
    for (int l = 0; l < m; ++l) s = fma(K[static_cast<long long>(l) * m + a], 0.5 * R[static_cast<long long>(b) * m + l], s);
    V[e] = s;
  }
  ex.sync();
  unsigned long long mx = 0;
  for (long long e = tid; e < m2; e += nth) {  // K ← sym(V); max |K| (exact, order-free)
    const int a = static_cast<int>(e % m), b = static_cast<int>(e / m);
    const double x = 0.5 * (V[e] + V[static_cast<long long>(a) * m + b]);
    K[e] = x;
    mx = max(mx, static_cast<unsigned long long>(__double_as_longlong(fabs(x))));
  }
  if (mx) atomicMax(amax, mx);
  ex.sync();
  for (long long e = tid; e < m2; e += nth) V[e] = ((e % m) == (e / m)) ? 1.0 : 0.0;
  const double tiny = 1e-18 * __longlong_as_double(static_cast<long long>(*reinterpret_cast<volatile unsigned long long*>(amax)));
  int sweeps = 0;
  for (int sw = 0; sw < 40; ++sw) {
    int rotated = 0;
    for (int r = 0; r < mm - 1; ++r) {
      for (int k = tid; k < np; k += nth) {  // rotation of pair k
        int p, q;
        rr_pair(k, r, mm, p, q);
        double c = 1.0, s = 0.0;
        if (q < m) {
          const double apq = K[static_cast<long long>(q) * m + p];
          if (fabs(apq) > tiny) {
            const double app = K[static_cast<long long>(p) * m + p], aqq = K[static_cast<long long>(q) * m + q];
            const double theta = (aqq - app) / (2.0 * apq);
            const double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(fma(theta, theta, 1.0)));
            c = 1.0 / sqrt(fma(t, t, 1.0));
            s = t * c;
            rotated = 1;
          }
        }
        cs[k] = c;
        sn[k] = s;
      }
      ex.sync();
      // K ← JᵀKJ as 2x2 blocks (rows of pair ka, columns of pair kb); V ← V·J (columns of pair kb)
      const long long nb = static_cast<long long>(np) * np, nv = static_cast<long long>(np) * m;
      for (long long e = tid; e < nb + nv; e += nth) {
        if (e < nb) {
          const int ka = static_cast<int>(e % np), kb = static_cast<int>(e / np);
          const double ca = cs[ka], sa = sn[ka], cb = cs[kb], sb = sn[kb];
          if (sa == 0.0 && sb == 0.0) continue;
          int p1, q1, p2, q2;
          rr_pair(ka, r, mm, p1, q1);
          rr_pair(kb, r, mm, p2, q2);
          const bool q1v = q1 < m, q2v = q2 < m;
          double* cp = K + static_cast<long long>(p2) * m;
          double* cq = K + static_cast<long long>(q2) * m;
          double x11 = cp[p1], x21 = q1v ? cp[q1] : 0.0;
          double x12 = q2v ? cq[p1] : 0.0, x22 = (q1v && q2v) ? cq[q1] : 0.0;
          // columns: [x·1, x·2] ← [c x·1 − s x·2, s x·1 + c x·2]
          double y11 = cb * x11 - sb * x12, y12 = sb * x11 + cb * x12;
          double y21 = cb * x21 - sb * x22, y22 = sb * x21 + cb * x22;
          // rows: [y1·; y2·] ← [c y1· − s y2·; s y1· + c y2·]
          cp[p1] = ca * y11 - sa * y21;
          if (q1v) cp[q1] = sa * y11 + ca * y21;
          if (q2v) {
            cq[p1] = ca * y12 - sa * y22;
            if (q1v) cq[q1] = sa * y12 + ca * y22;
          }
        } else {
          const long long e2 = e - nb;
          const int kb = static_cast<int>(e2 / m), row = static_cast<int>(e2 % m);
          const double sb = sn[kb];
          if (sb == 0.0) continue;
          const double cb = cs[kb];
          int p2, q2;
          rr_pair(kb, r, mm, p2, q2);
          double* vp = V + static_cast<long long>(p2) * m + row;
          double* vq = V + static_cast<long long>(q2) * m + row;
          const double x = *vp, y = *vq;
          *vp = cb * x - sb * y;
          *vq = sb * x + cb * y;
        }
      }
      ex.sync();
    }
    sweeps = sw + 1;
    if (!ex.any(rotated, flags + sw)) break;
  }
  // ascending Θ (ties by index), y_kk ≥ 0, Z = C·Y, λ̂_J = μ + Θ
  for (int k = tid; k < m; k += nth) th[k] = K[static_cast<long long>(k) * m + k];
  ex.sync();
  for (int k = tid; k < m; k += nth) {
    int rk = 0;
    const double x = th[k];
    for (int l = 0; l < m; ++l) rk += (th[l] < x || (th[l] == x && l < k)) ? 1 : 0;
    perm[rk] = k;
  }
  ex.sync();
  for (int k = tid; k < m; k += nth) {  // sign of sorted column k
    const int src = perm[k];
    double piv = V[static_cast<long long>(src) * m + k];
    if (piv == 0.0) {
      double best = -1.0;
      for (int l = 0; l < m; ++l) {
        const double v = V[static_cast<long long>(src) * m + l];
        if (fabs(v) > best) {
          best = fabs(v);
          piv = v;
        }
      }
    }
    sg[k] = piv < 0 ? -1.0 : 1.0;
  }
  ex.sync();
  for (long long e = tid; e < m2; e += nth) {  // Z[a,k] = Σ_l C[a,l] y_lk
    const int a = static_cast<int>(e % m), k = static_cast<int>(e / m);
    const double* y = V + static_cast<long long>(perm[k]) * m;
    double s = y[a];
    for (int l = 0; l < m; ++l) s = fma(0.5 * R[static_cast<long long>(l) * m + a], y[l], s);
    Z[e] = sg[k] * s;
  }
  for (int k = tid; k < m; k += nth) lam[J[k]] = mu + th[perm[k]];
  if (tid == 0) *sweeps_out = sweeps;
}

__global__ void __launch_bounds__(JT)
    k_cluster_jacobi(const int* __restrict__ goff, const int* __restrict__ gsq, const int* __restrict__ gm,
                     const int* __restrict__ mem, const double* __restrict__ mu, const double* __restrict__ Mbuf,
                     const double* __restrict__ Rbuf, double* __restrict__ Kbuf, double* __restrict__ Vbuf,
                     double* __restrict__ Zbuf, double* __restrict__ lam, int* __restrict__ sweeps_out,
                     int dense_min) {
  extern __shared__ double jsm[];  // cs[np] sn[np] th[m] sg[m] perm[m] | amax
  const int grp = blockIdx.x;
  const int m = gm[grp];
  if (m >= kCoopMin || m >= dense_min) return;  // solved by the cooperative kernel / the dense solver
  const int mm = m + (m & 1), np = mm / 2;
  double* cs = jsm;
  double* sn = cs + np;
  double* th = sn + np;
  double* sg = th + m;
  int* perm = reinterpret_cast<int*>(sg + m);
  unsigned long long* amax = reinterpret_cast<unsigned long long*>(jsm + 2 * np + 2 * m + (m + 1) / 2 + 1);
  if (threadIdx.x == 0) *amax = 0;
  __syncthreads();
  const long long o = gsq[grp];
  jacobi_group(CtaExec{}, m, Mbuf + o, Rbuf + o, Kbuf + o, Vbuf + o, Zbuf + o, cs, sn, th, sg, perm, nullptr, amax,
               mu[grp], mem + goff[grp], lam, sweeps_out + grp);
}

// One large group on the whole GPU (cooperative launch; grid-wide syncs between the phases).
__global__ void __launch_bounds__(JT)
    k_cluster_jacobi_coop(int grp, const int* __restrict__ goff, const int* __restrict__ gsq, const int* __restrict__ gm,
                          const int* __restrict__ mem, const double* __restrict__ mu, const double* __restrict__ Mbuf,
                          const double* __restrict__ Rbuf, double* __restrict__ Kbuf, double* __restrict__ Vbuf,
                          double* __restrict__ Zbuf, double* __restrict__ lam, int* __restrict__ sweeps_out,
                          double* __restrict__ scratch, int* __restrict__ flags) {
  const int m = gm[grp];
  const int mm = m + (m & 1), np = mm / 2;
  double* cs = scratch;
  double* sn = cs + np;
  double* th = sn + np;
  double* sg = th + m;
  int* perm = reinterpret_cast<int*>(sg + m);
  unsigned long long* amax = reinterpret_cast<unsigned long long*>(flags + 64);
  const long long o = gsq[grp];
  jacobi_group(GridExec{}, m, Mbuf + o, Rbuf + o, Kbuf + o, Vbuf + o, Zbuf + o, cs, sn, th, sg, perm, flags, amax, mu[grp],
               mem + goff[grp], lam, sweeps_out + grp);
}

__global__ void k_cluster_gather(const int* __restrict__ mem, int nmembers, const double* __restrict__ Ep, long long lde,
                                 int rows, double* __restrict__ T, int col0, int ncols) {
  const int c = blockIdx.x;  // member index over all groups
  if (c >= nmembers) return;
  const int jl = mem[c] - col0;
  const bool own = jl >= 0 && jl < ncols;  // other ranks' columns arrive by the all-reduce
  for (int i = blockIdx.y * blockDim.x + threadIdx.x; i < rows; i += gridDim.y * blockDim.x)
    T[static_cast<long long>(c) * rows + i] = own ? Ep[static_cast<long long>(jl) * lde + i] : 0.0;
}

constexpr int AK = 32;  // output columns per apply CTA

__global__ void __launch_bounds__(256)
    k_cluster_apply(const int* __restrict__ goff, const int* __restrict__ gsq, const int* __restrict__ gm,
                    const int* __restrict__ mem, const int* __restrict__ grp_of, const int* __restrict__ pos_of,
                    const double* __restrict__ T, const double* __restrict__ Zbuf, const int32_t* __restrict__ gexp,
                    int rows, double* __restrict__ Ep, long long lde, int col0, int ncols, int dense_min) {
  const int grp = blockIdx.z;
  const int m = gm[grp];
  const int k0 = blockIdx.y * AK;
  if (k0 >= m || m >= dense_min) return;  // dense groups: launch_dense_scatter
  const int kn = min(AK, m - k0);
  const double* Z = Zbuf + gsq[grp];
  const int* J = mem + goff[grp];
  const double* Tg = T + static_cast<long long>(goff[grp]) * rows;
  __shared__ double zs[64][AK];
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  double acc[AK];
#pragma unroll
  for (int q = 0; q < AK; ++q) acc[q] = 0.0;
  for (int l0 = 0; l0 < m; l0 += 64) {
    __syncthreads();
    for (int e = threadIdx.x; e < 64 * AK; e += blockDim.x) {
      const int l = l0 + e / AK, q = e % AK;
      zs[e / AK][q] = (l < m && q < kn) ? Z[static_cast<long long>(k0 + q) * m + l] : 0.0;
    }
    __syncthreads();
    if (i < rows) {
      const int lmax = min(64, m - l0);
      for (int l = 0; l < lmax; ++l) {
        const double t = Tg[static_cast<long long>(l0 + l) * rows + i];
#pragma unroll
        for (int q = 0; q < AK; ++q) acc[q] = fma(t, zs[l][q], acc[q]);
      }
    }
  }
  if (i >= rows) return;
  const bool in = grp_of[i] == grp;
  const int a = in ? pos_of[i] : 0;
#pragma unroll
  for (int q = 0; q < AK; ++q) {
    if (q >= kn) break;
    const int k = k0 + q;
    const int jl = J[k] - col0;
    if (jl < 0 || jl >= ncols) continue;  // owned by another rank
    double v = acc[q];
    if (in) v = ldexp_fast(Z[static_cast<long long>(k) * m + a] - (a == k ? 1.0 : 0.0), gexp[i]);
    Ep[static_cast<long long>(jl) * lde + i] = v;
  }
}

__global__ void __launch_bounds__(256)
    k_cluster_colstats(const int* __restrict__ mem, const double* __restrict__ Ep, long long lde, int rows,
                       const int32_t* __restrict__ gexp, double* __restrict__ nrm2, int32_t* __restrict__ eE_col,
                       int* __restrict__ eE_max, int col0, int ncols) {
  __shared__ double sh[2][8];
  const int jg = mem[blockIdx.x];
  const int j = jg - col0;  // local column
  if (j < 0 || j >= ncols) return;
  double m = 0.0, s2 = 0.0;
  for (int i = threadIdx.x; i < rows; i += 256) {
    const double ep = Ep[static_cast<long long>(j) * lde + i];
    const double e = ldexp_fast(ep, -gexp[i]);
    s2 = fma(e, e, s2);
    m = fmax(m, fabs(ep));
  }
  for (int o = 16; o > 0; o >>= 1) {
    m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    s2 = __dadd_rn(s2, __shfl_xor_sync(0xffffffffu, s2, o));
  }
  if ((threadIdx.x & 31) == 0) {
    sh[0][threadIdx.x >> 5] = m;
    sh[1][threadIdx.x >> 5] = s2;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double mx = sh[0][0], ss = sh[1][0];
    for (int w = 1; w < 8; ++w) {
      mx = fmax(mx, sh[0][w]);
      ss = __dadd_rn(ss, sh[1][w]);
    }
    nrm2[jg] = ss;
    const int e = (mx > 0.0) ? ceil_log2_d(mx) : -100000;
    eE_col[j] = e;
    if (mx > 0.0) atomicMax(eE_max, e);
  }
}

__global__ void k_gather_digit_cols(const int8_t* __restrict__ dig, long long ld, long long pstride, const int* __restrict__ J,
                                    int8_t* __restrict__ out, long long opstride, const int32_t* __restrict__ g,
                                    int32_t* __restrict__ gJ) {
  const int a = blockIdx.x, p = blockIdx.y;  // ld % 16 == 0: 16-byte copies
  const int4* src = reinterpret_cast<const int4*>(dig + p * pstride + static_cast<long long>(J[a]) * ld);
  int4* dst = reinterpret_cast<int4*>(out + p * opstride + static_cast<long long>(a) * ld);
  for (long long e = threadIdx.x; e < ld / 16; e += blockDim.x) dst[e] = src[e];
  if (p == 0 && threadIdx.x == 0) gJ[a] = g[J[a]];
}

}  // namespace

void launch_gather_digit_cols(const int8_t* dig, long long ld, long long pstride, int k, const int* J, int m,
                              int8_t* out, long long opstride, const int32_t* g, int32_t* gJ, cudaStream_t s) {
  k_gather_digit_cols<<<dim3(m, k), 256, 0, s>>>(dig, ld, pstride, J, out, opstride, g, gJ);
}

size_t cluster_jacobi_smem(int mmax) {
  const int m = std::min(mmax, kCoopMin);
  return sizeof(double) * (2 * (m + 1) + 2 * m + (m + 1) / 2 + 2) + 64;
}

int cluster_dot_splits(int ntiles, int rows) {
  const int want = (4 * 148 + ntiles - 1) / ntiles;          // ~4 CTAs per SM in total
  const int maxs = std::max(1, (rows + KC - 1) / KC);          // at least one row chunk each
  return std::max(1, std::min(std::min(want, 64), maxs));
}

cudaError_t launch_cluster_build(const ClusterLaunch& L, cudaStream_t s) {
  if (L.ntiles_dot > 0)
    k_cluster_dot<<<dim3(L.ntiles_dot, L.nsplit), TB * TB, 0, s>>>(L.tiles, L.goff, L.mem, L.xdig, L.ldd, L.pstride,
                                                                   L.kx, L.rows, L.nsplit, L.part);
  if (L.ntiles > 0)
    k_cluster_build<<<L.ntiles, TB * TB, 0, s>>>(L.tiles, L.goff, L.gsq, L.mem, L.mu, L.nsplit, L.part, L.rows,
                                                 L.gexp, L.r_hi, L.r_lo, L.wplanes, L.wpstride, *L.rpW, L.ellR,
                                                 L.scale8, L.lam, L.Mbuf, L.Rbuf, L.col0, L.ncols, L.ntiles_dot,
                                                 L.Gbuf);
  dim3 gg(L.nmembers, (L.rows + 255) / 256 < 64 ? (L.rows + 255) / 256 : 64);
  k_cluster_gather<<<gg, 256, 0, s>>>(L.mem, L.nmembers, L.Ep, L.lde, L.rows, L.T, L.col0, L.ncols);
  return cudaGetLastError();
}

cudaError_t launch_cluster_solve(const ClusterLaunch& L, cudaStream_t s) {
  const size_t sm = cluster_jacobi_smem(L.mmax);
  k_cluster_jacobi<<<L.ngroups, JT, sm, s>>>(L.goff, L.gsq, L.gm, L.mem, L.mu, L.Mbuf, L.Rbuf, L.Kbuf, L.Vbuf, L.Zbuf,
                                              L.lam, L.sweeps, L.dense_min);
  // large groups: one cooperative whole-GPU launch each
  int per = 0;  // per call: the occupancy is a property of the current device
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_cluster_jacobi_coop, JT, 0);
  const int coop_grid = sm_count() * std::max(1, std::min(per, 2));
  for (int q = 0; q < L.ngroups; ++q) {
    if (L.hgm[q] < kCoopMin || L.hgm[q] >= L.dense_min) continue;
    cudaError_t e = cudaMemsetAsync(L.coop_flags, 0, 128 * sizeof(int), s);
    if (e != cudaSuccess) return e;
    int grp = q;
    void* args[] = {&grp, (void*)&L.goff, (void*)&L.gsq, (void*)&L.gm, (void*)&L.mem, (void*)&L.mu, (void*)&L.Mbuf,
                    (void*)&L.Rbuf, (void*)&L.Kbuf, (void*)&L.Vbuf, (void*)&L.Zbuf, (void*)&L.lam, (void*)&L.sweeps,
                    (void*)&L.coop_scratch, (void*)&L.coop_flags};
    e = cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_cluster_jacobi_coop), dim3(coop_grid), dim3(JT), args, 0,
                                    s);
    if (e != cudaSuccess) return e;
  }
  return cudaGetLastError();
}

cudaError_t launch_cluster_apply(const ClusterLaunch& L, cudaStream_t s) {
  dim3 ga((L.rows + 255) / 256, (L.mmax + AK - 1) / AK, L.ngroups);
  k_cluster_apply<<<ga, 256, 0, s>>>(L.goff, L.gsq, L.gm, L.mem, L.grp_of, L.pos_of, L.T, L.Zbuf, L.gexp, L.rows,
                                     L.Ep, L.lde, L.col0, L.ncols, L.dense_min);
  return cudaGetLastError();
}

cudaError_t launch_cluster_colstats(const ClusterLaunch& L, cudaStream_t s) {
  k_cluster_colstats<<<L.nmembers, 256, 0, s>>>(L.mem, L.Ep, L.lde, L.rows, L.gexp, L.nrm2, L.eE_col, L.eE_max,
                                                L.col0, L.ncols);
  return cudaGetLastError();
}

}  // namespace ozr
