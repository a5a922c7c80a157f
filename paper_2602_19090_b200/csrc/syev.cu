// syev.cu — the hand-written dense symmetric eigensolver of the Rayleigh–Ritz sub-solve of large unresolved
// groups (R13: K = C·sym(M)·C = YΘYᵀ). Replaces a library eigensolver on the cluster path.
//
//   (1) Householder tridiagonalisation Qᴴᵀ K Qᴴ = T (lower storage, LAPACK dsytrd/dlatrd blocking): panels of
//       NB columns, each a persistent cooperative kernel (3 grid-wide barriers per column: the updated column
//       and its norm; the reflector, the symmetric product w = K₂₂v over 64 x 64 lower-triangle tiles — each
//       tile read ONCE and used for both of its row and column contributions, partials reduced in a fixed
//       order — and Vᵀv, Wᵀv; then w's last correction), followed by the rank-2·NB trailing update
//       K₂₂ −= VWᵀ + WVᵀ on the lower tiles.
//   (2) T = QᵀΘQᵀᵀ by Cuppen's divide and conquer with Gu–Eisenstat eigenvectors (syev_dc.cu).
//   (3) Y = Qᴴ·Qᵀ: the reflectors applied blockwise (compact WY, I − V T Vᵀ).
// Every reduction has a fixed order (no floating-point atomics): the result is deterministic.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <string>
#include <vector>

#include "ozr_internal.h"
#include "syev.h"

namespace ozr {

namespace cg = cooperative_groups;

namespace {

constexpr int NB = 32;   // panel width
constexpr int TB = 64;   // symv / update tile
constexpr int TT = 256;  // threads per CTA

__device__ __forceinline__ double block_sum256(double v, double* sh) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    v = (threadIdx.x < TT / 32) ? sh[threadIdx.x] : 0.0;
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (threadIdx.x == 0) sh[0] = v;
  }
  __syncthreads();
  v = sh[0];
  __syncthreads();
  return v;
}

// Four sums at once (fixed order; every thread receives the results): two block barriers instead of eight.
__device__ __forceinline__ void block_sum4(double (&v)[4], double* sh /* ≥ 4·(TT/32) + 4 */) {
#pragma unroll
  for (int k = 0; k < 4; ++k)
    for (int o = 16; o; o >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0)
#pragma unroll
    for (int k = 0; k < 4; ++k) sh[4 * w + k] = v[k];
  __syncthreads();
  if (threadIdx.x < 4) {
    double a = 0.0;
    for (int ww = 0; ww < TT / 32; ++ww) a += sh[4 * ww + threadIdx.x];
    sh[4 * (TT / 32) + threadIdx.x] = a;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < 4; ++k) v[k] = sh[4 * (TT / 32) + k];
  __syncthreads();
}

// linear index t of the active lower tiles (I ≥ J ≥ J0, I < mt) → (I, J), row-major over I
__device__ __forceinline__ void tile_of(int t, int J0, int& I, int& J) {
  // rows I' = I − J0 hold I' + 1 tiles: t = I'(I'+1)/2 + (J − J0)
  int Ip = static_cast<int>((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
  while ((Ip + 1) * (Ip + 2) / 2 <= t) ++Ip;
  while (Ip * (Ip + 1) / 2 > t) --Ip;
  I = J0 + Ip;
  J = J0 + (t - Ip * (Ip + 1) / 2);
}
__device__ __forceinline__ long long tslot(int I, int J) { return static_cast<long long>(I) * (I + 1) / 2 + J; }

struct PanelArgs {
  double* A;        // m x m, lda = m (lower triangle maintained)
  int m;
  int k0;           // first column of the panel
  int nb;           // columns in this panel
  double* V;        // m x NB (reflectors of the panel, v_{c+1} = 1)
  double* W;        // m x NB
  double* d;        // diagonal of T
  double* e;        // sub-diagonal of T
  double* tau;      // reflector scalars
  double* part;     // G x (5 + 2·NB) scalar partials
  double* yp;       // tile partials: slot(I, J) x 2 x TB
  double* gam;      // NB: γ_j of the panel's columns (W = W' + V·diag(γ); W' is what W holds)
  unsigned long long* dbg;  // OZR_SYEV_PROBE: accumulated ns per phase (CTA 0), or null
};
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Sum of the G per-CTA partials part[g·PS + off] in a fixed order (every CTA gets the same value): thread t sums
// g ≡ t (mod TT) ascending, then a fixed tree over the threads.
__device__ __forceinline__ double grid_partial_sum(const double* __restrict__ part, int PS, int off, int G, double* sh) {
  double a = 0.0;
  for (int g = threadIdx.x; g < G; g += TT) a += part[static_cast<long long>(g) * PS + off];
  return block_sum256(a, sh);
}

// Row block b (TB rows) is owned by CTA b (G ≥ mt is guaranteed by syev_trd_grid). The CTA keeps its rows of the
// panel's V and W in shared memory (vs, ws), so every per-row dot product of the panel reads shared memory.
struct PanelSmem {
  double tile[TB][TB + 1];  // tile[col][row]
  double vs[NB][TB], ws[NB][TB];
  double vr[TB], vc[TB], vloc[TB];
  double rowc[2 * NB];      // V(c, 0:i) | W(c, 0:i−1) (corrected)
  double gam[NB];           // γ_j of the finished columns
  double dots[2 * NB];      // Vᵀv | Wᵀv (reduced over the grid)
  double sh[4 * (TT / 32) + 4];
};

// Two grid-wide barriers per column. W(:, i)'s last correction γ_i·V(:, i) (γ_i = −½τ_i·w'ᵀv, a grid reduction)
// is never written back during the panel: W holds W', the γ_j are kept, and every use forms W' + γ_j V on the fly.
// Column i+1's phase A leaves out the terms of column i's W (unknown γ_i, and W'(c, i) of another CTA's row not yet
// visible); after the first barrier x = x'' − κ·V(r, i), κ = W'(c, i) + 2γ_i V(c, i), so σ = Σx''² − 2κΣx''b + κ²Σb²
// (b_r = V(r, i)), α and d_c follow from x'', and v_r = x_r·scale is formed on the fly.
__device__ __forceinline__ void trd_tile_load(const double* __restrict__ A, int m, int c, int I, int J, int tid,
                                              double (&reg)[TB * TB / TT]) {
  const int rt0 = I * TB, qt0 = J * TB;
#pragma unroll
  for (int u = 0; u < TB * TB / TT; ++u) {
    const int e2 = tid + u * TT;
    const int rho = e2 & (TB - 1), kap = e2 >> 6;
    const int r = rt0 + rho, q = qt0 + kap;
    const bool in = r < m && q < m && r >= c + 1 && q >= c + 1;
    const long long idx = (r >= q) ? r + static_cast<long long>(q) * m : q + static_cast<long long>(r) * m;
    reg[u] = in ? __ldcg(A + idx) : 0.0;
  }
}

__global__ void __launch_bounds__(TT, 2) k_trd_panel(PanelArgs P) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) unsigned char smraw[];
  PanelSmem& S = *reinterpret_cast<PanelSmem*>(smraw);
  const int G = gridDim.x, b = blockIdx.x, tid = threadIdx.x;
  const int m = P.m;
  const int mt = (m + TB - 1) / TB;
  double* A = P.A;
  const int PS = 5 + 2 * NB;  // per CTA: Σx''², Σx''b, Σb², w'ᵀv, Σx² (exact, rare) | Vᵀv (NB) | Wᵀv (NB)
  const int r0own = b * TB;
  const bool owner = b < mt;
  // every partial of the column reductions (Σx''², Σx''b, Σb², w'ᵀv, Vᵀv, Wᵀv) comes from the owners' rows: the
  // CTAs b ≥ mt write zeros, so the sums run over the GP = min(G, mt) owners only (2.8× fewer L2 loads at m = 6628)
  const int GP = min(G, mt);
  double tau_prev = 0.0;
  unsigned long long tlast = gtimer();
#define PROBE(k)                                          \
  if (P.dbg && b == 0 && tid == 0) {                      \
    const unsigned long long tn_ = gtimer();              \
    P.dbg[k] += tn_ - tlast;                              \
    tlast = tn_;                                          \
  }
  for (int i = 0; i < P.nb; ++i) {
    const int c = P.k0 + i;
    // ---- phase A: x''_r = A(r,c) − Σ_{j<i−1} [V(r,j)W(c,j) + W(r,j)V(c,j)] − W'(r,i−1)V(c,i−1), own rows r ≥ c
    if (tid < 2 * i) {
      const int j = tid < i ? tid : tid - i;
      const double vcj = P.V[c + static_cast<long long>(j) * m];
      if (tid < i) S.rowc[j] = vcj;
      else if (j < i - 1) S.rowc[NB + j] = fma(S.gam[j], vcj, P.W[c + static_cast<long long>(j) * m]);
    }
    __syncthreads();
    double ss = 0.0, sxb = 0.0, sbb = 0.0;
    if (owner && tid < TB) {
      const int r = r0own + tid;
      if (r < m && r >= c) {
        double x = A[r + static_cast<long long>(c) * m];
        double x2 = 0.0;
        for (int j = 0; j + 1 < i; j += 2) {
          x -= S.vs[j][tid] * S.rowc[NB + j] + S.ws[j][tid] * S.rowc[j];
          if (j + 2 < i) x2 -= S.vs[j + 1][tid] * S.rowc[NB + j + 1] + S.ws[j + 1][tid] * S.rowc[j + 1];
        }
        if (i > 0) x2 -= S.ws[i - 1][tid] * S.rowc[i - 1];  // W'(r, i−1) V(c, i−1)
        x += x2;
        A[r + static_cast<long long>(c) * m] = x;
        if (r >= c + 2) {
          const double bb = (i > 0) ? S.vs[i - 1][tid] : 0.0;
          ss = x * x;
          sxb = x * bb;
          sbb = bb * bb;
        }
      }
    }
    {
      double v4[4] = {ss, sxb, sbb, 0.0};
      block_sum4(v4, S.sh);
      if (tid < 3) P.part[static_cast<long long>(b) * PS + tid] = v4[tid];
    }
    PROBE(6);
    grid.sync();
    PROBE(0);
    // ---- phase B: γ_{i−1}, the reflector (every CTA, the same fixed-order sums), V(:, i), the tile products, Vᵀv, Wᵀv
    // every global value phase B needs, loaded at once (independent of the reductions below)
    const double w_ci = (i > 0) ? __ldcg(P.W + c + static_cast<long long>(i - 1) * m) : 0.0;
    const double a_cc = __ldcg(A + c + static_cast<long long>(c) * m);
    const double a_c1 = (c + 1 < m) ? __ldcg(A + c + 1 + static_cast<long long>(c) * m) : 0.0;
    const double v_c1 = (i > 0 && c + 1 < m) ? __ldcg(P.V + c + 1 + static_cast<long long>(i - 1) * m) : 0.0;
    const int rown = r0own + (tid & (TB - 1));
    const bool ownrow = owner && tid < TB && rown < m;
    const double a_rc = ownrow ? __ldcg(A + rown + static_cast<long long>(c) * m) : 0.0;
    double kap = 0.0;
    double sums[4] = {0.0, 0.0, 0.0, 0.0};  // Σ_g of slots 0..3, fixed order (g ≡ tid mod TT, then the block tree)
    for (int g = tid; g < GP; g += TT) {
      const double* pg = P.part + static_cast<long long>(g) * PS;
      sums[0] += pg[0];
      sums[1] += pg[1];
      sums[2] += pg[2];
      sums[3] += pg[3];
    }
    block_sum4(sums, S.sh);
    if (i > 0) {
      const double gam = -0.5 * tau_prev * sums[3];
      kap = fma(2.0 * gam, S.rowc[i - 1], w_ci);
      if (tid == 0) S.gam[i - 1] = gam;
      if (tid < TB) S.ws[i - 1][tid] = fma(gam, S.vs[i - 1][tid], S.ws[i - 1][tid]);  // private rows
    }
    const double sig0 = sums[0], sig1 = sums[1], sig2 = sums[2];
    double sigma = sig0 - 2.0 * kap * sig1 + kap * kap * sig2;
    // the expansion's rounding error (≈ u·(Σx''² + κ²Σb²)) enters the reflector's orthogonality as δσ/σ (τ·vᵀv =
    // 2 + δσ/(β(β − α))), so it is trusted only without cancellation; otherwise Σ x_r² exactly, one more barrier
    if (i > 0 && !(sigma >= 0.5 * (sig0 + kap * kap * sig2))) {
      double sx = 0.0;
      if (owner && tid < TB) {
        const int r = r0own + tid;
        if (r < m && r >= c + 2) {
          const double x = fma(-kap, S.vs[i - 1][tid], A[r + static_cast<long long>(c) * m]);
          sx = x * x;
        }
      }
      sx = block_sum256(sx, S.sh);
      if (tid == 0) P.part[static_cast<long long>(b) * PS + 4] = sx;
      grid.sync();
      sigma = grid_partial_sum(P.part, PS, 4, GP, S.sh);
    }
    sigma = fmax(sigma, 0.0);
    auto xfin = [&](int r) -> double {  // x_r = x''_r − κ V(r, i−1)
      const double x = A[r + static_cast<long long>(c) * m];
      return (i > 0) ? fma(-kap, P.V[r + static_cast<long long>(i - 1) * m], x) : x;
    };
    const double ccdiag = (i > 0) ? fma(-kap, S.rowc[i - 1], a_cc) : a_cc;  // V(c, i−1) = rowc[i−1]
    double alpha = 0.0, beta = 0.0, tau = 0.0, scale = 0.0;
    if (c + 1 < m) {
      alpha = (i > 0) ? fma(-kap, v_c1, a_c1) : a_c1;
      if (sigma == 0.0) {
        beta = alpha;  // H = I
      } else {
        beta = -copysign(sqrt(fma(alpha, alpha, sigma)), alpha);
        tau = (beta - alpha) / beta;
        scale = 1.0 / (alpha - beta);
      }
    }
    if (b == 0 && tid == 0) {
      P.d[c] = ccdiag;
      if (c + 1 < m) {
        P.e[c] = beta;
        P.tau[c] = tau;
      }
    }
    if (c + 1 >= m) break;  // the last column: only its diagonal
    auto vof = [&](int r) -> double { return r == c + 1 ? 1.0 : (r > c + 1 ? xfin(r) * scale : 0.0); };
    if (owner && tid < TB) {
      const int r = r0own + tid;
      // v_r from the hoisted x''_r (own row; V(r, i−1) is the CTA's own shared copy)
      const double xr = (i > 0) ? fma(-kap, S.vs[i - 1][tid], a_rc) : a_rc;
      const double v = (r >= m) ? 0.0 : (r == c + 1 ? 1.0 : (r > c + 1 ? xr * scale : 0.0));
      S.vloc[tid] = v;
      S.vs[i][tid] = v;
      if (r < m && r >= c + 1) P.V[r + static_cast<long long>(i) * m] = v;
    }
    PROBE(1);
    if (tau != 0.0) {
      const int J0 = (c + 1) / TB;
      const int na = mt - J0;
      const int ntiles = na * (na + 1) / 2;
      double reg[TB * TB / TT];
      int t = b, I = 0, J = 0;
      if (t < ntiles) {
        tile_of(t, J0, I, J);
        trd_tile_load(A, m, c, I, J, tid, reg);
      }
      while (t < ntiles) {
        const int rt0 = I * TB, qt0 = J * TB;
        __syncthreads();  // the previous tile's readers are done with shared memory
#pragma unroll
        for (int u = 0; u < TB * TB / TT; ++u) {
          const int e2 = tid + u * TT;
          S.tile[e2 >> 6][e2 & (TB - 1)] = reg[u];
        }
        if (tid < TB) S.vr[tid] = (rt0 + tid < m) ? vof(rt0 + tid) : 0.0;
        else if (tid < 2 * TB) S.vc[tid - TB] = (qt0 + tid - TB < m) ? vof(qt0 + tid - TB) : 0.0;
        __syncthreads();
        const int tn = t + G;  // prefetch the next tile while this one is reduced
        int In = 0, Jn = 0;
        if (tn < ntiles) {
          tile_of(tn, J0, In, Jn);
          trd_tile_load(A, m, c, In, Jn, tid, reg);
        }
        double* out = P.yp + tslot(I, J) * 2 * TB;
        const int half = tid & 1;
        if (tid < 2 * TB) {  // row ρ = tid/2: Σ_κ tile[κ][ρ] vc[κ], κ ≡ half (mod 2)
          const int rho = tid >> 1;
          double acc = 0.0;
#pragma unroll 8
          for (int kap = half; kap < TB; kap += 2) acc = fma(S.tile[kap][rho], S.vc[kap], acc);
          acc += __shfl_xor_sync(0xffffffffu, acc, 1);
          if (!half) out[rho] = acc;
        } else {  // column κ = (tid − 128)/2: Σ_ρ tile[κ][ρ] vr[ρ] (off-diagonal tiles)
          const int kap = (tid - 2 * TB) >> 1;
          double acc = 0.0;
          if (I != J) {
#pragma unroll 8
            for (int rho = half; rho < TB; rho += 2) acc = fma(S.tile[kap][rho], S.vr[rho], acc);
          }
          acc += __shfl_xor_sync(0xffffffffu, acc, 1);
          if (!half) out[TB + kap] = acc;
        }
        t = tn;
        I = In;
        J = Jn;
      }
      PROBE(2);
      // Vᵀv and Wᵀv over own rows: 2i dot products of length TB from shared memory, 4 threads each
      __syncthreads();
      if (owner && i > 0) {
        const int q = tid >> 2, part = tid & 3;
        if (q < 2 * NB) {
          const int j = q < NB ? q : q - NB;
          double acc = 0.0;
          if (j < i) {
            const double* row = q < NB ? S.vs[j] : S.ws[j];
            for (int t2 = part; t2 < TB; t2 += 4) acc = fma(row[t2], S.vloc[t2], acc);
          }
          acc += __shfl_xor_sync(0xffffffffu, acc, 1);
          acc += __shfl_xor_sync(0xffffffffu, acc, 2);
          if (part == 0 && j < i) P.part[static_cast<long long>(b) * PS + 5 + q] = acc;
        }
      } else if (i > 0 && tid < 2 * NB) {
        const int j = tid < NB ? tid : tid - NB;
        if (j < i) P.part[static_cast<long long>(b) * PS + 5 + tid] = 0.0;
      }
    }
    PROBE(3);
    grid.sync();
    // ---- phase C: y_r from the tile partials, w'_r = τ(y − V(Wᵀv) − W(Vᵀv)), partial of w'ᵀv (its γ: next column)
    double p3 = 0.0;
    PROBE(4);
    if (tau != 0.0) {
      if (i > 0) {  // Vᵀv, Wᵀv reduced over the grid: 4 threads per value, fixed order
        const int q = tid >> 2, part = tid & 3;
        double acc = 0.0;
        if (q < 2 * NB && (q < NB ? q : q - NB) < i) {
          double a8[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // independent partial sums: the loads stay in flight
          int g = part;
          for (; g + 28 < GP; g += 32)
#pragma unroll
            for (int u = 0; u < 8; ++u) a8[u] += __ldcg(P.part + static_cast<long long>(g + 4 * u) * PS + 5 + q);
          for (; g < GP; g += 4) a8[0] += __ldcg(P.part + static_cast<long long>(g) * PS + 5 + q);
          acc = ((a8[0] + a8[1]) + (a8[2] + a8[3])) + ((a8[4] + a8[5]) + (a8[6] + a8[7]));
        }
        acc += __shfl_xor_sync(0xffffffffu, acc, 1);
        acc += __shfl_xor_sync(0xffffffffu, acc, 2);
        if (part == 0 && q < 2 * NB) S.dots[q] = acc;
      }
      __syncthreads();
      if (owner) {
        const int J0 = (c + 1) / TB;
        const int R = b, t4 = tid & 3, row = tid >> 2;  // 4 threads per own row
        const int r = r0own + row;
        double y = 0.0;
        if (r < m && r >= c + 1) {
          // eight independent partial sums per thread: the L2 loads of a row's tile partials all stay in flight
          double a8[8] = {0, 0, 0, 0, 0, 0, 0, 0};
          int J = J0 + t4;
          for (; J + 28 <= R; J += 32)
#pragma unroll
            for (int u = 0; u < 8; ++u) a8[u] += __ldcg(P.yp + tslot(R, J + 4 * u) * 2 * TB + row);
          for (; J <= R; J += 4) a8[0] += __ldcg(P.yp + tslot(R, J) * 2 * TB + row);
          int I = R + 1 + t4;
          for (; I + 28 < mt; I += 32)
#pragma unroll
            for (int u = 0; u < 8; ++u) a8[u] += __ldcg(P.yp + tslot(I + 4 * u, R) * 2 * TB + TB + row);
          for (; I < mt; I += 4) a8[0] += __ldcg(P.yp + tslot(I, R) * 2 * TB + TB + row);
          y = ((a8[0] + a8[1]) + (a8[2] + a8[3])) + ((a8[4] + a8[5]) + (a8[6] + a8[7]));
        }
        y += __shfl_xor_sync(0xffffffffu, y, 1);
        y += __shfl_xor_sync(0xffffffffu, y, 2);
        if (t4 == 0 && r < m && r >= c + 1) {
          double y2 = 0.0;
          for (int j = 0; j < i; j += 2) {
            y -= S.vs[j][row] * S.dots[NB + j] + S.ws[j][row] * S.dots[j];
            if (j + 1 < i) y2 -= S.vs[j + 1][row] * S.dots[NB + j + 1] + S.ws[j + 1][row] * S.dots[j + 1];
          }
          const double w = tau * (y + y2);
          S.ws[i][row] = w;
          P.W[r + static_cast<long long>(i) * m] = w;
          p3 = w * S.vloc[row];
        } else if (t4 == 0 && row < TB) {
          S.ws[i][row] = 0.0;
        }
      }
    } else if (owner && tid < TB) {
      const int r = r0own + tid;
      S.ws[i][tid] = 0.0;
      if (r < m && r >= c + 1) P.W[r + static_cast<long long>(i) * m] = 0.0;
    }
    p3 = block_sum256(p3, S.sh);
    if (tid == 0) P.part[static_cast<long long>(b) * PS + 3] = p3;
    tau_prev = tau;
    PROBE(5);
  }
  // the last column's γ (one more barrier for its w'ᵀv); the γ_j go to the trailing update
  const int ilast = P.nb - 1, clast = P.k0 + ilast;
  if (clast + 1 < m) {
    grid.sync();
    const double gam = -0.5 * tau_prev * grid_partial_sum(P.part, PS, 3, GP, S.sh);
    if (tid == 0) S.gam[ilast] = gam;
  } else if (tid == 0) {
    S.gam[ilast] = 0.0;
  }
  __syncthreads();
  if (b == 0 && tid < P.nb) P.gam[tid] = S.gam[tid];
}

// Trailing update of the lower tiles of A(k1:m, k1:m): A −= V Wᵀ + W Vᵀ (nb columns); also stores the panel's
// reflectors below the sub-diagonal: A(r, k0 + j) = V(r, j) for r ≥ k0 + j + 2 (tiles with J == -1: the copy).
__global__ void __launch_bounds__(TT) k_trd_update(double* __restrict__ A, int m, int k0, int nb,
                                                   const double* __restrict__ V, const double* __restrict__ W,
                                                   const double* __restrict__ gam) {
  __shared__ double vR[NB][TB], wR[NB][TB], vC[NB][TB / 2], wC[NB][TB / 2];  // 48 KB: columns in two halves
  const int k1 = k0 + nb;
  const int J0 = k1 / TB, mt = (m + TB - 1) / TB;
  const int na = (k1 < m) ? mt - J0 : 0;
  const int t = blockIdx.x;
  if (t >= na * (na + 1) / 2) {  // the reflector copy: one CTA per panel column
    const int j = t - na * (na + 1) / 2;
    if (j >= nb) return;
    const int c = k0 + j;
    for (int r = c + 2 + threadIdx.x; r < m; r += TT) A[r + static_cast<long long>(c) * m] = V[r + static_cast<long long>(j) * m];
    return;
  }
  int I, J;
  tile_of(t, J0, I, J);
  const int r0 = I * TB, q0 = J * TB;
  for (int e2 = threadIdx.x; e2 < NB * TB; e2 += TT) {
    const int rho = e2 & (TB - 1), j = e2 >> 6;
    const int r = r0 + rho;
    const bool jr = j < nb && r < m && r >= k1;
    const double vv = jr ? V[r + static_cast<long long>(j) * m] : 0.0;
    vR[j][rho] = vv;
    wR[j][rho] = jr ? fma(gam[j], vv, W[r + static_cast<long long>(j) * m]) : 0.0;
  }
  const int rho = threadIdx.x & (TB - 1);
  const int r = r0 + rho;
  for (int h = 0; h < 2; ++h) {
    const int qh = q0 + h * (TB / 2);
    __syncthreads();
    for (int e2 = threadIdx.x; e2 < NB * (TB / 2); e2 += TT) {
      const int kap = e2 & (TB / 2 - 1), j = e2 >> 5;
      const int q = qh + kap;
      const bool jq = j < nb && q < m && q >= k1;
      const double vv = jq ? V[q + static_cast<long long>(j) * m] : 0.0;
      vC[j][kap] = vv;
      wC[j][kap] = jq ? fma(gam[j], vv, W[q + static_cast<long long>(j) * m]) : 0.0;
    }
    __syncthreads();
    for (int kk = threadIdx.x >> 6; kk < TB / 2; kk += TT / TB) {
      const int q = qh + kk;
      if (r >= m || q >= m || r < k1 || q < k1 || r < q) continue;
      double acc = 0.0;
#pragma unroll 8
      for (int j = 0; j < NB; ++j) acc = fma(vR[j][rho], wC[j][kk], fma(wR[j][rho], vC[j][kk], acc));
      A[r + static_cast<long long>(q) * m] -= acc;
    }
  }
}

// ================================================================ (2) divide and conquer on T
constexpr int LEAF = 32;

// Leaf: implicit QL with Wilkinson-type shifts (tqli) on an L ≤ 32 tridiagonal; thread t owns row t of the
// eigenvector block, every thread runs the scalar recurrence (identical values). Output: eigenvalues (unsorted)
// into lamo[lo..hi), eigenvectors into Q (block rows/columns lo..hi, ld = m).
__global__ void __launch_bounds__(LEAF) k_dc_leaf(const int* __restrict__ leaf_lo, const int* __restrict__ leaf_hi,
                                                  const double* __restrict__ dmod, const double* __restrict__ e,
                                                  double* __restrict__ lamo, double* __restrict__ Q, int m,
                                                  int* __restrict__ err) {
  const int lo = leaf_lo[blockIdx.x], n = leaf_hi[blockIdx.x] - lo;
  const int t = threadIdx.x;
  double d[LEAF], ee[LEAF], z[LEAF];
  for (int i = 0; i < LEAF; ++i) {
    d[i] = i < n ? dmod[lo + i] : 0.0;
    ee[i] = (i + 1 < n) ? e[lo + i] : 0.0;
    z[i] = (i == t) ? 1.0 : 0.0;
  }
  const double eps = 1.1102230246251565e-16;
  for (int l = 0; l < n; ++l) {
    int iter = 0, mm;
    do {
      for (mm = l; mm < n - 1; ++mm) {
        const double dd = fabs(d[mm]) + fabs(d[mm + 1]);
        if (fabs(ee[mm]) <= eps * dd) break;
      }
      if (mm != l) {
        if (++iter > 60) {
          if (t == 0) atomicOr(err, 1);
          break;
        }
        double g = (d[l + 1] - d[l]) / (2.0 * ee[l]);
        double r = hypot(g, 1.0);
        g = d[mm] - d[l] + ee[l] / (g + copysign(r, g));
        double s = 1.0, c = 1.0, p = 0.0;
        int i;
        bool early = false;
        for (i = mm - 1; i >= l; --i) {
          double f = s * ee[i];
          const double b = c * ee[i];
          ee[i + 1] = (r = hypot(f, g));
          if (r == 0.0) {
            d[i + 1] -= p;
            ee[mm] = 0.0;
            early = true;
            break;
          }
          s = f / r;
          c = g / r;
          g = d[i + 1] - p;
          r = (d[i] - g) * s + 2.0 * c * b;
          d[i + 1] = g + (p = s * r);
          g = c * r - b;
          f = z[i + 1];
          z[i + 1] = s * z[i] + c * f;
          z[i] = c * z[i] - s * f;
        }
        if (early) continue;
        d[l] -= p;
        ee[l] = g;
        ee[mm] = 0.0;
      }
    } while (mm != l);
  }
  if (t < n) {
    for (int j = 0; j < n; ++j) Q[static_cast<long long>(lo + j) * m + lo + t] = z[j];
    if (t == 0)
      for (int j = 0; j < n; ++j) lamo[lo + j] = d[j];
  }
}

// z of a merge: [Q1(last row, :) ; s·Q2(first row, :)] / √2 for node q (cols of the node's block)
__global__ void k_dc_zvec(const int* __restrict__ nlo, const int* __restrict__ nmid, const int* __restrict__ nhi,
                          const double* __restrict__ sgn, const double* __restrict__ Q, int m, double* __restrict__ z) {
  const int q = blockIdx.y;
  const int lo = nlo[q], mid = nmid[q], hi = nhi[q];
  for (int j = lo + blockIdx.x * blockDim.x + threadIdx.x; j < hi; j += gridDim.x * blockDim.x) {
    const double v = (j < mid) ? Q[static_cast<long long>(j) * m + mid - 1] : sgn[q] * Q[static_cast<long long>(j) * m + mid];
    z[j] = v * 0.70710678118654752440;
  }
}

// Qp (node block, ld = m) column jj = Q column lo + src[jj] (block-diagonal halves), then the deflation
// rotations of the node in order (each thread one row: the rotations only mix columns).
__global__ void k_dc_permrot(const int* __restrict__ nlo, const int* __restrict__ nmid, const int* __restrict__ nhi,
                             const int* __restrict__ src, const int* __restrict__ rot_off, const int4* __restrict__ rot_idx,
                             const double2* __restrict__ rot_cs, const double* __restrict__ Q, double* __restrict__ Qp,
                             int m) {
  const int q = blockIdx.y;
  const int lo = nlo[q], nn = nhi[q] - lo, n1 = nmid[q] - lo;
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nn) return;
  for (int jj = 0; jj < nn; ++jj) {  // diag(Q1, Q2): the off-diagonal child blocks are zero (never stored)
    const int c = src[lo + jj];
    Qp[static_cast<long long>(lo + jj) * m + lo + r] =
        ((r < n1) == (c < n1)) ? Q[static_cast<long long>(lo + c) * m + lo + r] : 0.0;
  }
  for (int k = rot_off[q]; k < rot_off[q + 1]; ++k) {
    const int a = rot_idx[k].x, b = rot_idx[k].y;  // node-local columns of Qp
    const double c = rot_cs[k].x, s = rot_cs[k].y;
    double* pa = Qp + static_cast<long long>(lo + a) * m + lo + r;
    double* pb = Qp + static_cast<long long>(lo + b) * m + lo + r;
    const double x = *pa, y = *pb;
    *pa = c * x + s * y;  // LAPACK drot(Q(:,PJ), Q(:,NJ), C, S): x' = c x + s y, y' = c y − s x
    *pb = c * y - s * x;
  }
}

// Secular equation of node q, root j (k non-deflated, d ascending, ρ > 0, z unit-ish): f(λ) = 1/ρ + Σ z_i²/(d_i − λ).
// Origin at the nearer pole (o = j or j + 1), τ = λ − d_o; Gragg's two-pole rational model with a bisection guard.
__device__ void secular_root(int k, const double* __restrict__ d, const double* __restrict__ z, double rho, int j,
                             int& o_out, double& tau_out) {
  const double eps = 1.1102230246251565e-16;
  const double ir = 1.0 / rho;
  double zz = 0.0;
  for (int i = 0; i < k; ++i) zz = fma(z[i], z[i], zz);
  int o = j;
  double a, b;  // bracket of τ
  if (j < k - 1) {
    const double del = d[j + 1] - d[j];
    double f = ir;
    for (int i = 0; i < k; ++i) f += z[i] * z[i] / ((d[i] - d[j]) - 0.5 * del);
    if (f >= 0.0) {
      o = j;
      a = 0.0;
      b = 0.5 * del;
    } else {
      o = j + 1;
      a = -0.5 * del;
      b = 0.0;
    }
  } else {
    a = 0.0;
    b = rho * zz;
  }
  const double dO = d[o];
  double t = 0.5 * (a + b);
  for (int it = 0; it < 80; ++it) {
    double psi = 0.0, dpsi = 0.0, phi = 0.0, dphi = 0.0, erre = 0.0;
    for (int i = 0; i < k; ++i) {
      const double del = (d[i] - dO) - t;
      const double q = z[i] / del;
      if (i <= j) {
        psi = fma(z[i], q, psi);
        dpsi = fma(q, q, dpsi);
      } else {
        phi = fma(z[i], q, phi);
        dphi = fma(q, q, dphi);
      }
      erre += fabs(z[i] * q);
    }
    const double f = ir + psi + phi;
    if (f > 0.0) b = t; else a = t;
    // LAPACK dlaed4's stop: |f| within the rounding error of its own evaluation, ε(8(|ψ| + |φ|) + 1/ρ + |τ|·f')
    if (fabs(f) <= eps * (8.0 * erre + ir + fabs(t) * (dpsi + dphi)) || b - a <= 2.0 * eps * fmax(fabs(a), fabs(b)) ||
        f == 0.0)
      break;
    // model c + sL/(ΔL − η) + sR/(ΔR − η) matching f and f' at η = 0
    double tn;
    const double dL = (d[j] - dO) - t;
    if (j < k - 1) {
      const double dR = (d[j + 1] - dO) - t;
      const double sL = dpsi * dL * dL, sR = dphi * dR * dR;
      const double c = f - dpsi * dL - dphi * dR;
      // c η² − (c(ΔL + ΔR) + sL + sR) η + (cΔLΔR + sLΔR + sRΔL) = 0, root in (ΔL, ΔR)
      const double A2 = c, B2 = c * (dL + dR) + sL + sR, C2 = c * dL * dR + sL * dR + sR * dL;
      double eta;
      if (A2 == 0.0) {
        eta = C2 / B2;
      } else {
        const double disc = fmax(B2 * B2 - 4.0 * A2 * C2, 0.0);
        const double sq = sqrt(disc);
        const double e1 = (B2 >= 0.0) ? (B2 + sq) / (2.0 * A2) : 2.0 * C2 / (B2 - sq);
        const double e2 = (B2 >= 0.0) ? 2.0 * C2 / (B2 + sq) : (B2 - sq) / (2.0 * A2);
        eta = (e1 > dL && e1 < dR) ? e1 : e2;
      }
      tn = t + eta;
    } else {
      const double sL = dpsi * dL * dL;
      const double c = f - dpsi * dL;
      tn = (c != 0.0) ? t + dL + sL / c : 0.5 * (a + b);
    }
    if (!(tn > a && tn < b)) tn = 0.5 * (a + b);
    t = tn;
  }
  o_out = o;
  tau_out = t;
}

struct DcNode {
  int lo, k;       // node start; non-deflated count
  double rho;      // ρ (> 0) of the normalised problem
};

// One thread per (node, root): origin and τ of every root
__global__ void k_dc_secular(const DcNode* __restrict__ nodes, const int* __restrict__ root_node,
                             const int* __restrict__ root_j, int nroots, const double* __restrict__ dk,
                             const double* __restrict__ zk, int* __restrict__ org, double* __restrict__ tau) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= nroots) return;
  const DcNode nd = nodes[root_node[g]];
  int o;
  double t;
  secular_root(nd.k, dk + nd.lo, zk + nd.lo, nd.rho, root_j[g], o, t);
  org[nd.lo + root_j[g]] = o;
  tau[nd.lo + root_j[g]] = t;
}

// Gu–Eisenstat: ẑ_i = sign(z_i)·sqrt(−W_i/ρ), W_i = (d_i − λ_i)·Π_{j≠i} (d_i − λ_j)/(d_i − d_j), with
// d_i − λ_j = (d_i − d_{o_j}) − τ_j. Then U (node block of Up, ld = m): u_ij = ẑ_i/(d_i − λ_j), normalised per column
// (one CTA per column j, after every ẑ is known: two kernels).
__global__ void k_dc_zhat(const DcNode* __restrict__ nodes, const int* __restrict__ root_node,
                          const int* __restrict__ root_j, int nroots, const double* __restrict__ dk,
                          const double* __restrict__ zk, const int* __restrict__ org, const double* __restrict__ tau,
                          double* __restrict__ zhat) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= nroots) return;
  const DcNode nd = nodes[root_node[g]];
  const int i = root_j[g], k = nd.k;
  const double* d = dk + nd.lo;
  const int* o = org + nd.lo;
  const double* ta = tau + nd.lo;
  double w = (d[i] - d[o[i]]) - ta[i];
  for (int j = 0; j < k; ++j)
    if (j != i) w *= ((d[i] - d[o[j]]) - ta[j]) / (d[i] - d[j]);
  const double zi = zk[nd.lo + i];
  zhat[nd.lo + i] = copysign(sqrt(fmax(-w / nd.rho, 0.0)), zi);
}

__global__ void __launch_bounds__(256) k_dc_umat(const DcNode* __restrict__ nodes, const int* __restrict__ root_node,
                                                 const int* __restrict__ root_j, const double* __restrict__ dk,
                                                 const int* __restrict__ org, const double* __restrict__ tau,
                                                 const double* __restrict__ zhat, double* __restrict__ U, int m,
                                                 double* __restrict__ lam_out) {
  __shared__ double sh[8];
  const int g = blockIdx.x;  // one CTA per (node, column j)
  const DcNode nd = nodes[root_node[g]];
  const int j = root_j[g], k = nd.k, lo = nd.lo;
  const double* d = dk + lo;
  const double dj = d[org[lo + j]], tj = tau[lo + j];
  double ss = 0.0;
  for (int i = threadIdx.x; i < k; i += 256) {
    const double u = zhat[lo + i] / ((d[i] - dj) - tj);
    U[static_cast<long long>(lo + j) * m + lo + i] = u;
    ss = fma(u, u, ss);
  }
  for (int o = 16; o; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t += sh[w];
    sh[0] = 1.0 / sqrt(t);
    lam_out[lo + j] = dj + tj;
  }
  __syncthreads();
  const double inv = sh[0];
  for (int i = threadIdx.x; i < k; i += 256) U[static_cast<long long>(lo + j) * m + lo + i] *= inv;
}

// Batched SIMT GEMM on node blocks: Qn[:, lo .. lo+k) (rows lo .. lo+nn) = Qp[:, lo .. lo+k) · U (k x k block), and
// the deflated columns copied: Qn[:, lo+k .. lo+nn) = Qp[:, lo+k .. lo+nn). 64 x 64 output tiles.
struct DcTile {
  int lo, nn, k, r0, c0;  // node, tile origin (node-local row, column)
};
__global__ void __launch_bounds__(256) k_dc_gemm(const DcTile* __restrict__ tiles, const double* __restrict__ Qp,
                                                 const double* __restrict__ U, double* __restrict__ Qn, int m) {
  __shared__ double as[16][65], bs[16][65];
  const DcTile T = tiles[blockIdx.x];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  double acc[4][4] = {};
  const int lo = T.lo;
  if (T.c0 >= T.k) {  // copy tile of deflated columns
    for (int e2 = threadIdx.x; e2 < 64 * 64; e2 += 256) {
      const int rr = T.r0 + (e2 & 63), cc = T.c0 + (e2 >> 6);
      if (rr < T.nn && cc < T.nn) Qn[static_cast<long long>(lo + cc) * m + lo + rr] = Qp[static_cast<long long>(lo + cc) * m + lo + rr];
    }
    return;
  }
  for (int l0 = 0; l0 < T.k; l0 += 16) {
    for (int e2 = threadIdx.x; e2 < 16 * 64; e2 += 256) {
      const int a = e2 & 63, l = e2 >> 6;
      const int rr = T.r0 + a, ll = l0 + l;
      as[l][a] = (rr < T.nn && ll < T.k) ? Qp[static_cast<long long>(lo + ll) * m + lo + rr] : 0.0;
      const int lq = e2 & 15, bcol = e2 >> 4;
      const int cc = T.c0 + bcol;
      bs[lq][bcol] = (l0 + lq < T.k && cc < T.k) ? U[static_cast<long long>(lo + cc) * m + lo + l0 + lq] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int l = 0; l < 16; ++l) {
      double pa[4], pb[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) pa[r] = as[l][tx + 16 * r];
#pragma unroll
      for (int c = 0; c < 4; ++c) pb[c] = bs[l][ty + 16 * c];
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[r][c] = fma(pa[r], pb[c], acc[r][c]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int rr = T.r0 + tx + 16 * r, cc = T.c0 + ty + 16 * c;
      if (rr < T.nn && cc < T.k) Qn[static_cast<long long>(lo + cc) * m + lo + rr] = acc[r][c];
    }
}

// ================================================================ (3) back-transformation helpers
// Vb (m x nbb, ld = m): the reflectors c0 .. c0+nbb of the tridiagonalisation (v_{c+1} = 1, v_r = A(r, c) below)
__global__ void k_bt_vblock(const double* __restrict__ A, int m, int c0, int nbb, double* __restrict__ Vb) {
  const int j = blockIdx.y, c = c0 + j;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < m; r += gridDim.x * blockDim.x) {
    double v = 0.0;
    if (c + 1 < m) v = (r == c + 1) ? 1.0 : (r > c + 1 ? A[r + static_cast<long long>(c) * m] : 0.0);
    Vb[r + static_cast<long long>(j) * m] = v;
  }
}
// Diagonal block q (columns q·TBT .. +nq) of T (upper, ld = ldt) of the compact WY form, from S = VbᵀVb (ld = ldt)
// and τ: T_ii = τ_i, T(r, i) = −τ_i Σ_{l=r}^{i−1} T(r, l) S(l, i) within the block. One CTA per block.
constexpr int TBT = 128;
__global__ void k_bt_tmat(const double* __restrict__ S, const double* __restrict__ tau, int c0, int nbb, int ldt,
                          double* __restrict__ T) {
  __shared__ double col[TBT];
  const int q0 = blockIdx.x * TBT, nq = min(TBT, nbb - q0);
  for (int ii = 0; ii < nq; ++ii) {
    const int i = q0 + ii;
    const double ti = tau[c0 + i];
    for (int r = q0 + threadIdx.x; r < i; r += blockDim.x) {
      double acc = 0.0;
      for (int l = r; l < i; ++l) acc = fma(T[r + static_cast<long long>(l) * ldt], S[l + static_cast<long long>(i) * ldt], acc);
      col[r - q0] = -ti * acc;
    }
    __syncthreads();
    for (int r = q0 + threadIdx.x; r < q0 + nq; r += blockDim.x)
      T[r + static_cast<long long>(i) * ldt] = (r < i) ? col[r - q0] : (r == i ? ti : 0.0);
    __syncthreads();
  }
}


// C = alpha·op(A)·B + beta·C (column-major; op(A) = A (M x K, lda) or Aᵀ with A stored K x M), 64 x 64 tiles,
// 4 x 4 per thread, K-slabs of 16; one fma chain per output over l ascending (deterministic).
__global__ void __launch_bounds__(256) k_dgemm(int M, int N, int K, double alpha, const double* __restrict__ A, int lda,
                                               int ta, const double* __restrict__ B, int ldb, double beta,
                                               double* __restrict__ C, int ldc) {
  __shared__ double as[16][65], bs[16][65];
  const int a0 = blockIdx.x * 64, b0 = blockIdx.y * 64;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  double acc[4][4] = {};
  for (int l0 = 0; l0 < K; l0 += 16) {
    for (int e2 = threadIdx.x; e2 < 16 * 64; e2 += 256) {
      int a, l;
      if (ta) {  // Aᵀ: element (a, l) = A[l + a·lda]: consecutive threads along l
        l = e2 & 15;
        a = e2 >> 4;
      } else {
        a = e2 & 63;
        l = e2 >> 6;
      }
      const int ra = a0 + a, ll = l0 + l;
      double v = 0.0;
      if (ra < M && ll < K) v = ta ? A[ll + static_cast<long long>(ra) * lda] : A[ra + static_cast<long long>(ll) * lda];
      as[l][a] = v;
      const int lq = e2 & 15, bc = e2 >> 4;
      bs[lq][bc] = (l0 + lq < K && b0 + bc < N) ? B[l0 + lq + static_cast<long long>(b0 + bc) * ldb] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int l = 0; l < 16; ++l) {
      double pa[4], pb[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) pa[r] = as[l][tx + 16 * r];
#pragma unroll
      for (int c = 0; c < 4; ++c) pb[c] = bs[l][ty + 16 * c];
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[r][c] = fma(pa[r], pb[c], acc[r][c]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int ra = a0 + tx + 16 * r, cb = b0 + ty + 16 * c;
      if (ra < M && cb < N) {
        double* p = C + ra + static_cast<long long>(cb) * ldc;
        *p = (beta == 0.0) ? alpha * acc[r][c] : fma(alpha, acc[r][c], beta * *p);
      }
    }
}

// Y_sorted[:, j] = Q[:, perm[j]] (ld = m), θ_j = lam[perm[j]]
__global__ void k_dc_final(const int* __restrict__ perm, const double* __restrict__ Q, const double* __restrict__ lam,
                           int m, double* __restrict__ Y, double* __restrict__ theta, int unscale) {
  const int j = blockIdx.y;
  const int p = perm[j];
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < m; r += gridDim.x * blockDim.x)
    Y[r + static_cast<long long>(j) * m] = Q[r + static_cast<long long>(p) * m];
  if (blockIdx.x == 0 && threadIdx.x == 0) theta[j] = ldexp(lam[p], unscale);
}

// Y(0:rows, 0:cols) −= P (Y with leading dimension ldy, P with ldp)
__global__ void k_sub_strided(double* __restrict__ Y, int ldy, const double* __restrict__ P, int ldp, int rows, int cols) {
  const int j = blockIdx.y;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += gridDim.x * blockDim.x)
    Y[r + static_cast<long long>(j) * ldy] -= P[r + static_cast<long long>(j) * ldp];
}

// ---------------------------------------------------------------- (1b) the trailing matrix in one thread-block cluster
// Once the trailing matrix A(k0:m, k0:m) fits in the distributed shared memory of one cluster of CS CTAs, the rest
// of the tridiagonalisation runs unblocked (LAPACK dsytd2 order: reflector of column c, y = τ·A₂₂v,
// y' = y − ½τ(yᵀv)v, A₂₂ −= v y'ᵀ + y' vᵀ) with every matrix element in shared memory: CTA k holds the columns
// q ≡ k (mod CS) of the trailing matrix in full (both triangles, so y_q = τ·A(:, q)ᵀv needs no cross-CTA
// reduction) and updates them itself. Per column c: (B1) the reflector of column c is in every CTA — its owner
// computed it from its own copy of the column (no grid reduction) and pushed v and τ into every CTA over DSMEM;
// every CTA forms y_q for its columns (one warp per column) and pushes y_q and its partial Σ y_q v_q into every
// CTA; (B2) y' = y − ½τ(yᵀv)v locally (the partials summed in a fixed order), then the rank-2 update of the CTA's
// columns. Look-ahead: the owner of column c + 1 updates that column first, forms and pushes its reflector and
// arrives at B1(c + 1) before updating its other columns (split arrive / wait), so the reflector and the v
// transfer overlap the other CTAs' updates. v, y, the partials and τ are double-buffered by column parity. Two
// cluster barriers and no global-memory round trip per column, against two grid-wide barriers and the tile
// partials of the panel kernel (which stays in charge while the trailing matrix is larger). Same reflector
// convention as k_trd_panel (β = −sign(α)·sqrt(α² + σ), τ = (β − α)/β, v_{c+1} = 1, v_r = x_r/(α − β)); every sum
// in a fixed order (deterministic).
constexpr int CT = 512;  // threads per cluster CTA
__device__ __forceinline__ void st_dsmem(double* p, uint32_t rank, double v) {
  uint32_t a;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;"
               : "=r"(a)
               : "r"(static_cast<uint32_t>(__cvta_generic_to_shared(p))), "r"(rank));
  asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
}
__device__ __forceinline__ uint32_t cl_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cl_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__host__ __device__ constexpr size_t trd_cluster_smem(int mp, int cs) {
  return sizeof(double) * (static_cast<size_t>((mp + cs - 1) / cs) * mp + 4 * static_cast<size_t>(mp) + 4 +
                           CT / 32 + 2 * cs + 8);
}
__device__ __forceinline__ double block_sum_ct(double v, double* red) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[w] = v;
  __syncthreads();
  double a = 0.0;
  for (int k = 0; k < CT / 32; ++k) a += red[k];
  return a;
}

template <int CS>
__global__ void __launch_bounds__(CT, 1) k_trd_cluster(double* __restrict__ A, int m, int k0, double* __restrict__ d,
                                                       double* __restrict__ e, double* __restrict__ tau,
                                                       unsigned long long* __restrict__ dbg) {
  extern __shared__ __align__(16) double csm[];
  const int mp = m - k0, NS = (mp + CS - 1) / CS;
  const int rank = static_cast<int>(cl_rank());
  // OZR_SYEV_PROBE: accumulated ns per phase as seen by CTA 1 (an owner one column in CS)
  unsigned long long tl = gtimer();
#define CPROBE(k)                                           \
  if (dbg && rank == 1 && threadIdx.x == 0) {              \
    const unsigned long long tn_ = gtimer();               \
    dbg[8 + (k)] += tn_ - tl;                              \
    tl = tn_;                                              \
  }
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  double* cols = csm;                                   // NS x mp: slot s = column q = s·CS + rank, rows 0..mp−1
  double* vbuf = cols + static_cast<size_t>(NS) * mp;   // [2][mp] v of the pivot column (pushed by its owner)
  double* ybuf = vbuf + 2 * static_cast<size_t>(mp);    // [2][mp] y, then y' (y_q pushed by q's owner)
  double* misc = ybuf + 2 * static_cast<size_t>(mp);    // [parity] τ of the pivot column (pushed by its owner)
  double* red = misc + 4;                               // CT/32 block partials
  double* redc = red + CT / 32;                         // [2][CS] Σ y_q v_q per CTA (pushed, slot = CTA rank)
  const long long ld = m;
  // the trailing matrix, both triangles from the stored lower one (row r, column q relative to k0)
  for (int s = 0; s < NS; ++s) {
    const int q = s * CS + rank;
    if (q >= mp) break;
    for (int r = tid; r < mp; r += CT) {
      const int hi = r >= q ? r : q, lo = r >= q ? q : r;
      cols[static_cast<size_t>(s) * mp + r] = A[(k0 + hi) + (k0 + lo) * ld];
    }
  }
  __syncthreads();
  cl_sync();  // every CTA's shared memory is live before any remote access
  // Reflector of column c (its owner, the column already updated): β, τ, v into the column (the stored reflector)
  // and into vbuf[c & 1] of every CTA; τ into misc[c & 1] of every CTA; d, e, τ out.
  auto reflector = [&](int c) {
    double* col = cols + static_cast<size_t>(c / CS) * mp;
    const int par = c & 1;
    double ss = 0.0;
    for (int r = c + 2 + tid; r < mp; r += CT) ss = fma(col[r], col[r], ss);
    const double sigma = block_sum_ct(ss, red);
    const double alpha = col[c + 1];
    double beta = alpha, tc = 0.0, scale = 0.0;
    if (sigma != 0.0) {
      beta = -copysign(sqrt(fma(alpha, alpha, sigma)), alpha);
      tc = (beta - alpha) / beta;
      scale = 1.0 / (alpha - beta);
    }
    double* vb = vbuf + par * static_cast<size_t>(mp);
    for (int r = c + 1 + tid; r < mp; r += CT) {
      double v = 1.0;
      if (r > c + 1) {
        v = col[r] * scale;
        col[r] = v;
      }
#pragma unroll 4
      for (int k = 0; k < CS; ++k) st_dsmem(vb + r, k, v);
    }
    if (tid == 0) {
      d[k0 + c] = col[c];
      e[k0 + c] = beta;
      tau[k0 + c] = tc;
    }
    if (tid < CS) st_dsmem(misc + par, tid, tc);
    __syncthreads();
  };
  auto arrive = [] { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); };
  auto wait = [] { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); };
  // A₂₂ −= v y'ᵀ + y' vᵀ on this CTA's columns in [qa, qb) (threads over rows r > c, every such column)
  auto update = [&](int c, int sa, int sb) {
    const int par = c & 1;
    const double* vb = vbuf + par * static_cast<size_t>(mp);
    const double* yb = ybuf + par * static_cast<size_t>(mp);
    for (int r = c + 1 + tid; r < mp; r += CT) {
      const double vr = vb[r], yr = yb[r];
      for (int s = sa; s < sb; ++s) {
        const int q = s * CS + rank;
        double* x = cols + static_cast<size_t>(s) * mp + r;
        *x = fma(-vr, yb[q], fma(-yr, vb[q], *x));
      }
    }
    __syncthreads();
  };
  if (rank == 0 && mp >= 2) reflector(0);
  if (mp >= 2) arrive();  // B1(0)
  for (int c = 0; c + 1 < mp; ++c) {
    const int par = c & 1;
    wait();  // B1(c): the reflector of column c is in every CTA, and every CTA has finished column c − 1
    CPROBE(1);
    const double tc = misc[par];
    double* vb = vbuf + par * static_cast<size_t>(mp);
    double* yb = ybuf + par * static_cast<size_t>(mp);
    const int s0 = (c + 1 - rank + CS - 1) / CS;  // first slot with column q > c
    const int s1 = (mp - rank + CS - 1) / CS;     // slots of real columns
    if (tc != 0.0) {
      // y_q = τ·A(c+1:, q)ᵀ v for this CTA's columns q > c: one warp per column, lanes over rows (four chains)
      double part = 0.0;
      for (int s = s0 + wid; s < s1; s += CT / 32) {
        const int q = s * CS + rank;
        const double* col = cols + static_cast<size_t>(s) * mp;
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
        int r = c + 1 + lane;
        for (; r + 96 < mp; r += 128) {
          a0 = fma(col[r], vb[r], a0);
          a1 = fma(col[r + 32], vb[r + 32], a1);
          a2 = fma(col[r + 64], vb[r + 64], a2);
          a3 = fma(col[r + 96], vb[r + 96], a3);
        }
        for (; r < mp; r += 32) a0 = fma(col[r], vb[r], a0);
        double a = (a0 + a1) + (a2 + a3);
        for (int o = 16; o; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
        const double y = tc * a;
        if (lane < CS) st_dsmem(yb + q, lane, y);  // y_q into every CTA (same value in every lane)
        part = fma(y, vb[q], part);                 // lane 0's counts
      }
      if (lane != 0) part = 0.0;
      const double sp = block_sum_ct(part, red);
      if (tid < CS) st_dsmem(redc + par * CS + rank, tid, sp);
    }
    CPROBE(3);
    // B2(c): every y_q and every CTA's Σ y_q v_q have landed. Also when τ = 0: the owner of column c arrived at
    // B1(c) before its deferred update of column c − 1, which reads vbuf[(c − 1) & 1] — the buffer the reflector
    // of column c + 1 is about to fill
    cl_sync();
    CPROBE(4);
    if (tc != 0.0) {
      double yv = 0.0;
      for (int k = 0; k < CS; ++k) yv += redc[par * CS + k];  // fixed order
      const double a2 = -0.5 * tc * yv;
      for (int q = c + 1 + tid; q < mp; q += CT) yb[q] = fma(a2, vb[q], yb[q]);
      __syncthreads();
      CPROBE(5);
    }
    const int c1 = c + 1;
    if (c1 + 1 < mp) {
      if (rank == c1 % CS) {
        // look-ahead: column c + 1 first, its reflector published, the barrier arrived at, then the rest
        const int sp1 = c1 / CS;
        if (tc != 0.0) update(c, sp1, sp1 + 1);
        reflector(c1);
        CPROBE(0);
        arrive();  // B1(c + 1)
        if (tc != 0.0) update(c, sp1 + 1, s1);
      } else {
        if (tc != 0.0) update(c, s0, s1);
        arrive();  // B1(c + 1)
      }
    } else if (tc != 0.0) {
      update(c, s0, s1);
    }
    CPROBE(6);
  }
  // the last diagonal element, and the reflectors back to global memory (rows r ≥ c + 2 of column c)
  if (rank == (mp - 1) % CS && tid == 0) d[k0 + mp - 1] = cols[static_cast<size_t>((mp - 1) / CS) * mp + mp - 1];
  for (int s = 0; s < NS; ++s) {
    const int q = s * CS + rank;
    if (q + 2 >= mp) break;
    for (int r = q + 2 + tid; r < mp; r += CT) A[(k0 + r) + (k0 + q) * ld] = cols[static_cast<size_t>(s) * mp + r];
  }
  cl_sync();  // no CTA leaves while another may still read its shared memory
#undef CPROBE
}


// The largest trailing size k_trd_cluster takes (0: unavailable on this device), and its cluster size. CS = 16
// (non-portable) where the device can co-schedule it, else 8. OZR_TRD_CLUSTER=0 disables it (A/B).
struct TrdCluster {
  int cs = 0, maxmp = 0;
};
TrdCluster trd_cluster_caps() {
  static int dev_seen[64];
  static TrdCluster cap[64];
  static std::mutex mu;
  if (const char* f = getenv("OZR_TRD_CLUSTER"))
    if (f[0] == '0') return {};
  std::lock_guard<std::mutex> g(mu);
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return {};
  if (dev_seen[dev]) return cap[dev];
  dev_seen[dev] = 1;
  int smax = 0;
  cudaDeviceGetAttribute(&smax, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  auto largest = [&](int cs) {
    int mp = 0;
    while (trd_cluster_smem(mp + 1, cs) <= static_cast<size_t>(smax)) ++mp;
    return mp;
  };
  for (int cs : {16, 8}) {
    const void* fn = cs == 16 ? reinterpret_cast<const void*>(k_trd_cluster<16>) : reinterpret_cast<const void*>(k_trd_cluster<8>);
    if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smax) != cudaSuccess) {
      cudaGetLastError();
      continue;
    }
    if (cs == 16 && cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) {
      cudaGetLastError();
      continue;
    }
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(cs);
    cfg.blockDim = dim3(CT);
    cfg.dynamicSmemBytes = smax;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int ncl = 0;
    if (cudaOccupancyMaxActiveClusters(&ncl, fn, &cfg) != cudaSuccess || ncl < 1) {
      cudaGetLastError();
      continue;
    }
    cap[dev] = {cs, largest(cs)};
    break;
  }
  return cap[dev];
}
cudaError_t launch_trd_cluster(const TrdCluster& tc, double* A, int m, int k0, double* d, double* e, double* tau,
                               cudaStream_t s, unsigned long long* dbg) {
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = tc.cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3(tc.cs);
  cfg.blockDim = dim3(CT);
  cfg.dynamicSmemBytes = trd_cluster_smem(m - k0, tc.cs);
  cfg.stream = s;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  if (tc.cs == 16) return cudaLaunchKernelEx(&cfg, k_trd_cluster<16>, A, m, k0, d, e, tau, dbg);
  return cudaLaunchKernelEx(&cfg, k_trd_cluster<8>, A, m, k0, d, e, tau, dbg);
}
}  // namespace

size_t syev_trd_partials(int m, int G) {
  const int mt = (m + TB - 1) / TB;
  return static_cast<size_t>(G) * (5 + 2 * NB) + static_cast<size_t>(mt) * (mt + 1) / 2 * 2 * TB;
}

int syev_trd_grid(int m) {
  // the >48 KB opt-in applies to the current device only: set once per device (ozr_internal.h)
  once_per_device(9, [] {
    return cudaFuncSetAttribute(k_trd_panel, cudaFuncAttributeMaxDynamicSharedMemorySize, sizeof(PanelSmem));
  });
  int per = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_trd_panel, TT, sizeof(PanelSmem));
  per = std::max(per, 1);
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const int mt = (m + TB - 1) / TB;
  // one CTA per row block at least (each owns one); more for the tile products (~mt²/2 tiles), bounded by
  // co-residency; fewer CTAs = cheaper barriers
  // (measured, tools/dev/syev_time.py: m = 2734 tridiagonalisation 56.6 ms at 3·mt CTAs, 64.3 at 5·mt, 66.6 at
  // 2·mt; m = 739 within 4 %; m = 6628 at the co-residency cap either way)
  int want = std::max(mt, std::min(mt * (mt + 1) / 2, 3 * mt));
  if (const char* g = getenv("OZR_SYEV_G")) want = std::max(mt, std::min(mt * (mt + 1) / 2, atoi(g) * mt / 8));  // A/B: G = g/8 · mt
  return std::min(want, nsm * per);
}

// Tridiagonalise A (m x m, lda = m, lower triangle read; overwritten: reflectors below the sub-diagonal).
cudaError_t syev_tridiag(double* A, int m, double* d, double* e, double* tau, double* V, double* W, double* part,
                         int G, cudaStream_t s) {
  unsigned long long* dbg = nullptr;
  if (getenv("OZR_SYEV_PROBE")) {
    cudaMalloc(&dbg, 16 * sizeof(unsigned long long));
    cudaMemsetAsync(dbg, 0, 16 * sizeof(unsigned long long), s);
  }
  const int mt = (m + TB - 1) / TB;
  if (G < mt) return cudaErrorInvalidConfiguration;  // every row block needs its owner CTA (m ≤ ~28000)
  double* yp = part + static_cast<size_t>(G) * (5 + 2 * NB);
  // OZR_SYEV_GDIV = d (A/B only): CTAs per panel from the panel's trailing size, clamp(m'/d, mt, G) — measured
  // no better than the fixed G (m = 2734: 77-85 ms for d = 12..28 against 73 ms fixed)
  static int gfac = -1;
  if (gfac < 0) {
    const char* f = getenv("OZR_SYEV_GDIV");  // A/B: G_panel = m'/GDIV (0: the fixed G)
    gfac = f ? atoi(f) : 0;
  }
  const TrdCluster tcl = trd_cluster_caps();
  for (int k0 = 0; k0 < m; k0 += NB) {
    if (m - k0 <= tcl.maxmp && m - k0 >= 2) {  // the rest inside one cluster's shared memory
      cudaError_t err = launch_trd_cluster(tcl, A, m, k0, d, e, tau, s, dbg);
      if (err != cudaSuccess) return err;
      break;
    }
    const int nb = std::min(NB, m - k0);
    const int Gk = gfac > 0 ? std::max(mt, std::min(G, (m - k0) / gfac)) : G;
    PanelArgs P{A, m, k0, nb, V, W, d, e, tau, part, yp, part + syev_trd_partials(m, G), dbg};
    void* args[] = {&P};
    cudaError_t err = cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_trd_panel), dim3(Gk), dim3(TT), args,
                                                  sizeof(PanelSmem), s);
    if (err != cudaSuccess) return err;
    const int k1 = k0 + nb;
    if (k1 < m) {
      const int J0 = k1 / TB, na = mt - J0;
      k_trd_update<<<na * (na + 1) / 2 + nb, TT, 0, s>>>(A, m, k0, nb, V, W, P.gam);
    } else {
      k_trd_update<<<nb, TT, 0, s>>>(A, m, k0, nb, V, W, P.gam);  // only the reflector copy (na = 0 tiles)
    }
  }
  if (dbg) {
    unsigned long long h[16];
    cudaMemcpyAsync(h, dbg, sizeof h, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    fprintf(stderr, "[ozr syev probe] m=%d G=%d ms: A %.2f sync1 %.2f B-head %.2f tiles %.2f dots %.2f sync2 %.2f C %.2f\n", m, G,
            h[6] * 1e-6, h[0] * 1e-6, h[1] * 1e-6, h[2] * 1e-6, h[3] * 1e-6, h[4] * 1e-6, h[5] * 1e-6);
    fprintf(stderr, "[ozr syev probe] cluster tail (CTA 1) ms: own-reflector %.2f B1-wait %.2f - %.2f y %.2f B2 %.2f y' %.2f update %.2f\n",
            h[8] * 1e-6, h[9] * 1e-6, h[10] * 1e-6, h[11] * 1e-6, h[12] * 1e-6, h[13] * 1e-6, h[14] * 1e-6);
    cudaFree(dbg);
  }
  return cudaGetLastError();
}

}  // namespace ozr

namespace ozr {

void* SyevWorkspace::get(int slot, size_t bytes) {
  if (static_cast<int>(bufs.size()) <= slot) bufs.resize(slot + 1, {nullptr, 0});
  auto& b = bufs[slot];
  if (bytes == 0) bytes = 16;
  if (b.second < bytes) {
    if (b.first) cudaFree(b.first);
    b.first = nullptr;
    b.second = 0;
    if (cudaMalloc(&b.first, bytes) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    b.second = bytes;
  }
  return b.first;
}
SyevWorkspace::~SyevWorkspace() {
  for (auto& b : bufs)
    if (b.first) cudaFree(b.first);
}

void syev_dgemm(int M, int N, int K, double alpha, const double* A, int lda, bool ta, const double* B, int ldb,
                double beta, double* C, int ldc, cudaStream_t s) {
  if (M <= 0 || N <= 0) return;
  k_dgemm<<<dim3((M + 63) / 64, (N + 63) / 64), 256, 0, s>>>(M, N, K, alpha, A, lda, ta ? 1 : 0, B, ldb, beta, C, ldc);
}

namespace {
enum { W_D, W_E, W_TAU, W_V, W_W, W_PART, W_Q0, W_Q1, W_QP, W_U, W_DMOD, W_LAMO, W_LAMN, W_DK, W_ZK, W_ZH, W_TS,
       W_ORG, W_Z, W_I, W_D2, W_NODE, W_TILE, W_ERR, W_VB, W_S, W_T, W_WT, W_WT2, W_P, W_STAGE, W_TT };

struct Node {
  int lo, mid, hi;
};

bool cuda_ok(cudaError_t e, std::string* err, const char* what) {
  if (e == cudaSuccess) return true;
  if (err) *err = std::string(what) + ": " + cudaGetErrorString(e);
  return false;
}
}  // namespace

// K (m x m, ld = m; the lower triangle is read) → eigenvalues θ ascending (device, m) and eigenvectors Y (device,
// m x m, ld = m; may alias K). gemm: the large products of the D&C merges and the back-transformation.
int dense_syev(SyevWorkspace& w, int m, double* K, double* theta, double* Y, const SyevGemm& gemm, int big_gemm_min,
               cudaStream_t s, std::string* err, const SyevDebug* dbg) {
#define SY_ALLOC(ptr, slot, T, cnt)                                        \
  T* ptr = static_cast<T*>(w.get(slot, sizeof(T) * static_cast<size_t>(cnt))); \
  if (!ptr) {                                                              \
    if (err) *err = "dense eigensolver: out of device memory";             \
    return 8;                                                              \
  }
  const size_t mm = static_cast<size_t>(m) * m;
  const int G = syev_trd_grid(m);
  SY_ALLOC(d, W_D, double, m);
  SY_ALLOC(e, W_E, double, m);
  SY_ALLOC(tau, W_TAU, double, m);
  SY_ALLOC(V, W_V, double, static_cast<size_t>(m) * NB);
  SY_ALLOC(Wp, W_W, double, static_cast<size_t>(m) * NB);
  SY_ALLOC(part, W_PART, double, syev_trd_partials(m, G) + NB);  // + the panel's γ_j
  SY_ALLOC(Q0, W_Q0, double, mm);
  SY_ALLOC(Q1, W_Q1, double, mm);
  SY_ALLOC(Qp, W_QP, double, mm);
  SY_ALLOC(U, W_U, double, mm);
  SY_ALLOC(dmod, W_DMOD, double, m);
  SY_ALLOC(lamo, W_LAMO, double, m);
  SY_ALLOC(dk, W_DK, double, m);
  SY_ALLOC(zk, W_ZK, double, m);
  SY_ALLOC(zh, W_ZH, double, m);
  SY_ALLOC(ts, W_TS, double, m);
  SY_ALLOC(org, W_ORG, int, m);
  SY_ALLOC(zv, W_Z, double, m);
  SY_ALLOC(derr, W_ERR, int, 4);
  // staging for the per-level host decisions: pinned host memory
  std::vector<double> hd(m), he(m), hlam(m), hz(m);
  if (!cuda_ok(cudaMemsetAsync(derr, 0, 4 * sizeof(int), s), err, "memset")) return 6;
  const bool trace = getenv("OZR_TRACE") != nullptr;
  cudaEvent_t tev[4] = {};
  if (trace)
    for (auto& ev : tev) cudaEventCreate(&ev);
  if (trace) cudaEventRecord(tev[0], s);
  const bool only_dc = dbg && dbg->d_in;
  if (only_dc) {  // stage (2) alone on a given tridiagonal
    if (!cuda_ok(cudaMemcpyAsync(hd.data(), dbg->d_in, m * sizeof(double), cudaMemcpyDeviceToHost, s), err, "D2H") ||
        (m > 1 && !cuda_ok(cudaMemcpyAsync(he.data(), dbg->e_in, (m - 1) * sizeof(double), cudaMemcpyDeviceToHost, s),
                           err, "D2H")) ||
        !cuda_ok(cudaStreamSynchronize(s), err, "sync"))
      return 6;
    he[m - 1] = 0.0;
    if (!cuda_ok(cudaMemcpyAsync(e, he.data(), m * sizeof(double), cudaMemcpyHostToDevice, s), err, "H2D")) return 6;
  } else {
    // ---- (1) tridiagonalise
    if (!cuda_ok(syev_tridiag(K, m, d, e, tau, V, Wp, part, G, s), err, "tridiagonalisation")) return 6;
    if (dbg && dbg->d_out) {  // stage (1) alone: d, e, τ out (K holds the reflectors)
      if (!cuda_ok(cudaMemcpyAsync(dbg->d_out, d, m * sizeof(double), cudaMemcpyDeviceToDevice, s), err, "copy") ||
          !cuda_ok(cudaMemcpyAsync(dbg->e_out, e, m * sizeof(double), cudaMemcpyDeviceToDevice, s), err, "copy") ||
          !cuda_ok(cudaMemcpyAsync(dbg->tau_out, tau, m * sizeof(double), cudaMemcpyDeviceToDevice, s), err, "copy") ||
          !cuda_ok(cudaStreamSynchronize(s), err, "sync"))
        return 6;
      return 0;
    }
    if (!cuda_ok(cudaMemcpyAsync(hd.data(), d, m * sizeof(double), cudaMemcpyDeviceToHost, s), err, "D2H")) return 6;
    if (m > 1 && !cuda_ok(cudaMemcpyAsync(he.data(), e, (m - 1) * sizeof(double), cudaMemcpyDeviceToHost, s), err, "D2H"))
      return 6;
    if (!cuda_ok(cudaStreamSynchronize(s), err, "sync")) return 6;
    he[m - 1] = 0.0;
  }
  if (trace) cudaEventRecord(tev[1], s);
  // ---- (2) divide and conquer on T·2^s with max|T_ij| ∈ [½, 1) (an exact power-of-two scaling, as LAPACK's dstedc
  // scales to unit norm): the deflation tolerance 8ε·max(|D|, |z|) compares quantities of the same scale only then
  double tnrm = 0.0;
  for (int a = 0; a < m; ++a) tnrm = std::max(tnrm, std::max(std::fabs(hd[a]), std::fabs(he[a])));
  const int sexp = (tnrm > 0.0) ? -std::ilogb(tnrm) - 1 : 0;
  for (int a = 0; a < m; ++a) {
    hd[a] = std::ldexp(hd[a], sexp);
    he[a] = std::ldexp(he[a], sexp);
  }
  if (!cuda_ok(cudaMemcpyAsync(e, he.data(), m * sizeof(double), cudaMemcpyHostToDevice, s), err, "H2D")) return 6;
  // the tree (levels of internal nodes, leaves)
  std::vector<std::vector<Node>> levels;
  std::vector<int> llo, lhi;
  std::vector<double> dm(hd);
  {
    struct Item { int lo, hi, depth; };
    std::vector<Item> stack{{0, m, 0}};
    while (!stack.empty()) {
      Item it = stack.back();
      stack.pop_back();
      if (it.hi - it.lo <= LEAF) {
        llo.push_back(it.lo);
        lhi.push_back(it.hi);
        continue;
      }
      const int mid = (it.lo + it.hi) / 2;
      if (static_cast<int>(levels.size()) <= it.depth) levels.resize(it.depth + 1);
      levels[it.depth].push_back({it.lo, mid, it.hi});
      const double ab = std::fabs(he[mid - 1]);
      dm[mid - 1] -= ab;  // tearing: T = diag(T1', T2') + |β| v vᵀ, v = e_{mid−1} + sign(β) e_mid
      dm[mid] -= ab;
      stack.push_back({it.lo, mid, it.depth + 1});
      stack.push_back({mid, it.hi, it.depth + 1});
    }
  }
  const int nleaf = static_cast<int>(llo.size());
  SY_ALLOC(ibuf, W_I, int, 16 * static_cast<size_t>(m) + 4 * nleaf + 64);
  SY_ALLOC(dbuf, W_D2, double, 4 * static_cast<size_t>(m) + 64);
  {
    std::vector<int> li(2 * nleaf);
    for (int q = 0; q < nleaf; ++q) {
      li[q] = llo[q];
      li[nleaf + q] = lhi[q];
    }
    if (!cuda_ok(cudaMemcpyAsync(ibuf, li.data(), li.size() * sizeof(int), cudaMemcpyHostToDevice, s), err, "H2D") ||
        !cuda_ok(cudaMemcpyAsync(dmod, dm.data(), m * sizeof(double), cudaMemcpyHostToDevice, s), err, "H2D"))
      return 6;
    k_dc_leaf<<<nleaf, LEAF, 0, s>>>(ibuf, ibuf + nleaf, dmod, e, lamo, Q0, m, derr);
    if (!cuda_ok(cudaGetLastError(), err, "leaf solve")) return 6;
    if (!cuda_ok(cudaStreamSynchronize(s), err, "sync")) return 6;  // li is about to go out of scope
  }
  double* Q = Q0;  // node blocks on the diagonal; every merge rewrites its block in place (from the Qp copy)
  const double eps = 1.1102230246251565e-16;
  for (int lev = static_cast<int>(levels.size()) - 1; lev >= 0; --lev) {
    const std::vector<Node>& nodes = levels[lev];
    const int nn_nodes = static_cast<int>(nodes.size());
    // z of every merge, and the current eigenvalues, to the host
    std::vector<int> ni(3 * nn_nodes);
    std::vector<double> sg(nn_nodes);
    for (int q = 0; q < nn_nodes; ++q) {
      ni[q] = nodes[q].lo;
      ni[nn_nodes + q] = nodes[q].mid;
      ni[2 * nn_nodes + q] = nodes[q].hi;
      sg[q] = he[nodes[q].mid - 1] < 0 ? -1.0 : 1.0;
    }
    if (!cuda_ok(cudaMemcpyAsync(ibuf, ni.data(), ni.size() * sizeof(int), cudaMemcpyHostToDevice, s), err, "H2D") ||
        !cuda_ok(cudaMemcpyAsync(dbuf, sg.data(), nn_nodes * sizeof(double), cudaMemcpyHostToDevice, s), err, "H2D"))
      return 6;
    k_dc_zvec<<<dim3(8, nn_nodes), 256, 0, s>>>(ibuf, ibuf + nn_nodes, ibuf + 2 * nn_nodes, dbuf, Q, m, zv);
    if (!cuda_ok(cudaMemcpyAsync(hz.data(), zv, m * sizeof(double), cudaMemcpyDeviceToHost, s), err, "D2H") ||
        !cuda_ok(cudaMemcpyAsync(hlam.data(), lamo, m * sizeof(double), cudaMemcpyDeviceToHost, s), err, "D2H") ||
        !cuda_ok(cudaStreamSynchronize(s), err, "sync"))
      return 6;
    if (getenv("OZR_SYEV_DUMP")) {  // debugging aid: the inputs of every merge level
      FILE* f = fopen((std::string(getenv("OZR_SYEV_DUMP")) + "_lev" + std::to_string(lev) + ".bin").c_str(), "wb");
      if (f) {
        fwrite(hlam.data(), sizeof(double), m, f);
        fwrite(hz.data(), sizeof(double), m, f);
        std::vector<double> hq(mm);
        cudaMemcpy(hq.data(), Q, mm * sizeof(double), cudaMemcpyDeviceToHost);
        fwrite(hq.data(), sizeof(double), mm, f);
        fclose(f);
      }
    }
    // host: sort, deflation (LAPACK dlaed2's rules), the Qp column sources and rotations
    std::vector<int> src(m, 0), rot_off(nn_nodes + 1, 0), root_node, root_j;
    std::vector<int4> rot_idx;
    std::vector<double2> rot_cs;
    std::vector<double> hdk(m, 0.0), hzk(m, 0.0), hlamn(hlam);
    std::vector<DcNode> dn(nn_nodes);
    std::vector<DcTile> tiles;
    std::vector<int> big;  // nodes whose merge product goes to the big GEMM
    for (int q = 0; q < nn_nodes; ++q) {
      const int lo = nodes[q].lo, n = nodes[q].hi - lo;
      const double rho = 2.0 * std::fabs(he[nodes[q].mid - 1]);
      std::vector<int> idx(n);
      for (int a = 0; a < n; ++a) idx[a] = a;
      std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) { return hlam[lo + a] < hlam[lo + b]; });
      std::vector<double> D(n), Z(n);
      double dmax = 0.0, zmax = 0.0;
      for (int a = 0; a < n; ++a) {
        D[a] = hlam[lo + idx[a]];
        Z[a] = hz[lo + idx[a]];
        dmax = std::max(dmax, std::fabs(D[a]));
        zmax = std::max(zmax, std::fabs(Z[a]));
      }
      const double tol = 8.0 * eps * std::max(dmax, zmax);
      std::vector<int> keep, defl;
      std::vector<std::pair<int, int>> rots;
      std::vector<double2> cs;
      int pj = -1;
      for (int j = 0; j < n; ++j) {
        if (rho * std::fabs(Z[j]) <= tol) {
          defl.push_back(j);
          continue;
        }
        if (pj < 0) {
          pj = j;
          continue;
        }
        double sv = Z[pj], cv = Z[j];
        const double tv = std::hypot(cv, sv);
        const double t = D[j] - D[pj];
        cv /= tv;
        sv = -sv / tv;
        if (std::fabs(t * cv * sv) <= tol) {
          Z[j] = tv;
          Z[pj] = 0.0;
          rots.push_back({pj, j});
          cs.push_back(make_double2(cv, sv));
          const double t2 = D[pj] * cv * cv + D[j] * sv * sv;
          D[j] = D[pj] * sv * sv + D[j] * cv * cv;
          D[pj] = t2;
          defl.push_back(pj);
          pj = j;
        } else {
          keep.push_back(pj);
          pj = j;
        }
      }
      if (pj >= 0) keep.push_back(pj);
      const int k = static_cast<int>(keep.size());
      std::vector<int> pos(n);
      for (int a = 0; a < k; ++a) pos[keep[a]] = a;
      for (int a = 0; a < static_cast<int>(defl.size()); ++a) pos[defl[a]] = k + a;
      for (int a = 0; a < n; ++a) src[lo + pos[a]] = idx[a];
      for (size_t r = 0; r < rots.size(); ++r) {
        rot_idx.push_back(make_int4(pos[rots[r].first], pos[rots[r].second], 0, 0));
        rot_cs.push_back(cs[r]);
      }
      rot_off[q + 1] = static_cast<int>(rot_idx.size());
      for (int a = 0; a < k; ++a) {
        hdk[lo + a] = D[keep[a]];
        hzk[lo + a] = Z[keep[a]];
      }
      for (int a = 0; a < static_cast<int>(defl.size()); ++a) hlamn[lo + k + a] = D[defl[a]];
      dn[q] = DcNode{lo, k, rho};
      for (int j = 0; j < k; ++j) {
        root_node.push_back(q);
        root_j.push_back(j);
      }
      const bool use_big = k >= big_gemm_min && gemm;
      if (use_big) big.push_back(q);
      // GEMM tiles (columns [c0, min(c0 + 64, k))) unless the big product takes the node; copy tiles (origin ≥ k)
      // for the deflated columns: one starting at k, then the 64-aligned ones above it (overlaps copy twice)
      for (int r0 = 0; r0 < n; r0 += 64) {
        if (!use_big)
          for (int c0 = 0; c0 < k; c0 += 64) tiles.push_back(DcTile{lo, n, k, r0, c0});
        if (k < n) tiles.push_back(DcTile{lo, n, k, r0, k});
        for (int c0 = (k / 64 + 1) * 64; c0 < n; c0 += 64) tiles.push_back(DcTile{lo, n, k, r0, c0});
      }
    }
    const int nroots = static_cast<int>(root_node.size());
    // upload: ints [src m | rot_off | root_node | root_j], int4 rot_idx, double2 rot_cs, dk, zk, lamn (deflated)
    std::vector<int> pk;
    pk.insert(pk.end(), src.begin(), src.end());
    const size_t o_roff = pk.size();
    pk.insert(pk.end(), rot_off.begin(), rot_off.end());
    const size_t o_rn = pk.size();
    pk.insert(pk.end(), root_node.begin(), root_node.end());
    const size_t o_rj = pk.size();
    pk.insert(pk.end(), root_j.begin(), root_j.end());
    while (pk.size() % 4) pk.push_back(0);
    const size_t o_ri = pk.size();
    for (const int4& v : rot_idx) {
      pk.push_back(v.x); pk.push_back(v.y); pk.push_back(v.z); pk.push_back(v.w);
    }
    const size_t o_nodes = pk.size();
    const int* dnp = reinterpret_cast<const int*>(dn.data());
    pk.insert(pk.end(), dnp, dnp + dn.size() * sizeof(DcNode) / sizeof(int));
    const size_t o_tiles = pk.size();
    const int* tp = reinterpret_cast<const int*>(tiles.data());
    pk.insert(pk.end(), tp, tp + tiles.size() * sizeof(DcTile) / sizeof(int));
    int* dpk = static_cast<int*>(w.get(W_NODE, pk.size() * sizeof(int) + 16));
    double2* dcs = static_cast<double2*>(w.get(W_TILE, (rot_cs.size() + 1) * sizeof(double2)));
    if (!dpk || !dcs) {
      if (err) *err = "dense eigensolver: out of device memory";
      return 8;
    }
    if (!cuda_ok(cudaMemcpyAsync(dpk, pk.data(), pk.size() * sizeof(int), cudaMemcpyHostToDevice, s), err, "H2D") ||
        (!rot_cs.empty() && !cuda_ok(cudaMemcpyAsync(dcs, rot_cs.data(), rot_cs.size() * sizeof(double2),
                                                     cudaMemcpyHostToDevice, s), err, "H2D")) ||
        !cuda_ok(cudaMemcpyAsync(dk, hdk.data(), m * sizeof(double), cudaMemcpyHostToDevice, s), err, "H2D") ||
        !cuda_ok(cudaMemcpyAsync(zk, hzk.data(), m * sizeof(double), cudaMemcpyHostToDevice, s), err, "H2D") ||
        !cuda_ok(cudaMemcpyAsync(lamo, hlamn.data(), m * sizeof(double), cudaMemcpyHostToDevice, s), err, "H2D"))
      return 6;
    const DcNode* dnd = reinterpret_cast<const DcNode*>(dpk + o_nodes);
    int maxn = 0;
    for (const Node& nd : nodes) maxn = std::max(maxn, nd.hi - nd.lo);
    // the node lo/hi arrays for permrot: reuse ibuf (still holds lo | mid | hi)
    k_dc_permrot<<<dim3((maxn + 127) / 128, nn_nodes), 128, 0, s>>>(ibuf, ibuf + nn_nodes, ibuf + 2 * nn_nodes, dpk, dpk + o_roff,
                                                                   reinterpret_cast<const int4*>(dpk + o_ri), dcs, Q, Qp, m);
    if (nroots > 0) {
      k_dc_secular<<<(nroots + 127) / 128, 128, 0, s>>>(dnd, dpk + o_rn, dpk + o_rj, nroots, dk, zk, org, ts);
      k_dc_zhat<<<(nroots + 127) / 128, 128, 0, s>>>(dnd, dpk + o_rn, dpk + o_rj, nroots, dk, zk, org, ts, zh);
      k_dc_umat<<<nroots, 256, 0, s>>>(dnd, dpk + o_rn, dpk + o_rj, dk, org, ts, zh, U, m, lamo);
    }
    if (!tiles.empty())
      k_dc_gemm<<<static_cast<int>(tiles.size()), 256, 0, s>>>(reinterpret_cast<const DcTile*>(dpk + o_tiles), Qp, U, Q, m);
    if (!cuda_ok(cudaGetLastError(), err, "merge")) return 6;
    for (int q : big) {  // Qn[:, lo .. lo+k) = Qp[:, lo .. lo+k) · U_kk (node block)
      const int lo = nodes[q].lo, n = nodes[q].hi - lo, k = dn[q].k;
      const size_t off = static_cast<size_t>(lo) * m + lo;
      if (gemm(n, k, k, Qp + off, m, false, U + off, m, Q + off, m) != 0) {
        if (err) *err = "dense eigensolver: merge product failed";
        return 6;
      }
    }
    if (!cuda_ok(cudaStreamSynchronize(s), err, "sync")) return 6;  // the staging vectors go out of scope
  }
  if (getenv("OZR_SYEV_DUMP")) {
    FILE* f = fopen((std::string(getenv("OZR_SYEV_DUMP")) + "_final.bin").c_str(), "wb");
    if (f) {
      std::vector<double> hq(mm), hl(m);
      cudaMemcpy(hq.data(), Q, mm * sizeof(double), cudaMemcpyDeviceToHost);
      cudaMemcpy(hl.data(), lamo, m * sizeof(double), cudaMemcpyDeviceToHost);
      fwrite(hl.data(), sizeof(double), m, f);
      fwrite(hq.data(), sizeof(double), mm, f);
      fclose(f);
    }
  }
  // eigenvalues ascending, columns permuted accordingly
  if (!cuda_ok(cudaMemcpyAsync(hlam.data(), lamo, m * sizeof(double), cudaMemcpyDeviceToHost, s), err, "D2H") ||
      !cuda_ok(cudaStreamSynchronize(s), err, "sync"))
    return 6;
  std::vector<int> perm(m);
  for (int a = 0; a < m; ++a) perm[a] = a;
  std::stable_sort(perm.begin(), perm.end(), [&](int a, int b) { return hlam[a] < hlam[b]; });
  if (!cuda_ok(cudaMemcpyAsync(ibuf, perm.data(), m * sizeof(int), cudaMemcpyHostToDevice, s), err, "H2D")) return 6;
  double* Yt = Q1;  // Q_T sorted
  k_dc_final<<<dim3(std::max(1, std::min(16, (m + 255) / 256)), m), 256, 0, s>>>(ibuf, Q, lamo, m, Yt, theta, -sexp);
  if (only_dc) {
    if (!cuda_ok(cudaMemcpyAsync(Y, Yt, mm * sizeof(double), cudaMemcpyDeviceToDevice, s), err, "copy") ||
        !cuda_ok(cudaStreamSynchronize(s), err, "sync"))
      return 6;
    return 0;
  }
  if (trace) cudaEventRecord(tev[2], s);
  // ---- (3) back-transformation Y = Qᴴ·Q_T, blocks of NBB reflectors from the last to the first
  constexpr int NBB = 512;  // reflectors per pass over Y (blocks of TBT = 128 merged into one compact WY T)
  SY_ALLOC(Vb, W_VB, double, static_cast<size_t>(m) * NBB);
  SY_ALLOC(S, W_S, double, NBB * NBB);
  SY_ALLOC(Tm, W_T, double, NBB * NBB);
  SY_ALLOC(Tt, W_TT, double, NBB * TBT);
  SY_ALLOC(Wt, W_WT, double, static_cast<size_t>(NBB) * m);
  SY_ALLOC(Wt2, W_WT2, double, static_cast<size_t>(NBB) * m);
  double* Pb = nullptr;
  const bool bigbt = gemm && m >= big_gemm_min;
  if (bigbt) {
    Pb = static_cast<double*>(w.get(W_P, sizeof(double) * mm));
    if (!Pb) {
      if (err) *err = "dense eigensolver: out of device memory";
      return 8;
    }
  }
  const int nref = m - 1;  // reflectors c = 0 .. m−2 (the last is the identity)
  for (int c0 = ((nref - 1) / NBB) * NBB; c0 >= 0; c0 -= NBB) {
    const int nbb = std::min(NBB, nref - c0);
    if (nbb <= 0) continue;
    const int r0 = c0 + 1, rows = m - r0;  // rows of Vb that can be nonzero
    k_bt_vblock<<<dim3(std::max(1, std::min(32, (m + 255) / 256)), nbb), 256, 0, s>>>(K, m, c0, nbb, Vb);
    syev_dgemm(nbb, nbb, rows, 1.0, Vb + r0, m, true, Vb + r0, m, 0.0, S, nbb, s);  // S = VbᵀVb
    if (!cuda_ok(cudaMemsetAsync(Tm, 0, sizeof(double) * nbb * nbb, s), err, "memset")) return 6;
    const int nsub = (nbb + TBT - 1) / TBT;
    k_bt_tmat<<<nsub, 128, 0, s>>>(S, tau, c0, nbb, nbb, Tm);
    for (int q = 1; q < nsub; ++q) {  // T(0:k, q) = −T(0:k, 0:k)·S(0:k, q)·T_qq, k = q·TBT
      const int k = q * TBT, nq = std::min(TBT, nbb - k);
      syev_dgemm(k, nq, nq, 1.0, S + static_cast<size_t>(k) * nbb, nbb, false, Tm + k + static_cast<size_t>(k) * nbb, nbb,
                 0.0, Tt, k, s);
      syev_dgemm(k, nq, k, -1.0, Tm, nbb, false, Tt, k, 0.0, Tm + static_cast<size_t>(k) * nbb, nbb, s);
    }
    if (bigbt) {
      if (gemm(nbb, m, rows, Vb + r0, m, true, Yt + r0, m, Wt, nbb) != 0) {  // Wt = VbᵀY
        if (err) *err = "dense eigensolver: back-transformation product failed";
        return 6;
      }
    } else {
      syev_dgemm(nbb, m, rows, 1.0, Vb + r0, m, true, Yt + r0, m, 0.0, Wt, nbb, s);
    }
    syev_dgemm(nbb, m, nbb, 1.0, Tm, nbb, false, Wt, nbb, 0.0, Wt2, nbb, s);  // Wt2 = T·Wt
    if (bigbt) {
      if (gemm(rows, m, nbb, Vb + r0, m, false, Wt2, nbb, Pb, rows) != 0) {  // P = Vb·Wt2
        if (err) *err = "dense eigensolver: back-transformation product failed";
        return 6;
      }
      k_sub_strided<<<dim3(std::max(1, std::min(16, (rows + 255) / 256)), m), 256, 0, s>>>(Yt + r0, m, Pb, rows, rows, m);
    } else {
      syev_dgemm(rows, m, nbb, -1.0, Vb + r0, m, false, Wt2, nbb, 1.0, Yt + r0, m, s);  // Y −= Vb·Wt2
    }
  }
  if (!cuda_ok(cudaGetLastError(), err, "back-transformation")) return 6;
  if (Y != Yt && !cuda_ok(cudaMemcpyAsync(Y, Yt, mm * sizeof(double), cudaMemcpyDeviceToDevice, s), err, "copy")) return 6;
  int herr = 0;
  if (!cuda_ok(cudaMemcpyAsync(&herr, derr, sizeof(int), cudaMemcpyDeviceToHost, s), err, "D2H") ||
      !cuda_ok(cudaStreamSynchronize(s), err, "sync"))
    return 6;
  if (trace) {
    cudaEventRecord(tev[3], s);
    cudaEventSynchronize(tev[3]);
    float t1 = 0, t2 = 0, t3 = 0;
    cudaEventElapsedTime(&t1, tev[0], tev[1]);
    cudaEventElapsedTime(&t2, tev[1], tev[2]);
    cudaEventElapsedTime(&t3, tev[2], tev[3]);
    fprintf(stderr, "[ozr syev] m=%d G=%d tridiag %.3f ms, divide-and-conquer %.3f ms, back-transformation %.3f ms\n", m, G,
            t1, t2, t3);
    for (auto& ev : tev) cudaEventDestroy(ev);
  }
  if (herr) {
    if (err) *err = "dense eigensolver: a leaf QL iteration did not converge";
    return 6;
  }
  return 0;
#undef SY_ALLOC
}

}  // namespace ozr
