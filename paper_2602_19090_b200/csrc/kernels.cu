// kernels.cu — the HBM-bound kernels of one ozr sweep. Each is "one CTA per column": the column
// is re-read from L2 between passes, every reduction has a fixed shape (deterministic; integer
// reductions are exact), and a column is produced by exactly one CTA (the block-column partition
// of X̂ across GPUs changes nothing).
//
//   k_colmax          w_j = max_i |x_ij|
//   k_x1_split        X̂ → X̂^(1) by the τ trick (eq. tau/x, s = 1), its INT8
//                     digits, g_j, and r_j = 1 − x̂_jᵀx̂_j EXACTLY (Alg. 1 line 2)
//   k_split_fixed     column-wise fixed-point digits of an fp64 or double-double matrix (R5/R6)
//   k_transpose_i8    digit planes [p][col][row] → [p][row][col] (A operand of X̂^(1)·Ẽ)
//   k_transpose_f64   fp64 transpose (ROWWISE splits of ozr_split / ozr_gemm)
//   k_recombine_V     V = Σ slice products (exact) → dd; λ̂_j = x̂_jᵀv_j/(1−r_j); Res = V − X̂D̂;
//                     column maxima of Res                            (Alg. 1 lines 1,3,4)
//   k_recombine_E     W → Ẽ (Alg. 1 line 5), scaled Ẽ' = diag(2^g)Ẽ, column maxima, ‖Ẽ‖_F parts
//   k_final           U = X̂^(1)Ẽ → X̂ ← RN(X̂^(1) + U) (Alg. 1 line 6, accsum), ν, column maxima
//   k_recombine_dd    generic recombination for ozr_gemm
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#include "ddmath.cuh"
#include "kernels.h"
#include "ozr_internal.h"
#include "ptx.cuh"

namespace ozr {

namespace {

constexpr int BS = 256;  // threads per CTA of every column kernel

// ---------------------------------------------------------------- deterministic block reductions
__device__ __forceinline__ double block_max(double v, double* sh) {
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  double r = sh[0];
  for (int i = 1; i < BS / 32; ++i) r = fmax(r, sh[i]);
  __syncthreads();
  return r;
}

__device__ __forceinline__ double block_sum(double v, double* sh) {  // fixed butterfly + fixed order
  for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  double r = sh[0];
  for (int i = 1; i < BS / 32; ++i) r = __dadd_rn(r, sh[i]);
  __syncthreads();
  return r;
}

__device__ __forceinline__ dd block_sum_dd(dd v, double* sh) {
  for (int o = 16; o > 0; o >>= 1) {
    dd u;
    u.hi = __shfl_xor_sync(0xffffffffu, v.hi, o);
    u.lo = __shfl_xor_sync(0xffffffffu, v.lo, o);
    v = dd_add(v, u);
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) {
    sh[2 * w] = v.hi;
    sh[2 * w + 1] = v.lo;
  }
  __syncthreads();
  dd r{sh[0], sh[1]};
  for (int i = 1; i < BS / 32; ++i) r = dd_add(r, dd{sh[2 * i], sh[2 * i + 1]});
  __syncthreads();
  return r;
}

__device__ __forceinline__ i128 block_sum_i128(i128 v, i128* sh) {  // exact: order irrelevant
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  for (int o = 16; o > 0; o >>= 1) {
    uint64_t lo = static_cast<uint64_t>(v), hi = static_cast<uint64_t>(static_cast<u128>(v) >> 64);
    uint64_t lo2 = __shfl_xor_sync(0xffffffffu, lo, o), hi2 = __shfl_xor_sync(0xffffffffu, hi, o);
    v += static_cast<i128>((static_cast<u128>(hi2) << 64) | lo2);
  }
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  i128 r = 0;
  for (int i = 0; i < BS / 32; ++i) r += sh[i];
  __syncthreads();
  return r;
}

// ---------------------------------------------------------------- recombination of one element
// value = Σ_chunks T_c · 2^{8(L − dhi_c) + e}, T_c = Horner over the chunk's groups (exact int128).
__device__ __forceinline__ void flush_chunk(dd& acc, bool& first, i128 T, int dlast, int L, int e) {
  dd v = i128_to_dd(T);
  const int sc = 8 * (L - dlast) + e;
  v.hi = ldexp_fast(v.hi, sc);
  v.lo = ldexp_fast(v.lo, sc);
  acc = first ? v : dd_add(acc, v);
  first = false;
}

// c0·2^24 + c1·2^16 + c2·2^8 + c3 exactly (|c| < 2^31, |limb| < 2^55), as a depth-2 tree of 64-bit adds (the
// Horner form is a dependent chain of three 64-bit multiply-adds)
__device__ __forceinline__ long long limb4(int32_t c0, int32_t c1, int32_t c2, int32_t c3) {
  const long long a = (static_cast<long long>(c0) << 24) + (static_cast<long long>(c1) << 16);
  const long long b = (static_cast<long long>(c2) << 8) + static_cast<long long>(c3);
  return a + b;
}

constexpr int kRegGroups = 24;  // plans up to this many groups keep every plane value in registers
constexpr int kFastGroups = 12;  // consecutive-diagonal plans up to this many groups: 64-bit limb Horner

__device__ __forceinline__ dd recombine_elem(const int32_t* __restrict__ planes, long long pstride, long long off,
                                             const RecombPlan& rp, int e, int Lj) {
  dd acc{0.0, 0.0};
  bool first = true;
  if (rp.consecutive) {
    // one group per diagonal d0, d0+1, ...: T = Σ_g c_g·256^{4·nl−1−g} (zero-padded to whole limbs),
    // four groups per exact int64 limb (|limb| < 2^55), limbs joined with constant 32-bit shifts — the
    // same exact integer as the general Horner below, without variable 128-bit shifts
    const int d0 = rp.diag[0];
    const int nact = min(rp.ngroups, Lj - d0 + 1);
    int32_t c[kFastGroups];
#pragma unroll
    for (int g = 0; g < kFastGroups; ++g) c[g] = (g < nact) ? __ldg(planes + g * pstride + off) : 0;
    long long Lm[kFastGroups / 4];
#pragma unroll
    for (int k = 0; k < kFastGroups / 4; ++k)
      Lm[k] = ((static_cast<long long>(c[4 * k]) * 256 + c[4 * k + 1]) * 256 + c[4 * k + 2]) * 256 + c[4 * k + 3];
    const int nl = (rp.ngroups + 3) >> 2;
    i128 T = Lm[0];
#pragma unroll
    for (int k = 1; k < kFastGroups / 4; ++k)
      if (k < nl) T = static_cast<i128>(static_cast<u128>(T) << 32) + static_cast<i128>(Lm[k]);
    flush_chunk(acc, first, T, d0 + 4 * nl - 1, rp.L, e);
    return acc;
  }
  if (rp.nchunks == 1 && rp.ngroups <= kRegGroups) {
    // one int128 chunk (the common case): issue every plane load first (memory-level parallelism),
    // then an unrolled Horner
    int32_t c[kRegGroups];
#pragma unroll
    for (int g = 0; g < kRegGroups; ++g)
      c[g] = (g < rp.ngroups && rp.diag[g] <= Lj) ? __ldg(planes + g * pstride + off) : 0;
    i128 T = 0;
    int dprev = rp.diag[0];
#pragma unroll
    for (int g = 0; g < kRegGroups; ++g) {
      if (g < rp.ngroups) {
        const int d = rp.diag[g];
        T = static_cast<i128>(static_cast<u128>(T) << (8 * (d - dprev))) + static_cast<i128>(c[g]);
        dprev = d;
      }
    }
    flush_chunk(acc, first, T, dprev, rp.L, e);
    return acc;
  }
  for (int c = 0; c < rp.nchunks; ++c) {
    i128 T = 0;
    int dprev = rp.diag[rp.chunk_first[c]];
    for (int g = rp.chunk_first[c]; g < rp.chunk_first[c + 1]; ++g) {
      const int d = rp.diag[g];
      const int32_t cv = (d <= Lj) ? __ldg(planes + g * pstride + off) : 0;
      T = static_cast<i128>(static_cast<u128>(T) << (8 * (d - dprev))) + static_cast<i128>(cv);
      dprev = d;
    }
    flush_chunk(acc, first, T, dprev, rp.L, e);
  }
  return acc;
}

__device__ int g_fastdd = 1;  // OZR_FASTDD=0 (A/B only): the limb → double-double fast paths off

// Column sweep (register path): f(i, v) for every row i of the column at `coloff`, e(i) its exponent.
template <class EF, class F>
__device__ __forceinline__ void for_column(const int32_t* __restrict__ planes, long long pstride, long long coloff,
                                           int rows, const RecombPlan& rp, int Lj, EF e, F f) {
  if (!rp.consecutive) {
    for (int i = threadIdx.x; i < rows; i += BS) f(i, recombine_elem(planes, pstride, coloff + i, rp, e(i), Lj));
    return;
  }
  const int d0 = rp.diag[0];
  const int nact = min(rp.ngroups, Lj - d0 + 1);
  const int nl = (rp.ngroups + 3) >> 2;
  const int dlast = d0 + 4 * nl - 1;
  auto fetch = [&](int i, int32_t (&c)[kFastGroups]) {
#pragma unroll
    for (int g = 0; g < kFastGroups; ++g) c[g] = (g < nact && i < rows) ? __ldg(planes + g * pstride + coloff + i) : 0;
  };
  auto combine = [&](const int32_t (&c)[kFastGroups], int ee) {
    long long Lm[kFastGroups / 4];
#pragma unroll
    for (int k = 0; k < kFastGroups / 4; ++k)
      Lm[k] = ((static_cast<long long>(c[4 * k]) * 256 + c[4 * k + 1]) * 256 + c[4 * k + 2]) * 256 + c[4 * k + 3];
    i128 T = Lm[0];
#pragma unroll
    for (int k = 1; k < kFastGroups / 4; ++k)
      if (k < nl) T = static_cast<i128>(static_cast<u128>(T) << 32) + static_cast<i128>(Lm[k]);
    dd acc{0.0, 0.0};
    bool first = true;
    flush_chunk(acc, first, T, dlast, rp.L, ee);
    return acc;
  };
  // one row at a time: the two-rows-in-flight form of this loop (row i + BS's plane loads issued before row i is
  // combined) gave run-to-run different results in the first row of each pair on sm_100a when compiled at the
  // register budget of the 2-CTA-per-SM variants (measured: tools/dev/tma_ab.py, OZR_NO_TMA=4); this path is the
  // fallback for unaligned operands and the experimental column bands, so it takes the plain form
  int32_t ca[kFastGroups];
  for (int i0 = threadIdx.x; i0 < rows; i0 += BS) {
    fetch(i0, ca);
    f(i0, combine(ca, e(i0)));
  }
}

// TMA-staged column sweep (HBM-bound recombination kernels): the column's plane segments and up to two
// fp64 side columns stream through a shared-memory ring filled by 1-D bulk copies (cp.async.bulk + mbarrier),
// one stage = TR rows = two rows per thread. A stage holds only the column's ACTIVE planes (nact ≤ NG: the
// per-tile budgets skip the groups above the tile's L), so its size follows the column, and the ring takes as
// many stages as the launch's shared-memory budget holds (≤ kMaxStages): with few active planes more stages —
// more bytes in flight — keep the copies ahead of the element loop. f(i, v, xv) gets the recombined element and
// the side-column values of row i. Requires rp.consecutive and 16-byte aligned segments (rows % 4 == 0, even
// leading dimensions) — checked by the host (`use_tma`); else the register path.
constexpr int RPT = 2;         // rows per thread per stage (two independent element chains per thread)

constexpr int kMaxStages = 8;
// dynamic shared memory of a TMA launch: the ring budget + the stage barriers. Per kernel (measured, n = 8192):
// recombine_V and final 70 KB (3 CTAs per SM: V's second pass and final's element chain want the extra bytes in
// flight), recombine_E 54 KB (4 CTAs per SM: its FP64 division wants the warps)
constexpr int kRingV = 70 * 1024, kRingE = 54 * 1024, kRingF = 70 * 1024;
// the ring actually allocated: at least two stages of the largest layout of NG planes + NX fp64 sides + the
// int32 side (so ts ≥ 2 always fits)
__host__ __device__ constexpr int ring_for(int ring, int ng, int nx, int rpt = RPT) {
  return ring > 2 * (((ng + 1) * rpt * BS * 4 + nx * rpt * BS * 8 + rpt * BS * 4 + 127) / 128 * 128)
             ? ring
             : 2 * (((ng + 1) * rpt * BS * 4 + nx * rpt * BS * 8 + rpt * BS * 4 + 127) / 128 * 128);
}
__host__ __device__ constexpr int tma_smem(int ring) { return ring + 2 * kMaxStages * 8; }

// icol (nullable): an int32 per-row vector staged beside the planes (the row exponents); e(i, icol[i]).
template <int NX, bool HI_ONLY = false, int NG = kFastGroups, int RING = kRingV, int RPTT = RPT, class EF, class F>
__device__ __forceinline__ void for_column_x(const int32_t* __restrict__ planes, long long pstride, long long coloff,
                                             int rows, const RecombPlan& rp, int Lj, const double* const* xcol,
                                             const int32_t* __restrict__ icol, int use_tma, unsigned char* tsm, EF e,
                                             F f) {
  if (!use_tma) {
    for_column(planes, pstride, coloff, rows, rp, Lj, [&](int i) { return e(i, icol ? icol[i] : 0); },
               [&](int i, const dd& v) {
                 double xv[NX > 0 ? NX : 1];
#pragma unroll
                 for (int x = 0; x < NX; ++x) xv[x] = xcol[x][i];
                 f(i, v, xv);
               });
    return;
  }
  constexpr int TRL = RPTT * BS;  // rows per stage
  const int tid = threadIdx.x;
  const int d0 = rp.diag[0];
  const int nact = max(0, min(rp.ngroups, Lj - d0 + 1));
  const int nl = (rp.ngroups + 3) >> 2;
  const int dlast = d0 + 4 * nl - 1;
  const int sc0 = 8 * (rp.L - dlast);
  const int nch = (rows + TRL - 1) / TRL;
  // this column's stage layout: nact planes | one zero plane (read for the slots nact..NG−1, branch-free) |
  // NX fp64 sides | the int32 side
  const int kSideX = (nact + 1) * TRL * 4, kSideI = kSideX + NX * TRL * 8;
  const int kStageBytes = (kSideI + (icol ? TRL * 4 : 0) + 127) & ~127;
  constexpr int kRing = ring_for(RING, NG, NX, RPTT);
  const int ts = max(2, min(kMaxStages, kRing / kStageBytes));  // kRing ≥ 2·kStageBytes by construction
  uint64_t* bar = reinterpret_cast<uint64_t*>(tsm + kRing);  // full[st]: the stage's copies landed
  uint64_t* ebar = bar + kMaxStages;                          // empty[st]: every warp is done with it
  if (tid == 0) {
    for (int st = 0; st < ts; ++st) {
      mbar_init(&bar[st], 1);
      mbar_init(&ebar[st], BS / 32);
    }
    fence_mbar_init();
  }
  for (int st = 0; st < ts; ++st)  // the zero planes (never written by the copies)
    for (int r = tid; r < TRL; r += BS) reinterpret_cast<int32_t*>(tsm + st * kStageBytes + nact * TRL * 4)[r] = 0;
  __syncthreads();
  auto issue = [&](int c, int st) {  // chunk c into stage st
    const int r0 = c * TRL, nr = min(TRL, rows - r0);
    unsigned char* base = tsm + st * kStageBytes;
    const uint32_t pb = static_cast<uint32_t>(nr) * 4u, xb = static_cast<uint32_t>(nr) * 8u;
    mbar_arrive_expect_tx(&bar[st], nact * pb + NX * xb + (icol ? pb : 0u));
    for (int g = 0; g < nact; ++g) bulk_g2s(base + g * TRL * 4, planes + g * pstride + coloff + r0, pb, &bar[st]);
    for (int x = 0; x < NX; ++x) bulk_g2s(base + kSideX + x * TRL * 8, xcol[x] + r0, xb, &bar[st]);
    if (icol) bulk_g2s(base + kSideI, icol + r0, pb, &bar[st]);
  };
  if (tid == 0)
    for (int c = 0; c < ts - 1 && c < nch; ++c) issue(c, c);
  int st = 0, ph = 0;  // stage and mbarrier parity of chunk c (no per-chunk division by the runtime ts)
  for (int c = 0; c < nch; ++c) {
    // chunk c + ts − 1 goes into the stage chunk c − 1 used, once every warp has released it (its empty
    // barrier; the other warps do not wait for one another)
    if (tid == 0 && c + ts - 1 < nch) {
      const int sp = st == 0 ? ts - 1 : st - 1;
      if (c > 0) mbar_wait(&ebar[sp], st == 0 ? (ph ^ 1) : ph);
      issue(c + ts - 1, sp);
    }
    mbar_wait(&bar[st], ph);
    const unsigned char* base = tsm + st * kStageBytes;
    const int st_used = st;
    if (++st == ts) {
      st = 0;
      ph ^= 1;
    }
#pragma unroll
    for (int h = 0; h < RPTT; ++h) {
    const int tl = tid + h * BS;  // row within the stage
    const int i = c * TRL + tl;
    if (i < rows) {
      // NG: groups compiled for this launch (4, 8 or 12 ≥ ngroups); the slots above nact read the zero plane
      int32_t cv[NG];
      const int32_t* pl = reinterpret_cast<const int32_t*>(base) + tl;
#pragma unroll
      for (int g = 0; g < NG; ++g) cv[g] = pl[min(g, nact) * TRL];
      long long Lm[NG / 4];
#pragma unroll
      for (int k = 0; k < NG / 4; ++k)
        Lm[k] = limb4(cv[4 * k], cv[4 * k + 1], cv[4 * k + 2], cv[4 * k + 3]);
      dd v{0.0, 0.0};
      const int ee = e(i, icol ? reinterpret_cast<const int32_t*>(base + kSideI)[tl] : 0);
      if (HI_ONLY && NG <= 8) {  // RN(value) from the one or two limbs, without 128-bit arithmetic
        const double hv = (nl == 1) ? __ll2double_rn(Lm[0]) : limbs2_rn(Lm[0], Lm[NG / 4 - 1]);
        v.hi = ldexp_fast(hv, sc0 + ee);
      } else if (g_fastdd && (NG == 4 || (NG <= 8 && nl == 1))) {  // one limb (|T| < 2^55): hi = RN(T), lo = T − hi exactly
        const double hv = __ll2double_rn(Lm[0]);
        const double lv = static_cast<double>(Lm[0] - __double2ll_rz(hv));
        v.hi = ldexp_fast(hv, sc0 + ee);
        v.lo = ldexp_fast(lv, sc0 + ee);
      } else if (g_fastdd && NG == 8) {  // two limbs: T = s·2^32 + b (s = L0 + ⌊L1/2^32⌋, 0 ≤ b < 2^32)
        const long long sL = Lm[0] + (Lm[1] >> 32);
        const double bd = static_cast<double>(static_cast<unsigned long long>(Lm[1]) & 0xFFFFFFFFull);
        if (sL > -(1LL << 47) && sL < (1LL << 47)) {
          // |T| < 2^79: hi = RN(s·2^32 + b) in one fma; T − hi = (s·2^32 − hi) + b with s·2^32 − hi exact in
          // the fma (|T − hi| ≤ ulp(hi)/2 < 2^26, b < 2^32: the sum is an exact integer below 2^34)
          const double sd = static_cast<double>(sL);
          const double hv = fma(sd, 4294967296.0, bd);
          const double lv = fma(sd, 4294967296.0, -hv) + bd;
          v.hi = ldexp_fast(hv, sc0 + ee);
          v.lo = ldexp_fast(lv, sc0 + ee);
        } else {
          const i128 T = static_cast<i128>(static_cast<u128>(static_cast<i128>(Lm[0])) << 32) + static_cast<i128>(Lm[1]);
          bool first = true;
          flush_chunk(v, first, T, dlast, rp.L, ee);
        }
      } else {
        i128 T = Lm[0];
#pragma unroll
        for (int k = 1; k < NG / 4; ++k)
          if (k < nl) T = static_cast<i128>(static_cast<u128>(T) << 32) + static_cast<i128>(Lm[k]);
        if (HI_ONLY) {  // the caller uses RN(value) only (its hi part is the same correctly rounded double)
          v.hi = ldexp_fast(i128_to_f64(T), sc0 + ee);
        } else {
          bool first = true;
          flush_chunk(v, first, T, dlast, rp.L, ee);
        }
      }
      double xv[NX > 0 ? NX : 1];
#pragma unroll
      for (int x = 0; x < NX; ++x) xv[x] = reinterpret_cast<const double*>(base + kSideX + x * TRL * 8)[tl];
      f(i, v, xv);
    }
    }
    __syncwarp();
    if ((tid & 31) == 0) mbar_arrive(&ebar[st_used]);
  }
  __syncthreads();  // the caller's block reductions reuse shared memory
}

// ---------------------------------------------------------------- device union-find (cluster branch)
__device__ __forceinline__ int uf_find(int* parent, int a) {
  int p = parent[a];
  while (p != a) {
    const int gp = parent[p];
    parent[a] = gp;  // path halving (a benign race: any ancestor is a valid parent)
    a = p;
    p = gp;
  }
  return a;
}
// link the larger root under the smaller one; retried until both are in one set
__device__ __forceinline__ void uf_unite(int* parent, int a, int b) {
  while (true) {
    a = uf_find(parent, a);
    b = uf_find(parent, b);
    if (a == b) return;
    if (a > b) {
      const int t = a;
      a = b;
      b = t;
    }
    if (atomicCAS(parent + b, b, a) == b) return;
  }
}

__global__ void k_iota(int* p, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = i;
}
__global__ void k_uf_flatten(int* parent, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    int a = i;
    while (parent[a] != a) a = parent[a];
    parent[i] = a;
  }
}

// ---------------------------------------------------------------- kernels
__global__ void __launch_bounds__(BS) k_colmax(const double* __restrict__ X, long long ldx, int rows,
                                               double* __restrict__ w, int* __restrict__ err) {
  __shared__ double sh[BS / 32];
  const double* col = X + blockIdx.x * ldx;
  double m = 0.0;
  bool bad = false;
  for (int i = threadIdx.x; i < rows; i += BS) {
    const double x = col[i];
    bad |= !isfinite(x);
    m = fmax(m, fabs(x));
  }
  if (bad) atomicOr(err, ERR_NONFINITE);
  m = block_max(m, sh);
  if (threadIdx.x == 0) w[blockIdx.x] = m;
}

// Digits of four consecutive rows, packed per plane into one 32-bit store (byte r = row i0 + r).
// k <= 8 with |p| ≤ 2^{8(k−1)+6} + 1 (every split of R5/R6): the excess-128 digits are the bytes of
// w = p + 0x8080808080808080 (mod 2^64) XOR 0x80 — the top digit is |d| ≤ 65, so nothing carries past byte
// k−1 — gathered across the four rows with byte permutes.
__device__ __forceinline__ void store_digits4_prmt(const long long (&p)[4], int k, int8_t* __restrict__ base,
                                                   long long pstride) {
  uint32_t lo[4], hi[4];
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const unsigned long long w = static_cast<unsigned long long>(p[r]) + 0x8080808080808080ULL;
    lo[r] = static_cast<uint32_t>(w);
    hi[r] = static_cast<uint32_t>(w >> 32);
  }
#pragma unroll
  for (int t = 0; t < 8; ++t) {
    if (t < k) {
      const unsigned sel = (t & 3) | (((t & 3) + 4) << 4);
      const uint32_t a = __byte_perm(t < 4 ? lo[0] : hi[0], t < 4 ? lo[1] : hi[1], sel);
      const uint32_t b = __byte_perm(t < 4 ? lo[2] : hi[2], t < 4 ? lo[3] : hi[3], sel);
      *reinterpret_cast<uint32_t*>(base + static_cast<long long>(k - 1 - t) * pstride) =
          __byte_perm(a, b, 0x5410) ^ 0x80808080u;
    }
  }
}

// Integer type T: long long when |p| < 2^62 (k <= 7), i128 otherwise.
template <typename T>
__device__ __forceinline__ void store_digits4(const T (&p)[4], int k, int8_t* __restrict__ base, long long pstride) {
  T off = 0;
  for (int s = 1; s < k; ++s) off = (off << 8) | 128;
  T w[4];
#pragma unroll
  for (int r = 0; r < 4; ++r) w[r] = p[r] + off;
  for (int q = 0; q < k; ++q) {
    const int sh = 8 * (k - 1 - q);
    uint32_t packed = 0;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      int d;
      if (q == 0) d = static_cast<int>(static_cast<long long>(w[r] >> sh));
      else d = static_cast<int>(static_cast<uint32_t>(w[r] >> sh) & 0xFFu) - 128;
      packed |= (static_cast<uint32_t>(d) & 0xFFu) << (8 * r);
    }
    *reinterpret_cast<uint32_t*>(base + q * pstride) = packed;
  }
}

__global__ void __launch_bounds__(BS)
    k_x1_split(const double* __restrict__ X, long long ldx, int rows, int beta, int kx, const double* __restrict__ w,
               double* __restrict__ X1, long long ldx1, int8_t* __restrict__ dig, long long ldd, long long pstride,
               int32_t* __restrict__ g_out, double* __restrict__ s_hi, double* __restrict__ s_lo,
               double* __restrict__ r_hi, double* __restrict__ r_lo, int* __restrict__ err) {
  __shared__ i128 shq[BS / 32];
  const int j = blockIdx.x;
  const double* col = X + j * ldx;
  double* x1c = X1 + j * ldx1;
  const double wj = w[j];
  const int c = ceil_log2_d(wj);
  const int g = c + beta - 53;
  const double tau = (wj == 0.0) ? 0.0 : scalbn(0.75, c + beta);  // eq. (tau)
  i128 sq = 0;
  // 4 consecutive rows per thread per group, two groups in flight (their loads issued together): the digit
  // planes get one 32-bit store per plane (ldd % 16 == 0, so rounding `rows` up to 4 stays inside the
  // column's padding). Σq² in two 64-bit halves per group (|q| ≤ 2^52: q² < 2^104 needs 128 bits).
  for (int i0 = 4 * threadIdx.x; i0 < rows; i0 += 8 * BS) {
    double xv[2][4];
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int i = i0 + h * 4 * BS + r;
        xv[h][r] = (i < rows) ? col[i] : 0.0;
      }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int ib = i0 + h * 4 * BS;
      if (ib >= rows) break;
      long long q[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const double x1 = __dsub_rn(__dadd_rn(tau, xv[h][r]), tau);  // eq. (x), s = 1: fl(fl(τ + x) − τ)
        if (ib + r < rows) x1c[ib + r] = x1;
        q[r] = __double2ll_rn(ldexp_fast(x1, -g));  // exact integer, |q| <= 2^{53-β}
        sq += static_cast<i128>(q[r]) * q[r];
      }
      store_digits4_prmt(q, kx, dig + j * ldd + ib, pstride);
    }
  }
  const i128 SQ = block_sum_i128(sq, shq);
  if (threadIdx.x == 0) {
    g_out[j] = g;
    // x̂_jᵀx̂_j = 2^{2g} SQ and r_j = 1 − 2^{2g} SQ = 2^{2g}(2^{−2g} − SQ), both exact integers scaled.
    const dd s = i128_to_dd(SQ);
    s_hi[j] = scalbn(s.hi, 2 * g);
    s_lo[j] = scalbn(s.lo, 2 * g);
    if (-2 * g <= 125 && -2 * g >= 0) {
      const dd r = i128_to_dd((static_cast<i128>(1) << (-2 * g)) - SQ);
      r_hi[j] = scalbn(r.hi, 2 * g);
      r_lo[j] = scalbn(r.lo, 2 * g);
    } else {  // a column far from unit norm (never an eigenvector estimate): r in double-double
      const dd r = dd_add(dd{1.0, 0.0}, dd{-s_hi[j], -s_lo[j]});
      r_hi[j] = r.hi;
      r_lo[j] = r.lo;
    }
    if (SQ == 0) atomicOr(err, ERR_DEGENERATE);
  }
}

// k_x1_split with 16 rows in flight per thread (four groups of four consecutive rows, 128-bit loads and
// stores) for 16-byte aligned columns (X, X1 16-byte aligned, ldx and ldx1 even): the same values, digits,
// g, s and r as k_x1_split, bit for bit. q = x̂^(1)/2^g is an exact integer with |q| ≤ 2^{53−β}; for β ≥ 3
// (|q| ≤ 2^50) it is read from the significand of q + 1.5·2^52 instead of a 64-bit float→int conversion.
// Σq² (exact, < 2^113 overall) accumulates per thread in three int64 parts of q = qh·2^26 + ql
// (0 ≤ ql < 2^26, |qh| ≤ 2^25): Σqh² (< 2^50 per term), Σqh·ql (< 2^51), Σql² (< 2^52), which stay below
// 2^63 for ≤ 2^11 rows per thread (rows ≤ 2^19, checked by the launcher).
constexpr int X1U = 4;  // groups of four rows per thread per iteration
__global__ void __launch_bounds__(BS)
    k_x1_split_v(const double* __restrict__ X, long long ldx, int rows, int beta, int kx, const double* __restrict__ w,
                 double* __restrict__ X1, long long ldx1, int8_t* __restrict__ dig, long long ldd, long long pstride,
                 int32_t* __restrict__ g_out, double* __restrict__ s_hi, double* __restrict__ s_lo,
                 double* __restrict__ r_hi, double* __restrict__ r_lo, int* __restrict__ err) {
  __shared__ i128 shq[BS / 32];
  const int j = blockIdx.x;
  const double* col = X + j * ldx;
  double* x1c = X1 + j * ldx1;
  const double wj = w[j];
  const int c = ceil_log2_d(wj);
  const int g = c + beta - 53;
  const double tau = (wj == 0.0) ? 0.0 : scalbn(0.75, c + beta);  // eq. (tau)
  const bool in_range = (-g >= -1022 && -g <= 1023);
  const double scale = in_range ? pow2i(-g) : 0.0;
  const bool magic = beta >= 3;
  long long qa = 0, qb = 0, qc = 0;  // Σqh², Σqh·ql, Σql²
  for (int i0 = 4 * threadIdx.x; i0 < rows; i0 += 4 * BS * X1U) {
    double xv[X1U][4];
#pragma unroll
    for (int u = 0; u < X1U; ++u) {
      const int ib = i0 + u * 4 * BS;
      if (ib + 3 < rows) {
        const double2 a = __ldg(reinterpret_cast<const double2*>(col + ib));
        const double2 b = __ldg(reinterpret_cast<const double2*>(col + ib + 2));
        xv[u][0] = a.x; xv[u][1] = a.y; xv[u][2] = b.x; xv[u][3] = b.y;
      } else {
#pragma unroll
        for (int r = 0; r < 4; ++r) xv[u][r] = (ib + r < rows) ? col[ib + r] : 0.0;
      }
    }
#pragma unroll
    for (int u = 0; u < X1U; ++u) {
      const int ib = i0 + u * 4 * BS;
      if (ib >= rows) break;
      long long q[4];
      double x1[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        x1[r] = __dsub_rn(__dadd_rn(tau, xv[u][r]), tau);  // eq. (x), s = 1: fl(fl(τ + x) − τ)
        const double qd = in_range ? x1[r] * scale : ldexp_fast(x1[r], -g);  // exact integer
        if (magic) q[r] = __double_as_longlong(__dadd_rn(qd, 6755399441055744.0)) - 0x4338000000000000LL;
        else q[r] = __double2ll_rn(qd);
        const long long qh = q[r] >> 26, ql = q[r] & 0x3FFFFFFLL;
        qa += qh * qh;
        qb += qh * ql;
        qc += ql * ql;
      }
      if (ib + 3 < rows) {
        *reinterpret_cast<double2*>(x1c + ib) = make_double2(x1[0], x1[1]);
        *reinterpret_cast<double2*>(x1c + ib + 2) = make_double2(x1[2], x1[3]);
      } else {
#pragma unroll
        for (int r = 0; r < 4; ++r)
          if (ib + r < rows) x1c[ib + r] = x1[r];
      }
      store_digits4_prmt(q, kx, dig + j * ldd + ib, pstride);
    }
  }
  const i128 sq = (static_cast<i128>(qa) << 52) + (static_cast<i128>(qb) << 27) + static_cast<i128>(qc);
  const i128 SQ = block_sum_i128(sq, shq);
  if (threadIdx.x == 0) {
    g_out[j] = g;
    const dd s = i128_to_dd(SQ);
    s_hi[j] = scalbn(s.hi, 2 * g);
    s_lo[j] = scalbn(s.lo, 2 * g);
    if (-2 * g <= 125 && -2 * g >= 0) {
      const dd r = i128_to_dd((static_cast<i128>(1) << (-2 * g)) - SQ);
      r_hi[j] = scalbn(r.hi, 2 * g);
      r_lo[j] = scalbn(r.lo, 2 * g);
    } else {
      const dd r = dd_add(dd{1.0, 0.0}, dd{-s_hi[j], -s_lo[j]});
      r_hi[j] = r.hi;
      r_lo[j] = r.lo;
    }
    if (SQ == 0) atomicOr(err, ERR_DEGENERATE);
  }
}

template <typename T>
__device__ __forceinline__ T rint_to(double x);
template <>
__device__ __forceinline__ long long rint_to<long long>(double x) { return __double2ll_rn(x); }
template <>
__device__ __forceinline__ i128 rint_to<i128>(double x) { return rint_to_i128(x); }

template <typename T>
__device__ __forceinline__ void split_fixed_body(const double* __restrict__ col, const double* __restrict__ cl, int rows,
                                                 int k, int S, int e, int8_t* __restrict__ base, long long pstride) {
  for (int i0 = 4 * threadIdx.x; i0 < rows; i0 += 4 * BS) {
    T p[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int i = i0 + r;
      p[r] = (i < rows) ? rint_to<T>(ldexp_fast(col[i], S - e)) : T(0);
      if (cl && i < rows) p[r] += rint_to<T>(ldexp_fast(cl[i], S - e));
    }
    if constexpr (sizeof(T) == 8) store_digits4_prmt(p, k, base + i0, pstride);
    else store_digits4<T>(p, k, base + i0, pstride);
  }
}

// k > 7 digits of a plain fp64 column (the A split, 15 digits): p = RNE(m·2^{S−e}) is an integer-valued
// double y = M·2^{8q + r} with |M| < 2^53, so p = x·256^q with x = M·2^r (|x| < 2^60): its q lowest digits
// are 0 and the others are the balanced base-256 digits of x, all in 64-bit arithmetic (the balanced
// recurrence d = ((x + 128) mod 256) − 128, x ← (x − d)/256 yields exactly the excess-128 digits of R5).
// With byte permutes: per row, the excess-128 digits
// at positions t = 0..k−1 (from the bottom) are the bytes of the 16-byte string
//   E = [0x80 × q] [bytes of w = x + 0x8080808080808080 (mod 2^64)] [0x80 ...]
// XOR 0x80 — positions below q are zero digits, the window holds x's eight balanced digits, and above it
// the digits are zero (|p| ≤ 2^{S_k} keeps x + 0x0080…80 in [0, 2^56), so no carry leaves the window).
// Four rows' digits of one plane are gathered with three PRMTs into one 32-bit store.
__device__ __forceinline__ void split_wide_body_prmt(const double* __restrict__ col, int rows, int k, int S, int e,
                                                    int8_t* __restrict__ base, long long pstride) {
  constexpr unsigned long long P80 = 0x8080808080808080ULL;
  double xin[4];  // the next group's rows are loaded while this group is packed
#pragma unroll
  for (int r = 0; r < 4; ++r) xin[r] = (4 * threadIdx.x + r < rows) ? col[4 * threadIdx.x + r] : 0.0;
  for (int i0 = 4 * threadIdx.x; i0 < rows; i0 += 4 * BS) {
    double xcur[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      xcur[r] = xin[r];
      const int inext = i0 + 4 * BS + r;
      xin[r] = (inext < rows) ? col[inext] : 0.0;
    }
    uint32_t E[4][4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const double y = rint(ldexp_fast(xcur[r], S - e));
      long long x;
      int q;
      if (fabs(y) < 9007199254740992.0) {
        x = static_cast<long long>(y);
        q = 0;
      } else {
        const long long bits = __double_as_longlong(y);
        const int ex = static_cast<int>((bits >> 52) & 0x7FF) - 1075;
        long long mant = (bits & 0xFFFFFFFFFFFFFLL) | 0x10000000000000LL;
        if (bits < 0) mant = -mant;
        q = ex >> 3;
        x = mant << (ex & 7);
      }
      const unsigned long long w = static_cast<unsigned long long>(x) + P80;
      unsigned long long lo, hi;
      if (q == 0) {
        lo = w;
        hi = P80;
      } else if (q >= 8) {  // S = 118 (k = 15) puts the window exactly on the upper word (a shift by 64 is UB)
        lo = P80;
        hi = w;
      } else {
        lo = (w << (8 * q)) | (P80 >> (64 - 8 * q));
        hi = (w >> (64 - 8 * q)) | (P80 << (8 * q));
      }
      E[r][0] = static_cast<uint32_t>(lo);
      E[r][1] = static_cast<uint32_t>(lo >> 32);
      E[r][2] = static_cast<uint32_t>(hi);
      E[r][3] = static_cast<uint32_t>(hi >> 32);
    }
#pragma unroll
    for (int t = 0; t < 16; ++t) {
      if (t < k) {
        const unsigned sel = (t & 3) | (((t & 3) + 4) << 4);
        const uint32_t a = __byte_perm(E[0][t >> 2], E[1][t >> 2], sel);
        const uint32_t b = __byte_perm(E[2][t >> 2], E[3][t >> 2], sel);
        const uint32_t packed = __byte_perm(a, b, 0x5410) ^ 0x80808080u;
        *reinterpret_cast<uint32_t*>(base + i0 + static_cast<long long>(k - 1 - t) * pstride) = packed;
      }
    }
  }
}

__global__ void __launch_bounds__(BS)
    k_split_fixed(const double* __restrict__ M, const double* __restrict__ Mlo, long long ldm, int rows, int k,
                  int8_t* __restrict__ dig, long long ldd, long long pstride, int32_t* __restrict__ ell_out,
                  int* __restrict__ err) {
  __shared__ double sh[BS / 32];
  const int j = blockIdx.x;
  const double* col = M + j * ldm;
  const double* cl = Mlo ? Mlo + j * ldm : nullptr;
  double m = 0.0;
  bool bad = false;
  for (int i = threadIdx.x; i < rows; i += BS) {
    const double x = col[i];
    bad |= !isfinite(x);
    m = fmax(m, fabs(x));
  }
  if (bad) atomicOr(err, ERR_NONFINITE);
  m = block_max(m, sh);
  const int e = ceil_log2_d(m);
  const int S = 8 * (k - 1) + 6;
  // |p| <= 2^S (+1 for a double-double): 64-bit arithmetic while S <= 54 (k <= 7)
  if (k <= 7) split_fixed_body<long long>(col, cl, rows, k, S, e, dig + j * ldd, pstride);
  else if (!cl) split_wide_body_prmt(col, rows, k, S, e, dig + j * ldd, pstride);
  else split_fixed_body<i128>(col, cl, rows, k, S, e, dig + j * ldd, pstride);
  if (threadIdx.x == 0) ell_out[j] = e - S;
}

// Digits of Res = V − X̂^(1)D̂ (Alg. 1 line 4, inner part), formed exactly as k_recombine_V's pass 2:
// r = dd_add(V, −TwoProd(x̂_ij, λ̂_j)); p = RNE(r_hi·2^{S−e}) + RNE(r_lo·2^{S−e}) (R6 for a double-double).
template <typename T>
__device__ __forceinline__ void split_res_body(const double* __restrict__ vh, const double* __restrict__ vl,
                                               const double* __restrict__ x1, double l, int rows, int k, int S, int e,
                                               int8_t* __restrict__ base, long long pstride) {
  for (int i0 = 4 * threadIdx.x; i0 < rows; i0 += 4 * BS) {
    T p[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int i = i0 + r;
      p[r] = T(0);
      if (i < rows) {
        double ph, pl;
        two_prod(x1[i], l, ph, pl);
        const dd rr = dd_add(dd{vh[i], vl[i]}, dd{-ph, -pl});
        p[r] = rint_to<T>(ldexp_fast(rr.hi, S - e)) + rint_to<T>(ldexp_fast(rr.lo, S - e));
      }
    }
    if constexpr (sizeof(T) == 8) store_digits4_prmt(p, k, base + i0, pstride);
    else store_digits4<T>(p, k, base + i0, pstride);
  }
}

__global__ void __launch_bounds__(BS)
    k_split_res(const double* __restrict__ Vh, const double* __restrict__ Vl, long long ldv,
                const double* __restrict__ X1, long long ldx1, const double* __restrict__ lam, int rows, int k,
                const int32_t* __restrict__ eR, int8_t* __restrict__ dig, long long ldd, long long pstride,
                int32_t* __restrict__ ell_out) {
  const int j = blockIdx.x;
  const int e = eR[j];  // ⌈log2 max_i |res_ij|⌉ from k_recombine_V (0 for a zero column)
  const int S = 8 * (k - 1) + 6;
  const double* vh = Vh + j * ldv;
  const double* vl = Vl + j * ldv;
  const double* x1 = X1 + j * ldx1;
  if (k <= 7) split_res_body<long long>(vh, vl, x1, lam[j], rows, k, S, e, dig + j * ldd, pstride);
  else split_res_body<i128>(vh, vl, x1, lam[j], rows, k, S, e, dig + j * ldd, pstride);
  if (threadIdx.x == 0) ell_out[j] = e - S;
}

__global__ void k_transpose_i8(const int8_t* __restrict__ src, long long lds, long long sps, int8_t* __restrict__ dst,
                               long long ldt, long long tps, int rows, int cols) {
  // src element (i,j) at src[p*sps + j*lds + i]; dst element (i,j) at dst[p*tps + i*ldt + j]
  // 64 x 64 byte tile, 32-bit global loads and stores (lds, ldt are multiples of 16, so the 4-byte
  // groups that straddle `rows` / `cols` stay inside each line's padding).
  __shared__ uint8_t t[64][68];
  const int p = blockIdx.z;
  const int i0 = blockIdx.x * 64, j0 = blockIdx.y * 64;
  for (int e = threadIdx.x; e < 64 * 16; e += blockDim.x) {
    const int i4 = (e & 15) * 4, jj = e >> 4;
    const int i = i0 + i4, j = j0 + jj;
    uint32_t v = 0;
    if (i < rows && j < cols) v = *reinterpret_cast<const uint32_t*>(src + p * sps + j * lds + i);
    *reinterpret_cast<uint32_t*>(&t[jj][i4]) = v;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < 64 * 16; e += blockDim.x) {
    const int j4 = (e & 15) * 4, ii = e >> 4;
    const int i = i0 + ii, j = j0 + j4;
    if (i < rows && j < cols) {
      const uint32_t v = static_cast<uint32_t>(t[j4][ii]) | (static_cast<uint32_t>(t[j4 + 1][ii]) << 8) |
                         (static_cast<uint32_t>(t[j4 + 2][ii]) << 16) | (static_cast<uint32_t>(t[j4 + 3][ii]) << 24);
      *reinterpret_cast<uint32_t*>(dst + p * tps + static_cast<long long>(i) * ldt + j) = v;
    }
  }
}

// The same transpose with 16-byte global loads and stores on 128 x 128-byte tiles: every global access of a warp
// covers whole 128-byte lines of the source columns / destination rows (the 64-byte tiles of the first form touched
// half lines: 56 % of the copy peak). For 16-byte aligned planes with lds, ldt, sps, tps multiples of 16 and rows,
// cols ≥ 1 (the 16-byte groups that straddle `rows` / `cols` stay inside each line's padding, as in
// k_transpose_i8). Shared memory: t[j][w ^ (j >> 4)] (32 words per column, pitch 33) — conflict-free for the
// column-wise stores (a warp: 4 columns x 8 quads) and the row-wise gathers (a warp: 4 rows x 8 column groups).
__global__ void __launch_bounds__(256) k_transpose_i8_v(const int8_t* __restrict__ src, long long lds, long long sps,
                                                        int8_t* __restrict__ dst, long long ldt, long long tps,
                                                        int rows, int cols) {
  __shared__ uint32_t t[128][33];
  const int p = blockIdx.z;
  const int i0 = blockIdx.x * 128, j0 = blockIdx.y * 128;
  const int tid = threadIdx.x;
  uint4 v[4];
#pragma unroll
  for (int r = 0; r < 4; ++r) {  // all four loads in flight before the first shared-memory store
    const int idx = tid + 256 * r;
    const int jj = idx >> 3, q = idx & 7;  // column j0 + jj, bytes [16q, 16q + 16) of the tile's rows
    const int i = i0 + 16 * q, j = j0 + jj;
    v[r] = make_uint4(0u, 0u, 0u, 0u);
    if (i < rows && j < cols) v[r] = __ldcs(reinterpret_cast<const uint4*>(src + p * sps + j * lds + i));
  }
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int idx = tid + 256 * r;
    const int jj = idx >> 3, q = idx & 7, sw = jj >> 4;
    t[jj][(4 * q + 0) ^ sw] = v[r].x;
    t[jj][(4 * q + 1) ^ sw] = v[r].y;
    t[jj][(4 * q + 2) ^ sw] = v[r].z;
    t[jj][(4 * q + 3) ^ sw] = v[r].w;
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int idx = tid + 256 * r;
    const int ii = idx >> 3, q = idx & 7;  // output row i0 + ii, bytes [16q, 16q + 16) = columns j0 + 16q + ..
    const int i = i0 + ii, j = j0 + 16 * q;
    if (i < rows && j < cols) {
      const int w = (ii >> 2) ^ q;  // columns 16q .. 16q + 15 share the swizzle (jb >> 4 = q)
      const uint32_t b = ii & 3;
      const uint32_t s01 = b | ((4u + b) << 4);  // byte b of the first word, byte b of the second
      uint32_t o[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int jb = 16 * q + 4 * k;
        const uint32_t lo = __byte_perm(t[jb][w], t[jb + 1][w], s01);
        const uint32_t hi = __byte_perm(t[jb + 2][w], t[jb + 3][w], s01);
        o[k] = __byte_perm(lo, hi, 0x5410);
      }
      *reinterpret_cast<uint4*>(dst + p * tps + static_cast<long long>(i) * ldt + j) = make_uint4(o[0], o[1], o[2], o[3]);
    }
  }
}

__global__ void k_transpose_f64(const double* __restrict__ src, long long lds, double* __restrict__ dst,
                                long long ldt, int rows, int cols) {
  // dst (cols x rows) = srcᵀ, column-major both
  __shared__ double t[32][33];
  const int i0 = blockIdx.x * 32, j0 = blockIdx.y * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  for (int jj = ty; jj < 32; jj += 8) {
    const int i = i0 + tx, j = j0 + jj;
    t[jj][tx] = (i < rows && j < cols) ? src[static_cast<long long>(j) * lds + i] : 0.0;
  }
  __syncthreads();
  for (int ii = ty; ii < 32; ii += 8) {
    const int j = j0 + tx, i = i0 + ii;
    if (i < rows && j < cols) dst[static_cast<long long>(i) * ldt + j] = t[tx][ii];
  }
}

template <int NG, int TMA>
__global__ void __launch_bounds__(BS, 3)
    k_recombine_V(const int32_t* __restrict__ planes, long long pstride, int rows, const __grid_constant__ RecombPlan rp,
                  const int32_t* __restrict__ ellA, const int32_t* __restrict__ ellB, int scale8,
                  const double* __restrict__ X1, long long ldx1, const double* __restrict__ s_hi,
                  const double* __restrict__ s_lo, double* __restrict__ Vh, double* __restrict__ Vl, long long ldv,
                  double* __restrict__ lam_out, int32_t* __restrict__ eR, int* __restrict__ eR_max, int use_tma,
                  const double* __restrict__ lam0) {
  extern __shared__ __align__(128) unsigned char tsm[];
  __shared__ double sh[2 * BS / 32];
  const int j = blockIdx.x;
  const int Lj = rp.tile_budgets ? rp.tileL[j / 256] : rp.L;
  const int eb = ellB[j] + scale8;
  const double* x1 = X1 + j * ldx1;
  dd t{0.0, 0.0};
  // pass 1: V (Alg. 1 line 1) and x̂_jᵀ v_j (line 3). Beside them, the residual against the PREVIOUS estimate
  // λ0 (lam0, the sweep's input λ̂): m0 = max_i |RN(v_i − x̂_i λ0)|, with max |x̂_i| and max |v_i| — enough to
  // enclose the exact column max of |Res| for the new λ̂ (below) without reading the column a second time
  const double l0 = lam0 ? lam0[j] : 0.0;
  double m0 = 0.0, xm = 0.0, vm = 0.0;
  const double* xc[1] = {x1};
  for_column_x<1, false, NG, kRingV>(planes, pstride, static_cast<long long>(j) * rows, rows, rp, Lj, xc, ellA, TMA, tsm,
                  [&](int, int ea) { return ea + eb; },
                  [&](int i, const dd& v, const double* xv) {
                    Vh[j * ldv + i] = v.hi;
                    Vl[j * ldv + i] = v.lo;
                    t = dd_add(t, dd_mul_d(v, xv[0]));
                    m0 = fmax(m0, fabs(__fma_rn(-xv[0], l0, v.hi) + v.lo));
                    xm = fmax(xm, fabs(xv[0]));
                    vm = fmax(vm, fabs(v.hi));
                  });
  t = block_sum_dd(t, sh);
  const dd lam = dd_div(t, dd{s_hi[j], s_lo[j]});  // λ̂_j = x̂_jᵀv̂_j / (1 − r_j)
  const double l = lam.hi;
  // The split (k_split_res, R6) needs e = ⌈log2 m⌉, m = max_i |hi(dd_add(v_i, −TwoProd(x̂_i, λ̂)))|. Each such
  // hi is within 2^-52|ρ_i| + 2^-104(|v_i| + |x̂_i λ̂|) of the exact ρ_i(λ̂) = v_i − x̂_i λ̂; pass 1's value
  // RN(RN(v_hi − x̂λ0) + v_lo) is within 2^-51|ρ_i(λ0)| + 2^-105|v_i| of ρ_i(λ0); and
  // |ρ_i(λ̂) − ρ_i(λ0)| ≤ |x̂_i||λ̂ − λ0|. So m ∈ [lo, hi] below (constants rounded generously outward);
  // when ⌈log2⌉ agrees at both ends e is decided exactly, else (and without λ0) pass 2 computes m itself.
  m0 = block_max(m0, sh);
  xm = block_max(xm, sh);
  vm = block_max(vm, sh);
  const double dlt = xm * fabs(l - l0) * (1.0 + 0x1p-48);
  const double sl = 0x1p-96 * (vm + xm * (fabs(l) + fabs(l0)));
  const double mlo = (m0 * (1.0 - 0x1p-48) - dlt) * (1.0 - 0x1p-48) - sl;
  const double mhi = (m0 * (1.0 + 0x1p-48) + dlt) * (1.0 + 0x1p-48) + sl;
  if (lam0 && mlo > 0.0 && ceil_log2_d(mlo) == ceil_log2_d(mhi)) {
    if (threadIdx.x == 0) {
      lam_out[j] = l;
      const int e = ceil_log2_d(mhi);
      eR[j] = e;
      atomicMax(eR_max, e);
    }
    return;
  }
  // pass 2: column max of |Res|, Res = V − X̂ D̂ (line 4, inner part) in double-double — Res itself is
  // formed again, identically, by the digit split (k_split_res), so it is never written here
  double m = 0.0;
  const double* vh = Vh + j * ldv;
  const double* vl = Vl + j * ldv;
  constexpr int U2 = 4;  // four rows per thread in flight (12 independent loads; the column was just written, L2)
  int i = threadIdx.x;
  for (; i + (U2 - 1) * BS < rows; i += U2 * BS) {
    double a[U2], b[U2], c[U2];
#pragma unroll
    for (int u = 0; u < U2; ++u) {
      a[u] = x1[i + u * BS];
      b[u] = vh[i + u * BS];
      c[u] = vl[i + u * BS];
    }
#pragma unroll
    for (int u = 0; u < U2; ++u) {
      double ph, pl;
      two_prod(a[u], l, ph, pl);
      const dd r = dd_add(dd{b[u], c[u]}, dd{-ph, -pl});
      m = fmax(m, fabs(r.hi));
    }
  }
  for (; i < rows; i += BS) {
    double ph, pl;
    two_prod(x1[i], l, ph, pl);
    const dd r = dd_add(dd{vh[i], vl[i]}, dd{-ph, -pl});
    m = fmax(m, fabs(r.hi));
  }
  m = block_max(m, sh);
  if (threadIdx.x == 0) {
    lam_out[j] = l;
    const int e = ceil_log2_d(m);
    eR[j] = e;
    if (m > 0.0) atomicMax(eR_max, e);
  }
}

template <int NG, int TMA, int RPTE = RPT>
__global__ void __launch_bounds__(BS, NG <= 8 ? (RPTE == 4 ? 2 : 4) : 2)
    k_recombine_E(const int32_t* __restrict__ planes, long long pstride, int rows, const __grid_constant__ RecombPlan rp,
                  const int32_t* __restrict__ ellA, const int32_t* __restrict__ ellB, int scale8,
                  const double* __restrict__ r_hi, const double* __restrict__ lam, const int32_t* __restrict__ gX,
                  int col0, double* __restrict__ Ep, long long lde, double* __restrict__ nrm2,
                  int* __restrict__ eE_max, int32_t* __restrict__ eE_col, int* __restrict__ err,
                  const EdgeOut eo, int use_tma, double* __restrict__ nW2) {
  extern __shared__ __align__(128) unsigned char tsm[];
  __shared__ double sh[BS / 32];
  const int j = blockIdx.x;        // local column
  const int Lj = rp.tile_budgets ? rp.tileL[j / 256] : rp.L;
  const int jg = col0 + j;         // global index of column j (its λ̂)
  const int eb = ellB[j] + scale8;
  const double lj = lam[jg];
  double m = 0.0, s2 = 0.0, w2 = 0.0;
  bool bad = false, unresolved = false;
  // the row vectors λ̂_i and ℓ_i of the row operand (X̂^(1)ᵀ: g_i) ride in the shared-memory stages
  // with the planes
  const double* xc[1] = {lam};
  // the row exponent of the row operand X̂^(1)ᵀ is g_i (ellA == gX): it scales Ẽ' = diag(2^g)Ẽ too, so the
  // staged value is kept for the element (the exponent functor runs right before the element functor)
  int gcur = 0;
  for_column_x<1, true, NG, kRingE, RPTE>(planes, pstride, static_cast<long long>(j) * rows, rows, rp, Lj, xc, ellA, TMA, tsm,
                            [&](int, int gi) { gcur = gi; return gi + eb; }, [&](int i, const dd& wv, const double* xv) {
    double e;
    w2 = __fma_rn(wv.hi, wv.hi, w2);
    if (i == jg) {
      e = r_hi[j] * 0.5;  // ẽ_jj = r_j / 2
    } else {
      const double dl = __dsub_rn(lj, xv[0]);  // λ̃_j − λ̃_i
      if (eo.mode == 0) {
        if (dl == 0.0) bad = true;
        e = __ddiv_rn(wv.hi, dl);  // ẽ_ij = w_ij / (λ̃_j − λ̃_i)  (Alg. 1 line 5)
      } else {
        // cluster branch (R13): equal λ̂ or |ẽ_ij| > κ marks an unresolved pair; the group sub-solve
        // (cluster.cu) rewrites its columns
        e = (dl == 0.0) ? 0.0 : __ddiv_rn(wv.hi, dl);
        if (dl == 0.0 || fabs(e) > eo.kappa) {
          uf_unite(eo.parent, i, jg);
          unresolved = true;
        }
      }
    }
    s2 = __fma_rn(e, e, s2);
    const double ep = ldexp_fast(e, gcur);  // Ẽ' = diag(2^g) Ẽ (exact)
    Ep[j * lde + i] = ep;
    m = fmax(m, fabs(ep));
  });
  if (bad) atomicOr(err, ERR_DEGENERATE);
  if (__syncthreads_or(unresolved) && threadIdx.x == 0) atomicOr(eo.any, 1);
  m = block_max(m, sh);
  s2 = block_sum(s2, sh);
  w2 = block_sum(w2, sh);
  if (threadIdx.x == 0) {
    nrm2[j] = s2;
    if (nW2) nW2[j] = w2;
    eE_col[j] = (m > 0.0) ? ceil_log2_d(m) : -100000;
    if (m > 0.0) atomicMax(eE_max, ceil_log2_d(m));
  }
}

// R = I − X̂^(1)ᵀX̂^(1) for the local columns (form_R): r_ij = −RN(g_ij) off the diagonal, the exact
// r_j on it (R10); ‖r_j‖² per column (fixed-shape reduction).
__global__ void __launch_bounds__(BS)
    k_form_R(const int32_t* __restrict__ planes, long long pstride, int rows, const __grid_constant__ RecombPlan rp,
             const int32_t* __restrict__ g, int scale8, int col0, const double* __restrict__ r_hi,
             const double* __restrict__ r_lo, double* __restrict__ R, long long ldr, double* __restrict__ nR2) {
  __shared__ double sh[BS / 32];
  const int j = blockIdx.x;
  const int jg = col0 + j;
  const int Lj = rp.tile_budgets ? rp.tileL[j / 256] : rp.L;
  const int eb = g[jg] + scale8;
  double s2 = 0.0;
  for_column(planes, pstride, static_cast<long long>(j) * rows, rows, rp, Lj, [&](int i) { return g[i] + eb; },
             [&](int i, const dd& v) {
               const double r = (i == jg) ? (r_hi[jg] + r_lo[jg]) : -(v.hi + v.lo);
               R[static_cast<long long>(j) * ldr + i] = r;
               s2 = __fma_rn(r, r, s2);
             });
  s2 = block_sum(s2, sh);
  if (threadIdx.x == 0) nR2[j] = s2;
}

template <int NG, int TMA>
__global__ void __launch_bounds__(BS, NG <= 8 ? 3 : 2)
    k_final(const int32_t* __restrict__ planes, long long pstride, int rows, const __grid_constant__ RecombPlan rp,
            const int32_t* __restrict__ ellB, int scale8, const double* __restrict__ X1, long long ldx1,
            double* __restrict__ X, long long ldx, double* __restrict__ nu2, double* __restrict__ wnext, int use_tma,
            double* __restrict__ D) {
  extern __shared__ __align__(128) unsigned char tsm[];
  __shared__ double sh[BS / 32];
  const int j = blockIdx.x;
  const int Lj = rp.tile_budgets ? rp.tileL[j / 256] : rp.L;
  const int eb = ellB[j] + scale8;  // the Q operand (digits of X̂^(1)/2^g) has ℓ = 0 on every row
  double s2 = 0.0, m = 0.0;
  const double* xc[2] = {X1 + j * ldx1, X + j * ldx};
  for_column_x<2, false, NG, kRingF>(planes, pstride, static_cast<long long>(j) * rows, rows, rp, Lj, xc, nullptr, TMA, tsm,
                  [&](int, int) { return eb; }, [&](int i, const dd& u, const double* xv) {
    const double x1 = xv[0];
    double s, e;
    two_sum(x1, u.hi, s, e);
    const double xn = __dadd_rn(s, __dadd_rn(e, u.lo));  // accsum: RN(x^(1) + U)
    const double xo = xv[1];
    const double d = __dsub_rn(xn, xo);
    s2 = __fma_rn(d, d, s2);
    m = fmax(m, fabs(xn));
    X[j * ldx + i] = xn;
    if (D) D[static_cast<long long>(j) * rows + i] = d;  // the update, for its 2-norm estimate (R12)
  });
  s2 = block_sum(s2, sh);
  m = block_max(m, sh);
  if (threadIdx.x == 0) {
    nu2[j] = s2;
    wnext[j] = m;
  }
}

constexpr int kRingD = 54 * 1024;
template <int NG, int TMA>
__global__ void __launch_bounds__(BS, NG <= 8 ? 4 : 2)
    k_recombine_dd(const int32_t* __restrict__ planes, long long pstride, int rows, const __grid_constant__ RecombPlan rp,
                   const int32_t* __restrict__ ellA, const int32_t* __restrict__ ellB, int scale8,
                   double* __restrict__ Ch, double* __restrict__ Cl, long long ldc) {
  extern __shared__ __align__(128) unsigned char tsm[];
  const int j = blockIdx.x;
  const int Lj = rp.tile_budgets ? rp.tileL[j / 256] : rp.L;
  const int eb = ellB[j] + scale8;
  for_column_x<0, false, NG, kRingD>(planes, pstride, static_cast<long long>(j) * rows, rows, rp, Lj, nullptr, ellA, TMA,
                                     tsm, [&](int, int ea) { return ea + eb; }, [&](int i, const dd& v, const double*) {
                                       Ch[j * ldc + i] = v.hi;
                                       if (Cl) Cl[j * ldc + i] = v.lo;
                                     });
}

// ---------------------------------------------------------------- power-iteration vector helpers (certify.cu, R12)
// out[0] = Σ x_j² (one CTA, fixed order)
__global__ void __launch_bounds__(BS) k_sumsq(const double* __restrict__ x, int n, double* __restrict__ out) {
  __shared__ double sh[BS / 32];
  double acc = 0.0;
  for (int i = threadIdx.x; i < n; i += BS) acc = fma(x[i], x[i], acc);
  acc = block_sum(acc, sh);
  if (threadIdx.x == 0) out[0] = acc;
}
// v = z / sqrt(nrm2[0]) (nrm2[0] > 0), or a deterministic start vector (seed: the global column index)
__global__ void k_normalize(double* __restrict__ v, const double* __restrict__ z, int n, const double* __restrict__ nrm2,
                            int col0) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  if (!z) {
    unsigned int h = static_cast<unsigned int>(col0 + j) * 2654435761u;
    h ^= h >> 15;
    h *= 2246822519u;
    h ^= h >> 13;
    v[j] = (static_cast<double>(h & 0xFFFFFF) / 16777216.0) - 0.5;
    return;
  }
  const double s = nrm2[0];
  v[j] = s > 0.0 ? z[j] / sqrt(s) : 0.0;
}

// small host <-> device transfers through mapped pinned memory (no copy engine involved)
__global__ void k_copy_bytes(char* __restrict__ dst, const char* __restrict__ src, size_t bytes, int a8) {
  const size_t t = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x, st = static_cast<size_t>(gridDim.x) * blockDim.x;
  if (a8) {
    const size_t n8 = bytes / 8;
    for (size_t i = t; i < n8; i += st)
      reinterpret_cast<unsigned long long*>(dst)[i] = reinterpret_cast<const unsigned long long*>(src)[i];
  } else {
    for (size_t i = t; i < bytes; i += st) dst[i] = src[i];
  }
}

}  // namespace

// ---------------------------------------------------------------- launchers
namespace {
void init_attrs();
// OZR_NO_TMA (A/B only): bit 0 / 1 / 2 forces the register path of recombine_V / recombine_E / final
int no_tma_mask() {
  static int m = -1;
  if (m < 0) {
    const char* e = getenv("OZR_NO_TMA");
    m = e ? atoi(e) : 0;
    const char* f = getenv("OZR_FASTDD");
    if (f && f[0] == '0') {
      int z = 0;
      cudaMemcpyToSymbol(g_fastdd, &z, sizeof z);
    }
  }
  return m;
}
int tma_ok(const RecombPlan& rp, const int32_t* planes, long long pstride, int rows, const double* x0, long long ld0,
           const double* x1, long long ld1) {
  init_attrs();
  auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  if (!rp.consecutive || rows % 4 || pstride % 4 || !al(planes)) return 0;
  if (x0 && (ld0 % 2 || !al(x0))) return 0;
  if (x1 && (ld1 % 2 || !al(x1))) return 0;
  return 1;
}
// dynamic shared memory of the TMA paths; every recombination kernel prefers the largest carveout (the same
// SM configuration as the slice GEMM, with which its register path co-resides)
void init_attrs() {
  once_per_device(8, [] {
#define OZR_ATTR(K, R, NX)                                                                                 \
  cudaFuncSetAttribute(K<4, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, tma_smem(ring_for(R, 4, NX)));   \
  cudaFuncSetAttribute(K<8, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, tma_smem(ring_for(R, 8, NX)));   \
  cudaFuncSetAttribute(K<12, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, tma_smem(ring_for(R, 12, NX))); \
  cudaFuncSetAttribute(K<4, 1>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);                        \
  cudaFuncSetAttribute(K<8, 1>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);                        \
  cudaFuncSetAttribute(K<12, 1>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);                       \
  cudaFuncSetAttribute(K<12, 0>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    OZR_ATTR(k_recombine_V, kRingV, 1);
    OZR_ATTR(k_recombine_E, kRingE, 1);
    OZR_ATTR(k_final, kRingF, 2);
    OZR_ATTR(k_recombine_dd, kRingD, 0);
#undef OZR_ATTR
    return cudaPeekAtLastError();
  });
}
}  // namespace

void launch_split_res(const double* Vh, const double* Vl, long long ldv, const double* X1, long long ldx1,
                      const double* lam, int rows, int cols, int k, const int32_t* eR, int8_t* dig, long long ldd,
                      long long pstride, int32_t* ell, cudaStream_t s) {
  k_split_res<<<cols, BS, 0, s>>>(Vh, Vl, ldv, X1, ldx1, lam, rows, k, eR, dig, ldd, pstride, ell);
}
void launch_colmax(const double* X, long long ldx, int rows, int cols, double* w, int* err, cudaStream_t s) {
  k_colmax<<<cols, BS, 0, s>>>(X, ldx, rows, w, err);
}
void launch_x1_split(const double* X, long long ldx, int rows, int cols, int beta, int kx, const double* w, double* X1,
                     long long ldx1, int8_t* dig, long long ldd, long long pstride, int32_t* g, double* s_hi,
                     double* s_lo, double* r_hi, double* r_lo, int* err, cudaStream_t s) {
  auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  if (al(X) && al(X1) && ldx % 2 == 0 && ldx1 % 2 == 0 && rows <= (1 << 19) && kx <= 8)
    k_x1_split_v<<<cols, BS, 0, s>>>(X, ldx, rows, beta, kx, w, X1, ldx1, dig, ldd, pstride, g, s_hi, s_lo, r_hi,
                                     r_lo, err);
  else
    k_x1_split<<<cols, BS, 0, s>>>(X, ldx, rows, beta, kx, w, X1, ldx1, dig, ldd, pstride, g, s_hi, s_lo, r_hi, r_lo,
                                   err);
}
void launch_split_fixed(const double* M, const double* Mlo, long long ldm, int rows, int cols, int k, int8_t* dig,
                        long long ldd, long long pstride, int32_t* ell, int* err, cudaStream_t s) {
  k_split_fixed<<<cols, BS, 0, s>>>(M, Mlo, ldm, rows, k, dig, ldd, pstride, ell, err);
}
void launch_transpose_i8(const int8_t* src, long long lds, long long sps, int8_t* dst, long long ldt, long long tps,
                         int rows, int cols, int planes, cudaStream_t s) {
  dim3 grid((rows + 63) / 64, (cols + 63) / 64, planes);
  const bool al = ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0 &&
                  (lds | sps | ldt | tps) % 16 == 0;
  if (al) {
    dim3 gridv((rows + 127) / 128, (cols + 127) / 128, planes);
    k_transpose_i8_v<<<gridv, 256, 0, s>>>(src, lds, sps, dst, ldt, tps, rows, cols);
  } else {
    k_transpose_i8<<<grid, 256, 0, s>>>(src, lds, sps, dst, ldt, tps, rows, cols);
  }
}
void launch_transpose_f64(const double* src, long long lds, double* dst, long long ldt, int rows, int cols,
                          cudaStream_t s) {
  dim3 grid((rows + 31) / 32, (cols + 31) / 32);
  k_transpose_f64<<<grid, 256, 0, s>>>(src, lds, dst, ldt, rows, cols);
}
void launch_recombine_V(const int32_t* planes, long long pstride, int rows, int cols, const RecombPlan& rp,
                        const int32_t* ellA, const int32_t* ellB, int scale8, const double* X1, long long ldx1,
                        const double* s_hi, const double* s_lo, double* Vh, double* Vl, long long ldv,
                        double* lam_out, int32_t* eR, int* eR_max, cudaStream_t s, int allow_tma,
                        const double* lam0) {
  init_attrs();
  const int tma = allow_tma && !(no_tma_mask() & 1) && tma_ok(rp, planes, pstride, rows, X1, ldx1, X1, ldx1) && (reinterpret_cast<uintptr_t>(ellA) & 15) == 0;
  // OZR_RES_2PASS=1 (A/B and the bit-identity test): always re-read the column for the Res exponent
  if (const char* e2 = getenv("OZR_RES_2PASS"))
    if (e2[0] == '1') lam0 = nullptr;
#define OZR_RV(NG_, TMA_)                                                                                          \
  k_recombine_V<NG_, TMA_><<<cols, BS, TMA_ ? tma_smem(ring_for(kRingV, NG_, 1)) : 0, s>>>(planes, pstride, rows, rp, ellA, ellB, scale8, X1, ldx1, s_hi, \
                                                          s_lo, Vh, Vl, ldv, lam_out, eR, eR_max, tma, lam0)
  if (tma && rp.ngroups <= 4) OZR_RV(4, 1);
  else if (tma && rp.ngroups <= 8) OZR_RV(8, 1);
  else if (tma) OZR_RV(12, 1);
  else OZR_RV(12, 0);
#undef OZR_RV
}
void launch_recombine_E(const int32_t* planes, long long pstride, int rows, int cols, const RecombPlan& rp,
                        const int32_t* ellA, const int32_t* ellB, int scale8, const double* r_hi, const double* lam,
                        const int32_t* gX, int col0, double* Ep, long long lde, double* nrm2, int* eE_max,
                        int32_t* eE_col, int* err, const EdgeOut& eo, double* nW2, cudaStream_t s, int allow_tma) {
  init_attrs();
  if (gX != ellA) {  // Ẽ' takes its row scaling from the staged row exponents (k_recombine_E)
    fprintf(stderr, "ozr: launch_recombine_E: gX must be the row operand's exponents\n");
    abort();
  }
  const int tma = allow_tma && !(no_tma_mask() & 2) && tma_ok(rp, planes, pstride, rows, lam, 0, nullptr, 0) &&
                  (reinterpret_cast<uintptr_t>(ellA) & 15) == 0;
#define OZR_RE(NG_, TMA_, R_)                                                                                            \
  k_recombine_E<NG_, TMA_, R_><<<cols, BS, TMA_ ? tma_smem(ring_for(kRingE, NG_, 1, R_)) : 0, s>>>(planes, pstride, rows, rp, ellA, ellB, scale8, r_hi, lam, gX, \
                                                          col0, Ep, lde, nrm2, eE_max, eE_col, err, eo, tma, nW2)
  // (four rows per thread per stage — 2 CTAs per SM by registers and shared memory — measured 557 µs against
  // 461 µs at n = 8192: the division's latency wants the warps)
  if (tma && rp.ngroups <= 4) OZR_RE(4, 1, RPT);
  else if (tma && rp.ngroups <= 8) OZR_RE(8, 1, RPT);
  else if (tma) OZR_RE(12, 1, RPT);
  else OZR_RE(12, 0, RPT);
#undef OZR_RE
}
void launch_final(const int32_t* planes, long long pstride, int rows, int cols, const RecombPlan& rp,
                  const int32_t* ellB, int scale8, const double* X1, long long ldx1, double* X, long long ldx,
                  double* nu2, double* wnext, cudaStream_t s, int allow_tma, double* D) {
  init_attrs();
  const int tma = allow_tma && !(no_tma_mask() & 4) && tma_ok(rp, planes, pstride, rows, X1, ldx1, X, ldx);
#define OZR_FI(NG_, TMA_)                                                                                                 \
  k_final<NG_, TMA_><<<cols, BS, TMA_ ? tma_smem(ring_for(kRingF, NG_, 2)) : 0, s>>>(planes, pstride, rows, rp, ellB, scale8, X1, ldx1, X, ldx, nu2, wnext, \
                                                    tma, D)
  if (tma && rp.ngroups <= 4) OZR_FI(4, 1);
  else if (tma && rp.ngroups <= 8) OZR_FI(8, 1);
  else if (tma) OZR_FI(12, 1);
  else OZR_FI(12, 0);
#undef OZR_FI
}
void launch_form_R(const int32_t* planes, long long pstride, int rows, int cols, const RecombPlan& rp, const int32_t* g,
                   int scale8, int col0, const double* r_hi, const double* r_lo, double* R, long long ldr, double* nR2,
                   cudaStream_t s) {
  k_form_R<<<cols, BS, 0, s>>>(planes, pstride, rows, rp, g, scale8, col0, r_hi, r_lo, R, ldr, nR2);
}
void launch_sumsq(const double* x, int n, double* out, cudaStream_t s) { k_sumsq<<<1, BS, 0, s>>>(x, n, out); }
void launch_normalize(double* v, const double* z, int n, const double* nrm2, int col0, cudaStream_t s) {
  k_normalize<<<(n + 255) / 256, 256, 0, s>>>(v, z, n, nrm2, col0);
}
void launch_copy_bytes(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  if (bytes == 0) return;
  const bool a8 = ((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src) | bytes) & 7) == 0;
  const size_t units = a8 ? bytes / 8 : bytes;
  const int grid = static_cast<int>(std::min<size_t>((units + 255) / 256, 1024));
  k_copy_bytes<<<grid, 256, 0, s>>>(static_cast<char*>(dst), static_cast<const char*>(src), bytes, a8 ? 1 : 0);
}
void launch_iota(int* p, int n, cudaStream_t s) { k_iota<<<(n + 255) / 256, 256, 0, s>>>(p, n); }
void launch_uf_flatten(int* parent, int n, cudaStream_t s) { k_uf_flatten<<<(n + 255) / 256, 256, 0, s>>>(parent, n); }
void launch_recombine_dd(const int32_t* planes, long long pstride, int rows, int cols, const RecombPlan& rp,
                         const int32_t* ellA, const int32_t* ellB, int scale8, double* Ch, double* Cl, long long ldc,
                         cudaStream_t s) {
  init_attrs();
  const int tma = !(no_tma_mask() & 8) && tma_ok(rp, planes, pstride, rows, nullptr, 0, nullptr, 0) &&
                  (reinterpret_cast<uintptr_t>(ellA) & 15) == 0;
#define OZR_RD(NG_, TMA_)                                                                                        \
  k_recombine_dd<NG_, TMA_><<<cols, BS, TMA_ ? tma_smem(ring_for(kRingD, NG_, 0)) : 0, s>>>(planes, pstride, rows, rp, \
                                                                                          ellA, ellB, scale8, Ch, Cl, ldc)
  if (tma && rp.ngroups <= 4) OZR_RD(4, 1);
  else if (tma && rp.ngroups <= 8) OZR_RD(8, 1);
  else if (tma) OZR_RD(12, 1);
  else OZR_RD(12, 0);
#undef OZR_RD
}

}  // namespace ozr
