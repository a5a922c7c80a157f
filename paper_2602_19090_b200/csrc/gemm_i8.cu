// gemm_i8.cu — the slice-product kernel of the one-sided Ozaki product (§2.3 eq. (9)-(12),
// §3.3 eq. (38) "A X̂ = A^(1) X̂ + ... + A^(n_A) X̂"): every product of two digit planes is an exact
// INT8 x INT8 -> INT32 tensor-core GEMM (tcgen05.mma kind::i8, accumulator in TMEM), and all pairs
// (s,t) of one accumulation group are summed into the same TMEM accumulator by walking a "virtual K"
// = (pairs of the group) x K. Exactness: |digit| <= 128, so a group is exact while
// K * npairs * 2^14 < 2^31 (the host planner enforces it).
//
// Structure (one CTA = one 128 x 256 output tile of one group, 128 threads):
//   warp 0 lane 0 : TMA producer  (A tile 128 x 128 B, B tile 256 x 128 B per stage, SW128)
//   warp 1 lane 0 : MMA issuer    (4 x tcgen05.mma M128 N256 K32 per stage)
//   all 4 warps   : epilogue      (tcgen05.ld 32x32b -> int32 column-major plane, coalesced)
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cuda.h>
#include <cuda_runtime.h>

#include "ozr_internal.h"
#include "ptx.cuh"

namespace ozr {

namespace {

constexpr int BM = 128;
constexpr int BN = kTileN;
constexpr int BK = 128;  // bytes of K per stage (= one 128 B swizzle row)
constexpr int STAGES = 4;
constexpr int UMMA_K = 32;  // K per tcgen05.mma for 8-bit inputs
constexpr int A_STAGE_BYTES = BM * BK;
constexpr int B_STAGE_BYTES = BN * BK;
constexpr int SMEM_BYTES = STAGES * (A_STAGE_BYTES + B_STAGE_BYTES) + 1024 /*align*/ + 256 /*barriers*/;
constexpr int TMEM_COLS = 256;
constexpr int BAND = 3;  // n-tiles per rasterisation band (3 vs 4: same time, −8 % DRAM reads on V, −18 % on W)

// Persistent form: one CTA per SM; its first job is blockIdx.x, the next ones come from a global atomic
// counter, so the jobs in flight at any moment stay neighbours in the rasterised order (as with the
// hardware CTA scheduler). The producer fetches the job ids and passes them to the other roles through a
// small shared-memory queue. Warp roles:
//   warp 0 lane 0 : job fetch + TMA producer over every job of the CTA (the smem ring never drains)
//   warp 1 lane 0 : MMA issuer, accumulating job t into TMEM buffer t % 2 (2 x 256 columns)
//   warps 2..5    : epilogue of job t − 1 (tcgen05.ld → int32 plane) while job t is being multiplied
constexpr int NWARPS = 6;
constexpr int TMEM_ALLOC = 2 * TMEM_COLS;
constexpr int JQ = 4;  // job queue depth (the epilogue trails the MMA issuer by one job)

struct JobInfo {
  int g, m0, n0, skip;
};

__device__ __forceinline__ JobInfo job_info(int job, const PairTable& pt, int M, int N, int tiles_m) {
  const int G = pt.ngroups;
  JobInfo ji;
  ji.g = job % G;  // the groups of one tile run back to back (they share its operand rows)
  const int tile = job / G;
  // L2 rasterisation: bands of BAND n-tiles; inside a band, consecutive tiles sweep the band's n-tiles
  // for one m-tile, then the next m-tile — the band's B columns stay L2-resident while A streams once
  // per band (instead of once per n-tile)
  const int tiles_n = (N + BN - 1) / BN;
  const int band = tile / (BAND * tiles_m);
  const int r = tile - band * (BAND * tiles_m);
  const int nb = min(BAND, tiles_n - band * BAND);
  ji.m0 = (r / nb) * BM;
  ji.n0 = (band * BAND + r % nb) * BN;
  ji.skip = (pt.tile_budgets && pt.diag[ji.g] > pt.tileL[ji.n0 / BN]) ? 1 : 0;  // beyond the tile's budget
  return ji;
}

__global__ void __launch_bounds__(NWARPS * 32, 1)
    k_gemm_i8(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
              const __grid_constant__ PairTable pt, int32_t* __restrict__ out, long long out_plane_stride,
              long long ldo, int M, int N, int K, int tiles_m, int njobs, int* __restrict__ job_counter) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_STAGE_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * B_STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* acc_full = empty + STAGES;    // [2]
  uint64_t* acc_empty = acc_full + 2;     // [2]
  uint64_t* jq_full = acc_empty + 2;   // [JQ]
  uint64_t* jq_empty = jq_full + JQ;   // [JQ]
  int* jq = reinterpret_cast<int*>(jq_empty + JQ);  // [JQ] job ids (−1 = done)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(jq + JQ);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int nkb = (K + BK - 1) / BK;

  if (threadIdx.x == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], 128);  // the 128 epilogue threads
    }
    for (int q = 0; q < JQ; ++q) {
      mbar_init(&jq_full[q], 1);
      mbar_init(&jq_empty[q], 1 + 128);  // MMA issuer + epilogue threads
    }
    fence_mbar_init();
  }
  if (warp == 0) {
    tmem_alloc(tmem_slot, TMEM_ALLOC);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- job fetch + TMA producer
      int it = 0;  // ring position, continuous across jobs
      for (int jn = 0;; ++jn) {
        const int job = (jn == 0) ? static_cast<int>(blockIdx.x) : static_cast<int>(gridDim.x) + atomicAdd(job_counter, 1);
        const int slot = jn % JQ;
        mbar_wait(&jq_empty[slot], ((jn / JQ) & 1) ^ 1);
        jq[slot] = job < njobs ? job : -1;
        mbar_arrive(&jq_full[slot]);
        if (job >= njobs) break;
        const JobInfo ji = job_info(job, pt, M, N, tiles_m);
        if (ji.skip) continue;
        const int p0 = pt.first[ji.g];
        const int total = (pt.first[ji.g + 1] - p0) * nkb;
        for (int q = 0; q < total; ++q, ++it) {
          const int stage = it % STAGES;
          const uint32_t phase = (it / STAGES) & 1;
          mbar_wait(&empty[stage], phase ^ 1);
          const int p = p0 + q / nkb;
          const int kb = q - (q / nkb) * nkb;
          mbar_arrive_expect_tx(&full[stage], A_STAGE_BYTES + B_STAGE_BYTES);
          tma_load_3d(sA + stage * A_STAGE_BYTES, &tmA, &full[stage], kb * BK, ji.m0, pt.s[p]);
          tma_load_3d(sB + stage * B_STAGE_BYTES, &tmB, &full[stage], kb * BK, ji.n0, pt.t[p]);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer (single thread)
      constexpr uint32_t idesc = idesc_i8(BM, BN);
      int it = 0, t = 0;
      for (int jn = 0;; ++jn) {
        const int slot = jn % JQ;
        mbar_wait(&jq_full[slot], (jn / JQ) & 1);
        const int job = *reinterpret_cast<volatile int*>(&jq[slot]);
        mbar_arrive(&jq_empty[slot]);
        if (job < 0) break;
        const JobInfo ji = job_info(job, pt, M, N, tiles_m);
        if (ji.skip) continue;
        const int buf = t & 1;
        mbar_wait(&acc_empty[buf], ((t >> 1) & 1) ^ 1);  // the epilogue has drained this accumulator
        tc_fence_after();
        const uint32_t acc = tmem_base + static_cast<uint32_t>(buf * TMEM_COLS);
        const int total = (pt.first[ji.g + 1] - pt.first[ji.g]) * nkb;
        for (int q = 0; q < total; ++q, ++it) {
          const int stage = it % STAGES;
          const uint32_t phase = (it / STAGES) & 1;
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(sA + stage * A_STAGE_BYTES);
          const uint32_t b_addr = smem_u32(sB + stage * B_STAGE_BYTES);
#pragma unroll
          for (int k = 0; k < BK / UMMA_K; ++k) {
            const uint64_t ad = umma_desc_kmajor_sw128(a_addr + k * UMMA_K);
            const uint64_t bd = umma_desc_kmajor_sw128(b_addr + k * UMMA_K);
            mma_i8(acc, ad, bd, idesc, (q > 0 || k > 0) ? 1u : 0u);
          }
          mma_commit(&empty[stage]);  // frees the smem slot when these MMAs complete
        }
        mma_commit(&acc_full[buf]);  // accumulator complete (also when total == 0: the epilogue writes 0)
        ++t;
      }
    }
    __syncwarp();
  } else {
    // ---------------- epilogue warps 2..5: TMEM lane quarter (warp % 4) → int32 plane, column-major
    const int quarter = warp & 3;
    int t = 0;
    for (int jn = 0;; ++jn) {
      const int slot = jn % JQ;
      mbar_wait(&jq_full[slot], (jn / JQ) & 1);
      const int job = *reinterpret_cast<volatile int*>(&jq[slot]);
      mbar_arrive(&jq_empty[slot]);
      if (job < 0) break;
      const JobInfo ji = job_info(job, pt, M, N, tiles_m);
      if (ji.skip) continue;
      const int buf = t & 1;
      mbar_wait(&acc_full[buf], (t >> 1) & 1);
      tc_fence_after();
      __syncwarp();
      const bool total_zero = (pt.first[ji.g + 1] == pt.first[ji.g]);
      int32_t* op = out + static_cast<long long>(pt.out_plane[ji.g]) * out_plane_stride;
      const int row = ji.m0 + quarter * 32 + lane;
      const uint32_t acc = tmem_base + static_cast<uint32_t>(buf * TMEM_COLS) + (static_cast<uint32_t>(quarter * 32) << 16);
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 32) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(acc + c0, r);
        tmem_ld_wait();
        if (row < M) {
#pragma unroll
          for (int c = 0; c < 32; ++c) {
            const int col = ji.n0 + c0 + c;
            if (col < N) op[static_cast<long long>(col) * ldo + row] = total_zero ? 0 : static_cast<int32_t>(r[c]);
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&acc_empty[buf]);
      ++t;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem_base, TMEM_ALLOC);
}

// ---------------------------------------------------------------- CTA-pair form (cta_group::2)
// A cluster of 2 CTAs (one TPC) computes a 256 x 256 tile: each CTA stages ITS 128 rows of A and ITS half
// (128 of 256 rows) of B per K-block, the leader issues tcgen05.mma.cta_group::2 (M = 256) that reads the
// operands from both CTAs' shared memory and accumulates rows 0-127 in the leader's TMEM, 128-255 in the
// peer's. Per SM, the shared-memory fill per K-block drops from 48 KB to 32 KB for the same MMA work
// (the single-CTA form is bound by L2 → SM operand traffic). Roles per CTA as in the single-CTA form; the
// leader fetches the jobs and mirrors them into the peer's queue (DSMEM), the MMA warp is the leader's.
// A stage holds KH2 = 2 K-blocks of 128 B (two swizzle atoms per operand, loaded by separate TMA boxes): the
// MMA issuer commits the stage back to the producer once per 8 MMAs instead of once per 4 — a tcgen05.commit
// per 4 MMAs costs 37 % of the MMA rate, per 8 MMAs 16 % (tools/i8_peak.cu). Same 192 KB ring.
constexpr int KH2 = 2;
constexpr int STAGES2 = 3;
constexpr int B_HALF_BYTES = (BN / 2) * BK;
constexpr int A_STAGE2 = KH2 * A_STAGE_BYTES;
constexpr int B_STAGE2 = KH2 * B_HALF_BYTES;
constexpr int SMEM2_BYTES = STAGES2 * (A_STAGE2 + B_STAGE2) + 1024 /*align*/ + 512 /*barriers*/;

// order 0: (band, m-tile, n-tile, group) — a tile's groups back to back;
// order 1: (band, m-tile, group, n-tile) — the band's n-tiles of one group back to back: those jobs read the
// same A rows and planes at the same time (A is the larger operand: k_A planes vs k_X), so each A K-block is
// fetched from DRAM once and served to all BAND readers from L2.
__device__ __forceinline__ JobInfo job_info2(int job, const PairTable& pt, int N, int tiles_m2, int order, int BANDW) {
  const int G = pt.ngroups;
  const int tiles_n = (N + BN - 1) / BN;
  JobInfo ji;
  if (order & 1) {
    const int per_band = tiles_m2 * BANDW * G;
    const int band = job / per_band;
    const int r = job - band * per_band;
    const int nb = min(BANDW, tiles_n - band * BANDW);
    const int q = r / nb;
    ji.g = q % G;
    ji.m0 = (q / G) * (2 * BM);
    ji.n0 = (band * BANDW + r % nb) * BN;
  } else {
    ji.g = job % G;
    const int tile = job / G;
    const int band = tile / (BANDW * tiles_m2);
    const int r = tile - band * (BANDW * tiles_m2);
    const int nb = min(BANDW, tiles_n - band * BANDW);
    ji.m0 = (r / nb) * (2 * BM);  // the pair's 256 rows
    ji.n0 = (band * BANDW + r % nb) * BN;
  }
  ji.skip = (pt.tile_budgets && pt.diag[ji.g] > pt.tileL[ji.n0 / BN]) ? 1 : 0;
  return ji;
}

// KIND 0: int8 digit planes (kind::i8, exact int32); KIND 1: bf16 operands (kind::f16, f32 accumulator: the
// certificate's Q = ẼᵀC, certify.cu). Both consume 32 bytes of K per MMA from the same 128-byte swizzle rows, so
// the data movement is byte-for-byte the same; K is given in bytes.
template <int KIND>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NWARPS * 32, 1)
    k_gemm_i8_2sm(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                  const __grid_constant__ PairTable pt, int32_t* __restrict__ out, long long out_plane_stride,
                  long long ldo, int M, int N, int K, int tiles_m2, int njobs, int* __restrict__ job_counter,
                  int l2hint, int order, int bandw) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES2 * A_STAGE2;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES2 * B_STAGE2);
  uint64_t* empty = full + STAGES2;
  uint64_t* acc_full = empty + STAGES2;  // [2]
  uint64_t* acc_empty = acc_full + 2;    // [2] (leader's)
  uint64_t* jq_full = acc_empty + 2;     // [JQ]
  uint64_t* jq_empty = jq_full + JQ;     // [JQ] (leader's)
  int* jq = reinterpret_cast<int*>(jq_empty + JQ);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(jq + JQ);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = (rank == 0);
  const int nkb = (K + KH2 * BK - 1) / (KH2 * BK);  // stages of KH2 K-blocks

  if (threadIdx.x == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    for (int s = 0; s < STAGES2; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], 8);  // 4 epilogue warps x 2 CTAs
    }
    for (int q = 0; q < JQ; ++q) {
      mbar_init(&jq_full[q], 1);
      mbar_init(&jq_empty[q], 10);  // leader: MMA + 4 epilogue warps; peer: producer + 4 epilogue warps
    }
    fence_mbar_init();
  }
  if (warp == 0) {
    tmem_alloc_2sm(tmem_slot, TMEM_ALLOC);
    tmem_relinquish_2sm();
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // the peer's barriers are initialised before any remote arrive / multicast
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- job fetch (leader) + TMA producer (both CTAs)
      // L2 policies (l2hint bit 0: A rows evict-first — they are reused only by the jobs in flight on the same
      // m-tile; bit 1: the band's B columns evict-last — reused by every m-tile of the band)
      const uint64_t polA = (l2hint & 1) ? l2_policy_evict_first() : l2_policy_evict_normal();
      const uint64_t polB = (l2hint & 2) ? l2_policy_evict_last() : l2_policy_evict_normal();
      int it = 0;
      for (int jn = 0;; ++jn) {
        const int slot = jn % JQ;
        int job;
        if (leader) {
          job = (jn == 0) ? static_cast<int>(blockIdx.x >> 1)
                          : static_cast<int>(gridDim.x >> 1) + atomicAdd(job_counter, 1);
          if (job >= njobs) job = -1;
          mbar_wait_cluster(&jq_empty[slot], ((jn / JQ) & 1) ^ 1);
          jq[slot] = job;
          st_cluster_u32(mapa_u32(&jq[slot], 1), static_cast<uint32_t>(job));
          mbar_arrive(&jq_full[slot]);
          mbar_arrive_remote(mapa_u32(&jq_full[slot], 1));
        } else {
          mbar_wait_cluster(&jq_full[slot], (jn / JQ) & 1);
          job = *reinterpret_cast<volatile int*>(&jq[slot]);
          mbar_arrive_remote(mapa_u32(&jq_empty[slot], 0));
        }
        if (job < 0) break;
        const JobInfo ji = job_info2(job, pt, N, tiles_m2, order, bandw);
        if (ji.skip) continue;
        const int p0 = pt.first[ji.g];
        const int npg = pt.first[ji.g + 1] - p0;
        const int total = npg * nkb;
        const bool kouter = (order & 2) != 0;
        for (int q = 0; q < total; ++q, ++it) {
          const int stage = it % STAGES2;
          const uint32_t phase = (it / STAGES2) & 1;
          mbar_wait(&empty[stage], phase ^ 1);
          if (leader) mbar_arrive_expect_tx(&full[stage], 2 * (A_STAGE2 + B_STAGE2));
          // kouter: K-block outer, the group's pairs inner — at any moment every job of a tile's neighbourhood
          // reads the same K-block of the A planes, so L2 serves them all from one DRAM fetch
          int p, kb;
          if (kouter) {
            kb = q / npg;
            p = p0 + (q - kb * npg);
          } else {
            p = p0 + q / nkb;
            kb = q - (q / nkb) * nkb;
          }
          const uint32_t fb = mapa_u32(&full[stage], 0);  // the leader's barrier counts both CTAs' bytes
#pragma unroll
          for (int h = 0; h < KH2; ++h) {  // K beyond the extent is zero-filled by the tensor map
            tma_load_3d_2sm_hint(sA + stage * A_STAGE2 + h * A_STAGE_BYTES, &tmA, fb, (kb * KH2 + h) * BK,
                                 ji.m0 + static_cast<int>(rank) * BM, pt.s[p], polA);
            tma_load_3d_2sm_hint(sB + stage * B_STAGE2 + h * B_HALF_BYTES, &tmB, fb, (kb * KH2 + h) * BK,
                                 ji.n0 + static_cast<int>(rank) * (BN / 2), pt.t[p], polB);
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0 && leader) {
      // ---------------- MMA issuer (leader CTA, single thread): M = 256 over the pair
      constexpr uint32_t idesc = KIND == 0 ? idesc_i8(2 * BM, BN) : idesc_bf16(2 * BM, BN);
      int it = 0, t = 0;
      for (int jn = 0;; ++jn) {
        const int slot = jn % JQ;
        mbar_wait_cluster(&jq_full[slot], (jn / JQ) & 1);
        const int job = *reinterpret_cast<volatile int*>(&jq[slot]);
        mbar_arrive(&jq_empty[slot]);
        if (job < 0) break;
        const JobInfo ji = job_info2(job, pt, N, tiles_m2, order, bandw);
        if (ji.skip) continue;
        const int buf = t & 1;
        mbar_wait_cluster(&acc_empty[buf], ((t >> 1) & 1) ^ 1);  // both CTAs' epilogues drained it
        tc_fence_after();
        const uint32_t acc = tmem_base + static_cast<uint32_t>(buf * TMEM_COLS);
        const int total = (pt.first[ji.g + 1] - pt.first[ji.g]) * nkb;
        for (int q = 0; q < total; ++q, ++it) {
          const int stage = it % STAGES2;
          const uint32_t phase = (it / STAGES2) & 1;
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(sA + stage * A_STAGE2);
          const uint32_t b_addr = smem_u32(sB + stage * B_STAGE2);
#pragma unroll
          for (int h = 0; h < KH2; ++h)
#pragma unroll
            for (int k = 0; k < BK / UMMA_K; ++k) {
              const uint64_t ad = umma_desc_kmajor_sw128(a_addr + h * A_STAGE_BYTES + k * UMMA_K);
              const uint64_t bd = umma_desc_kmajor_sw128(b_addr + h * B_HALF_BYTES + k * UMMA_K);
              if constexpr (KIND == 0) mma_i8_2sm(acc, ad, bd, idesc, (q > 0 || h > 0 || k > 0) ? 1u : 0u);
              else mma_bf16_2sm(acc, ad, bd, idesc, (q > 0 || h > 0 || k > 0) ? 1u : 0u);
            }
          mma_commit_2sm(&empty[stage], 0x3);  // frees the stage in both CTAs
        }
        mma_commit_2sm(&acc_full[buf], 0x3);
        ++t;
      }
    }
    __syncwarp();
  } else {
    // ---------------- epilogue warps 2..5 of both CTAs: this CTA's 128 rows of the pair tile
    const int quarter = warp & 3;
    int t = 0;
    for (int jn = 0;; ++jn) {
      const int slot = jn % JQ;
      mbar_wait_cluster(&jq_full[slot], (jn / JQ) & 1);
      const int job = *reinterpret_cast<volatile int*>(&jq[slot]);
      __syncwarp();
      if (lane == 0) {
        if (leader) mbar_arrive(&jq_empty[slot]);
        else mbar_arrive_remote(mapa_u32(&jq_empty[slot], 0));
      }
      if (job < 0) break;
      const JobInfo ji = job_info2(job, pt, N, tiles_m2, order, bandw);
      if (ji.skip) continue;
      const int buf = t & 1;
      mbar_wait(&acc_full[buf], (t >> 1) & 1);
      tc_fence_after();
      __syncwarp();
      const bool total_zero = (pt.first[ji.g + 1] == pt.first[ji.g]);
      int32_t* op = out + static_cast<long long>(pt.out_plane[ji.g]) * out_plane_stride;
      const int row = ji.m0 + static_cast<int>(rank) * BM + quarter * 32 + lane;
      const uint32_t acc = tmem_base + static_cast<uint32_t>(buf * TMEM_COLS) + (static_cast<uint32_t>(quarter * 32) << 16);
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 32) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(acc + c0, r);
        tmem_ld_wait();
        if (row < M) {
#pragma unroll
          for (int c = 0; c < 32; ++c) {
            const int col = ji.n0 + c0 + c;
            if (col < N) op[static_cast<long long>(col) * ldo + row] = total_zero ? 0 : static_cast<int32_t>(r[c]);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (leader) mbar_arrive(&acc_empty[buf]);
        else mbar_arrive_remote(mapa_u32(&acc_empty[buf], 0));
      }
      ++t;
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // no CTA leaves while its peer may still signal its barriers or read its smem
  if (warp == 0) tmem_dealloc_2sm(tmem_base, TMEM_ALLOC);
}

// ---------------------------------------------------------------- SIMT cross-check kernel (dev only)
__global__ void k_gemm_i8_simt(DigitOperand A, DigitOperand B, PairTable pt, int32_t* out,
                               long long out_plane_stride, long long ldo, int M, int N, int K) {
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  const int col = blockIdx.y;
  const int g = blockIdx.z;
  if (row >= M || col >= N) return;
  if (pt.tile_budgets && pt.diag[g] > pt.tileL[col / kTileN]) return;
  int32_t acc = 0;
  for (int p = pt.first[g]; p < pt.first[g + 1]; ++p) {
    const int8_t* a = A.base + pt.s[p] * A.plane_stride + static_cast<long long>(row) * A.ld;
    const int8_t* b = B.base + pt.t[p] * B.plane_stride + static_cast<long long>(col) * B.ld;
    for (int k = 0; k < K; ++k) acc += static_cast<int32_t>(a[k]) * static_cast<int32_t>(b[k]);
  }
  out[pt.out_plane[g] * out_plane_stride + static_cast<long long>(col) * ldo + row] = acc;
}

typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

PFN_encodeTiled get_encode() {
  static PFN_encodeTiled fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return nullptr;
    fn = reinterpret_cast<PFN_encodeTiled>(p);
  }
  return fn;
}

// 3-D uint8 tensor map over digit planes: dims (K bytes, cols, planes), box (BK, box_rows, 1), SW128.
bool make_tmap(CUtensorMap* tm, const DigitOperand& op, int K, int cols, int box_rows) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(K), static_cast<cuuint64_t>(cols),
                        static_cast<cuuint64_t>(op.nplanes)};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(op.ld), static_cast<cuuint64_t>(op.plane_stride)};
  cuuint32_t box[3] = {static_cast<cuuint32_t>(BK), static_cast<cuuint32_t>(box_rows), 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<int8_t*>(op.base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

}  // namespace

cudaError_t launch_gemm_i8(const DigitOperand& A, const DigitOperand& B, int M, int N, int K,
                           const PairTable& pt, int32_t* out, int64_t out_plane_stride, int64_t ldo,
                           cudaStream_t stream, int* job_counter, int job_order, int kind) {
  if (M <= 0 || N <= 0 || pt.ngroups <= 0) return cudaSuccess;
  if (K <= 0 || (A.ld % 16) || (B.ld % 16) || (A.plane_stride % 16) || (B.plane_stride % 16))
    return cudaErrorInvalidValue;
  static int use2_env = -1;
  if (use2_env < 0) {
    const char* v = getenv("OZR_GEMM");
    use2_env = (v && v[0] == '1') ? 0 : 1;  // OZR_GEMM=1sm: the single-CTA form (A/B measurements)
  }
  const int use2 = (kind == 1) ? 1 : use2_env;  // the bf16 form exists only as the CTA pair
  CUtensorMap tmA, tmB;
  if (!make_tmap(&tmA, A, K, M, BM) || !make_tmap(&tmB, B, K, N, use2 ? BN / 2 : BN)) return cudaErrorInvalidValue;
  if (!use2) {
    cudaError_t e = once_per_device(0, [] {
      return cudaFuncSetAttribute(k_gemm_i8, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
    });
    if (e != cudaSuccess) return e;
  }
  const int tiles_m = (M + BM - 1) / BM;
  const int tiles_n = (N + BN - 1) / BN;
  const long long jobs = static_cast<long long>(tiles_m) * tiles_n * pt.ngroups;
  const int nsm = sm_count();
  if (use2) {
    auto kfn = (kind == 1) ? k_gemm_i8_2sm<1> : k_gemm_i8_2sm<0>;
    cudaError_t e2 = once_per_device(1 + (kind & 1), [kfn] {
      cudaError_t e3 = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM2_BYTES);
      if (e3 != cudaSuccess) return e3;
      // the largest shared-memory carveout (228 KB), so that the ~30 KB the GEMM leaves free on every SM can
      // host the register-path recombination CTAs of the previous column band (ozr_api.cu run_banded)
      return cudaFuncSetAttribute(kfn, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    });
    if (e2 != cudaSuccess) return e2;
    const int tiles_m2 = (M + 2 * BM - 1) / (2 * BM);
    const long long jobs2 = static_cast<long long>(tiles_m2) * tiles_n * pt.ngroups;
    const int clusters = static_cast<int>(std::min<long long>(jobs2, nsm / 2));
    if (!job_counter) return cudaErrorInvalidValue;
    cudaError_t e = cudaMemsetAsync(job_counter, 0, sizeof(int), stream);
    if (e != cudaSuccess) return e;
    // L2 policy: the band's B columns evict-last (measured: V launch DRAM read 30.3 → 18.2 GB with job order 1)
    static int l2hint = -1, env_order = -1, bandw = BAND;
    if (l2hint < 0) {
      const char* h = getenv("OZR_L2HINT");
      l2hint = h ? atoi(h) : 2;
      const char* o = getenv("OZR_GEMM_ORDER");
      env_order = o ? atoi(o) : -1;
      const char* b = getenv("OZR_GEMM_BAND");
      bandw = b ? atoi(b) : BAND;
    }
    const int order = env_order >= 0 ? env_order : (job_order >= 0 ? job_order : 1);
    kfn<<<2 * clusters, NWARPS * 32, SMEM2_BYTES, stream>>>(tmA, tmB, pt, out, out_plane_stride, ldo, M, N, K,
                                                             tiles_m2, static_cast<int>(jobs2), job_counter, l2hint,
                                                             order, bandw);
    return cudaGetLastError();
  }
  const int grid = static_cast<int>(std::min<long long>(jobs, nsm));
  if (!job_counter) return cudaErrorInvalidValue;
  int* counter = job_counter;  // the caller's (per context): launches on one stream are ordered, reset before each
  cudaError_t e = cudaMemsetAsync(counter, 0, sizeof(int), stream);
  if (e != cudaSuccess) return e;
  k_gemm_i8<<<grid, NWARPS * 32, SMEM_BYTES, stream>>>(tmA, tmB, pt, out, out_plane_stride, ldo, M, N, K, tiles_m,
                                                        static_cast<int>(jobs), counter);
  return cudaGetLastError();
}

cudaError_t launch_gemm_i8_simt(const DigitOperand& A, const DigitOperand& B, int M, int N, int K,
                                const PairTable& pt, int32_t* out, int64_t out_plane_stride, int64_t ldo,
                                cudaStream_t stream) {
  dim3 grid((M + 127) / 128, N, pt.ngroups);
  k_gemm_i8_simt<<<grid, 128, 0, stream>>>(A, B, pt, out, out_plane_stride, ldo, M, N, K);
  return cudaGetLastError();
}

}  // namespace ozr
