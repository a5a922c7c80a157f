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
#include <cstdio>
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
constexpr int BAND = 4;  // n-tiles per rasterisation band

__global__ void __launch_bounds__(128, 1)
    k_gemm_i8(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
              const __grid_constant__ PairTable pt, int32_t* __restrict__ out, long long out_plane_stride,
              long long ldo, int M, int N, int K, int tiles_m) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_STAGE_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * B_STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* accf = empty + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accf + 1);

  const int G = pt.ngroups;
  const int job = blockIdx.x;
  const int g = job % G;  // the groups of one tile run back to back (they share its operand rows)
  const int tile = job / G;
  // L2 rasterisation: bands of BAND n-tiles; inside a band, consecutive tiles sweep the band's n-tiles
  // for one m-tile, then the next m-tile — the band's B columns stay L2-resident while A streams once
  // per band (instead of once per n-tile)
  const int tiles_n = (N + BN - 1) / BN;
  const int band = tile / (BAND * tiles_m);
  const int r = tile - band * (BAND * tiles_m);
  const int nb = min(BAND, tiles_n - band * BAND);
  const int m0 = (r / nb) * BM;
  const int n0 = (band * BAND + r % nb) * BN;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if (pt.tile_budgets && pt.diag[g] > pt.tileL[n0 / BN]) return;  // beyond this column tile's budget

  if (threadIdx.x == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(accf, 1);
    fence_mbar_init();
  }
  if (warp == 0) {
    tmem_alloc(tmem_slot, TMEM_COLS);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int nkb = (K + BK - 1) / BK;
  const int p0 = pt.first[g];
  const int npairs = pt.first[g + 1] - p0;
  const int total = npairs * nkb;

  if (warp == 0) {
    if (lane == 0) {
    // ---------------- TMA producer
    for (int it = 0; it < total; ++it) {
      const int stage = it % STAGES;
      const uint32_t phase = (it / STAGES) & 1;
      mbar_wait(&empty[stage], phase ^ 1);
      const int p = p0 + it / nkb;
      const int kb = it - (it / nkb) * nkb;
      mbar_arrive_expect_tx(&full[stage], A_STAGE_BYTES + B_STAGE_BYTES);
      tma_load_3d(sA + stage * A_STAGE_BYTES, &tmA, &full[stage], kb * BK, m0, pt.s[p]);
      tma_load_3d(sB + stage * B_STAGE_BYTES, &tmB, &full[stage], kb * BK, n0, pt.t[p]);
    }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {
    // ---------------- MMA issuer (single thread)
    constexpr uint32_t idesc = idesc_i8(BM, BN);
    for (int it = 0; it < total; ++it) {
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
        mma_i8(tmem_base, ad, bd, idesc, (it > 0 || k > 0) ? 1u : 0u);
      }
      mma_commit(&empty[stage]);  // frees the smem slot when these MMAs complete
    }
    mma_commit(accf);  // accumulator complete
    }
    __syncwarp();
  }

  // ---------------- epilogue: TMEM -> registers -> int32 plane (column-major, coalesced per column)
  mbar_wait(accf, 0);
  tc_fence_after();
  __syncwarp();
  int32_t* op = out + static_cast<long long>(pt.out_plane[g]) * out_plane_stride;
  const int row = m0 + warp * 32 + lane;
  const bool total_zero = (total == 0);
#pragma unroll 1
  for (int c0 = 0; c0 < BN; c0 += 32) {
    uint32_t r[32];
    tmem_ld_32x32b_x32(tmem_base + (static_cast<uint32_t>(warp * 32) << 16) + c0, r);
    tmem_ld_wait();
    if (row < M) {
#pragma unroll
      for (int c = 0; c < 32; ++c) {
        const int col = n0 + c0 + c;
        if (col < N) op[static_cast<long long>(col) * ldo + row] = total_zero ? 0 : static_cast<int32_t>(r[c]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem_base, TMEM_COLS);
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
                           cudaStream_t stream) {
  if (M <= 0 || N <= 0 || pt.ngroups <= 0) return cudaSuccess;
  if (K <= 0 || (A.ld % 16) || (B.ld % 16) || (A.plane_stride % 16) || (B.plane_stride % 16))
    return cudaErrorInvalidValue;
  CUtensorMap tmA, tmB;
  if (!make_tmap(&tmA, A, K, M, BM) || !make_tmap(&tmB, B, K, N, BN)) return cudaErrorInvalidValue;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(k_gemm_i8, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  const int tiles_m = (M + BM - 1) / BM;
  const int tiles_n = (N + BN - 1) / BN;
  const long long jobs = static_cast<long long>(tiles_m) * tiles_n * pt.ngroups;
  k_gemm_i8<<<static_cast<unsigned>(jobs), 128, SMEM_BYTES, stream>>>(tmA, tmB, pt, out, out_plane_stride, ldo, M,
                                                                      N, K, tiles_m);
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
