// ozr_internal.h — internal (non-ABI) declarations shared by the ozr CUDA sources.
#pragma once
#include <cstdint>
#include <mutex>
#include <cuda_runtime.h>

namespace ozr {

// Runs f() once per (current device, key), under a lock: kernel attributes set with cudaFuncSetAttribute apply to
// the current device only, so they are set for every device a context runs on, and no thread launches before
// they are in place.
template <class F>
cudaError_t once_per_device(int key, F f) {
  static std::mutex mu;
  static unsigned long long seen[128] = {};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= 128 || key < 0 || key >= 64) return f();
  std::lock_guard<std::mutex> g(mu);
  const unsigned long long bit = 1ull << key;
  if (seen[dev] & bit) return cudaSuccess;
  e = f();
  if (e == cudaSuccess) seen[dev] |= bit;
  return e;
}
inline int sm_count() {
  int dev = 0, nsm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  return nsm > 0 ? nsm : 1;
}

constexpr int kMaxPairs = 256;   // digit pairs per product
constexpr int kMaxGroups = 96;   // int32 accumulation groups (output planes) per product
constexpr int kTileN = 256;      // N extent of one slice-GEMM tile
constexpr int kMaxNTiles = 256;  // per-N-tile pair budgets: N <= 65536

// A product C = Σ_groups Σ_{(s,t) in group} D^A_s · D^B_t is described by a pair table.
// Group g accumulates pairs [first[g], first[g+1]) into ONE int32 plane out_plane[g].
// s/t are 0-based digit-plane indices of the A / B operand.
struct PairTable {
  int ngroups;
  int first[kMaxGroups + 1];
  int out_plane[kMaxGroups];
  int diag[kMaxGroups];  // s+t (1-based digits) of the group: its weight 256^{-diag}
  unsigned char s[kMaxPairs];
  unsigned char t[kMaxPairs];
  // Per-N-tile budgets (R8b): when tile_budgets != 0, tile `nt` (columns [256 nt, 256 nt + 256))
  // only accumulates groups with diag <= tileL[nt]; the other CTAs exit without writing.
  int tile_budgets;
  unsigned char tileL[kMaxNTiles];
};

// Digit-plane operand: planes of int8, "column-major" i.e. plane[p][col][row] with row contiguous.
// For a GEMM operand the contiguous index is K (K-major); `rows` = K extent, `cols` = M or N extent.
struct DigitOperand {
  const int8_t* base;
  int64_t ld;            // bytes between consecutive columns (>= rows, multiple of 16)
  int64_t plane_stride;  // bytes between planes (multiple of 16)
  int nplanes;
};

// Launch the tcgen05 INT8 slice-product kernel: for each group g, out_planes[out_plane[g]] (M x N int32,
// column-major, leading dim ldo) = Σ_{pairs} A_s^T-tile products over K.
//   A: M "columns" of K bytes each (A operand, K-major), B: N columns of K bytes (B operand, K-major).
// job_counter: a device int owned by the caller (one per stream/context), reset by the launcher.
// job_order (CTA-pair form): bit 0 — the BAND n-tiles of one pair group run back to back (they read the same
// A rows and planes at the same time); bit 1 — K-block outer, the group's pairs inner (every job near a tile
// reads the same A K-block at once). Measured best: 3 when the A operand has more planes than B (V = A·X̂),
// else 1 (W, U). −1: 1 (OZR_GEMM_ORDER overrides for experiments).
// kind 0: int8 digit planes (exact int32 planes); kind 1: bf16 operands (2 bytes per K element; K and ld in
// BYTES), f32 accumulator written as raw 32-bit words (the certificate's Q = ẼᵀC, certify.cu).
cudaError_t launch_gemm_i8(const DigitOperand& A, const DigitOperand& B, int M, int N, int K,
                           const PairTable& pt, int32_t* out, int64_t out_plane_stride, int64_t ldo,
                           cudaStream_t stream, int* job_counter, int job_order = -1, int kind = 0);

// Reference (SIMT) version of the same contract; used only by the dev harness to cross-check the
// tensor-core kernel on the GPU. Not on the product path.
cudaError_t launch_gemm_i8_simt(const DigitOperand& A, const DigitOperand& B, int M, int N, int K,
                                const PairTable& pt, int32_t* out, int64_t out_plane_stride, int64_t ldo,
                                cudaStream_t stream);

}  // namespace ozr
