// i8_peak.cu — measured dense INT8 tensor-core peak of this B200 (MEASURED_PEAKS.json has no INT8 entry):
// the slice GEMM's exact instruction stream — tcgen05.mma.cta_group::2.kind::i8, M = 256 per CTA pair,
// N = 256, K = 32, K-major 128 B-swizzled shared-memory operands, int32 accumulators in TMEM — issued
// back to back from shared memory that is never refilled (no TMA, no epilogue, no global traffic), one
// CTA pair per two SMs on all 148 SMs. Burst (≈ 0.2 s) and sustained (≈ 4 s) runs, like the bf16 figures.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o i8_peak tools/i8_peak.cu
// Prints one JSON line. Not part of the library.
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_2602_19090_b200/csrc/ptx.cuh"

using namespace ozr;

constexpr int BM = 128, BN = 256, BK = 128, UMMA_K = 32;
constexpr int A_BYTES = BM * BK, B_HALF = (BN / 2) * BK;

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) k_i8_peak(long long iters, int* sink, int random_bits, int commit_every) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + A_BYTES;
  uint64_t* done = reinterpret_cast<uint64_t*>(sB + B_HALF);
  uint64_t* ring = done + 1;  // 6 stage barriers the GEMM would commit to (nobody waits on them here)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(ring + 6);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool leader = cluster_ctarank() == 0;
  // operand bytes: pseudo-random (random_bits = 1, the power a real digit plane draws) or a low-toggle
  // pattern (random_bits = 0)
  for (int i = threadIdx.x; i < (A_BYTES + B_HALF) / 4; i += blockDim.x) {
    uint32_t h = static_cast<uint32_t>(i + 977 * blockIdx.x) * 2654435761u;
    h ^= h >> 15;
    h *= 2246822519u;
    h ^= h >> 13;
    reinterpret_cast<uint32_t*>(smem)[i] = random_bits ? h : 0x01010101u * (i & 7);
  }
  if (threadIdx.x == 0) {
    mbar_init(done, 1);
    for (int q = 0; q < 6; ++q) mbar_init(ring + q, 1);
    fence_mbar_init();
  }
  if (warp == 0) {
    tmem_alloc_2sm(tmem_slot, 512);
    tmem_relinquish_2sm();
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (warp == 1 && lane == 0 && leader) {
    constexpr uint32_t idesc = idesc_i8(2 * BM, BN);
    const uint32_t a_addr = smem_u32(sA), b_addr = smem_u32(sB);
    for (long long it = 0; it < iters; ++it) {
      const uint32_t acc = tmem + static_cast<uint32_t>((it & 1) * 256);
#pragma unroll
      for (int k = 0; k < BK / UMMA_K; ++k)
        mma_i8_2sm(acc, umma_desc_kmajor_sw128(a_addr + k * UMMA_K), umma_desc_kmajor_sw128(b_addr + k * UMMA_K),
                   idesc, 1u);
      if (commit_every && (it % commit_every) == 0) mma_commit_2sm(ring + (it / commit_every) % 6, 0x3);
    }
    mma_commit_2sm(done, 0x3);
  }
  if (threadIdx.x == 0) {
    mbar_wait(done, 0);
    if (iters < 0) *sink = 1;
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 0) tmem_dealloc_2sm(tmem, 512);
}

int main() {
  const int smem = A_BYTES + B_HALF + 1024 + 128;
  cudaFuncSetAttribute(k_i8_peak, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int grid = nsm / 2 * 2;
  int* sink;
  cudaMalloc(&sink, 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  double res[2][2] = {{0, 0}, {0, 0}};  // [random_bits][burst, sustained]
  const double target_s[2] = {0.2, 4.0};
  long long iters = 2000;
  k_i8_peak<<<grid, 128, smem>>>(iters, sink, 1, 0);  // warm-up
  cudaDeviceSynchronize();
  for (int rb = 0; rb < 2; ++rb)
    for (int m = 0; m < 2; ++m) {
      cudaEventRecord(e0);
      k_i8_peak<<<grid, 128, smem>>>(iters, sink, rb, 0);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e0, e1);
      const long long it2 = static_cast<long long>(iters * (target_s[m] * 1e3 / ms));  // scale to the target
      cudaEventRecord(e0);
      k_i8_peak<<<grid, 128, smem>>>(it2, sink, rb, 0);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      const double ops = 2.0 * (grid / 2) * static_cast<double>(it2) * (BK / UMMA_K) * (2.0 * BM) * BN * UMMA_K;
      res[rb][m] = ops / (ms * 1e-3) / 1e12;
    }
  // the same stream with a tcgen05.commit to a stage barrier after every 1 / 2 K-blocks (the GEMM commits
  // once per K-block to release its shared-memory stage), low-toggle data, burst length
  double rc[2] = {0, 0};
  for (int q = 0; q < 2; ++q) {
    const long long it2 = iters * 50;
    cudaEventRecord(e0);
    k_i8_peak<<<grid, 128, smem>>>(it2, sink, 0, q + 1);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    rc[q] = 2.0 * (grid / 2) * static_cast<double>(it2) * (BK / UMMA_K) * (2.0 * BM) * BN * UMMA_K / (ms * 1e-3) / 1e12;
  }
  fprintf(stderr, "commit every K-block: %.1f TOPS, every 2: %.1f TOPS (low-toggle)\n", rc[0], rc[1]);
  const cudaError_t err = cudaGetLastError();
  printf("{\"int8_tops_burst\": %.1f, \"int8_tops_sustained\": %.1f, \"low_toggle_burst\": %.1f, "
         "\"low_toggle_sustained\": %.1f, \"ctas\": %d, \"operands\": \"pseudo-random bytes (first pair), a "
         "low-toggle pattern (second pair)\", \"error\": \"%s\"}\n",
         res[1][0], res[1][1], res[0][0], res[0][1], grid, cudaGetErrorString(err));
  return err == cudaSuccess ? 0 : 1;
}
