// Dev harness (not product, not a test): cross-check the tcgen05 INT8 slice-product kernel against the
// SIMT reference kernel on random digit planes, then time it on a large case.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <cuda_runtime.h>
#include "../ozr_internal.h"

using namespace ozr;

#define CK(x)                                                                       \
  do {                                                                              \
    cudaError_t e_ = (x);                                                           \
    if (e_ != cudaSuccess) {                                                        \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      exit(1);                                                                      \
    }                                                                               \
  } while (0)

__global__ void k_fill(int8_t* p, long long n, unsigned seed) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  unsigned x = (unsigned)(i * 2654435761ull) ^ seed;
  x ^= x >> 13; x *= 0x5bd1e995u; x ^= x >> 15;
  p[i] = (int8_t)(x & 0xFF);
}

static PairTable make_table(int kA, int kB, int L, int maxpairs) {
  PairTable pt;
  memset(&pt, 0, sizeof(pt));
  int np = 0, ng = 0;
  for (int d = 2; d <= L; ++d) {
    int cnt = 0;
    for (int s = 1; s <= kA; ++s) {
      int t = d - s;
      if (t < 1 || t > kB) continue;
      if (cnt == 0 || cnt == maxpairs) {
        pt.first[ng] = np;
        pt.out_plane[ng] = ng;
        pt.diag[ng] = d;
        ng++;
        cnt = 0;
      }
      pt.s[np] = s - 1;
      pt.t[np] = t - 1;
      np++;
      cnt++;
    }
  }
  pt.first[ng] = np;
  pt.ngroups = ng;
  return pt;
}

static int run_check(int M, int N, int K, int kA, int kB, int L, int maxpairs) {
  int64_t ldA = (K + 15) / 16 * 16;
  DigitOperand A{nullptr, ldA, ldA * M, kA}, B{nullptr, ldA, ldA * N, kB};
  int8_t *dA, *dB;
  CK(cudaMalloc(&dA, A.plane_stride * kA));
  CK(cudaMalloc(&dB, B.plane_stride * kB));
  k_fill<<<(A.plane_stride * kA + 255) / 256, 256>>>(dA, A.plane_stride * kA, 1234u);
  k_fill<<<(B.plane_stride * kB + 255) / 256, 256>>>(dB, B.plane_stride * kB, 987u);
  A.base = dA;
  B.base = dB;
  PairTable pt = make_table(kA, kB, L, maxpairs);
  int64_t ldo = M, ps = (int64_t)M * N;
  int32_t *o1, *o2;
  int* counter = nullptr;
  CK(cudaMalloc(&counter, sizeof(int)));
  CK(cudaMalloc(&o1, ps * pt.ngroups * 4));
  CK(cudaMalloc(&o2, ps * pt.ngroups * 4));
  CK(cudaMemset(o1, 0x55, ps * pt.ngroups * 4));
  CK(launch_gemm_i8(A, B, M, N, K, pt, o1, ps, ldo, 0, counter));
  CK(launch_gemm_i8_simt(A, B, M, N, K, pt, o2, ps, ldo, 0));
  CK(cudaDeviceSynchronize());
  std::vector<int32_t> h1(ps * pt.ngroups), h2(ps * pt.ngroups);
  CK(cudaMemcpy(h1.data(), o1, h1.size() * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(h2.data(), o2, h2.size() * 4, cudaMemcpyDeviceToHost));
  long long bad = 0;
  for (size_t i = 0; i < h1.size(); ++i)
    if (h1[i] != h2[i]) {
      if (bad < 5) printf("  mismatch at %zu: tc=%d simt=%d\n", i, h1[i], h2[i]);
      bad++;
    }
  printf("check M=%d N=%d K=%d kA=%d kB=%d L=%d groups=%d: %s (%lld bad of %zu)\n", M, N, K, kA, kB, L, pt.ngroups,
         bad ? "FAIL" : "OK", bad, h1.size());
  cudaFree(dA); cudaFree(dB); cudaFree(o1); cudaFree(o2);
  return bad ? 1 : 0;
}

static void run_time(int n, int npairs) {
  int64_t ld = n;
  DigitOperand A{nullptr, ld, ld * n, npairs}, B{nullptr, ld, ld * n, 1};
  int8_t *dA, *dB;
  CK(cudaMalloc(&dA, A.plane_stride * npairs));
  CK(cudaMalloc(&dB, B.plane_stride));
  k_fill<<<(A.plane_stride * npairs + 255) / 256, 256>>>(dA, A.plane_stride * npairs, 1u);
  k_fill<<<(B.plane_stride + 255) / 256, 256>>>(dB, B.plane_stride, 2u);
  A.base = dA; B.base = dB;
  PairTable pt;
  memset(&pt, 0, sizeof(pt));
  pt.ngroups = 1; pt.first[0] = 0; pt.first[1] = npairs; pt.out_plane[0] = 0; pt.diag[0] = 2;
  for (int p = 0; p < npairs; ++p) { pt.s[p] = p; pt.t[p] = 0; }
  int32_t* o;
  int* counter = nullptr;
  CK(cudaMalloc(&counter, sizeof(int)));
  CK(cudaMalloc(&o, (int64_t)n * n * 4));
  for (int w = 0; w < 3; ++w) CK(launch_gemm_i8(A, B, n, n, n, pt, o, (int64_t)n * n, n, 0, counter));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int reps = 10;
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) CK(launch_gemm_i8(A, B, n, n, n, pt, o, (int64_t)n * n, n, 0, counter));
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  ms /= reps;
  double ops = 2.0 * n * (double)n * n * npairs;
  printf("time n=%d pairs=%d: %.3f ms  %.1f TOPS (int8)\n", n, npairs, ms, ops / ms / 1e9);
  cudaFree(dA); cudaFree(dB); cudaFree(o);
}

int main(int argc, char** argv) {
  int bad = 0;
  bad += run_check(128, 256, 128, 1, 1, 2, 16);
  bad += run_check(256, 512, 384, 2, 2, 3, 16);
  bad += run_check(300, 200, 1000, 4, 3, 5, 16);
  bad += run_check(1024, 1024, 1024, 6, 5, 7, 3);
  if (bad) { printf("FAILED\n"); return 1; }
  run_time(4096, 8);
  run_time(8192, 8);
  run_time(8192, 16);
  printf("ALL OK\n");
  return 0;
}
