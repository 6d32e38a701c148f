// Standalone check of the tcgen05 encodings in csrc/umma.cuh on B200:
// D[128 x N] = A[128 x 256] * B[N x 256]^T (bf16 in, fp32 out) with operands
// written into K-major SW128 shared memory, accumulated over 16 K=16 MMAs,
// read back with tcgen05.ld, compared with a host fp64 reference. Also times
// the MMA chain. Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o
// umma_test umma_test.cu
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../../paper_2011_01383_b200/csrc/umma.cuh"

using namespace cx::umma;

constexpr int M = 128, K = 256;

template <int N>
__global__ void __launch_bounds__(128, 1) k_mma(const __nv_bfloat16 *A, const __nv_bfloat16 *B,
                                               float *D, long long *cyc) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char *smem = (unsigned char *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  unsigned char *sA = smem;                 // 4 K-atoms x 16 KB
  unsigned char *sB = smem + 4 * M * 128;   // 4 K-atoms x N*128 B
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid / 32;
  // fill: each 16-byte chunk = 8 bf16 of one row
  for (int idx = tid; idx < M * (K / 8); idx += 128) {
    int r = idx / (K / 8), c = idx % (K / 8), ka = c / 8, ch = c % 8;
    uint4 v = *reinterpret_cast<const uint4 *>(A + (size_t)r * K + c * 8);
    *reinterpret_cast<uint4 *>(sA + ka * M * 128 + sw128_off(r, ch)) = v;
  }
  for (int idx = tid; idx < N * (K / 8); idx += 128) {
    int r = idx / (K / 8), c = idx % (K / 8), ka = c / 8, ch = c % 8;
    uint4 v = *reinterpret_cast<const uint4 *>(B + (size_t)r * K + c * 8);
    *reinterpret_cast<uint4 *>(sB + ka * N * 128 + sw128_off(r, ch)) = v;
  }
  fence_proxy_async();
  if (warp == 0) tmem_alloc<(N < 32 ? 32 : N)>(&tbase);
  if (tid == 0) mbar_init(&bar, 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tm = tbase;
  long long t0 = clock64();
  if (tid == 0) {
    constexpr uint32_t id = idesc_bf16(M, N);
    for (int ka = 0; ka < 4; ka++)
      for (int kk = 0; kk < 4; kk++) {
        uint64_t a = sdesc_sw128(smem_u32(sA + ka * M * 128 + kk * 32));
        uint64_t b = sdesc_sw128(smem_u32(sB + ka * N * 128 + kk * 32));
        mma_bf16(tm, a, b, id, (ka | kk) != 0);
      }
    mma_commit(&bar);
  }
  __syncwarp();
  mbar_wait(&bar, 0);
  fence_after();
  long long t1 = clock64();
  for (int c0 = 0; c0 < N; c0 += 32) {
    float v[32];
    tmem_ld32(tm + ((uint32_t)(warp * 32) << 16) + c0, v);
    for (int j = 0; j < 32; j++) D[(size_t)tid * N + c0 + j] = v[j];
  }
  if (tid == 0) cyc[0] = t1 - t0;
  fence_before();
  __syncthreads();
  if (warp == 0) tmem_free<(N < 32 ? 32 : N)>(tm);
}

template <int N>
int run() {
  std::vector<__nv_bfloat16> hA(M * K), hB(N * K);
  std::vector<float> fA(M * K), fB(N * K);
  srand(1234 + N);
  for (int i = 0; i < M * K; i++) {
    float x = (rand() / (float)RAND_MAX) * 2 - 1;
    hA[i] = __float2bfloat16(x);
    fA[i] = __bfloat162float(hA[i]);
  }
  for (int i = 0; i < N * K; i++) {
    float x = (rand() / (float)RAND_MAX) * 2 - 1;
    hB[i] = __float2bfloat16(x);
    fB[i] = __bfloat162float(hB[i]);
  }
  __nv_bfloat16 *dA, *dB;
  float *dD;
  long long *dc;
  cudaMalloc(&dA, M * K * 2);
  cudaMalloc(&dB, N * K * 2);
  cudaMalloc(&dD, M * N * 4);
  cudaMalloc(&dc, 8);
  cudaMemcpy(dA, hA.data(), M * K * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB.data(), N * K * 2, cudaMemcpyHostToDevice);
  size_t smem = 1024 + 4 * M * 128 + 4 * N * 128;
  cudaFuncSetAttribute(k_mma<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_mma<N><<<1, 128, smem>>>(dA, dB, dD, dc);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("N=%d: CUDA error %s\n", N, cudaGetErrorString(e));
    return 1;
  }
  std::vector<float> hD(M * N);
  long long cyc;
  cudaMemcpy(hD.data(), dD, M * N * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
  double maxerr = 0;
  for (int m = 0; m < M; m++)
    for (int n = 0; n < N; n++) {
      double r = 0;
      for (int k = 0; k < K; k++) r += (double)fA[m * K + k] * fB[n * K + k];
      maxerr = fmax(maxerr, fabs(r - hD[m * N + n]));
    }
  printf("N=%3d: max abs err %.3e  (%s)  mma chain %lld cycles\n", N, maxerr,
         maxerr < 1e-3 ? "OK" : "FAIL", cyc);
  cudaFree(dA);
  cudaFree(dB);
  cudaFree(dD);
  return maxerr < 1e-3 ? 0 : 1;
}

int main() {
  int bad = 0;
  bad += run<32>();
  bad += run<64>();
  bad += run<128>();
  bad += run<256>();
  printf(bad ? "UMMA TEST FAILED\n" : "UMMA TEST PASSED\n");
  return bad;
}
