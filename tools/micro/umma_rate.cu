// tcgen05.mma throughput on one SM: one thread issues REPS x 16 MMAs
// (M = 128, N, K = 16, bf16 SS operands: A and B both in shared memory,
// K-major SW128) into one TMEM accumulator, one commit at the end; cycles per
// MMA vs N. Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o umma_rate umma_rate.cu
#include <cuda_runtime.h>

#include <cstdio>

#include "../../paper_2011_01383_b200/csrc/umma.cuh"

using namespace cx::umma;
constexpr int M = 128, REPS = 64;

template <int N>
__global__ void __launch_bounds__(128, 1) k_rate(long long *cyc) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char *smem = (unsigned char *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  unsigned char *sA = smem, *sB = smem + 4 * M * 128;
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid / 32;
  for (int i = tid; i < (4 * M * 128 + 4 * N * 128) / 16; i += 128)
    reinterpret_cast<uint4 *>(smem)[i] = make_uint4(0x3f803f80u, 0, 0x3f803f80u, 0);
  if (warp == 0) tmem_alloc<N < 32 ? 32 : N>(&tbase);
  if (tid == 0) mbar_init(&bar, 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  fence_proxy_async();
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tm = tbase;
  long long t0 = clock64();
  if (tid == 0) {
    constexpr uint32_t id = idesc_bf16(M, N);
    for (int r = 0; r < REPS; r++)
      for (int ka = 0; ka < 4; ka++)
#pragma unroll
        for (int kk = 0; kk < 4; kk++) {
          uint64_t a = sdesc_sw128(smem_u32(sA + ka * M * 128 + kk * 32));
          uint64_t b = sdesc_sw128(smem_u32(sB + ka * N * 128 + kk * 32));
          mma_bf16(tm, a, b, id, (r | ka | kk) != 0);
        }
    mma_commit(&bar);
  }
  __syncwarp();
  mbar_wait(&bar, 0);
  fence_after();
  long long t1 = clock64();
  if (tid == 0) cyc[0] = t1 - t0;
  __syncthreads();
  if (warp == 0) tmem_free<N < 32 ? 32 : N>(tm);
}

template <int N>
void run() {
  long long *d, h = 0;
  cudaMalloc(&d, 8);
  auto k = k_rate<N>;
  const int smem = 1024 + 4 * M * 128 + 4 * N * 128;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int it = 0; it < 3; it++) k<<<1, 128, smem>>>(d);
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  cudaError_t e = cudaGetLastError();
  const double per = (double)h / (REPS * 16);
  printf("N=%3d: %lld cycles for %d MMAs = %.1f cycles/MMA = %.0f flop/clk/SM (%s)\n", N, h, REPS * 16,
         per, 2.0 * M * N * 16 / per, cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  run<32>();
  run<64>();
  run<128>();
  run<256>();
  return 0;
}
