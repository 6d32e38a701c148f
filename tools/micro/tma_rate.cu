// TMA 2D tile-load throughput per SM (148 CTAs, one lane issuing, S boxes in
// flight, a consumer lane re-arming): box = 64 bf16 (128 B, SWIZZLE_128B) x
// BOXR rows from a [rows][RW] bf16 tensor, consecutive row blocks (as the
// tensor-core kernel's parent-slot operands). Reports GB/s per SM and chip.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tma_rate tma_rate.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#include "../../paper_2011_01383_b200/csrc/umma.cuh"

using namespace cx::umma;

struct alignas(64) Desc { unsigned long long d[16]; };

template <int S>
__global__ void __launch_bounds__(64, 1) k_tma(const __grid_constant__ Desc dsc, int boxr, int rw,
                                               long long rows, int iters, long long *cyc) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char *sm = (unsigned char *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t full[S];
  const int box_bytes = 128 * boxr;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; s++) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int katoms = rw / 64;
  const long long nblk = rows / boxr;
  long long t0 = clock64();
  if (threadIdx.x == 0) {
    for (int it = 0; it < iters; it++) {
      const int st = it % S;
      if (it >= S) mbar_wait(&full[st], ((it / S) - 1) & 1);  // slot consumed (landed)
      const long long b = ((long long)blockIdx.x * 7919 + it / katoms) % nblk;
      mbar_arrive_expect_tx(&full[st], box_bytes);
      tma_tile2d(smem_u32(sm + (size_t)st * box_bytes), &dsc, &full[st], (it % katoms) * 64, (int)(b * boxr));
    }
    for (int it = iters; it < iters + S; it++) {
      const int st = it % S;
      mbar_wait(&full[st], ((it / S) - 1) & 1);
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// 3D: dims {64 cols, rows, atoms} (strides: row = rw*2 B, atom = 128 B), box
// {64, 128, NA}: NA K-atoms of 128 rows in ONE instruction, laid out in shared
// memory atom after atom (each a 16 KB K-major SW128 block)
template <int S>
__global__ void __launch_bounds__(64, 1) k_tma3(const __grid_constant__ Desc dsc, int na, int rw,
                                                long long rows, int iters, int producers) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char *sm = (unsigned char *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t full[S];
  const int box_bytes = 128 * 128 * na;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; s++) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int groups = rw / 64 / na;
  const long long nblk = rows / 128;
  // producer p (lane 0 of warp p) issues iterations it = p, p + producers, ...
  // producers > 0: lane 0 of warps 0..producers-1; producers < 0: lanes
  // 0..-producers-1 of warp 0 (issuing in lockstep)
  const int p = producers > 0 ? threadIdx.x / 32 : threadIdx.x;
  const bool prod = producers > 0 ? ((threadIdx.x & 31) == 0 && p < producers) : (threadIdx.x < -producers);
  if (producers < 0) producers = -producers;
  if (prod) {
    for (int it = p; it < iters; it += producers) {
      const int st = it % S;
      if (it >= S) mbar_wait(&full[st], ((it / S) - 1) & 1);
      const long long b = ((long long)blockIdx.x * 7919 + it / groups) % nblk;
      mbar_arrive_expect_tx(&full[st], box_bytes);
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%2, %3, %4}], [%5];"
          ::"r"(smem_u32(sm + (size_t)st * box_bytes)), "l"(&dsc), "r"(0), "r"((int)(b * 128)),
            "r"((it % groups) * na), "r"(smem_u32(&full[st])) : "memory");
    }
  }
  __syncthreads();
  if (threadIdx.x == 0)
    for (int it = iters - S; it < iters; it++) mbar_wait(&full[it % S], (it / S) & 1);
  __syncthreads();
}

using EncodeFn = CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                              const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <int S>
void run(EncodeFn enc, void *base, long long rows, int rw, int boxr, const char *what) {
  Desc d;
  cuuint64_t dims[2] = {(cuuint64_t)rw, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)rw * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)boxr}, es[2] = {1, 1};
  enc(reinterpret_cast<CUtensorMap *>(&d), CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides, box, es,
      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  long long *cyc;
  cudaMalloc(&cyc, 148 * 8);
  const int smem = 1024 + S * 128 * boxr;
  cudaFuncSetAttribute(k_tma<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 2048;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_tma<S><<<148, 64, smem>>>(d, boxr, rw, rows, iters, cyc);
  cudaEventRecord(e0);
  k_tma<S><<<148, 64, smem>>>(d, boxr, rw, rows, iters, cyc);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double bytes = 148.0 * iters * 128 * boxr;
  printf("%-5s rw=%4d box=64x%3d S=%2d: %7.1f GB/s chip, %5.1f GB/s/SM (%s)\n", what, rw, boxr, S,
         bytes / (ms * 1e-3) / 1e9, bytes / 148 / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
  cudaFree(cyc);
}

template <int S>
void run3(EncodeFn enc, void *base, long long rows, int rw, int na, int producers) {
  Desc d;
  cuuint64_t dims[3] = {64, (cuuint64_t)rows, (cuuint64_t)(rw / 64)};
  cuuint64_t strides[2] = {(cuuint64_t)rw * 2, 128};
  cuuint32_t box[3] = {64, 128, (cuuint32_t)na}, es[3] = {1, 1, 1};
  CUresult r = enc(reinterpret_cast<CUtensorMap *>(&d), CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, base, dims, strides,
                   box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const int smem = 1024 + S * 128 * 128 * na;
  cudaFuncSetAttribute(k_tma3<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 1024;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_tma3<S><<<148, 64, smem>>>(d, na, rw, rows, iters, producers);
  cudaEventRecord(e0);
  k_tma3<S><<<148, 64, smem>>>(d, na, rw, rows, iters, producers);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double bytes = 148.0 * iters * 128 * 128 * na;
  printf("3D    rw=%4d box=64x128x%d S=%d producers=%d: %7.1f GB/s chip, %5.1f GB/s/SM (encode %d, %s)\n", rw, na, S,
         producers, bytes / (ms * 1e-3) / 1e9, bytes / 148 / (ms * 1e-3) / 1e9, (int)r,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  void *p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  EncodeFn enc = reinterpret_cast<EncodeFn>(p);
  void *big;
  const size_t nbytes = (size_t)512 << 20;
  cudaMalloc(&big, nbytes);
  cudaMemset(big, 0, nbytes);
  {
    const long long rows_l2 = (48ll << 20) / (512 * 2);
    run3<4>(enc, big, rows_l2, 512, 1, -2);
    run3<4>(enc, big, rows_l2, 512, 1, -4);
    run3<4>(enc, big, rows_l2, 512, 2, -2);
    run3<4>(enc, big, rows_l2, 512, 1, 4);
    run3<4>(enc, big, rows_l2, 512, 1, 1);
    run3<4>(enc, big, rows_l2, 512, 1, 2);
    run3<4>(enc, big, rows_l2, 512, 2, 1);
    run3<3>(enc, big, rows_l2, 512, 4, 1);
    run3<2>(enc, big, rows_l2, 512, 4, 2);
    run3<4>(enc, big, rows_l2, 256, 2, 1);
  }
  for (int rw : {256, 512}) {
    const long long rows_l2 = (48ll << 20) / (rw * 2), rows_dram = (long long)(nbytes / (rw * 2));
    for (int boxr : {64, 128, 256}) {
      run<4>(enc, big, rows_l2, rw, boxr, "L2");
      if (boxr <= 128) run<8>(enc, big, rows_l2, rw, boxr, "L2");
      if (boxr <= 128) run<12>(enc, big, rows_l2, rw, boxr, "L2");
      run<4>(enc, big, rows_dram, rw, boxr, "HBM");
      if (boxr <= 128) run<8>(enc, big, rows_dram, rw, boxr, "HBM");
    }
  }
  return 0;
}
