// Row-gather throughput on B200: every CTA (one per SM) gathers random 128-byte
// row pieces of a bf16 table into shared-memory stages, the way the tensor-core
// forward feeds its MMAs. Modes:
//   0  TMA tile::gather4 (one warp issues 32 x 4 rows per 16 KB stage), S stages in flight
//   1  cp.async 16 B by 128 threads, S stages in flight (commit groups)
//   2  TMA 2D tile loads of contiguous rows (box 64 x 128) -- the non-gather reference
// Table rows: `rows` x 256 bf16 (512 B per row); each stage = 128 rows x one
// 64-column K-atom. Reports GB/s over the whole grid and per SM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_bench gather_bench.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../../paper_2011_01383_b200/csrc/umma.cuh"

using namespace cx::umma;

constexpr int H = 256, TM = 128, STAGE = TM * 128;

struct alignas(64) Desc { unsigned long long d[16]; };
struct Args {
  Desc tm;
  const unsigned short *tab;
  const int *idx;  // [ctas][iters][128] row ids
  int iters, S, mode;
  unsigned long long *cyc;
};

__global__ void __launch_bounds__(160, 1) k_gather(const __grid_constant__ Args a) {
  extern __shared__ __align__(1024) unsigned char sm_raw[];
  unsigned char *sm = (unsigned char *)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t full[16];
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const int S = a.S;
  if (tid == 0)
    for (int s = 0; s < S; s++) mbar_init(&full[s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  const int *idx = a.idx + (size_t)blockIdx.x * a.iters * TM;
  unsigned long long t0 = clock64();
  if (a.mode == 0 || a.mode == 2) {
    if (warp == 0) {
      for (int it = 0; it < a.iters; it++) {
        const int s = it % S;
        if (it >= S) mbar_wait(&full[s], ((it / S) - 1) & 1);  // consume: previous use landed
        if (lane == 0) mbar_arrive_expect_tx(&full[s], STAGE);
        __syncwarp();
        const int ka = it & 3;
        if (a.mode == 0) {
          const int4 r = *reinterpret_cast<const int4 *>(idx + (size_t)it * TM + 4 * lane);
          tma_gather4(smem_u32(sm + s * STAGE + lane * 512), &a.tm, &full[s], ka * 64, r.x, r.y, r.z, r.w);
        } else if (lane == 0) {
          const int r0 = idx[(size_t)it * TM] & ~127;
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
              " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(sm + s * STAGE)), "l"(&a.tm),
              "r"(ka * 64), "r"(r0), "r"(smem_u32(&full[s])) : "memory");
        }
      }
      for (int it = a.iters - S; it < a.iters; it++) mbar_wait(&full[it % S], (it / S) & 1);
    }
  } else {
    if (tid < 128) {
      int pend = 0;
      for (int it = 0; it < a.iters; it++) {
        const int s = it % S, ka = it & 3;
        for (int e = 0; e < 8; e++) {
          const int q = tid + 128 * e, r = q >> 3, c = q & 7;
          const int row = idx[(size_t)it * TM + r];
          const unsigned short *g = a.tab + (size_t)row * H + ka * 64 + c * 8;
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(sm + s * STAGE + sw128_off(r, c))),
                       "l"(g) : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
        if (++pend >= S) {
          asm volatile("cp.async.wait_group 0;" ::: "memory");  // conservative: S in flight
          pend = 0;
        }
      }
      asm volatile("cp.async.wait_all;" ::: "memory");
    }
  }
  __syncthreads();
  if (tid == 0) a.cyc[blockIdx.x] = clock64() - t0;
}

using EncodeFn = CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                              const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char **argv) {
  const long long rows = argc > 1 ? atoll(argv[1]) : 20000;
  const int iters = 256;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned short *tab;
  int *idx;
  unsigned long long *cyc;
  cudaMalloc(&tab, rows * H * 2);
  cudaMemset(tab, 0, rows * H * 2);
  std::vector<int> hidx((size_t)sms * iters * TM);
  srand(1);
  for (auto &v : hidx) v = (int)(((unsigned long long)rand() * rand()) % rows);
  cudaMalloc(&idx, hidx.size() * 4);
  cudaMemcpy(idx, hidx.data(), hidx.size() * 4, cudaMemcpyHostToDevice);
  cudaMalloc(&cyc, sms * 8);
  void *fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  for (int mode = 0; mode < 3; mode++) {
    Desc d;
    cuuint64_t dims[2] = {(cuuint64_t)H, (cuuint64_t)rows}, str[1] = {(cuuint64_t)H * 2};
    cuuint32_t box[2] = {64, (cuuint32_t)(mode == 2 ? 128 : 1)}, es[2] = {1, 1};
    CUresult r = ((EncodeFn)fn)((CUtensorMap *)&d, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, tab, dims, str, box, es,
                                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("encode failed %d\n", r); return 1; }
    for (int S : {2, 4, 6, 8, 12}) {
      Args a{d, tab, idx, iters, S, mode, cyc};
      size_t smem = 1024 + (size_t)S * STAGE;
      cudaFuncSetAttribute(k_gather, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      k_gather<<<sms, 160, smem>>>(a);
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0);
      for (int rep = 0; rep < 5; rep++) k_gather<<<sms, 160, smem>>>(a);
      cudaEventRecord(e1);
      cudaError_t err = cudaDeviceSynchronize();
      if (err != cudaSuccess) { printf("mode %d S %d: %s\n", mode, S, cudaGetErrorString(err)); return 1; }
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      double bytes = 5.0 * sms * iters * STAGE;
      printf("mode %d (%s) rows %lld S %2d: %7.1f GB/s total, %6.1f GB/s per SM, %.2f us per stage\n", mode,
             mode == 0 ? "tma gather4" : mode == 1 ? "cp.async16" : "tma tile   ", rows, S,
             bytes / (ms * 1e-3) / 1e9, bytes / (ms * 1e-3) / 1e9 / sms, ms * 1e3 / 5 / iters);
    }
  }
  return 0;
}
