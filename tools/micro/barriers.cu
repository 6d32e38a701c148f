// Microbenchmarks on B200: cost of __syncthreads (512 threads), of a dependent
// shared-memory load chain, of reading %globaltimer, of a grid barrier
// (release/acquire counter, 144 co-resident CTAs) and of barrier.cluster.
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__global__ void k_bar(long long *out, int iters) {
  __shared__ int s[1024];
  s[threadIdx.x] = threadIdx.x;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; i++) __syncthreads();
  long long t1 = clock64();
  int x = threadIdx.x;
  for (int i = 0; i < iters; i++) x = s[(x + 1) & 511];  // dependent LDS chain
  long long t2 = clock64();
  unsigned long long g;
  for (int i = 0; i < iters; i++) { asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g)); x += (int)g; }
  long long t3 = clock64();
  for (int i = 0; i < iters; i++) x += __syncthreads_or(x == 12345);
  long long t4 = clock64();
  if (threadIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t1; out[2] = t3 - t2; out[3] = t4 - t3; out[9] = x; }
}

__device__ unsigned int g_count;
__global__ void k_grid(long long *out, int iters) {
  long long t0 = clock64();
  unsigned epoch = 0;
  for (int i = 0; i < iters; i++) {
    __syncthreads();
    epoch++;
    if (threadIdx.x == 0) {
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(&g_count) : "memory");
      unsigned v;
      do { asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(&g_count) : "memory"); } while (v < epoch * gridDim.x);
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(&g_count) : "memory");
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (blockIdx.x == 0 && threadIdx.x == 0) out[4] = t1 - t0;
}

__global__ void k_cg(long long *out, int iters) {
  cg::grid_group g = cg::this_grid();
  long long t0 = clock64();
  for (int i = 0; i < iters; i++) g.sync();
  long long t1 = clock64();
  if (blockIdx.x == 0 && threadIdx.x == 0) out[5] = t1 - t0;
}

__global__ void __cluster_dims__(16, 1, 1) k_cluster(long long *out, int iters) {
  long long t0 = clock64();
  for (int i = 0; i < iters; i++) {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  }
  long long t1 = clock64();
  if (blockIdx.x == 0 && threadIdx.x == 0) out[6] = t1 - t0;
}

int main() {
  long long *d, h[10] = {0};
  cudaMalloc(&d, 80);
  cudaMemset(d, 0, 80);
  const int it = 1000;
  k_bar<<<1, 512>>>(d, it);
  cudaDeviceSynchronize();
  void *args[] = {&d, (void *)&it};
  int itv = it;
  void *args2[] = {&d, &itv};
  cudaLaunchCooperativeKernel((void *)k_grid, 144, 512, args2, 0, 0);
  cudaDeviceSynchronize();
  cudaLaunchCooperativeKernel((void *)k_cg, 144, 512, args2, 0, 0);
  cudaDeviceSynchronize();
  cudaFuncSetAttribute(k_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  int ncl = 0;
  {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(16 * 8); cfg.blockDim = dim3(512);
    cudaOccupancyMaxActiveClusters(&ncl, (void *)k_cluster, &cfg);
  }
  k_cluster<<<16 * (ncl > 0 ? ncl : 1), 512>>>(d, it);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(h, d, 80, cudaMemcpyDeviceToHost);
  printf("syncthreads(512 thr): %.1f cyc | dep LDS: %.1f cyc | globaltimer read: %.1f cyc | syncthreads_or: %.1f cyc\n",
         h[0] / (double)it, h[1] / (double)it, h[2] / (double)it, h[3] / (double)it);
  printf("grid barrier (144 CTA, red.release/ld.acquire): %.1f cyc | cg grid.sync: %.1f cyc | cluster16 barrier: %.1f cyc (max active 16-clusters %d, err %s)\n",
         h[4] / (double)it, h[5] / (double)it, h[6] / (double)it, ncl, cudaGetErrorString(e));
  int n8 = 0;
  {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(8 * 18); cfg.blockDim = dim3(512);
    cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = 8; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    cudaOccupancyMaxActiveClusters(&n8, (void *)k_bar, &cfg);
  }
  printf("max active 8-clusters (512 thr): %d\n", n8);
  return 0;
}
