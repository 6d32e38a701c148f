// diag.cu -- measurement kernels behind cx_diag_sync_cycles (include/cx.h):
// the per-level synchronisation and dependent-arithmetic costs that make up
// the critical-path bound of SURVEY.md §8(d),
//   T_cp = t_launch + (L - 1) t_sync + L t_chain,
// measured in the same process and on the same device as the bench (the
// paper's own accounting of barrier cost per batch: App. A.4 P:2010-2040;
// "the cost of a barrier cannot be amortized").
//
// kind 0  push hand-off (the cluster kernel's level-to-level path): in a
//         16-CTA cluster every CTA sends a 64-byte slice to every CTA
//         (st.async + mbarrier complete_tx) and waits for the 16 slices of the
//         next level on its mbarrier.
// kind 1  barrier.cluster arrive.release / wait.acquire (16-CTA cluster).
// kind 2  grid barrier: release add + acquire poll on a global counter, one
//         CTA per SM (co-resident, cooperative launch).
// kind 3  the dependent arithmetic of one level for one node on one warp, the
//         shortest chain any implementation of a level needs at H = 256 with a
//         warp-wide dot product: shared-memory load -> 4 dependent FFMA2
//         (8 k per lane) -> 5 shuffle-add steps (32 lanes) -> sigma and tanh
//         (MUFU ex2 + rcp each) -> shared-memory store feeding the next level.
// out[0] = cycles per level (CTA 0, clock64), out[1] = levels timed.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include "common.cuh"

namespace cx {
namespace {

constexpr int kDiagCluster = 16;

__global__ void __cluster_dims__(kDiagCluster, 1, 1) diag_push(unsigned long long *out, int levels) {
  __shared__ __align__(16) float rows[2][kDiagCluster * 16];
  __shared__ __align__(8) unsigned long long mb[2];
  const int tid = threadIdx.x;
  if (tid < 2) mbar_init(&mb[tid], 1);
  fence_mbar_init_cluster();
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  unsigned crank;
  asm("mov.u32 %0, %%cluster_ctarank;" : "=r"(crank));
  const long long t0 = clock64();
  for (int l = 0; l < levels; l++) {
    const int b = l & 1;
    if (tid == 0) mbar_expect_tx(&mb[b], kDiagCluster * 64u);
    // lane hu < 16 of warp 0 sends this CTA's 64-byte slice to CTA hu
    if (tid < kDiagCluster) {
      const unsigned dst = mapa_rank(smem_addr(&rows[b][crank * 16]), (unsigned)tid);
      const unsigned bar = mapa_rank(smem_addr(&mb[b]), (unsigned)tid);
      const float4 v = make_float4((float)l, 1.f, 2.f, 3.f);
#pragma unroll
      for (int q = 0; q < 4; q++) st_async_v4(dst + 16u * q, v, bar);
    }
    while (!mbar_try_wait_cluster(&mb[b], (unsigned)((l >> 1) & 1))) {
    }
    __syncthreads();  // the level's consumers (all warps) may proceed
  }
  const long long t1 = clock64();
  if (tid == 0 && blockIdx.x == 0) {
    out[0] = (unsigned long long)((t1 - t0) / levels);
    out[1] = (unsigned long long)levels;
  }
  // nobody may exit while a peer can still write into its shared memory
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__global__ void __cluster_dims__(kDiagCluster, 1, 1) diag_cluster_bar(unsigned long long *out, int levels) {
  const long long t0 = clock64();
  for (int l = 0; l < levels; l++)
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  const long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    out[0] = (unsigned long long)((t1 - t0) / levels);
    out[1] = (unsigned long long)levels;
  }
}

__global__ void diag_grid_bar(unsigned long long *out, int levels, GridBar *bar) {
  unsigned epoch = 0;
  const long long t0 = clock64();
  for (int l = 0; l < levels; l++) grid_sync(bar, gridDim.x, epoch);
  const long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    out[0] = (unsigned long long)((t1 - t0) / levels);
    out[1] = (unsigned long long)levels;
  }
  grid_exit(bar, gridDim.x);
}

__global__ void diag_chain(unsigned long long *out, int levels) {
  __shared__ __align__(16) float buf[32 * 8 + 32];
  const int lane = threadIdx.x & 31;
  for (int i = lane; i < 32 * 8 + 32; i += 32) buf[i] = 0.001f * i;
  __syncwarp();
  float w[8];
#pragma unroll
  for (int j = 0; j < 8; j++) w[j] = 0.01f * (j + 1) + 1e-4f * lane;
  int idx = lane * 8;
  const long long t0 = clock64();
  for (int l = 0; l < levels; l++) {
    const float4 a = *reinterpret_cast<const float4 *>(&buf[idx & ~3]);
    const float4 b = *reinterpret_cast<const float4 *>(&buf[(idx & ~3) + 4]);
    float2 acc = make_float2(0.f, 0.f);
    acc = ffma2(make_float2(w[0], w[1]), make_float2(a.x, a.y), acc);
    acc = ffma2(make_float2(w[2], w[3]), make_float2(a.z, a.w), acc);
    acc = ffma2(make_float2(w[4], w[5]), make_float2(b.x, b.y), acc);
    acc = ffma2(make_float2(w[6], w[7]), make_float2(b.z, b.w), acc);
    float s = acc.x + acc.y;
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    const float h = sigmoidf_(s) * tanhf_(s);
    buf[256 + lane] = h;
    __syncwarp();
    idx = (lane * 8 + (__float_as_int(buf[256 + (lane ^ 1)]) & 8)) & 255;  // depends on h
  }
  const long long t1 = clock64();
  if (lane == 0 && blockIdx.x == 0) {
    out[0] = (unsigned long long)((t1 - t0) / levels);
    out[1] = (unsigned long long)levels;
  }
}

}  // namespace
}  // namespace cx

extern "C" cx_status cx_diag_sync_cycles(int32_t kind, int32_t levels, unsigned long long *out,
                                          void *workspace, void *stream) {
  using namespace cx;
  if (!out || levels < 1 || kind < 0 || kind > 3) return CX_E_ARG;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e = cudaSuccess;
  switch (kind) {
    case 0:
      cudaFuncSetAttribute(diag_push, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      diag_push<<<kDiagCluster, 512, 0, s>>>(out, levels);
      e = cudaGetLastError();
      break;
    case 1:
      cudaFuncSetAttribute(diag_cluster_bar, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      diag_cluster_bar<<<kDiagCluster, 512, 0, s>>>(out, levels);
      e = cudaGetLastError();
      break;
    case 2: {
      if (!workspace) return CX_E_ARG;
      int dev = 0, sms = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      GridBar *bar = static_cast<GridBar *>(workspace);
      void *params[] = {&out, &levels, &bar};
      e = cudaLaunchCooperativeKernel((const void *)diag_grid_bar, sms, 512, params, 0, s);
      break;
    }
    case 3:
      diag_chain<<<1, 32, 0, s>>>(out, levels);
      e = cudaGetLastError();
      break;
  }
  return e == cudaSuccess ? CX_OK : CX_E_CUDA;
}
