// Microbenchmark of the cluster kernel's warp-per-unit contraction engine
// (csrc/warp_engine.cuh): cycles per tile of T nodes for the TreeLSTM leaf
// (3 gates on x) and level (U_iou h~ + U_f h_k, 2 children) products, 148
// CTAs x 512 threads, each tile followed by a lead-lane store and a
// __syncthreads as in the kernel. FMA floor per node: leaf 3*16*256/128 = 96
// cycles, level 5*16*256/128 = 160 cycles per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2011_01383_b200/csrc \
//        tools/micro/warp_engine_bench.cu -o /tmp/web && /tmp/web
#include <cstdio>
#include <cuda_runtime.h>

#include "warp_engine.cuh"

using namespace cx;
using namespace cx::wq;

template <class PH, int T, int ROWS, int UW>
__global__ void __launch_bounds__(512, 1) k_bench(long long *out, int iters, float *sink, const float *wsrc) {
  constexpr int H = 256, KC = 8;
  __shared__ __align__(16) float X[ROWS * H];
  __shared__ float res[16 * 32];
  __shared__ float xs[2][16 * 3 * 8 * 8];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const Roles<UW> ro(warp, lane);
  for (int i = tid; i < ROWS * H; i += 512) X[i] = 0.001f * (i % 97);
  WRegs<H> w;  // from global memory, as in the kernel (no constant folding)
  rw::Gate gs[4];
  for (int g = 0; g < 4; g++) gs[g] = {wsrc, g * 16, H, 0};
  load_wregs_w<4, H, UW>(w, gs, 4, ro.unit(), ro);
  __syncthreads();
  float accum = 0.f;
  long long t0 = clock64();
  for (int it = 0; it < iters; it++) {
    float r[PH::NA];
    // rotate the tile base so the loads cannot be hoisted out of the loop
    const bool act = contract_w<PH, H, T, UW>(X + (size_t)((it & 1) * PH::NV) * H, w, r, ro, xs[it & 1]);
    const int tn = node_of_lane<T, UW>(lane);
    if (act) {
      float s = 0.f;
#pragma unroll
      for (int a = 0; a < PH::NA; a++) s += r[a];
      res[ro.unit() * 32 + tn] = s;
    }
    __syncthreads();
    accum += res[(warp * 32 + it) & 511];
  }
  long long t1 = clock64();
  if (tid == 0) out[blockIdx.x] = t1 - t0;
  if (accum == 12345.f) sink[0] = accum;
}

template <class PH, int T, int UW>
void run(const char *name, double floor_per_node) {
  long long *d;
  float *sink;
  cudaMalloc(&d, 148 * 8);
  cudaMalloc(&sink, 4);
  float *wsrc;
  cudaMalloc(&wsrc, 64 * 256 * 4);
  cudaMemset(wsrc, 0, 64 * 256 * 4);
  const int iters = 2000;
  constexpr int ROWS = (T + 1) * PH::NV;
  k_bench<PH, T, ROWS, UW><<<148, 512>>>(d, 10, sink, wsrc);
  k_bench<PH, T, ROWS, UW><<<148, 512>>>(d, iters, sink, wsrc);
  cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  double m = 0;
  for (int i = 0; i < 148; i++) m += h[i];
  m /= 148.0 * iters;
  printf("%-10s UW=%d T=%2d  %7.0f cycles/tile  %6.0f cycles/node  floor %4.0f  eff %.2f  (%s)\n", name, UW, T, m,
         m / T, floor_per_node, floor_per_node * T / m, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  run<rw::RLstmLeaf, 1, 1>("leaf", 96);
  run<rw::RLstmLeaf, 8, 1>("leaf", 96);
  run<rw::RLstmLeaf, 1, 2>("leaf", 96);
  run<rw::RLstmLeaf, 4, 2>("leaf", 96);
  run<rw::RLstmLeaf, 8, 2>("leaf", 96);
  run<rw::RLstmLeaf, 8, 4>("leaf", 96);
  run<rw::RLstmLevel<2>, 1, 1>("level", 160);
  run<rw::RLstmLevel<2>, 4, 1>("level", 160);
  run<rw::RLstmLevel<2>, 1, 2>("level", 160);
  run<rw::RLstmLevel<2>, 2, 2>("level", 160);
  run<rw::RLstmLevel<2>, 4, 2>("level", 160);
  run<rw::RLstmLevel<2>, 1, 4>("level", 160);
  run<rw::RLstmLevel<2>, 4, 4>("level", 160);
  run<rw::RLstmLevel<2>, 8, 4>("level", 160);
  return 0;
}
