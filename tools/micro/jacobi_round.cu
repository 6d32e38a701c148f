// Cycles per Jacobi height round in one 512-thread CTA (10 grid DAGs of
// 10x10, n = 1000): variants of the round body.
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>

template <int V>
__global__ void rounds(const int *gch, int n, int maxc, long long *out) {
  extern __shared__ int sm[];
  int *ch = sm, *hgt = sm + maxc * n;
  const int tid = threadIdx.x, nthr = blockDim.x;
  for (int i = tid; i < maxc * n; i += nthr) ch[i] = gch[i];
  for (int v = tid; v < n; v += nthr) hgt[v] = ch[v] == -1 ? 0 : -1;
  __syncthreads();
  long long t0 = clock64();
  int r = 0;
  bool progress = true;
  while (progress) {
    r++;
    bool any = false;
    if (V == 0) {
#pragma unroll 1
      for (int v = tid; v < n; v += nthr) {
        if (hgt[v] >= 0) continue;
        bool ok = true;
#pragma unroll 1
        for (int k = 0; k < maxc; k++) {
          int c = ch[k * n + v];
          if (c == -1) break;
          int hc = hgt[c];
          if (hc < 0 || hc >= r) { ok = false; break; }
        }
        if (ok) { hgt[v] = r; any = true; }
      }
    } else if (V == 1) {  // branch-free children check, maxc == 2
      for (int v = tid; v < n; v += nthr) {
        const int h = hgt[v];
        const int c0 = ch[v], c1 = ch[n + v];
        const int h0 = c0 >= 0 ? hgt[c0] : 0, h1 = c1 >= 0 ? hgt[c1] : 0;
        const bool ok = h < 0 && h0 >= 0 && h0 < r && h1 >= 0 && h1 < r;
        if (ok) { hgt[v] = r; any = true; }
      }
    } else {  // V == 2: same, volatile-free plus __syncthreads + flag
      for (int v = tid; v < n; v += nthr) {
        const int h = hgt[v];
        const int c0 = ch[v], c1 = ch[n + v];
        const int h0 = c0 >= 0 ? hgt[c0] : 0, h1 = c1 >= 0 ? hgt[c1] : 0;
        if (h < 0 && h0 >= 0 && h0 < r && h1 >= 0 && h1 < r) { hgt[v] = r; any = true; }
      }
    }
    progress = __syncthreads_or(any);
  }
  long long t1 = clock64();
  if (tid == 0) { out[0] = t1 - t0; out[1] = r; }
}

int main() {
  const int n = 1000, maxc = 2;
  std::vector<int> ch(2 * n, -1);
  for (int g = 0; g < 10; g++)
    for (int i = 0; i < 10; i++)
      for (int j = 0; j < 10; j++) {
        int me = g * 100 + i * 10 + j, s = 0;
        if (i > 0) ch[s++ * n + me] = me - 10;
        if (j > 0) ch[s++ * n + me] = me - 1;
      }
  int *d;
  long long *o, h[2];
  cudaMalloc(&d, 8 * n);
  cudaMalloc(&o, 16);
  cudaMemcpy(d, ch.data(), 8 * n, cudaMemcpyHostToDevice);
  for (int rep = 0; rep < 2; rep++) {
    rounds<0><<<1, 512, 12 * n>>>(d, n, maxc, o); cudaMemcpy(h, o, 16, cudaMemcpyDeviceToHost);
    printf("V0 (lin_single loop)   %lld cycles, %lld rounds, %.0f / round\n", h[0], h[1], (double)h[0] / h[1]);
    rounds<1><<<1, 512, 12 * n>>>(d, n, maxc, o); cudaMemcpy(h, o, 16, cudaMemcpyDeviceToHost);
    printf("V1 (branch-free)       %lld cycles, %lld rounds, %.0f / round\n", h[0], h[1], (double)h[0] / h[1]);
    rounds<1><<<1, 1024, 12 * n>>>(d, n, maxc, o); cudaMemcpy(h, o, 16, cudaMemcpyDeviceToHost);
    printf("V1 1024 threads        %lld cycles, %lld rounds, %.0f / round\n", h[0], h[1], (double)h[0] / h[1]);
  }
  return 0;
}
