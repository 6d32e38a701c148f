// Cost of one "Jacobi round" (3 dependent LDS + __syncthreads_or) in a single
// 512-thread CTA, and of one walk-up step (atomics + fences), in cycles.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void rounds(int R, int mode, long long *out) {
  __shared__ int s[1024];
  __shared__ int pend[1024];
  const int tid = threadIdx.x;
  for (int i = tid; i < 1024; i += blockDim.x) { s[i] = (i * 7 + 3) & 1023; pend[i] = 1 << 20; }
  __syncthreads();
  long long t0 = clock64();
  int acc = 0;
  if (mode == 0) {
    for (int r = 0; r < R; r++) {
      int x = s[tid];
      int y = s[x];
      int z = s[y];
      if (z == r) s[tid] = z;
      acc += __syncthreads_or(z > 5000);
    }
  } else if (mode == 1) {  // walk-up step: atomicMax, fence, atomicSub, fence, atomicAdd read
    int cur = tid;
    for (int r = 0; r < R; r++) {
      int p = s[cur];
      atomicMax(&s[p], r);
      __threadfence_block();
      acc += atomicSub(&pend[p], 1);
      __threadfence_block();
      cur = atomicAdd(&s[p], 0) & 1023;
    }
  } else if (mode == 2) {  // same without fences
    int cur = tid;
    for (int r = 0; r < R; r++) {
      int p = s[cur];
      atomicMax(&s[p], r);
      acc += atomicSub(&pend[p], 1);
      cur = atomicAdd(&s[p], 0) & 1023;
    }
  } else {  // plain __syncthreads rounds
    for (int r = 0; r < R; r++) { acc += s[(tid + r) & 1023]; __syncthreads(); }
  }
  long long t1 = clock64();
  if (tid == 0) { out[0] = t1 - t0; out[1] = acc; }
}

int main() {
  long long *d, h[2];
  cudaMalloc(&d, 16);
  const char *names[] = {"jacobi round (3 LDS + bar.red.or)", "walk step (atom+fence)", "walk step (no fence)", "bar.sync round"};
  for (int mode = 0; mode < 4; mode++)
    for (int threads : {32, 512})
      for (int R : {1, 10, 100}) {
        rounds<<<1, threads>>>(R, mode, d);
        rounds<<<1, threads>>>(R, mode, d);
        cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
        printf("%-36s threads %3d R %4d: %8lld cycles  (%.0f / round)\n", names[mode], threads, R, h[0], (double)h[0] / R);
      }
  return 0;
}
