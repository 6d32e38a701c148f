// Cold vs warm cost of the single-CTA linearizer body (lin_single.cuh): the
// same CTA runs it three times back to back on a 10-grid (10x10) DAG and on a
// 390-node forest-like tree set; clock64 around each run. If the later runs
// are much faster, first-touch effects (instruction fetch, cold loads) and not
// the algorithm set the linearizer's time.
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>
#include "../../paper_2011_01383_b200/csrc/lin_single.cuh"

using namespace cx;

__global__ void run3(LinArgs a, long long *t) {
  extern __shared__ int sm[];
  for (int r = 0; r < 3; r++) {
    __syncthreads();
    long long t0 = clock64();
    LinOut o = lin_single_body(a, sm, 2048, r == 2, nullptr, LinPrefetch{});  // run 2 traced
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) { t[2 * r] = t1 - t0; t[2 * r + 1] = o.L; }
  }
}

int main() {
  for (int kind = 0; kind < 2; kind++) {
    int n, maxc = 2;
    std::vector<int> ch;
    if (kind == 0) {  // 10 grids 10x10: child slots [up, left]
      n = 1000;
      ch.assign(2 * n, -1);
      for (int g = 0; g < 10; g++)
        for (int i = 0; i < 10; i++)
          for (int j = 0; j < 10; j++) {
            int me = g * 100 + i * 10 + j, s = 0;
            if (i > 0) ch[s++ * n + me] = me - 10;
            if (j > 0) ch[s++ * n + me] = me - 1;
          }
    } else {  // 10 complete-ish binary trees of 39 nodes, pre-order ids
      n = 390;
      ch.assign(2 * n, -1);
      for (int g = 0; g < 10; g++)
        for (int v = 0; v < 39; v++) {
          int l = 2 * v + 1, r = 2 * v + 2;
          if (r < 39) { ch[g * 39 + v] = g * 39 + l; ch[n + g * 39 + v] = g * 39 + r; }
        }
    }
    int *d_ch, *bufs;
    cx_lin_header *hdr;
    cudaMalloc(&d_ch, 4 * ch.size());
    cudaMemcpy(d_ch, ch.data(), 4 * ch.size(), cudaMemcpyHostToDevice);
    cudaMalloc(&bufs, 4 * 16 * n);
    cudaMalloc(&hdr, sizeof(cx_lin_header));
    long long *d_t, h_t[6];
    cudaMalloc(&d_t, sizeof h_t);
    unsigned long long *d_tr, h_tr[32];
    cudaMalloc(&d_tr, sizeof h_tr);
    cudaMemset(d_tr, 0, sizeof h_tr);
    LinArgs a = {};
    a.ch = d_ch; a.n = n; a.maxc = maxc; a.kind = kind == 0 ? CX_DAG : CX_TREE; a.hdr = hdr;
    a.perm = bufs; a.inv = bufs + n; a.chn = bufs + 2 * n; a.hnew = bufs + 4 * n; a.lbeg = bufs + 5 * n;
    a.lsize = bufs + 6 * n; a.roots = bufs + 7 * n; a.sid = bufs + 8 * n; a.trace = d_tr;
    size_t smem = sizeof(int) * lin_sm_ints(n, maxc, 2048);
    cudaFuncSetAttribute(run3, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int rep = 0; rep < 2; rep++) {
      run3<<<1, 512, smem>>>(a, d_t);
      cudaMemcpy(h_t, d_t, sizeof h_t, cudaMemcpyDeviceToHost);
      printf("%s launch %d: cycles per run %lld %lld %lld (L = %lld)\n", kind == 0 ? "DAG 10x(10x10)" : "trees 10x39",
             rep, h_t[0], h_t[2], h_t[4], h_t[1]);
    }
    cudaMemcpy(h_tr, d_tr, sizeof h_tr, cudaMemcpyDeviceToHost);
    const char *nm[] = {"load+init+a1", "a2 heights", "a3 counts", "a3 scans", "a4 scatter", "a5+a6 remap, structures"};
    for (int k = 1; k <= 6; k++) printf("   warm %-26s %8lld cycles\n", nm[k - 1], (long long)(h_tr[16 + k] - h_tr[16 + k - 1]));
  }
  return 0;
}
