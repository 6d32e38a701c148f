// lin_kernels.cuh -- internal interface between api.cu and linearize.cu.
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#include "common.cuh"

namespace cx {

// shared-memory budget of the single-CTA linearizer (int entries / bytes)
constexpr int kLinSmemCnt = 8192;              // per-(level, segment) count table
constexpr size_t kLinSmemMax = 200 * 1024;     // heights + in-degree + children copy + table

struct LinArgs {
  const int32_t *ch;  // [maxc][n] input ids
  int n, maxc, kind;
  cx_lin_header *hdr;
  int32_t *perm, *inv, *chn, *hnew, *lbeg, *lsize, *roots, *sid;
  // workspace
  GridBar *bar;
  int32_t *misc;   // 32 ints
  int32_t *indeg;  // n
  int32_t *hgt;    // n
  int32_t *cnt;    // budget
  int budget;
  unsigned long long *trace;  // debug: %globaltimer per phase (CTA 0), NULL = off
  int hjacobi;  // single-CTA path: Jacobi rounds for trees too (CX_LIN_JACOBI=1, measurement)
};

// debug timeline (trace build only, see trace_mark in fwd_kernels.cuh)
__device__ __forceinline__ void lin_mark(const LinArgs &a, int s) {
#ifdef CX_TRACE
  if (a.trace && threadIdx.x == 0 && blockIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.trace[s] = t;
    a.trace[16 + s] = clock64();
  }
#else
  (void)a;
  (void)s;
#endif
}

// multi-CTA path: parent pointers [n] + per-block level-count table
inline size_t lin_budget_entries(int n) { return 2 * (size_t)n + 40960; }

inline size_t lin_workspace_bytes(int n) {
  return sizeof(GridBar) + 32 * sizeof(int32_t) + sizeof(int32_t) * (2 * (size_t)n) +
         sizeof(int32_t) * lin_budget_entries(n) + 256;
}

bool lin_use_single(int n, int maxc);
size_t lin_single_smem_bytes(int n, int maxc);
cudaError_t launch_linearize(const LinArgs &a, int num_sms, cudaStream_t stream);
cudaError_t launch_empty(int ctas, int threads, int coop, unsigned long long *t, cudaStream_t stream);

}  // namespace cx
