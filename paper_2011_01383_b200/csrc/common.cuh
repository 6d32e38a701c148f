// common.cuh -- device primitives shared by the linearizer and forward kernels.
//
// The paper's global barrier (draft P:514-521; GRNN comparison P:1535-1545)
// becomes a release/acquire counter barrier on B200: one red.release.gpu per
// CTA, one thread spinning on ld.acquire.gpu. Data written by other CTAs is
// read with ld.global.cg (L2) so no stale L1 line is ever used.
#pragma once
#include <cstdint>

#include "../../include/cx.h"

namespace cx {

constexpr uint64_t kNoError = ~0ull;

// Host: per-device slot for the lazily filled kernel-attribute caches
// (cudaFuncSetAttribute applies per device context). -1 when unavailable.
constexpr int kMaxDevices = 64;
inline int device_slot() {
  int dev = -1;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return -1;
  return dev;
}

// 128-byte aligned synchronisation words kept in the caller's workspace.
struct GridBar {
  unsigned int count;   // arrivals, monotonic within one launch
  unsigned int exit;    // blocks that left the kernel
  unsigned int pad[30];
};

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned *p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_add_u32(unsigned *p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ unsigned ld_relaxed_u32(const unsigned *p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Grid-wide barrier for a co-resident (cooperatively launched) grid, split in
// two halves so a CTA can prefetch data that does not depend on the level
// being completed while it waits. `epoch` counts barriers passed so far.
// Arrive: bar.sync orders the CTA's writes before thread 0's red.release.gpu.
// Wait: thread 0 polls with relaxed loads and finishes with one ld.acquire.gpu;
// the trailing bar.sync publishes the acquire to the whole CTA. Data written
// by other CTAs is then read with ld.global.cg (L2), never a stale L1 line.
__device__ __forceinline__ void grid_arrive(GridBar *bar, unsigned &epoch) {
  __syncthreads();
  epoch += 1;
  if (threadIdx.x == 0) red_release_add_u32(&bar->count, 1u);
}
__device__ __forceinline__ void grid_wait(GridBar *bar, unsigned nblocks, unsigned epoch) {
  if (threadIdx.x == 0) {
    const unsigned target = epoch * nblocks;
    // watchdog: a grid that is not co-resident would spin forever; trap
    // (sticky launch error, reported as CX_E_CUDA) instead of hanging
    unsigned long long spins = 0;
    while (ld_relaxed_u32(&bar->count) < target) {
      if (++spins > (1ull << 26)) __trap();
    }
    (void)ld_acquire_u32(&bar->count);
  }
  __syncthreads();
}
__device__ __forceinline__ void grid_sync(GridBar *bar, unsigned nblocks, unsigned &epoch) {
  grid_arrive(bar, epoch);
  grid_wait(bar, nblocks, epoch);
}

// Called once by every CTA at kernel end: the last CTA out resets the words
// so the workspace is reusable without a memset (all CTAs have passed all
// barriers by the time the exit count is complete).
__device__ __forceinline__ void grid_exit(GridBar *bar, unsigned nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    unsigned prev = atomicAdd(&bar->exit, 1u);
    if (prev == nblocks - 1) {
      bar->count = 0;
      bar->exit = 0;
      __threadfence();
    }
  }
}

// Programmatic dependent launch (PDL): cx_linearize lets the dependent
// cx_forward grid start early; the forward stages its weights, then waits for
// the linearization (and its memory) before reading it. Without a PDL edge
// (standalone launch) the wait returns immediately.
__device__ __forceinline__ void griddep_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void griddep_wait() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

// Latch a data error: lowest (code, node) wins.
__device__ __forceinline__ void latch_error(cx_lin_header *h, int code, int node) {
  unsigned long long key = ((unsigned long long)(unsigned)code << 32) | (unsigned)node;
  atomicMin(reinterpret_cast<unsigned long long *>(&h->err_key), key);
}

__device__ __forceinline__ float4 ldcg4(const float *p) {
  return __ldcg(reinterpret_cast<const float4 *>(p));
}
__device__ __forceinline__ int ldcg_i(const int *p) { return __ldcg(p); }

// Gate nonlinearities on the MUFU pipe (ex2 + rcp): sigma(x) = 1 / (1 + e^-x),
// tanh(x) = (e^2x - 1) / (e^2x + 1) with |x| clamped at 15 (tanh(15) rounds to
// 1 in fp32). __expf's error is <= 2 + 1.16|x| ulp; over the clamp range the
// result stays within ~5e-6 relative (absolute near 0), far inside the fp32
// path's 1e-4 tolerance (Q10).
__device__ __forceinline__ float sigmoidf_(float x) { return __fdividef(1.0f, 1.0f + __expf(-x)); }
__device__ __forceinline__ float tanhf_(float x) {
  x = fminf(fmaxf(x, -15.f), 15.f);
  float e = __expf(2.f * x);
  return __fdividef(e - 1.f, e + 1.f);
}

// ---- cluster dataflow primitives (forward_cluster.cu push mode) ------------
// A producer writes a row piece straight into a consumer CTA's shared memory
// with st.async; each store signals the consumer's mbarrier with its byte
// count (complete_tx, release at cluster scope). The consumer posts the bytes
// it expects once (arrive.expect_tx) and waits with acquire at cluster scope:
// no fence and no cluster-wide barrier on the level-to-level path.
__device__ __forceinline__ unsigned smem_addr(const void *p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long *m, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(m)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init_cluster() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long *m, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;"
               ::"r"(smem_addr(m)), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait_cluster(unsigned long long *m, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_addr(m)), "r"(parity)
      : "memory");
  return ok != 0;
}
// shared::cluster address of the local shared-memory address `a` in CTA `rank`
__device__ __forceinline__ unsigned mapa_rank(unsigned a, unsigned rank) {
  unsigned r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_async_v4(unsigned dst, const float4 &v, unsigned mbar) {
  asm volatile(
      "st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1, %2, %3, %4}, [%5];"
      ::"r"(dst), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "r"(mbar)
      : "memory");
}
__device__ __forceinline__ unsigned dynamic_smem_bytes() {
  unsigned r;
  asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(r));
  return r;
}

// packed fp32x2 FMA (sm_100: FFMA2): d = a * b + c element-wise
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  float2 d;
  asm("{\n\t.reg .b64 ra, rb, rc, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\tmov.b64 rc, {%6, %7};\n\t"
      "fma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return d;
}

}  // namespace cx
