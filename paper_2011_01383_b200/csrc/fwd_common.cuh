// fwd_common.cuh -- device helpers shared by the forward kernel families
// (forward.cu: weights staged in shared memory; forward_rw.cu: weights
// resident in registers).
#pragma once
#include <cuda_runtime.h>

#include "common.cuh"
#include "fwd_kernels.cuh"

namespace cx {
namespace fwd {

constexpr int kMaxC = 4;  // largest max_children instantiated for child-sum cells

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

__device__ __forceinline__ void fma4(float &acc, const float4 &w, const float4 &v) {
  acc = fmaf(w.x, v.x, acc);
  acc = fmaf(w.y, v.y, acc);
  acc = fmaf(w.z, v.z, acc);
  acc = fmaf(w.w, v.w, acc);
}
__device__ __forceinline__ float4 add4(const float4 &a, const float4 &b) {
  return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
}

// contiguous chunk of [0, M) owned by node group g of Gn
__device__ __forceinline__ void chunk_of(int M, int Gn, int g, int &lo, int &hi) {
  int q = M / Gn, r = M % Gn;
  lo = g * q + min(g, r);
  hi = lo + q + (g < r ? 1 : 0);
}
__device__ __forceinline__ int owner_of(int pos, int M, int Gn) {
  int q = M / Gn, r = M % Gn, big = r * (q + 1);
  return pos < big ? pos / (q + 1) : r + (pos - big) / q;
}

template <int TM>
struct TileMetaT {
  int own[TM];          // input id of each node of the tile
  int cin[TM][kMaxC];   // input ids of children, -1 absent
  int nch[TM];          // present children
  int word[TM];         // clamped word id (phases that read Emb)
  int root[TM];         // index in roots[] if the node is a root, else -1
};

// Write h (column col) of tile node t to h_out, and to root_out when the node
// is a root (no separate pass over the roots).
template <class M>
__device__ __forceinline__ void put_h(const FwdArgs &a, const M &m, int t, int col, float v) {
  a.h_out[(size_t)m.own[t] * a.H + col] = v;
  if (a.root_out) {
    const int r = m.root[t];
    if (r >= 0) a.root_out[(size_t)r * a.H + col] = v;
  }
}

// Tile bookkeeping for nodes with new ids [i0, i0 + cnt): depends only on the
// linearization, so it can be loaded while the CTA waits at a barrier.
template <class M>
__device__ void load_meta(const FwdArgs &a, M &m, int i0, int cnt, bool want_children,
                          bool want_word, bool binary, bool latch) {
  const int t = threadIdx.x;
  if (t < cnt) {
    int i = i0 + t;
    int own = __ldg(a.perm + i);
    m.own[t] = own;
    if (a.root_out) {
      const int r = __ldg(a.sid + i);
      m.root[t] = __ldg(a.roots + r) == i ? r : -1;
    } else {
      m.root[t] = -1;
    }
    if (want_word) {
      int w = __ldg(a.words + own);
      if (w < 0 || w >= a.V) {
        if (latch) latch_error(a.hdr, CX_E_WORD_RANGE, own);
        w = 0;
      }
      m.word[t] = w;
    }
    if (want_children) {
      int nc = 0;
      for (int k = 0; k < a.maxc; k++) {
        int c = __ldg(a.chn + (size_t)k * a.n + i);
        if (c < 0) break;
        if (k < kMaxC) m.cin[t][k] = __ldg(a.perm + c);
        nc++;
      }
      for (int k = nc; k < kMaxC; k++) m.cin[t][k] = -1;
      if (binary && nc != 2) {
        if (latch) latch_error(a.hdr, CX_E_ARITY, own);
        if (nc < 2) m.cin[t][1] = m.cin[t][0];  // clamp for memory safety
        nc = 2;
      }
      m.nch[t] = nc;
    }
  }
}

// X[t][j][:] = row src(t, j) (H floats) or zeros, for t < cnt. The pieces are
// cp.async.cg copies (L2, no register round trip): every iteration's copy is
// in flight at once and the thread waits once at the end -- a loaded-value
// loop would pay one dependent L2/HBM round trip per iteration. The caller's
// __syncthreads publishes the rows to the CTA.
template <int NV, int H, class SRC>
__device__ __forceinline__ void gather_rows_c(float *X, int cnt, SRC src) {
  constexpr int q = H / 4;
  const int total = cnt * NV * q;
  for (int idx = threadIdx.x; idx < total; idx += blockDim.x) {
    int row = idx / q, c = idx - row * q;
    int t = row / NV, j = row - t * NV;
    const float *p = src(t, j);
    float *d = X + (size_t)row * H + 4 * c;
    if (p) cp_async16(d, p + 4 * c);
    else *reinterpret_cast<float4 *>(d) = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  cp_async_wait_all();
}

// Walk [lo, hi) in tiles of at most TMAX nodes; a tile of cnt nodes runs the
// smallest instantiation T in {1, 2, 4, ..., TMAX} with T >= cnt
// (warp-uniform branch).
template <int TMAX, class F>
__device__ __forceinline__ void for_tiles(int lo, int hi, F &f) {
  for (int i0 = lo; i0 < hi; i0 += TMAX) {
    int cnt = min(TMAX, hi - i0);
    if constexpr (TMAX >= 32) {
      if (cnt > 16) { f.template run<32>(i0, cnt); continue; }
    }
    if constexpr (TMAX >= 16) {
      if (cnt > 8) { f.template run<16>(i0, cnt); continue; }
    }
    if constexpr (TMAX >= 8) {
      if (cnt > 4) { f.template run<8>(i0, cnt); continue; }
    }
    if constexpr (TMAX >= 4) {
      if (cnt > 2) { f.template run<4>(i0, cnt); continue; }
    }
    if (cnt == 2) f.template run<2>(i0, cnt);
    else f.template run<1>(i0, cnt);
  }
}

// The last CTA out publishes the latched status and resets the barrier words.
__device__ __forceinline__ void publish_and_exit(const FwdArgs &a) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    unsigned prev = atomicAdd(&a.bar->exit, 1u);
    if (prev == gridDim.x - 1) {
      unsigned long long key = atomicAdd(reinterpret_cast<unsigned long long *>(&a.hdr->err_key), 0ull);
      if (key != kNoError) {
        a.hdr->status = (int)(key >> 32);
        a.hdr->bad_node = (int)(key & 0xffffffffu);
      }
      a.bar->count = 0;
      a.bar->exit = 0;
      a.bar->pad[2] = 0;  // the tensor-core kernel's DAG in-degree overflow flag
      __threadfence();
    }
  }
}

// Fused linearize + forward: data errors of the forward phase are latched into
// `ferr` (a workspace word, inverted key: 0 = none, atomicMax keeps the lowest
// key) because CTA 0 writes the header with plain stores while the other CTAs
// already run. The last CTA out -- after CTA 0's header stores, ordered by the
// exit counter -- merges it into the header and resets the words.
__device__ __forceinline__ void fused_exit(const FwdArgs &a, unsigned long long *ferr) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    unsigned prev = atomicAdd(&a.bar->exit, 1u);
    if (prev == gridDim.x - 1) {
      __threadfence();
      const unsigned long long f = atomicExch(ferr, 0ull);
      unsigned long long *hk = reinterpret_cast<unsigned long long *>(&a.hdr->err_key);
      if (f) atomicMin(hk, ~f);
      const unsigned long long key = atomicAdd(hk, 0ull);
      if (key != kNoError) {
        a.hdr->status = (int)(key >> 32);
        a.hdr->bad_node = (int)(key & 0xffffffffu);
        // (num_levels stays as the linearization wrote it: the header equals
        // the two separate calls', cx.h)
      }
      a.bar->count = 0;
      a.bar->exit = 0;
      a.bar->pad[2] = 0;  // the tensor-core kernel's DAG in-degree overflow flag
      __threadfence();
    }
  }
}

}  // namespace fwd
}  // namespace cx
