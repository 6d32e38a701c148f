// forward.cu -- the persistent forward kernel.
//
// What Cortex generates (Listing 2, App. A.4):
//   for n in leaf_batch:           rnn[n] = leaf_case(n)          (specialised)
//   for b in internal_batches:     barrier                        (batch loop carries the dependence)
//     for n in batch:              rnn[n] = recursive_case(n, rnn[children(n)])
// as ONE kernel launch with the weights persisted on chip.
//
// B200 design:
//   * grid = Gn node groups x Gu unit groups, one 256-thread CTA per SM,
//     cooperatively launched so a release/acquire grid barrier is legal;
//   * CTA (gn, gu) owns hidden units [32 gu, 32 gu + 32) of every gate: the
//     recurrent weight rows of those units stay resident in shared memory
//     for the whole level loop (leaf-phase weights are staged first and then
//     replaced while the CTA waits at the first barrier);
//   * each level is split into contiguous chunks, one per node group; a
//     chunk is processed in tiles of T <= 8 nodes: the tile's child rows are
//     gathered (whole H-vectors, float4, L2) into shared memory -- the
//     paper's dense per-iteration cache rnn_cache[b, n, i, k];
//   * lane = hidden unit, the 8 warps split the contraction dimension; a
//     product table per cell phase says which weight gate multiplies which
//     gathered vector (children h_k, or their child-sum h~, or the leaf x);
//   * partial sums are reduced through shared memory and the gate algebra is
//     fused into the epilogue, which writes h (and c / z / s) of the owned
//     units straight into the caller's INPUT-numbered h_out.
// fp32 throughout: FMA on CUDA cores (the 1e-4 bound rules out TF32/bf16
// tensor cores for this path; the bf16 tensor-core path is separate).
#include <cuda_runtime.h>

#include <cstdlib>

#include "common.cuh"
#include "fwd_common.cuh"
#include "fwd_kernels.cuh"
#include "smem_engine.cuh"

namespace cx {
namespace {
using namespace sme;

constexpr int kWarps = kFwdThreads / 32;
constexpr int kMaxC = 4;

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

// ---------------------------------------------------------------------------
// Per-cell shape traits, shared by host (smem sizing) and device.
// NG: resident weight gates; NV: gathered vectors per node; NA: accumulators
// per node; TMAX: node tile.
// ---------------------------------------------------------------------------
template <int CELL, int MAXC>
struct Traits;
template <int MAXC>
struct Traits<CX_TREELSTM, MAXC> {
  static constexpr int NG = 4, NV = MAXC, NA = 3 + MAXC, TMAX = 8;
};
template <int MAXC>
struct Traits<CX_TREEGRU, MAXC> {
  static constexpr int NG = 3, NV = MAXC, NA = 1 + MAXC, TMAX = 4;
};
template <int MAXC>
struct Traits<CX_TREEFC, MAXC> {
  static constexpr int NG = 2, NV = 2, NA = 1, TMAX = 8;
};
template <int MAXC>
struct Traits<CX_DAGRNN, MAXC> {
  static constexpr int NG = 1, NV = MAXC, NA = 1, TMAX = 8;
};
template <int MAXC>
struct Traits<CX_TREERNN, MAXC> {
  static constexpr int NG = 0, NV = 0, NA = 0, TMAX = 8;
};

template <int CELL, int MAXC>
struct Layout {
  using Tr = Traits<CELL, MAXC>;
  // float offsets into dynamic shared memory
  static __host__ __device__ size_t w_floats(int H) { return (size_t)Tr::NG * kUG * (H + 4); }
  static __host__ __device__ size_t x_floats(int H) {
    size_t xs = (size_t)Tr::TMAX * (Tr::NV > 0 ? Tr::NV : 1) * H;
    size_t rs = (size_t)kWarps * Tr::NA * Tr::TMAX * 32;
    return xs > rs ? xs : rs;
  }
  static __host__ __device__ size_t cv_floats() { return (size_t)Tr::TMAX * kMaxC * 32; }
  static __host__ __device__ size_t bytes(int H) {
    if (Tr::NG == 0) return 0;
    return sizeof(float) * (w_floats(H) + x_floats(H) + cv_floats());
  }
};

using TileMeta = fwd::TileMetaT<8>;

struct GateSrc {
  const float *base;
  int r0, ld, c0;
};

// Stage rows (units unit0..unit0+31) of NG gates into Ws with cp.async:
// warp w copies rows w, w+8, ..., lanes stride over the row's 16-byte chunks.
__device__ void load_gates(float *Ws, const GateSrc *gs, int NG, int unit0, int H) {
  const int HP = H + 4, q = H >> 2;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int row = warp; row < NG * kUG; row += kWarps) {
    const int g = row >> 5, u = row & 31;
    const float *src = gs[g].base + (size_t)(gs[g].r0 + unit0 + u) * gs[g].ld + gs[g].c0;
    float *dst = Ws + (size_t)row * HP;
    for (int c = lane; c < q; c += 32) cp_async16(dst + 4 * c, src + 4 * c);
  }
  cp_async_commit();
}

using fwd::load_meta;
using fwd::put_h;

// X[t][j][:] = row src(t, j) (H floats) or zeros; rows of t >= cnt untouched.
template <class SRC>
__device__ __forceinline__ void gather_rows(float *X, int NV, int H, int cnt, SRC src) {
  const int q = H >> 2, total = cnt * NV * q;
  for (int idx = threadIdx.x; idx < total; idx += blockDim.x) {
    int row = idx / q, c = idx - row * q;
    int t = row / NV, j = row - t * NV;
    const float *p = src(t, j);
    float4 v = p ? ldcg4(p + 4 * c) : make_float4(0.f, 0.f, 0.f, 0.f);
    *reinterpret_cast<float4 *>(X + (size_t)row * H + 4 * c) = v;
  }
}

// Walk [lo, hi) in tiles of at most TMAX nodes; a tile of cnt nodes runs the
// smallest instantiation T in {1, 2, 4, 8} with T >= cnt (warp-uniform branch).
template <int TMAX, class F>
__device__ __forceinline__ void tiles_T(int lo, int hi, F &f) {
  for (int i0 = lo; i0 < hi; i0 += TMAX) {
    int cnt = min(TMAX, hi - i0);
    if constexpr (TMAX >= 8) {
      if (cnt > 4) {
        f.template run<8>(i0, cnt);
        continue;
      }
    }
    if (cnt > 2) f.template run<4>(i0, cnt);
    else if (cnt == 2) f.template run<2>(i0, cnt);
    else f.template run<1>(i0, cnt);
  }
}

// ---------------------------------------------------------------------------
// Cell bodies. Each provides leaf_range(), leaf weights, level weights,
// phases per level, and the tile functors.
// ---------------------------------------------------------------------------
struct Ctx {
  const FwdArgs *a;
  float *Ws, *X, *cv;
  const float *bias;  // shared memory [gate][32]: biases of the owned units
  TileMeta *m;
  int gn, gu, unit0, H;
  bool latch;  // only unit group 0 latches data errors (avoid duplicate atomics)
  int tslot;   // debug trace: first trace slot of this level's first tile, -1 = off
};

// ----- TreeLSTM (Q1: child-sum, [Tai et al.]) -------------------------------
template <int MAXC>
struct TreeLstm {
  static constexpr int kPhases = 1;
  struct Leaf {
    Ctx c;
    int pre;
    __device__ void meta(int i0, int cnt) { load_meta(*c.a, *c.m, i0, cnt, false, true, false, c.latch); }
    template <int T>
    __device__ void run(int i0, int cnt) {
      const FwdArgs &a = *c.a;
      const int H = c.H;
      if (i0 != pre) {
        meta(i0, cnt);
        __syncthreads();
      }
      gather_rows(c.X, 1, H, cnt, [&](int t, int) { return a.emb + (size_t)c.m->word[t] * H; });
      cp_async_wait_all();  // leaf weights (staged asynchronously at kernel start)
      __syncthreads();
      float acc[3][T], s[3];
      fma_engine<PhLstmLeaf, T>(c.Ws, c.X, H, acc);
      reduce_acc<3, T>(c.X, acc, s);
      const int lane = threadIdx.x & 31;
      const int t = threadIdx.x >> 5, unit = c.unit0 + lane;
      if (t < cnt) {
        float ig = s[0] + c.bias[0 * 32 + lane], og = s[1] + c.bias[1 * 32 + lane],
              ug = s[2] + c.bias[2 * 32 + lane];
        float cc = sigmoidf_(ig) * tanhf_(ug);
        float hh = sigmoidf_(og) * tanhf_(cc);
        size_t o = (size_t)c.m->own[t] * H + unit;
        put_h(a, *c.m, t, unit, hh);
        a.cbuf[o] = cc;
      }
      __syncthreads();
    }
  };
  struct Level {
    Ctx c;
    int phase, pre;
    __device__ void meta(int i0, int cnt) { load_meta(*c.a, *c.m, i0, cnt, true, false, false, c.latch); }
    template <int T>
    __device__ void run(int i0, int cnt) {
      const FwdArgs &a = *c.a;
      const int H = c.H;
      const int lane = threadIdx.x & 31;
      if (i0 != pre) {
        meta(i0, cnt);
        __syncthreads();
      }
      if (c.tslot >= 0) trace_mark(a, c.tslot);
      gather_rows(c.X, MAXC, H, cnt, [&](int t, int j) {
        int ci = c.m->cin[t][j];
        return ci >= 0 ? a.h_out + (size_t)ci * H : (const float *)nullptr;
      });
      // children's memory cells for the owned units
      for (int idx = threadIdx.x; idx < cnt * MAXC * 32; idx += blockDim.x) {
        int t = idx / (MAXC * 32), r = idx - t * MAXC * 32, k = r >> 5, u = r & 31;
        int ci = c.m->cin[t][k];
        c.cv[(t * kMaxC + k) * 32 + u] = ci >= 0 ? __ldcg(a.cbuf + (size_t)ci * H + c.unit0 + u) : 0.f;
      }
      __syncthreads();
      if (c.tslot >= 0) trace_mark(a, c.tslot + 1);
      float acc[3 + MAXC][T], s[3 + MAXC];
      fma_engine<PhLstmLevel<MAXC>, T>(c.Ws, c.X, H, acc);
      if (c.tslot >= 0) trace_mark(a, c.tslot + 2);
      reduce_acc<3 + MAXC, T>(c.X, acc, s);
      if (c.tslot >= 0) trace_mark(a, c.tslot + 3);
      const int t = threadIdx.x >> 5, unit = c.unit0 + lane;
      if (t < cnt) {
        float ig = s[0] + c.bias[0 * 32 + lane], og = s[1] + c.bias[1 * 32 + lane],
              ug = s[2] + c.bias[2 * 32 + lane], bfu = c.bias[3 * 32 + lane];
        float cc = sigmoidf_(ig) * tanhf_(ug);
        const int nc = c.m->nch[t];
#pragma unroll
        for (int k = 0; k < MAXC; k++)
          if (k < nc) cc += sigmoidf_(s[3 + k] + bfu) * c.cv[(t * kMaxC + k) * 32 + lane];
        float hh = sigmoidf_(og) * tanhf_(cc);
        size_t o = (size_t)c.m->own[t] * H + unit;
        put_h(a, *c.m, t, unit, hh);
        a.cbuf[o] = cc;
      }
      __syncthreads();
      if (c.tslot >= 0) trace_mark(a, c.tslot + 4);
      c.tslot = -1;
    }
  };
  // biases [gate][unit]: b_i, b_o, b_u, b_f
  __device__ static int biases(const FwdArgs &a, const float **b, int *off) {
    b[0] = b[1] = b[2] = a.w[2];
    off[0] = 0; off[1] = a.H; off[2] = 2 * a.H;
    b[3] = a.w[4]; off[3] = 0;
    return 4;
  }
  __device__ static int leaf_lo(const FwdArgs &, int first_leaf) { return first_leaf; }
  __device__ static int leaf_gates(const FwdArgs &a, GateSrc *gs) {
    const int H = a.H;
    gs[0] = {a.w[0], 0, H, 0};
    gs[1] = {a.w[0], H, H, 0};
    gs[2] = {a.w[0], 2 * H, H, 0};
    return 3;
  }
  __device__ static int level_gates(const FwdArgs &a, GateSrc *gs) {
    const int H = a.H;
    gs[0] = {a.w[1], 0, H, 0};
    gs[1] = {a.w[1], H, H, 0};
    gs[2] = {a.w[1], 2 * H, H, 0};
    gs[3] = {a.w[3], 0, H, 0};
    return 4;
  }
};

// ----- TreeGRU (Q3: child-sum, reset gate per child before U_h) -------------
template <int MAXC>
struct TreeGru {
  static constexpr int kPhases = 2;
  struct Leaf {
    Ctx c;
    int pre;
    __device__ void meta(int i0, int cnt) { load_meta(*c.a, *c.m, i0, cnt, false, true, false, c.latch); }
    template <int T>
    __device__ void run(int i0, int cnt) {
      const FwdArgs &a = *c.a;
      const int H = c.H;
      if (i0 != pre) {
        meta(i0, cnt);
        __syncthreads();
      }
      gather_rows(c.X, 1, H, cnt, [&](int t, int) { return a.emb + (size_t)c.m->word[t] * H; });
      cp_async_wait_all();
      __syncthreads();
      float acc[2][T], s[2];
      fma_engine<PhGruLeaf, T>(c.Ws, c.X, H, acc);
      reduce_acc<2, T>(c.X, acc, s);
      const int lane = threadIdx.x & 31;
      const int t = threadIdx.x >> 5, unit = c.unit0 + lane;
      if (t < cnt) {
        float z = sigmoidf_(s[0] + c.bias[0 * 32 + lane]);
        float g = tanhf_(s[1] + c.bias[2 * 32 + lane]);
        put_h(a, *c.m, t, unit, (1.f - z) * g);
      }
      __syncthreads();
    }
  };
  struct Level {
    Ctx c;
    int phase, pre;
    __device__ void meta(int i0, int cnt) {
      if (phase == 0) load_meta(*c.a, *c.m, i0, cnt, true, false, false, c.latch);
      else load_meta(*c.a, *c.m, i0, cnt, false, false, false, false);
    }
    template <int T>
    __device__ void run(int i0, int cnt) {
      const FwdArgs &a = *c.a;
      const int H = c.H;
      const int lane = threadIdx.x & 31;
      const int t = threadIdx.x >> 5, unit = c.unit0 + lane;
      if (i0 != pre) {
        meta(i0, cnt);
        __syncthreads();
      }
      if (phase == 0) {
        gather_rows(c.X, MAXC, H, cnt, [&](int tt, int j) {
          int ci = c.m->cin[tt][j];
          return ci >= 0 ? a.h_out + (size_t)ci * H : (const float *)nullptr;
        });
        __syncthreads();
        if (t < cnt) {  // stash h_k[unit] before the reduction overwrites X
#pragma unroll
          for (int k = 0; k < MAXC; k++)
            c.cv[(t * kMaxC + k) * 32 + lane] = c.X[(size_t)(t * MAXC + k) * H + unit];
        }
        float acc[1 + MAXC][T], s[1 + MAXC];
        fma_engine<PhGruA<MAXC>, T>(c.Ws, c.X, H, acc);
        reduce_acc<1 + MAXC, T>(c.X, acc, s);
        if (t < cnt) {
          float z = sigmoidf_(s[0] + c.bias[0 * 32 + lane]);
          float br = c.bias[1 * 32 + lane];
          float sum = 0.f, ht = 0.f;
          const int nc = c.m->nch[t];
#pragma unroll
          for (int k = 0; k < MAXC; k++)
            if (k < nc) {
              float hk = c.cv[(t * kMaxC + k) * 32 + lane];
              sum += sigmoidf_(s[1 + k] + br) * hk;
              ht += hk;
            }
          size_t o = (size_t)c.m->own[t] * H + unit;
          a.sbuf[o] = sum;
          a.zbuf[o] = z;
          a.h_out[o] = ht;  // stash h~ for phase B (overwritten there)
        }
        __syncthreads();
      } else {
        gather_rows(c.X, 1, H, cnt, [&](int tt, int) { return a.sbuf + (size_t)c.m->own[tt] * H; });
        __syncthreads();
        float acc[1][T], s[1];
        fma_engine<PhGruB, T>(c.Ws, c.X, H, acc);
        reduce_acc<1, T>(c.X, acc, s);
        if (t < cnt) {
          size_t o = (size_t)c.m->own[t] * H + unit;
          float g = tanhf_(s[0] + c.bias[2 * 32 + lane]);
          float z = __ldcg(a.zbuf + o), ht = __ldcg(a.h_out + o);
          put_h(a, *c.m, t, unit, z * ht + (1.f - z) * g);
        }
        __syncthreads();
      }
    }
  };
  __device__ static int biases(const FwdArgs &a, const float **b, int *off) {
    b[0] = a.w[4]; b[1] = a.w[5]; b[2] = a.w[6];
    off[0] = off[1] = off[2] = 0;
    return 3;
  }
  __device__ static int leaf_lo(const FwdArgs &, int first_leaf) { return first_leaf; }
  __device__ static int leaf_gates(const FwdArgs &a, GateSrc *gs) {
    gs[0] = {a.w[0], 0, a.H, 0};
    gs[1] = {a.w[0], a.H, a.H, 0};
    return 2;
  }
  __device__ static int level_gates(const FwdArgs &a, GateSrc *gs) {
    gs[0] = {a.w[1], 0, a.H, 0};
    gs[1] = {a.w[2], 0, a.H, 0};
    gs[2] = {a.w[3], 0, a.H, 0};
    return 3;
  }
};

// ----- TreeFC (Q2: h = tanh(W [h_l; h_r] + b), leaf = Emb) -----------------
template <int MAXC>
struct TreeFc {
  static constexpr int kPhases = 1;
  struct Leaf {  // pure gather (no weights): h = x
    Ctx c;
    int pre;
    __device__ void meta(int i0, int cnt) { load_meta(*c.a, *c.m, i0, cnt, false, true, false, c.latch); }
    template <int T>
    __device__ void run(int i0, int cnt) {
      const FwdArgs &a = *c.a;
      if (i0 != pre) {
        meta(i0, cnt);
        __syncthreads();
      }
      const int t = threadIdx.x >> 5, unit = c.unit0 + (threadIdx.x & 31);
      if (t < cnt)
        put_h(a, *c.m, t, unit, __ldg(a.emb + (size_t)c.m->word[t] * c.H + unit));
      __syncthreads();
    }
  };
  struct Level {
    Ctx c;
    int phase, pre;
    __device__ void meta(int i0, int cnt) { load_meta(*c.a, *c.m, i0, cnt, true, false, true, c.latch); }
    template <int T>
    __device__ void run(int i0, int cnt) {
      const FwdArgs &a = *c.a;
      const int H = c.H;
      if (i0 != pre) {
        meta(i0, cnt);
        __syncthreads();
      }
      gather_rows(c.X, 2, H, cnt, [&](int t, int j) { return a.h_out + (size_t)c.m->cin[t][j] * H; });
      __syncthreads();
      float acc[1][T], s[1];
      fma_engine<PhFcLevel, T>(c.Ws, c.X, H, acc);
      reduce_acc<1, T>(c.X, acc, s);
      const int t = threadIdx.x >> 5, unit = c.unit0 + (threadIdx.x & 31);
      if (t < cnt) put_h(a, *c.m, t, unit, tanhf_(s[0] + c.bias[threadIdx.x & 31]));
      __syncthreads();
    }
  };
  __device__ static int biases(const FwdArgs &a, const float **b, int *off) {
    b[0] = a.w[1];
    off[0] = 0;
    return 1;
  }
  __device__ static int leaf_lo(const FwdArgs &, int first_leaf) { return first_leaf; }
  __device__ static int leaf_gates(const FwdArgs &, GateSrc *) { return 0; }
  __device__ static int level_gates(const FwdArgs &a, GateSrc *gs) {
    gs[0] = {a.w[0], 0, 2 * a.H, 0};
    gs[1] = {a.w[0], 0, 2 * a.H, a.H};
    return 2;
  }
};

// ----- DAG-RNN (Q8: h = tanh(W_x x + U sum_pred h + b), every node has x) --
template <int MAXC>
struct DagRnn {
  static constexpr int kPhases = 1;
  // "leaf" phase = input projection of EVERY node (GRNN-style input GEMM at the
  // start); leaves finish here.
  struct Leaf {
    Ctx c;
    int pre;
    __device__ void meta(int i0, int cnt) { load_meta(*c.a, *c.m, i0, cnt, false, true, false, c.latch); }
    template <int T>
    __device__ void run(int i0, int cnt) {
      const FwdArgs &a = *c.a;
      const int H = c.H;
      if (i0 != pre) {
        meta(i0, cnt);
        __syncthreads();
      }
      gather_rows(c.X, 1, H, cnt, [&](int t, int) { return a.emb + (size_t)c.m->word[t] * H; });
      cp_async_wait_all();
      __syncthreads();
      float acc[1][T], s[1];
      fma_engine<PhDagProj, T>(c.Ws, c.X, H, acc);
      reduce_acc<1, T>(c.X, acc, s);
      const int t = threadIdx.x >> 5, unit = c.unit0 + (threadIdx.x & 31);
      if (t < cnt) {
        float p = s[0] + c.bias[threadIdx.x & 31];
        size_t o = (size_t)c.m->own[t] * H + unit;
        a.pbuf[o] = p;
        if (i0 + t >= a.hdr->first_leaf) put_h(a, *c.m, t, unit, tanhf_(p));
      }
      __syncthreads();
    }
  };
  struct Level {
    Ctx c;
    int phase, pre;
    __device__ void meta(int i0, int cnt) { load_meta(*c.a, *c.m, i0, cnt, true, false, false, c.latch); }
    template <int T>
    __device__ void run(int i0, int cnt) {
      const FwdArgs &a = *c.a;
      const int H = c.H;
      const int lane = threadIdx.x & 31;
      if (i0 != pre) {
        meta(i0, cnt);
        __syncthreads();
      }
      gather_rows(c.X, MAXC, H, cnt, [&](int t, int j) {
        int ci = c.m->cin[t][j];
        return ci >= 0 ? a.h_out + (size_t)ci * H : (const float *)nullptr;
      });
      for (int idx = threadIdx.x; idx < cnt * 32; idx += blockDim.x)
        c.cv[idx] = __ldcg(a.pbuf + (size_t)c.m->own[idx >> 5] * H + c.unit0 + (idx & 31));
      __syncthreads();
      float acc[1][T], s[1];
      fma_engine<PhDagLevel<MAXC>, T>(c.Ws, c.X, H, acc);
      reduce_acc<1, T>(c.X, acc, s);
      const int t = threadIdx.x >> 5, unit = c.unit0 + lane;
      if (t < cnt) put_h(a, *c.m, t, unit, tanhf_(s[0] + c.cv[t * 32 + lane]));
      __syncthreads();
    }
  };
  __device__ static int biases(const FwdArgs &a, const float **b, int *off) {
    b[0] = a.w[2];
    off[0] = 0;
    return 1;
  }
  __device__ static int leaf_lo(const FwdArgs &, int) { return 0; }
  __device__ static int leaf_gates(const FwdArgs &a, GateSrc *gs) {
    gs[0] = {a.w[0], 0, a.H, 0};
    return 1;
  }
  __device__ static int level_gates(const FwdArgs &a, GateSrc *gs) {
    gs[0] = {a.w[1], 0, a.H, 0};
    return 1;
  }
};

// ----- TreeRNN (Listing 1: leaf Emb[words[n]], internal tanh(lh + rh)) ------
template <int MAXC>
struct TreeRnn {
  static constexpr int kPhases = 1;
  struct Leaf {
    Ctx c;
    int pre;
    __device__ void meta(int i0, int cnt) { load_meta(*c.a, *c.m, i0, cnt, false, true, false, c.latch); }
    template <int T>
    __device__ void run(int i0, int cnt) {
      const FwdArgs &a = *c.a;
      if (i0 != pre) {
        meta(i0, cnt);
        __syncthreads();
      }
      const int ug = min(kUG, c.H);
      for (int idx = threadIdx.x; idx < cnt * ug; idx += blockDim.x) {
        int t = idx / ug, unit = c.unit0 + idx % ug;
        put_h(a, *c.m, t, unit, __ldg(a.emb + (size_t)c.m->word[t] * c.H + unit));
      }
      __syncthreads();
    }
  };
  struct Level {
    Ctx c;
    int phase, pre;
    __device__ void meta(int i0, int cnt) { load_meta(*c.a, *c.m, i0, cnt, true, false, true, c.latch); }
    template <int T>
    __device__ void run(int i0, int cnt) {
      const FwdArgs &a = *c.a;
      if (i0 != pre) {
        meta(i0, cnt);
        __syncthreads();
      }
      const int ug = min(kUG, c.H);
      for (int idx = threadIdx.x; idx < cnt * ug; idx += blockDim.x) {
        int t = idx / ug, unit = c.unit0 + idx % ug;
        float l = __ldcg(a.h_out + (size_t)c.m->cin[t][0] * c.H + unit);
        float r = __ldcg(a.h_out + (size_t)c.m->cin[t][1] * c.H + unit);
        put_h(a, *c.m, t, unit, tanhf_(l + r));
      }
      __syncthreads();
    }
  };
  __device__ static int biases(const FwdArgs &, const float **, int *) { return 0; }
  __device__ static int leaf_lo(const FwdArgs &, int first_leaf) { return first_leaf; }
  __device__ static int leaf_gates(const FwdArgs &, GateSrc *) { return 0; }
  __device__ static int level_gates(const FwdArgs &, GateSrc *) { return 0; }
};

// ---------------------------------------------------------------------------
// The persistent kernel skeleton shared by the unit-split cells.
// ---------------------------------------------------------------------------
template <int CELL, int MAXC, class C>
__global__ void __launch_bounds__(kFwdThreads, 1) fwd_kernel(FwdArgs a) {
  extern __shared__ __align__(16) float smem[];
  __shared__ TileMeta meta;
  GateSrc gsrc[4];
  using Lay = Layout<CELL, MAXC>;
  using Tr = Traits<CELL, MAXC>;

  griddep_wait();
  if (*reinterpret_cast<volatile int *>(&a.hdr->status) != CX_OK) return;
  const int L = a.hdr->num_levels, first_leaf = a.hdr->first_leaf, n = a.n;
  const int gn = blockIdx.x / a.Gu, gu = blockIdx.x % a.Gu;
  const int H = a.H;

  Ctx ctx;
  ctx.a = &a;
  ctx.Ws = smem;
  ctx.X = smem + Lay::w_floats(H);
  ctx.cv = ctx.X + Lay::x_floats(H);
  ctx.m = &meta;
  ctx.gn = gn;
  ctx.gu = gu;
  ctx.unit0 = gu * min(kUG, H);
  ctx.H = H;
  ctx.latch = gu == 0;
  ctx.tslot = -1;
  unsigned epoch = 0;
  trace_mark(a, 0);

  // biases of the owned units -> shared memory (read by every epilogue)
  __shared__ float s_bias[4 * kUG];
  {
    const float *bp[4];
    int off[4];
    int nb = C::biases(a, bp, off);
    const int ug = min(kUG, H);
    if (threadIdx.x < nb * kUG) {
      int g = threadIdx.x / kUG, u = threadIdx.x % kUG;
      s_bias[threadIdx.x] = u < ug ? __ldg(bp[g] + off[g] + ctx.unit0 + u) : 0.f;
    }
  }
  ctx.bias = s_bias;

  // ---- leaf phase (specialised leaf loop nest) ------------------
  // The leaf weights are staged with cp.async; the first tile's bookkeeping and
  // Emb gather overlap the copy (each leaf tile waits for it before its FMA).
  {
    int ng = C::leaf_gates(a, gsrc);
    if (ng) load_gates(ctx.Ws, gsrc, ng, ctx.unit0, H);
    __syncthreads();
    trace_mark(a, 1);
    int lo0 = C::leaf_lo(a, first_leaf);
    int lo, hi;
    chunk_of(n - lo0, a.Gn, gn, lo, hi);
    typename C::Leaf f{ctx, -1};
    tiles_T<Tr::TMAX>(lo0 + lo, lo0 + hi, f);
    cp_async_wait_all();
  }
  __syncthreads();
  trace_mark(a, 2);
  // recurrent weights: issued now, landed while the CTA waits at the barrier
  {
    int ng = C::level_gates(a, gsrc);
    if (ng) load_gates(ctx.Ws, gsrc, ng, ctx.unit0, H);
  }
  // ---- internal batches, one grid barrier per level (and phase) -----------
  // While waiting at a barrier the CTA already loads the bookkeeping of its
  // first tile of the next level (it depends only on the linearization).
  for (int l = 1; l < L; l++) {
    const int base = __ldg(a.lbeg + l), M = __ldg(a.lsize + l);
    int lo, hi;
    chunk_of(M, a.Gn, gn, lo, hi);
    for (int ph = 0; ph < C::kPhases; ph++) {
      const int slot = 3 + 2 * ((l - 1) * C::kPhases + ph);
      trace_mark(a, slot);
      grid_arrive(a.bar, epoch);
      typename C::Level f{ctx, ph, -1};
      if (hi > lo) {
        f.meta(base + lo, min(Tr::TMAX, hi - lo));
        f.pre = base + lo;
      }
      grid_wait(a.bar, gridDim.x, epoch);
      trace_mark(a, slot + 1);
      if (l == 1 && ph == 0) {
        cp_async_wait_all();
        __syncthreads();
      }
      f.c.tslot = a.trace ? 64 + 5 * ((l - 1) * C::kPhases + ph) : -1;
      tiles_T<Tr::TMAX>(base + lo, base + hi, f);
    }
  }
  cp_async_wait_all();
  trace_mark(a, a.trace_slots - 2);

  // ---- the last CTA out publishes the latched status -----------------------
  __syncthreads();
  trace_mark(a, a.trace_slots - 1);
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
      __threadfence();
    }
  }
}

}  // namespace

// MV-RNN lives in forward_mvrnn.cu, the register-weight path in forward_rw.cu
bool mvrnn_plan(int H, int num_sms, FwdPlan *plan, int *Gn, int *Gu);
bool rw_plan(int cell, int H, int maxc, int num_sms, FwdPlan *plan, int *Gn, int *Gu);
bool cluster_plan(int cell, int H, int maxc, int n, int roots, FwdPlan *plan, int *Gn, int *Gu);
bool big_plan(int cell, int H, int maxc, int num_sms, FwdPlan *plan, int *Gn, int *Gu);
size_t big_workspace_bytes(int cell, int H, int n, int V);

template <int CELL, int MAXC, class C>
static bool plan_for(int H, int num_sms, FwdPlan *p, int *Gn, int *Gu) {
  using Lay = Layout<CELL, MAXC>;
  int gu = H >= kUG ? H / kUG : 1;
  if (H >= kUG && H % kUG) return false;
  if (gu > num_sms) return false;
  size_t smem = Lay::bytes(H);
  if (smem > 227 * 1024) return false;
  auto k = fwd_kernel<CELL, MAXC, C>;
  static size_t smem_set[kMaxDevices];  // per device; callers serialise plans (api.cu mutex)
  const int dev = device_slot();
  if (dev < 0) return false;
  if (smem > smem_set[dev]) {
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return false;
    smem_set[dev] = smem;
    cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    cudaGetLastError();
  }
  *Gu = gu;
  *Gn = num_sms / gu;
  p->ctas = *Gn * gu;
  p->threads = kFwdThreads;
  p->smem = smem;
  p->kernel = (const void *)k;
  p->family = 1;
  return true;
}

bool fwd_plan(int cell, int H, int maxc, int n, int path, int num_sms, FwdPlan *plan, int *Gn,
              int *Gu) {
  if (H <= 0 || H > 1024 || H % 4) return false;
  // Register-resident weights (forward_rw.cu) for small and medium batches;
  // the shared-memory-weight kernel below for large batches, where 32 units
  // per CTA minimise the re-gathering of child rows across unit groups.
  const bool rw_ok = (cell == CX_TREELSTM || cell == CX_TREEGRU || cell == CX_TREEFC ||
                      cell == CX_DAGRNN || cell == CX_SIMPLETREEGRU) && (H == 64 || H == 128 || H == 256 || H == 512);
  if ((path == 0 || path == 3) && cluster_plan(cell, H, maxc, n, 0, plan, Gn, Gu)) return true;
  if ((path == 4 || (path == 0 && n > kRwMaxNodes)) && big_plan(cell, H, maxc, num_sms, plan, Gn, Gu))
    return true;
  const bool want_rw = path == 1 || (path == 0 && n <= kRwMaxNodes);
  if (rw_ok && want_rw && rw_plan(cell, H, maxc, num_sms, plan, Gn, Gu)) return true;
  const bool weighted = cell != CX_TREERNN && cell != CX_MVRNN;
  if (weighted && (H % kUG)) return false;
  switch (cell) {
    case CX_TREERNN:
      return plan_for<CX_TREERNN, 2, TreeRnn<2>>(H, num_sms, plan, Gn, Gu);
    case CX_TREEFC:
      return plan_for<CX_TREEFC, 2, TreeFc<2>>(H, num_sms, plan, Gn, Gu);
    case CX_TREELSTM:
      if (maxc <= 1) return plan_for<CX_TREELSTM, 1, TreeLstm<1>>(H, num_sms, plan, Gn, Gu);
      if (maxc <= 2) return plan_for<CX_TREELSTM, 2, TreeLstm<2>>(H, num_sms, plan, Gn, Gu);
      if (maxc <= 4) return plan_for<CX_TREELSTM, 4, TreeLstm<4>>(H, num_sms, plan, Gn, Gu);
      return false;
    case CX_TREEGRU:
      if (maxc <= 1) return plan_for<CX_TREEGRU, 1, TreeGru<1>>(H, num_sms, plan, Gn, Gu);
      if (maxc <= 2) return plan_for<CX_TREEGRU, 2, TreeGru<2>>(H, num_sms, plan, Gn, Gu);
      if (maxc <= 4) return plan_for<CX_TREEGRU, 4, TreeGru<4>>(H, num_sms, plan, Gn, Gu);
      return false;
    case CX_DAGRNN:
      if (maxc <= 1) return plan_for<CX_DAGRNN, 1, DagRnn<1>>(H, num_sms, plan, Gn, Gu);
      if (maxc <= 2) return plan_for<CX_DAGRNN, 2, DagRnn<2>>(H, num_sms, plan, Gn, Gu);
      if (maxc <= 4) return plan_for<CX_DAGRNN, 4, DagRnn<4>>(H, num_sms, plan, Gn, Gu);
      return false;
    case CX_MVRNN:
      return mvrnn_plan(H, num_sms, plan, Gn, Gu);
  }
  return false;
}

size_t fwd_workspace_bytes(int cell, int H, int n, int V) {
  size_t N = (size_t)(n > 0 ? n : 1), h = (size_t)H;
  size_t b = sizeof(GridBar);
  if (cell == CX_TREELSTM || cell == CX_DAGRNN) {  // large-batch path: hs, st + words
    size_t big = big_workspace_bytes(cell, H, (int)N, V);
    size_t other = 4 * N * h;
    return b + (big > other ? big : other) + 1024;
  }
  switch (cell) {
    case CX_TREELSTM: b += 4 * N * h; break;            // c (when aux_out == NULL)
    case CX_TREEGRU:
    case CX_SIMPLETREEGRU: b += 2 * 4 * N * h; break;   // z, s (refactored: m)
    case CX_DAGRNN: b += 4 * N * h; break;              // projections
    case CX_MVRNN: b += 4 * N * h * h; break;           // A (when aux_out == NULL)
    default: break;
  }
  return b + 1024;
}

// Programmatic dependent launch of cx_forward behind cx_linearize is opt-in
// (CX_PDL=1): measured on B200 it saves ~2 us eagerly and nothing under CUDA
// graph replay, and an early-resident cooperative forward slowed the fp32
// DAG-RNN b4096 step from 10.1 to 15.7 ms. The kernels are written for it
// either way (weights staged before griddepcontrol.wait).
bool pdl_enabled() {
  static const bool on = [] {
    const char *e = std::getenv("CX_PDL");
    return e && e[0] == '1';
  }();
  return on;
}

// Cooperative launch through cudaLaunchKernelEx so it can be captured into a
// CUDA graph (the bench replays linearize + forward as one graph).
cudaError_t fwd_launch(const FwdPlan &plan, FwdArgs &args, cudaStream_t stream) {
  void *params[] = {&args};
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(plan.ctas);
  cfg.blockDim = dim3(plan.threads);
  cfg.dynamicSmemBytes = plan.smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  if (plan.cluster > 1) {  // independent clusters: no grid barrier, no co-residency needed
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = plan.cluster;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
  } else {
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
  }
  // programmatic dependent launch: the kernel stages its weights while the
  // preceding cx_linearize runs (griddepcontrol.wait before reading it)
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  if (plan.family == 7) {  // fused single-CTA kernel: no grid-wide dependency, plain launch
    cfg.attrs = attr + 1;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
  }
  return cudaLaunchKernelExC(&cfg, plan.kernel, params);
}

}  // namespace cx
