// forward_rw.cu -- persistent forward with REGISTER-resident weights
// (the latency path: small and medium batches).
//
// Model persistence (App. C) keeps the
// recurrent weights on chip across all levels. Here they live in registers:
// CTA (gn, gu) owns 16 hidden units; its 512 threads split the contraction
// dimension into 32 chunks of KC = H/32 (warp w, half-warp s -> chunk 2w+s)
// and thread (u, chunk) holds W[g][unit0+u][chunk] for every gate g -- at
// H = 256 that is 4 gates x 8 = 32 floats per thread for TreeLSTM. A tile of
// T nodes therefore costs no weight traffic at all: the children's rows are
// gathered into shared memory (the paper's rnn_cache), every
// thread multiplies its register slice against its chunk of each row, the
// two half-warps are combined with one shuffle and the 16 warps through
// shared memory, and the gate algebra runs in the epilogue.
//
// Compared with forward.cu (32 units per CTA, weights streamed from shared
// memory every tile) this halves the units per CTA, doubles the node groups
// (Gn = 9 at H = 256) and removes the per-tile 128 KiB shared-memory weight
// sweep that dominated small levels.
#include <cuda_runtime.h>

#include <cuda_bf16.h>

#include <cstdlib>
#include <type_traits>

#include "rw_engine.cuh"

namespace cx {
namespace {
using namespace fwd;
using namespace rw;

constexpr bool kGruRefactorDefault = false;  // set from the measurement

// ---------------------------------------------------------------------------
// Cells
// ---------------------------------------------------------------------------
template <int H, int MAXC>
struct RTreeLstm {
  static constexpr int kPhases = 1;
  static constexpr bool kLeafPost = false;
  using M = TileMetaT<kLeafBlock>;
  __device__ static int leaf_gates(const FwdArgs &a, Gate *g) {
    g[0] = {a.w[0], 0, H, 0}; g[1] = {a.w[0], H, H, 0}; g[2] = {a.w[0], 2 * H, H, 0};
    return 3;
  }
  __device__ static int level_gates(const FwdArgs &a, Gate *g) {
    g[0] = {a.w[1], 0, H, 0}; g[1] = {a.w[1], H, H, 0}; g[2] = {a.w[1], 2 * H, H, 0};
    g[3] = {a.w[3], 0, H, 0};
    return 4;
  }
  __device__ static int biases(const FwdArgs &a, const float **b, int *off) {
    b[0] = b[1] = b[2] = a.w[2]; off[0] = 0; off[1] = H; off[2] = 2 * H;
    b[3] = a.w[4]; off[3] = 0;
    return 4;
  }
  __device__ static int leaf_lo(int first_leaf) { return first_leaf; }
  // Leaf blocks: bookkeeping and Emb rows of a block of up to 2 TMAX leaves are
  // loaded once (block()), then the block is contracted tile by tile (run()).
  struct Leaf {
    RCtx c; M *m; const float (*w)[RShape<H>::KC]; int b0;
    __device__ void meta(int i0, int cnt) { load_meta(*c.a, *m, i0, cnt, false, true, false, c.latch); }
    __device__ void block(int cnt) {
      const FwdArgs &a = *c.a;
      gather_rows_c<1, H>(c.X, cnt, [&](int t, int) { return a.emb + (size_t)m->word[t] * H; });
    }
    template <int T>
    __device__ __forceinline__ void run(int i0, int cnt) {
      const FwdArgs &a = *c.a;
      const int off = i0 - b0;
      if (c.tslot >= 0) trace_mark(a, c.tslot + 1);
      float s[3];
      contract<RLstmLeaf, H, T>(c, c.X + (size_t)(i0 - b0) * H, *reinterpret_cast<const float(*)[4][RShape<H>::KC]>(w), s);
      const int t = threadIdx.x >> 4, u = threadIdx.x & 15;
      if (t < cnt) {
        float cc = sigmoidf_(s[0] + c.bias[u]) * tanhf_(s[2] + c.bias[32 + u]);
        float hh = sigmoidf_(s[1] + c.bias[16 + u]) * tanhf_(cc);
        size_t o = (size_t)m->own[off + t] * H + c.unit0 + u;
        put_h(a, *m, off + t, c.unit0 + u, hh);
        a.cbuf[o] = cc;
      }
      __syncthreads();
      if (c.tslot >= 0) trace_mark(a, c.tslot + 4);
      c.tslot = -1;
    }
  };
  struct Level {
    RCtx c; M *m; const float (*w)[RShape<H>::KC]; int phase, pre;
    __device__ void meta(int i0, int cnt) { load_meta(*c.a, *m, i0, cnt, true, false, false, c.latch); }
    template <int T>
    __device__ __forceinline__ void run(int i0, int cnt) {
      const FwdArgs &a = *c.a;
      if (i0 != pre) { meta(i0, cnt); __syncthreads(); }
      if (c.tslot >= 0) trace_mark(a, c.tslot);
      gather_rows_c<MAXC, H>(c.X, cnt, [&](int t, int j) {
        int ci = m->cin[t][j];
        return ci >= 0 ? a.h_out + (size_t)ci * H : (const float *)nullptr;
      });
      for (int idx = threadIdx.x; idx < cnt * MAXC * kRUG; idx += blockDim.x) {
        int t = idx / (MAXC * kRUG), r = idx - t * MAXC * kRUG, k = r >> 4, u = r & 15;
        int ci = m->cin[t][k];
        c.cv[(t * kMaxC + k) * kRUG + u] = ci >= 0 ? __ldcg(a.cbuf + (size_t)ci * H + c.unit0 + u) : 0.f;
      }
      __syncthreads();
      if (c.tslot >= 0) trace_mark(a, c.tslot + 1);
      float s[3 + MAXC];
      contract<RLstmLevel<MAXC>, H, T>(c, c.X, *reinterpret_cast<const float(*)[4][RShape<H>::KC]>(w), s);
      const int t = threadIdx.x >> 4, u = threadIdx.x & 15;
      if (t < cnt) {
        float cc = sigmoidf_(s[0] + c.bias[u]) * tanhf_(s[2] + c.bias[32 + u]);
        const float bf = c.bias[48 + u];
        const int nc = m->nch[t];
#pragma unroll
        for (int k = 0; k < MAXC; k++)
          if (k < nc) cc += sigmoidf_(s[3 + k] + bf) * c.cv[(t * kMaxC + k) * kRUG + u];
        float hh = sigmoidf_(s[1] + c.bias[16 + u]) * tanhf_(cc);
        size_t o = (size_t)m->own[t] * H + c.unit0 + u;
        put_h(a, *m, t, c.unit0 + u, hh);
        a.cbuf[o] = cc;
      }
      __syncthreads();
      if (c.tslot >= 0) trace_mark(a, c.tslot + 4);
      c.tslot = -1;
    }
  };
};

// TreeGRU (reading Q3) and SimpleTreeGRU (SIMPLE, Q24: h = (1 - z) g at
// internal nodes, footnote P:1638-1640), ORIGINAL schedule: phase A gathers the
// children's h and forms z = sigma(U_z h~ + b_z) and s = sum_k sigma(U_r h_k +
// b_r) * h_k (3 matvecs); a grid barrier; phase B g = tanh(U_h s + b_h) (1
// matvec) and h; a grid barrier.
template <int H, int MAXC, bool SIMPLE = false>
struct RTreeGru {
  static constexpr int kPhases = 2;
  static constexpr bool kLeafPost = false;
  using M = TileMetaT<kLeafBlock>;
  __device__ static int leaf_gates(const FwdArgs &a, Gate *g) {
    g[0] = {a.w[0], 0, H, 0}; g[1] = {a.w[0], H, H, 0};
    return 2;
  }
  __device__ static int level_gates(const FwdArgs &a, Gate *g) {
    g[0] = {a.w[1], 0, H, 0}; g[1] = {a.w[2], 0, H, 0}; g[2] = {a.w[3], 0, H, 0};
    return 3;
  }
  __device__ static int biases(const FwdArgs &a, const float **b, int *off) {
    b[0] = a.w[4]; b[1] = a.w[5]; b[2] = a.w[6]; off[0] = off[1] = off[2] = 0;
    return 3;
  }
  __device__ static int leaf_lo(int first_leaf) { return first_leaf; }
  struct Leaf {
    RCtx c; M *m; const float (*w)[RShape<H>::KC]; int b0;
    __device__ void meta(int i0, int cnt) { load_meta(*c.a, *m, i0, cnt, false, true, false, c.latch); }
    __device__ void block(int cnt) {
      const FwdArgs &a = *c.a;
      gather_rows_c<1, H>(c.X, cnt, [&](int t, int) { return a.emb + (size_t)m->word[t] * H; });
    }
    template <int T>
    __device__ __forceinline__ void run(int i0, int cnt) {
      const FwdArgs &a = *c.a;
      const int off = i0 - b0;
      float s[2];
      contract<RGruLeaf, H, T>(c, c.X + (size_t)off * H, *reinterpret_cast<const float(*)[4][RShape<H>::KC]>(w), s);
      const int t = threadIdx.x >> 4, u = threadIdx.x & 15;
      if (t < cnt) {
        float z = sigmoidf_(s[0] + c.bias[u]);
        float g = tanhf_(s[1] + c.bias[32 + u]);
        put_h(a, *m, off + t, c.unit0 + u, (1.f - z) * g);
      }
      __syncthreads();
    }
  };
  struct Level {
    RCtx c; M *m; const float (*w)[RShape<H>::KC]; int phase, pre;
    __device__ void meta(int i0, int cnt) {
      if (phase == 0) load_meta(*c.a, *m, i0, cnt, true, false, false, c.latch);
      else load_meta(*c.a, *m, i0, cnt, false, false, false, false);
    }
    template <int T>
    __device__ __forceinline__ void run(int i0, int cnt) {
      const FwdArgs &a = *c.a;
      if (i0 != pre) { meta(i0, cnt); __syncthreads(); }
      const int t = threadIdx.x >> 4, u = threadIdx.x & 15;
      const auto &wr = *reinterpret_cast<const float(*)[4][RShape<H>::KC]>(w);
      if (phase == 0) {
        gather_rows_c<MAXC, H>(c.X, cnt, [&](int tt, int j) {
          int ci = m->cin[tt][j];
          return ci >= 0 ? a.h_out + (size_t)ci * H : (const float *)nullptr;
        });
        __syncthreads();
        float s[1 + MAXC];
        contract<RGruA<MAXC>, H, T>(c, c.X, wr, s);
        if (t < cnt) {
          const int unit = c.unit0 + u;
          float z = sigmoidf_(s[0] + c.bias[u]);
          float br = c.bias[16 + u];
          float sum = 0.f, ht = 0.f;
          const int nc = m->nch[t];
#pragma unroll
          for (int k = 0; k < MAXC; k++)
            if (k < nc) {
              float hk = c.X[(size_t)(t * MAXC + k) * H + unit];
              sum += sigmoidf_(s[1 + k] + br) * hk;
              ht += hk;
            }
          size_t o = (size_t)m->own[t] * H + unit;
          a.sbuf[o] = sum;
          a.zbuf[o] = z;
          a.h_out[o] = ht;  // stash h~ for phase B (overwritten there)
        }
        __syncthreads();
      } else {
        gather_rows_c<1, H>(c.X, cnt, [&](int tt, int) { return a.sbuf + (size_t)m->own[tt] * H; });
        __syncthreads();
        float s[1];
        contract<RGruB, H, T>(c, c.X, wr, s);
        if (t < cnt) {
          size_t o = (size_t)m->own[t] * H + c.unit0 + u;
          float g = tanhf_(s[0] + c.bias[32 + u]);
          float z = __ldcg(a.zbuf + o), ht = __ldcg(a.h_out + o);
          put_h(a, *m, t, c.unit0 + u, SIMPLE ? (1.f - z) * g : z * ht + (1.f - z) * g);
        }
        __syncthreads();
      }
    }
  };
};

// Recursive refactoring (§3.1, evaluated P:1632-1644) of the
// two GRU cells: the reset-gated contribution m_k = sigma(U_r h_k + b_r) * h_k
// depends on the child only, so it moves across the recursion backedge into
// the CHILD's step (A1 of Fig. rec_refactoring), right after its h is
// complete. A level then runs
//   phase 0: gather h~ = sum_k h_k and m~ = sum_k m_k (sums formed in the
//            gather), z = sigma(U_z h~ + b_z), g = tanh(U_h m~ + b_h), h (2 matvecs
//            on the critical path instead of 3); grid barrier;
//   phase 1: m = sigma(U_r h + b_r) * h of the level's own nodes (1 matvec);
//            grid barrier
// plus one extra phase for the leaves' m after the leaf phase. The barrier
// count per level is the same as the original schedule (each phase needs a
// complete vector of the one before); the work on the per-level critical path
// drops from 4 to 3 matvecs per node. Both schedules are measured.
template <int H, int MAXC, bool SIMPLE>
struct RTreeGruR {
  static constexpr int kPhases = 2;
  static constexpr bool kLeafPost = true;
  using M = TileMetaT<kLeafBlock>;
  // products: phase 0 U_z . h~ (vector 0) and U_h . m~ (vector 1); phase 1 U_r . h
  struct P0 : PhBase<3, 2, 0, 2, 2> {
    __device__ static constexpr int g(int p) { return p; }
    __device__ static constexpr int v(int p) { return p; }
    __device__ static constexpr int a(int p) { return p; }
  };
  struct P1 : PhBase<3, 1, 0, 1, 1> {
    __device__ static constexpr int g(int p) { return 2; }
    __device__ static constexpr int v(int p) { return 0; }
    __device__ static constexpr int a(int p) { return 0; }
  };
  __device__ static int leaf_gates(const FwdArgs &a, Gate *g) {
    g[0] = {a.w[0], 0, H, 0}; g[1] = {a.w[0], H, H, 0};
    return 2;
  }
  __device__ static int level_gates(const FwdArgs &a, Gate *g) {  // U_z, U_h, U_r
    g[0] = {a.w[1], 0, H, 0}; g[1] = {a.w[3], 0, H, 0}; g[2] = {a.w[2], 0, H, 0};
    return 3;
  }
  __device__ static int biases(const FwdArgs &a, const float **b, int *off) {
    b[0] = a.w[4]; b[1] = a.w[5]; b[2] = a.w[6]; off[0] = off[1] = off[2] = 0;
    return 3;
  }
  __device__ static int leaf_lo(int first_leaf) { return first_leaf; }
  using Leaf = typename RTreeGru<H, MAXC, SIMPLE>::Leaf;
  // m = sigma(U_r h + b_r) * h of the nodes [i0, i0 + cnt) (their h complete)
  __device__ static void m_phase(const RCtx &c, M *m, const float (*w)[RShape<H>::KC], int i0,
                                 int cnt, auto tt) {
    constexpr int T = decltype(tt)::value;
    const FwdArgs &a = *c.a;
    gather_rows_c<1, H>(c.X, cnt, [&](int t, int) { return a.h_out + (size_t)m->own[t] * H; });
    __syncthreads();
    float s[1];
    contract<P1, H, T>(c, c.X, *reinterpret_cast<const float(*)[4][RShape<H>::KC]>(w), s);
    const int t = threadIdx.x >> 4, u = threadIdx.x & 15;
    if (t < cnt) {
      const int unit = c.unit0 + u;
      const float h = c.X[(size_t)t * H + unit];
      a.sbuf[(size_t)m->own[t] * H + unit] = sigmoidf_(s[0] + c.bias[16 + u]) * h;
    }
    __syncthreads();
  }
  struct LeafPost {
    RCtx c; M *m; const float (*w)[RShape<H>::KC]; int pre;
    __device__ void meta(int i0, int cnt) { load_meta(*c.a, *m, i0, cnt, false, false, false, false); }
    template <int T>
    __device__ __forceinline__ void run(int i0, int cnt) {
      meta(i0, cnt);
      __syncthreads();
      m_phase(c, m, w, i0, cnt, std::integral_constant<int, T>{});
    }
  };
  struct Level {
    RCtx c; M *m; const float (*w)[RShape<H>::KC]; int phase, pre;
    __device__ void meta(int i0, int cnt) {
      if (phase == 0) load_meta(*c.a, *m, i0, cnt, true, false, false, c.latch);
      else load_meta(*c.a, *m, i0, cnt, false, false, false, false);
    }
    template <int T>
    __device__ __forceinline__ void run(int i0, int cnt) {
      const FwdArgs &a = *c.a;
      if (i0 != pre) { meta(i0, cnt); __syncthreads(); }
      if (phase == 1) {
        m_phase(c, m, w, i0, cnt, std::integral_constant<int, T>{});
        return;
      }
      // X rows per node: h~ then m~, summed over the present children
      constexpr int q = H / 4;
      for (int idx = threadIdx.x; idx < cnt * q; idx += blockDim.x) {
        const int t = idx / q, cq = idx - t * q;
        float4 hs = make_float4(0.f, 0.f, 0.f, 0.f), ms = hs;
#pragma unroll
        for (int k = 0; k < MAXC; k++) {
          const int ci = m->cin[t][k];
          if (ci >= 0) {
            hs = add4(hs, ldcg4(a.h_out + (size_t)ci * H + 4 * cq));
            ms = add4(ms, ldcg4(a.sbuf + (size_t)ci * H + 4 * cq));
          }
        }
        *reinterpret_cast<float4 *>(c.X + (size_t)(2 * t) * H + 4 * cq) = hs;
        *reinterpret_cast<float4 *>(c.X + (size_t)(2 * t + 1) * H + 4 * cq) = ms;
      }
      __syncthreads();
      float s[2];
      contract<P0, H, T>(c, c.X, *reinterpret_cast<const float(*)[4][RShape<H>::KC]>(w), s);
      const int t = threadIdx.x >> 4, u = threadIdx.x & 15;
      if (t < cnt) {
        const int unit = c.unit0 + u;
        const float z = sigmoidf_(s[0] + c.bias[u]);
        const float g = tanhf_(s[1] + c.bias[32 + u]);
        const float ht = c.X[(size_t)(2 * t) * H + unit];
        put_h(a, *m, t, unit, SIMPLE ? (1.f - z) * g : z * ht + (1.f - z) * g);
      }
      __syncthreads();
    }
  };
};

template <int H, int MAXC>
struct RTreeFc {
  static constexpr int kPhases = 1;
  static constexpr bool kLeafPost = false;
  using M = TileMetaT<kLeafBlock>;
  __device__ static int leaf_gates(const FwdArgs &, Gate *) { return 0; }
  __device__ static int level_gates(const FwdArgs &a, Gate *g) {
    g[0] = {a.w[0], 0, 2 * H, 0}; g[1] = {a.w[0], 0, 2 * H, H};
    return 2;
  }
  __device__ static int biases(const FwdArgs &a, const float **b, int *off) {
    b[0] = a.w[1]; off[0] = 0;
    return 1;
  }
  __device__ static int leaf_lo(int first_leaf) { return first_leaf; }
  struct Leaf {  // h = Emb[word] (pure gather, done for the whole block)
    RCtx c; M *m; const float (*w)[RShape<H>::KC]; int b0;
    __device__ void meta(int i0, int cnt) { load_meta(*c.a, *m, i0, cnt, false, true, false, c.latch); }
    __device__ void block(int cnt) {
      const FwdArgs &a = *c.a;
      for (int idx = threadIdx.x; idx < cnt * kRUG; idx += blockDim.x) {
        int t = idx >> 4, u = idx & 15;
        put_h(a, *m, t, c.unit0 + u, __ldg(a.emb + (size_t)m->word[t] * H + c.unit0 + u));
      }
    }
    template <int T>
    __device__ __forceinline__ void run(int, int) {}
  };
  struct Level {
    RCtx c; M *m; const float (*w)[RShape<H>::KC]; int phase, pre;
    __device__ void meta(int i0, int cnt) { load_meta(*c.a, *m, i0, cnt, true, false, true, c.latch); }
    template <int T>
    __device__ __forceinline__ void run(int i0, int cnt) {
      const FwdArgs &a = *c.a;
      if (i0 != pre) { meta(i0, cnt); __syncthreads(); }
      gather_rows_c<2, H>(c.X, cnt, [&](int t, int j) { return a.h_out + (size_t)m->cin[t][j] * H; });
      if (a.bf16ops) {  // dtype bf16 on FMA: the gathered operand rows rounded (reading Q18)
        __syncthreads();  // (the rows were copied by other threads' cp.async)
        for (int idx = threadIdx.x; idx < cnt * 2 * H; idx += blockDim.x)
          c.X[idx] = __bfloat162float(__float2bfloat16_rn(c.X[idx]));
      }
      __syncthreads();
      float s[1];
      contract<RFcLevel, H, T>(c, c.X, *reinterpret_cast<const float(*)[4][RShape<H>::KC]>(w), s);
      const int t = threadIdx.x >> 4, u = threadIdx.x & 15;
      if (t < cnt) put_h(a, *m, t, c.unit0 + u, tanhf_(s[0] + c.bias[u]));
      __syncthreads();
    }
  };
};

template <int H, int MAXC>
struct RDagRnn {
  static constexpr int kPhases = 1;
  static constexpr bool kLeafPost = false;
  using M = TileMetaT<kLeafBlock>;
  // gates {W_x, U} resident through leaves and levels (input projections are
  // fused into each level instead of a separate all-node GEMM)
  __device__ static int leaf_gates(const FwdArgs &a, Gate *g) {
    g[0] = {a.w[0], 0, H, 0}; g[1] = {a.w[1], 0, H, 0};
    return 2;
  }
  __device__ static int level_gates(const FwdArgs &a, Gate *g) { return leaf_gates(a, g); }
  __device__ static int biases(const FwdArgs &a, const float **b, int *off) {
    b[0] = a.w[2]; off[0] = 0;
    return 1;
  }
  __device__ static int leaf_lo(int first_leaf) { return first_leaf; }
  struct Leaf {  // h = tanh(W_x x + b)
    RCtx c; M *m; const float (*w)[RShape<H>::KC]; int b0;
    __device__ void meta(int i0, int cnt) { load_meta(*c.a, *m, i0, cnt, false, true, false, c.latch); }
    __device__ void block(int cnt) {
      const FwdArgs &a = *c.a;
      gather_rows_c<1, H>(c.X, cnt, [&](int t, int) { return a.emb + (size_t)m->word[t] * H; });
    }
    template <int T>
    __device__ __forceinline__ void run(int i0, int cnt) {
      const FwdArgs &a = *c.a;
      const int off = i0 - b0;
      float s[1];
      contract<RDagLeaf, H, T>(c, c.X + (size_t)off * H, *reinterpret_cast<const float(*)[4][RShape<H>::KC]>(w), s);
      const int t = threadIdx.x >> 4, u = threadIdx.x & 15;
      if (t < cnt) put_h(a, *m, off + t, c.unit0 + u, tanhf_(s[0] + c.bias[u]));
      __syncthreads();
    }
  };
  struct Level {  // h = tanh(W_x x + U h~ + b)
    RCtx c; M *m; const float (*w)[RShape<H>::KC]; int phase, pre;
    __device__ void meta(int i0, int cnt) { load_meta(*c.a, *m, i0, cnt, true, true, false, c.latch); }
    template <int T>
    __device__ __forceinline__ void run(int i0, int cnt) {
      const FwdArgs &a = *c.a;
      if (i0 != pre) { meta(i0, cnt); __syncthreads(); }
      gather_rows_c<MAXC + 1, H>(c.X, cnt, [&](int t, int j) {
        if (j == MAXC) return a.emb + (size_t)m->word[t] * H;
        int ci = m->cin[t][j];
        return ci >= 0 ? a.h_out + (size_t)ci * H : (const float *)nullptr;
      });
      __syncthreads();
      float s[1];
      contract<RDagLevel<MAXC>, H, T>(c, c.X, *reinterpret_cast<const float(*)[4][RShape<H>::KC]>(w), s);
      const int t = threadIdx.x >> 4, u = threadIdx.x & 15;
      if (t < cnt) put_h(a, *m, t, c.unit0 + u, tanhf_(s[0] + c.bias[u]));
      __syncthreads();
    }
  };
};

// ---------------------------------------------------------------------------
// Kernel skeleton
// ---------------------------------------------------------------------------
template <int CELL, int H, int MAXC, class C>
__global__ void __launch_bounds__(kRThreads, 1) rw_kernel(FwdArgs a) {
  using Cfg = RCfg<CELL, H, MAXC>;
  using Lay = RLayout<CELL, H, MAXC>;
  constexpr int KC = RShape<H>::KC;
  extern __shared__ __align__(16) float smem[];
  __shared__ typename C::M meta;
  __shared__ float s_bias[4 * kRUG];

  const int gn = blockIdx.x / a.Gu, gu = blockIdx.x % a.Gu;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int u = lane & 15, k0 = (warp * 2 + (lane >> 4)) * KC;

  RCtx ctx;
  ctx.a = &a;
  ctx.X = smem;
  ctx.red = smem + Lay::x_floats;
  ctx.red2 = ctx.red + Lay::red_floats;
  ctx.cv = ctx.red2 + Lay::red2_floats;
  ctx.gn = gn;
  ctx.gu = gu;
  ctx.unit0 = gu * kRUG;
  ctx.latch = gu == 0;
  ctx.tslot = -1;
  unsigned epoch = 0;
  trace_mark(a, 0);

  {
    const float *bp[4];
    int off[4];
    int nb = C::biases(a, bp, off);
    if (threadIdx.x < nb * kRUG) {
      int g = threadIdx.x / kRUG, uu = threadIdx.x % kRUG;
      s_bias[threadIdx.x] = __ldg(bp[g] + off[g] + ctx.unit0 + uu);
    }
  }
  ctx.bias = s_bias;

  float w[4][KC];
  Gate gs[4];
  // ---- leaf phase (specialised leaf loop nest) ------------------
  // Leaves are processed in blocks of up to kLeafBlock: one bookkeeping pass and one
  // Emb gather per block (the first block's overlap the weight loads).
  {
    int ng = C::leaf_gates(a, gs);
    load_wregs<Cfg::NG, KC>(w, gs, ng, ctx.unit0 + u, k0);
    trace_mark(a, 1);
  }
  // the linearization is read from here on (PDL: weights staged meanwhile)
  griddep_wait();
  if (*reinterpret_cast<volatile int *>(&a.hdr->status) != CX_OK) return;
  const int L = a.hdr->num_levels, first_leaf = a.hdr->first_leaf, n = a.n;
  {
    const int lo0 = C::leaf_lo(first_leaf);
    int lo, hi;
    chunk_of(n - lo0, a.Gn, gn, lo, hi);
    typename C::Leaf f{ctx, &meta, w, 0};
    f.c.tslot = a.trace ? 59 : -1;
    for (int b0 = lo0 + lo; b0 < lo0 + hi; b0 += kLeafBlock) {
      const int cntb = min(kLeafBlock, lo0 + hi - b0);
      __syncthreads();  // previous block's readers of meta / X are done
      f.meta(b0, cntb);
      __syncthreads();
      if (f.c.tslot >= 0) trace_mark(a, f.c.tslot);
      f.block(cntb);
      __syncthreads();
      f.b0 = b0;
      for_tiles<Cfg::TMAX>(b0, b0 + cntb, f);
    }
  }
  __syncthreads();
  trace_mark(a, 2);
  {
    int ng = C::level_gates(a, gs);
    load_wregs<Cfg::NG, KC>(w, gs, ng, ctx.unit0 + u, k0);
    if (a.bf16ops)  // dtype bf16 on FMA (TreeFC small batches): weights rounded
#pragma unroll
      for (int g = 0; g < 4; g++)
#pragma unroll
        for (int j = 0; j < KC; j++) w[g][j] = __bfloat162float(__float2bfloat16_rn(w[g][j]));
  }
  if constexpr (C::kLeafPost) {  // refactored GRU: the leaves' m once their h is complete
    grid_sync(a.bar, gridDim.x, epoch);
    const int lo0 = C::leaf_lo(first_leaf);
    int lo, hi;
    chunk_of(n - lo0, a.Gn, gn, lo, hi);
    typename C::LeafPost f{ctx, &meta, w, -1};
    for_tiles<Cfg::TMAX>(lo0 + lo, lo0 + hi, f);
  }
  // ---- internal batches: one grid barrier per level (and phase) -------------
  for (int l = 1; l < L; l++) {
    const int base = __ldg(a.lbeg + l), M = __ldg(a.lsize + l);
    int lo, hi;
    chunk_of(M, a.Gn, gn, lo, hi);
    for (int ph = 0; ph < C::kPhases; ph++) {
      if (C::kLeafPost && ph == 1 && l == L - 1) break;  // the top level's m feeds nobody
      const int slot = 3 + 2 * ((l - 1) * C::kPhases + ph);
      trace_mark(a, slot);
      grid_arrive(a.bar, epoch);
      typename C::Level f{ctx, &meta, w, ph, -1};
      if (hi > lo) {
        f.meta(base + lo, min(Cfg::TMAX, hi - lo));
        f.pre = base + lo;
      }
      grid_wait(a.bar, gridDim.x, epoch);
      trace_mark(a, slot + 1);
      f.c.tslot = a.trace ? 64 + 5 * ((l - 1) * C::kPhases + ph) : -1;
      for_tiles<Cfg::TMAX>(base + lo, base + hi, f);
    }
  }
  trace_mark(a, a.trace_slots - 2);
  trace_mark(a, a.trace_slots - 1);
  publish_and_exit(a);
}

template <int CELL, int H, int MAXC, class C>
bool rplan(int num_sms, FwdPlan *p, int *Gn, int *Gu) {
  constexpr size_t smem = RLayout<CELL, H, MAXC>::bytes;
  if (smem > 227 * 1024) return false;
  auto k = rw_kernel<CELL, H, MAXC, C>;
  static bool set_dev[kMaxDevices];  // per device (attributes are per context)
  const int dev = device_slot();
  if (dev < 0) return false;
  if (!set_dev[dev]) {
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return false;
    set_dev[dev] = true;
    cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    cudaGetLastError();
  }
  *Gu = H / kRUG;
  *Gn = num_sms / *Gu;
  if (*Gn < 1) return false;
  p->ctas = *Gn * *Gu;
  p->threads = kRThreads;
  p->smem = smem;
  p->kernel = (const void *)k;
  p->family = 2;
  return true;
}

template <int CELL, int H>
bool rplan_maxc(int maxc, int num_sms, FwdPlan *p, int *Gn, int *Gu, int variant = 0) {
  if constexpr (CELL == CX_TREEFC) {
    return rplan<CELL, H, 2, RTreeFc<H, 2>>(num_sms, p, Gn, Gu);
  } else {
    auto pick = [&](auto mc) {
      constexpr int MC = decltype(mc)::value;
      if constexpr (CELL == CX_TREELSTM) return rplan<CELL, H, MC, RTreeLstm<H, MC>>(num_sms, p, Gn, Gu);
      if constexpr (CELL == CX_TREEGRU) {
        // GRU cells share one configuration; the variant picks the schedule
        if (variant == 0) return rplan<CELL, H, MC, RTreeGru<H, MC, false>>(num_sms, p, Gn, Gu);
        if (variant == 1) return rplan<CELL, H, MC, RTreeGru<H, MC, true>>(num_sms, p, Gn, Gu);
        if (variant == 2) return rplan<CELL, H, MC, RTreeGruR<H, MC, false>>(num_sms, p, Gn, Gu);
        return rplan<CELL, H, MC, RTreeGruR<H, MC, true>>(num_sms, p, Gn, Gu);
      }
      if constexpr (CELL == CX_DAGRNN) return rplan<CELL, H, MC, RDagRnn<H, MC>>(num_sms, p, Gn, Gu);
      return false;
    };
    if (maxc <= 1) return pick(std::integral_constant<int, 1>{});
    if (maxc <= 2) return pick(std::integral_constant<int, 2>{});
    if (maxc <= 4) return pick(std::integral_constant<int, 4>{});
    return false;
  }
}

// GRU schedule: original (2 phases: 3 + 1 matvecs) or recursive refactoring
// (2 phases: 2 + 1 matvecs, plus the leaves' m) -- CX_GRU_REFACTOR=0/1
// overrides the default for measurement.
inline int gru_variant(bool simple) {
  const char *e = std::getenv("CX_GRU_REFACTOR");
  const bool refac = e ? e[0] == '1' : kGruRefactorDefault;
  return (simple ? 1 : 0) + (refac ? 2 : 0);
}

template <int H>
bool rplan_cell(int cell, int maxc, int num_sms, FwdPlan *p, int *Gn, int *Gu) {
  switch (cell) {
    case CX_TREELSTM: return rplan_maxc<CX_TREELSTM, H>(maxc, num_sms, p, Gn, Gu);
    // TreeGRU / SimpleTreeGRU x original / refactored schedule (gru_variant)
    case CX_TREEGRU: return rplan_maxc<CX_TREEGRU, H>(maxc, num_sms, p, Gn, Gu, gru_variant(false));
    case CX_SIMPLETREEGRU: return rplan_maxc<CX_TREEGRU, H>(maxc, num_sms, p, Gn, Gu, gru_variant(true));
    case CX_TREEFC: return rplan_maxc<CX_TREEFC, H>(maxc, num_sms, p, Gn, Gu);
    case CX_DAGRNN: return rplan_maxc<CX_DAGRNN, H>(maxc, num_sms, p, Gn, Gu);
  }
  return false;
}

}  // namespace

bool rw_plan(int cell, int H, int maxc, int num_sms, FwdPlan *p, int *Gn, int *Gu) {
  switch (H) {
    case 64: return rplan_cell<64>(cell, maxc, num_sms, p, Gn, Gu);
    case 128: return rplan_cell<128>(cell, maxc, num_sms, p, Gn, Gu);
    case 256: return rplan_cell<256>(cell, maxc, num_sms, p, Gn, Gu);
    case 512: return rplan_cell<512>(cell, maxc, num_sms, p, Gn, Gu);
  }
  return false;
}

}  // namespace cx
