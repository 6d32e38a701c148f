// rw_engine.cuh -- the register-resident-weight contraction engine shared by
// forward_rw.cu (grid of unit groups x node groups) and forward_cluster.cu
// (one thread-block cluster per group of structures).
//
// A CTA of 16 warps owns 16 hidden units; thread (u = lane & 15, chunk =
// 2 warp + lane / 16) holds W[g][unit0 + u][chunk * KC, +KC) of every gate g in
// registers (KC = H / 32). contract() multiplies a tile of gathered rows by
// those registers (packed FFMA2 over k pairs), reduces the two half-warps with
// one shuffle and the 16 warps through shared memory.
#pragma once
#include <cuda_runtime.h>

#include "fwd_common.cuh"

namespace cx {
namespace rw {
using namespace fwd;

constexpr int kRUG = 16;            // hidden units per CTA
constexpr int kRNW = 16;            // warps per CTA
constexpr int kRThreads = 32 * kRNW;
constexpr int kLeafBlock = 32;      // leaves per bookkeeping + gather block (rw kernel)

// ---------------------------------------------------------------------------
// Product tables. Vectors 0..NV-1 are gathered rows; vector NV is h~, the sum
// of the first NCH vectors (children). Product p adds W[g(p)] . vec[v(p)] into
// accumulator a(p).
// ---------------------------------------------------------------------------
template <int NG_, int NV_, int NCH_, int NA_, int NP_>
struct PhBase {
  static constexpr int NG = NG_, NV = NV_, NCH = NCH_, NA = NA_, NP = NP_;
};
struct RLstmLeaf : PhBase<3, 1, 0, 3, 3> {  // [i; o; u] = W_iou x
  __device__ static constexpr int g(int p) { return p; }
  __device__ static constexpr int v(int p) { return 0; }
  __device__ static constexpr int a(int p) { return p; }
};
template <int MAXC>
struct RLstmLevel : PhBase<4, MAXC, MAXC, 3 + MAXC, 3 + MAXC> {  // U_iou h~ ; U_f h_k
  __device__ static constexpr int g(int p) { return p < 3 ? p : 3; }
  __device__ static constexpr int v(int p) { return p < 3 ? MAXC : p - 3; }
  __device__ static constexpr int a(int p) { return p; }
};
struct RGruLeaf : PhBase<2, 1, 0, 2, 2> {  // W_z x ; W_h x
  __device__ static constexpr int g(int p) { return p; }
  __device__ static constexpr int v(int p) { return 0; }
  __device__ static constexpr int a(int p) { return p; }
};
template <int MAXC>
struct RGruA : PhBase<3, MAXC, MAXC, 1 + MAXC, 1 + MAXC> {  // U_z h~ ; U_r h_k
  __device__ static constexpr int g(int p) { return p < 1 ? 0 : 1; }
  __device__ static constexpr int v(int p) { return p < 1 ? MAXC : p - 1; }
  __device__ static constexpr int a(int p) { return p; }
};
struct RGruB : PhBase<3, 1, 0, 1, 1> {  // U_h s
  __device__ static constexpr int g(int p) { return 2; }
  __device__ static constexpr int v(int p) { return 0; }
  __device__ static constexpr int a(int p) { return 0; }
};
struct RFcLevel : PhBase<2, 2, 0, 1, 2> {  // W_l h_l + W_r h_r
  __device__ static constexpr int g(int p) { return p; }
  __device__ static constexpr int v(int p) { return p; }
  __device__ static constexpr int a(int p) { return 0; }
};
struct RDagLeaf : PhBase<2, 1, 0, 1, 1> {  // W_x x (gate 0 of {W_x, U})
  __device__ static constexpr int g(int p) { return 0; }
  __device__ static constexpr int v(int p) { return 0; }
  __device__ static constexpr int a(int p) { return 0; }
};
template <int MAXC>
struct RDagLevel : PhBase<2, MAXC + 1, MAXC, 1, 2> {  // W_x x + U h~  (x = vector MAXC)
  __device__ static constexpr int g(int p) { return p == 0 ? 1 : 0; }
  __device__ static constexpr int v(int p) { return p == 0 ? MAXC + 1 : MAXC; }
  __device__ static constexpr int a(int p) { return 0; }
};

// ---------------------------------------------------------------------------
// Per-cell configuration (host + device): level/leaf gates, node tile,
// gathered vectors, accumulators.
// ---------------------------------------------------------------------------
template <int CELL, int H, int MAXC>
struct RCfg;
template <int H, int MAXC>
struct RCfg<CX_TREELSTM, H, MAXC> {
  static constexpr int NG = 4, TMAX = H >= 512 ? 4 : 8, NVMAX = MAXC, NAMAX = 3 + MAXC;
};
template <int H, int MAXC>
struct RCfg<CX_TREEGRU, H, MAXC> {
  static constexpr int NG = 3, TMAX = 8, NVMAX = MAXC, NAMAX = 1 + MAXC;
};
template <int H, int MAXC>
struct RCfg<CX_TREEFC, H, MAXC> {
  static constexpr int NG = 2, TMAX = 16, NVMAX = 2, NAMAX = 1;
};
template <int H, int MAXC>
struct RCfg<CX_DAGRNN, H, MAXC> {
  static constexpr int NG = 2, TMAX = 16, NVMAX = MAXC + 1, NAMAX = 1;
};

template <int CELL, int H, int MAXC>
struct RLayout {
  using C = RCfg<CELL, H, MAXC>;
  // X holds a level tile's gathered rows, or a leaf block of kLeafBlock rows
  // (one bookkeeping pass + one Emb gather per block; fewer, larger blocks
  // put fewer dependent global round trips on the leaf phase's path)
  static constexpr size_t tile_rows = (size_t)C::TMAX * (C::NVMAX > 2 ? C::NVMAX : 2);
  static constexpr size_t x_floats = (tile_rows > kLeafBlock ? tile_rows : kLeafBlock) * H;
  static constexpr size_t red_floats = (size_t)kRNW * C::NAMAX * C::TMAX * kRUG;
  static constexpr size_t red2_floats = (size_t)C::NAMAX * C::TMAX * kRUG;
  static constexpr size_t cv_floats = (size_t)C::TMAX * kMaxC * kRUG;
  static constexpr size_t bytes = sizeof(float) * (x_floats + red_floats + red2_floats + cv_floats);
};

template <int H>
struct RShape {
  static constexpr int KC = H / (2 * kRNW);  // contraction chunk per thread
};

struct Gate {
  const float *base;
  int r0, ld, c0;
};

// wreg[g][j] = W_g[unit0 + u][k0 + j]   (global -> registers)
template <int NG, int KC>
__device__ __forceinline__ void load_wregs(float (&w)[4][KC], const Gate *gs, int ng, int row_u,
                                           int k0) {
#pragma unroll
  for (int g = 0; g < NG; g++) {
    if (g < ng) {
      const float *src = gs[g].base + (size_t)(gs[g].r0 + row_u) * gs[g].ld + gs[g].c0 + k0;
      if constexpr (KC % 4 == 0) {
#pragma unroll
        for (int j = 0; j < KC; j += 4) {
          float4 v = __ldg(reinterpret_cast<const float4 *>(src + j));
          w[g][j] = v.x; w[g][j + 1] = v.y; w[g][j + 2] = v.z; w[g][j + 3] = v.w;
        }
      } else {
#pragma unroll
        for (int j = 0; j < KC; j++) w[g][j] = __ldg(src + j);
      }
    }
  }
}

struct RCtx {
  const FwdArgs *a;
  float *X, *red, *red2, *cv;
  const float *bias;  // [gate][16]
  int gn, gu, unit0;
  bool latch;
  int tslot;  // debug trace slot base for this tile (-1 = off)
};

// Contraction of one tile against the register-resident weights, reduced to
// full sums: on return s[a] (threads tid < T*16: node t = tid/16, unit u =
// tid%16) holds accumulator a of that (node, unit).
// HTS: X already holds the child sum h~ as an extra row after the NV gathered
// rows of every node (computed once per tile instead of once per unit lane).
template <class PH, int H, int T, bool HTS = false>
__device__ __forceinline__ void contract(const RCtx &c, const float *X,
                                         const float (&w)[4][RShape<H>::KC], float (&s)[PH::NA]) {
  constexpr int KC = RShape<H>::KC;
  constexpr int NV = PH::NV;
  constexpr int NVX = HTS ? NV + 1 : NV;  // rows per node in X
  static_assert(KC % 2 == 0, "packed FFMA2 needs an even k chunk");
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int u = lane & 15, ksub = lane >> 4;
  const int k0 = (warp * 2 + ksub) * KC;
  // even/odd k partial sums packed in float2 -> one FFMA2 per two products
  float2 acc2[PH::NA][T];
#pragma unroll
  for (int a = 0; a < PH::NA; a++)
#pragma unroll
    for (int t = 0; t < T; t++) acc2[a][t] = make_float2(0.f, 0.f);
  constexpr int QB = KC < 4 ? KC : 4;  // k-block held in registers at a time
#pragma unroll
  for (int t = 0; t < T; t++) {
#pragma unroll
    for (int q = 0; q < KC; q += QB) {
      float x[NV + 1][QB];
#pragma unroll
      for (int j = 0; j < NVX; j++) {
        const float *p = X + (size_t)(t * NVX + j) * H + k0 + q;
        if constexpr (QB == 4) {
          float4 v = *reinterpret_cast<const float4 *>(p);
          x[j][0] = v.x; x[j][1] = v.y; x[j][2] = v.z; x[j][3] = v.w;
        } else {
          float2 v = *reinterpret_cast<const float2 *>(p);
          x[j][0] = v.x; x[j][1] = v.y;
        }
      }
      if constexpr (PH::NCH > 0 && !HTS) {
#pragma unroll
        for (int e = 0; e < QB; e++) {
          float sum = x[0][e];
#pragma unroll
          for (int j = 1; j < PH::NCH; j++) sum += x[j][e];
          x[NV][e] = sum;
        }
      }
#pragma unroll
      for (int p = 0; p < PH::NP; p++)
#pragma unroll
        for (int e = 0; e < QB; e += 2)
          acc2[PH::a(p)][t] = ffma2(make_float2(w[PH::g(p)][q + e], w[PH::g(p)][q + e + 1]),
                                    make_float2(x[PH::v(p)][e], x[PH::v(p)][e + 1]),
                                    acc2[PH::a(p)][t]);
    }
  }
  float acc[PH::NA][T];
#pragma unroll
  for (int a = 0; a < PH::NA; a++)
#pragma unroll
    for (int t = 0; t < T; t++) acc[a][t] = acc2[a][t].x + acc2[a][t].y;
  // half-warps hold the two chunks of each unit: combine with one shuffle, then
  // across the 16 warps through shared memory. Partials are laid out
  // [warp][acc][unit][node] so a lane stores its nodes with float4 stores; the
  // two half-warps (which hold identical sums) split the accumulators.
#pragma unroll
  for (int a = 0; a < PH::NA; a++)
#pragma unroll
    for (int t = 0; t < T; t++) acc[a][t] += __shfl_xor_sync(0xffffffffu, acc[a][t], 16);
#pragma unroll
  for (int a = 0; a < PH::NA; a++) {
    if ((a & 1) != ksub) continue;
    float *dst = c.red + ((size_t)(warp * PH::NA + a) * kRUG + u) * T;
    if constexpr (T % 4 == 0) {
#pragma unroll
      for (int t = 0; t < T; t += 4)
        *reinterpret_cast<float4 *>(dst + t) = make_float4(acc[a][t], acc[a][t + 1], acc[a][t + 2], acc[a][t + 3]);
    } else {
#pragma unroll
      for (int t = 0; t < T; t++) dst[t] = acc[a][t];
    }
  }
  __syncthreads();
  if (c.tslot >= 0) trace_mark(*c.a, c.tslot + 2);
  constexpr int QW = T % 4 == 0 ? 4 : 1;  // floats per partial-sum load
  constexpr int G = PH::NA * kRUG * T / QW;
  constexpr int WS = PH::NA * kRUG * T;     // floats per warp's block
  for (int g = threadIdx.x; g < G; g += blockDim.x) {
    if constexpr (QW == 4) {
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int ww = 0; ww < kRNW; ww++) {
        const float4 x = *reinterpret_cast<const float4 *>(c.red + (size_t)ww * WS + 4 * g);
        v.x += x.x; v.y += x.y; v.z += x.z; v.w += x.w;
      }
      *reinterpret_cast<float4 *>(c.red2 + 4 * g) = v;
    } else {
      float v = 0.f;
#pragma unroll
      for (int ww = 0; ww < kRNW; ww++) v += c.red[(size_t)ww * WS + g];
      c.red2[g] = v;
    }
  }
  __syncthreads();
  const int t = threadIdx.x >> 4, uu = threadIdx.x & 15;
#pragma unroll
  for (int a = 0; a < PH::NA; a++) s[a] = t < T ? c.red2[(a * kRUG + uu) * T + t] : 0.f;
  if (c.tslot >= 0) trace_mark(*c.a, c.tslot + 3);
}


}  // namespace rw
}  // namespace cx
