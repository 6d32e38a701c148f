// warp_engine.cuh -- warp-per-unit contraction engine of the cluster kernel
// (forward_cluster.cu), the latency path of small batches.
//
// A CTA of 16 warps owns 16 hidden units: warp w owns unit unit0 + w and lane c
// owns the k-chunk {128 m + 4 c + j : j < 4} (H >= 128) or {2 c, 2 c + 1}
// (H = 64) of EVERY gate row of that unit, held in registers (KC = H / 32
// floats per gate). A node's product W_g . vec is then a partial dot product
// per lane and a sum over the 32 lanes of ONE warp: the whole contraction of a
// tile -- and the gate epilogue that follows it -- needs no shared-memory
// reduction and no block barrier. The NA x T partial sums of a tile (T nodes)
// are reduced with a transposed butterfly: log2(T) halving steps (each lane
// keeps half of its values and adds its partner's other half: NA T / 2 + ...
// shuffles instead of 5 NA T), then 5 - log2(T) ordinary butterfly steps on NA
// values; afterwards the lanes of node t (t given by the halving bits) hold
// all NA sums of t and one of them runs t's epilogue.
//
// Reads of the gathered rows are conflict-free 128-bit loads (the 32 lanes of
// a load cover 512 contiguous bytes); every warp reads the whole tile, so a
// node costs 2 H rows x 16 warps of shared-memory bandwidth -- measured against
// the previous engine (k-chunk per half-warp, 16-warp shared-memory reduction,
// two __syncthreads per tile), see DESIGN.md §6.2d.
#pragma once
#include <cuda_runtime.h>

#include "rw_engine.cuh"

namespace cx {
namespace wq {
using namespace fwd;

template <int H>
struct WShape {
  static constexpr int KC = H / 32;  // floats per lane per row
  static_assert(KC == 2 || KC % 4 == 0, "H must be 64 or a multiple of 128");
};

// k index of register j of lane c
template <int KC>
__device__ __forceinline__ int kidx(int c, int j) {
  if constexpr (KC >= 4) return 128 * (j >> 2) + 4 * c + (j & 3);
  else return 2 * c + j;
}

// wreg[g][j] = W_g[row_u][kidx(lane, j)]   (global -> registers)
template <int NG, int KC>
__device__ __forceinline__ void load_wregs_w(float (&w)[4][KC], const rw::Gate *gs, int ng,
                                             int row_u, int lane) {
#pragma unroll
  for (int g = 0; g < NG; g++) {
    if (g < ng) {
      const float *src = gs[g].base + (size_t)(gs[g].r0 + row_u) * gs[g].ld + gs[g].c0;
      if constexpr (KC >= 4) {
#pragma unroll
        for (int m = 0; m < KC / 4; m++) {
          const float4 v = __ldg(reinterpret_cast<const float4 *>(src + 128 * m + 4 * lane));
          w[g][4 * m] = v.x; w[g][4 * m + 1] = v.y; w[g][4 * m + 2] = v.z; w[g][4 * m + 3] = v.w;
        }
      } else {
        const float2 v = __ldg(reinterpret_cast<const float2 *>(src + 2 * lane));
        w[g][0] = v.x; w[g][1] = v.y;
      }
    }
  }
}

template <int T>
struct Log2 {
  static constexpr int v = T <= 1 ? 0 : 1 + Log2<(T > 1 ? T / 2 : 1)>::v;
};
template <>
struct Log2<1> {
  static constexpr int v = 0;
};

// node of the tile whose sums this lane holds after wreduce<NA, T>
template <int T>
__device__ __forceinline__ int node_of_lane(int lane) {
  constexpr int LT = Log2<T>::v;
  int t = 0;
#pragma unroll
  for (int s = 0; s < LT; s++) t = (t << 1) | ((lane >> (4 - s)) & 1);
  return t;
}
// one lane per node runs the epilogue
template <int T>
__device__ __forceinline__ bool lead_lane(int lane) {
  constexpr int LT = Log2<T>::v;
  return (lane & ((32 >> LT) - 1)) == 0;
}

// The reduction needs no selects: lane l accumulates node t of the tile in
// slot t ^ g(l), g(l) = node_of_lane<T>(l) (it reads node t ^ g(l)'s rows
// when it fills slot t). At halving step S (mask 16 >> S) the live slots are
// [0, T >> S); every lane keeps the first half and sends the second, and the
// slot permutation makes the partner's second half exactly the nodes this lane
// keeps. The summation tree of a node is the same for every T (pairs over
// lane bit 4, then 3, ..., then 0), so results do not depend on the tile size.
template <int N, int S>
__device__ __forceinline__ void halve(float (&v)[N]) {
  constexpr int M = 16 >> S, Hf = (N >> S) / 2;
#pragma unroll
  for (int i = 0; i < Hf; i++) v[i] += __shfl_xor_sync(0xffffffffu, v[Hf + i], M);
}

template <int NA, int T>
__device__ __forceinline__ void wreduce(float (&v)[NA * T], float (&r)[NA]) {
  constexpr int LT = Log2<T>::v;
  static_assert((1 << LT) == T && LT <= 5, "T must be a power of two <= 32");
  if constexpr (LT >= 1) halve<NA * T, 0>(v);
  if constexpr (LT >= 2) halve<NA * T, 1>(v);
  if constexpr (LT >= 3) halve<NA * T, 2>(v);
  if constexpr (LT >= 4) halve<NA * T, 3>(v);
  if constexpr (LT >= 5) halve<NA * T, 4>(v);
#pragma unroll
  for (int s = LT; s < 5; s++) {
#pragma unroll
    for (int a = 0; a < NA; a++) v[a] += __shfl_xor_sync(0xffffffffu, v[a], 16 >> s);
  }
#pragma unroll
  for (int a = 0; a < NA; a++) r[a] = v[a];
}

// Contraction of a tile of T nodes (rows of X: NVX per node, H floats each)
// against this warp's register weights; on return r[a] holds accumulator a of
// (node node_of_lane<T>(lane), unit of this warp). HTS: X already carries h~
// (the sum of the NCH children) as row NV of every node; otherwise it is
// summed from the child rows in registers. Products are packed FFMA2 over
// (even, odd) k pairs -- half the FP32 issue slots of scalar FFMA, leaving
// room for the loads and shuffles (the FP32 pipe itself runs at the same
// rate either way); the two halves are added before the reduction.
template <class PH, int H, int T, bool HTS = false>
__device__ __forceinline__ void contract_w(const float *X, const float (&w)[4][WShape<H>::KC],
                                           float (&r)[PH::NA]) {
  constexpr int KC = WShape<H>::KC;
  constexpr int NV = PH::NV;
  constexpr int NVX = HTS ? NV + 1 : NV;
  constexpr int QB = KC >= 4 ? 4 : 2;  // k block held in registers at a time
  const int lane = threadIdx.x & 31;
  const int g = node_of_lane<T>(lane);
  float2 acc[PH::NA * T];
#pragma unroll
  for (int i = 0; i < PH::NA * T; i++) acc[i] = make_float2(0.f, 0.f);
#pragma unroll
  for (int t = 0; t < T; t++) {
    const float *Xt = X + (size_t)((t ^ g) * NVX) * H;  // slot t holds node t ^ g
#pragma unroll
    for (int q = 0; q < KC; q += QB) {
      float x[NV + 1][QB];
#pragma unroll
      for (int j = 0; j < NVX; j++) {
        const float *p = Xt + (size_t)j * H;
        if constexpr (QB == 4) {
          const float4 v = *reinterpret_cast<const float4 *>(p + 32 * q + 4 * lane);
          x[j][0] = v.x; x[j][1] = v.y; x[j][2] = v.z; x[j][3] = v.w;
        } else {
          const float2 v = *reinterpret_cast<const float2 *>(p + 2 * lane);
          x[j][0] = v.x; x[j][1] = v.y;
        }
      }
      if constexpr (PH::NCH > 0 && !HTS) {
#pragma unroll
        for (int e = 0; e < QB; e++) {
          float s = x[0][e];
#pragma unroll
          for (int j = 1; j < PH::NCH; j++) s += x[j][e];
          x[NV][e] = s;
        }
      }
#pragma unroll
      for (int p = 0; p < PH::NP; p++)
#pragma unroll
        for (int e = 0; e < QB; e += 2)
          acc[t * PH::NA + PH::a(p)] =
              ffma2(make_float2(w[PH::g(p)][q + e], w[PH::g(p)][q + e + 1]),
                    make_float2(x[PH::v(p)][e], x[PH::v(p)][e + 1]), acc[t * PH::NA + PH::a(p)]);
    }
  }
  float v[PH::NA * T];
#pragma unroll
  for (int i = 0; i < PH::NA * T; i++) v[i] = acc[i].x + acc[i].y;
  wreduce<PH::NA, T>(v, r);
}

}  // namespace wq
}  // namespace cx
