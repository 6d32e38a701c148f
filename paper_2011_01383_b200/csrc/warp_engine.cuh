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

// packed fp32 pairs (b64 registers) for the FFMA2 / FADD2 datapath
typedef unsigned long long f2;
__device__ __forceinline__ f2 f2pack(float lo, float hi) {
  f2 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ float f2sum(f2 a) {
  float lo, hi;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(a));
  return lo + hi;
}
__device__ __forceinline__ f2 f2fma(f2 a, f2 b, f2 c) {
  f2 d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ f2 f2add(f2 a, f2 b) {
  f2 d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}

template <int H>
struct WShape {
  static constexpr int KC = H / 32;  // floats per lane per row
  static_assert(KC == 2 || KC % 4 == 0, "H must be 64 or a multiple of 128");
};

// Thread roles, UW = units per warp (1, 2 or 4). The CTA's 16 units form
// 16 / UW unit groups of UW units; the UW warps of a group split K in UW
// parts (warp w: group w % (16 / UW), part w / (16 / UW)); inside a warp,
// lanes [LPU u, LPU (u + 1)) (LPU = 32 / UW lanes per unit) hold unit u of the
// group, lane c of them the conflict-free k-chunk
//   k = part * H / UW + 4 LPU m + 4 c + j   (H / UW >= 4 LPU; KC = 4 m + j)
//   k = part * H / UW + 2 c + j             (H = 64)
// Every warp then reads H / UW floats of each row (the UW units of a lane
// group share each load), i.e. 16 warps x H / UW per row instead of 16 x H.
template <int UW>
struct Roles {
  static_assert(UW == 1 || UW == 2 || UW == 4, "UW in {1, 2, 4}");
  static constexpr int LPU = 32 / UW, NGRP = 16 / UW;
  static constexpr int LG = UW == 1 ? 5 : UW == 2 ? 4 : 3;  // log2(LPU)
  int grp, part, ul, c;  // unit group, k part, unit in the group, lane in the unit
  __device__ __forceinline__ Roles(int warp, int lane)
      : grp(warp % NGRP), part(warp / NGRP), ul(lane >> LG), c(lane & (LPU - 1)) {}
  __device__ __forceinline__ int unit() const { return grp * UW + ul; }  // unit in the CTA
};

// offset of register block m (4 floats) / the float2 of lane c inside part p
template <int H, int UW>
__device__ __forceinline__ int koff(int part, int c, int m) {
  constexpr int KC = WShape<H>::KC, LPU = 32 / UW;
  if constexpr (KC >= 4) return part * (H / UW) + 4 * LPU * m + 4 * c;
  else return part * (H / UW) + 2 * c;
}

// wreg[g][j] = W_g[row_u][k(j)] for this thread's unit row and k-chunk
// (k pairs: w[g][i] = (W_g[.][k(2i)], W_g[.][k(2i + 1)]))
template <int H>
using WRegs = f2[4][WShape<H>::KC / 2];
template <int NG, int H, int UW>
__device__ __forceinline__ void load_wregs_w(WRegs<H> &w, const rw::Gate *gs, int ng, int row_u,
                                             const Roles<UW> &ro) {
  constexpr int KC = WShape<H>::KC;
#pragma unroll
  for (int g = 0; g < NG; g++) {
    if (g < ng) {
      const float *src = gs[g].base + (size_t)(gs[g].r0 + row_u) * gs[g].ld + gs[g].c0;
      if constexpr (KC >= 4) {
#pragma unroll
        for (int m = 0; m < KC / 4; m++) {
          const float4 v = __ldg(reinterpret_cast<const float4 *>(src + koff<H, UW>(ro.part, ro.c, m)));
          w[g][2 * m] = f2pack(v.x, v.y);
          w[g][2 * m + 1] = f2pack(v.z, v.w);
        }
      } else {
        const float2 v = __ldg(reinterpret_cast<const float2 *>(src + koff<H, UW>(ro.part, ro.c, 0)));
        w[g][0] = f2pack(v.x, v.y);
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

// node of the tile whose sums this lane holds after the reduction (bits of the
// lane inside its unit's lane group, most significant first)
template <int T, int UW>
__device__ __forceinline__ int node_of_lane(int lane) {
  constexpr int LT = Log2<T>::v, LG = Roles<UW>::LG;
  int t = 0;
#pragma unroll
  for (int s = 0; s < LT; s++) t = (t << 1) | ((lane >> (LG - 1 - s)) & 1);
  return t;
}
// one lane per (unit, node) holds the reduced sums
template <int T, int UW>
__device__ __forceinline__ bool lead_lane(int lane) {
  constexpr int LT = Log2<T>::v, LPU = Roles<UW>::LPU;
  return (lane & ((LPU >> LT) - 1)) == 0;
}

// The reduction needs no selects: lane l accumulates node t of the tile in
// slot t ^ g(l), g(l) = node_of_lane(l) (it reads node t ^ g(l)'s rows when
// it fills slot t). At halving step S (mask LPU / 2 >> S) the live slots are
// [0, T >> S); every lane keeps the first half and sends the second, and the
// slot permutation makes the partner's second half exactly the nodes this lane
// keeps. The summation tree of a node is the same for every T (pairs over the
// lane bits from the highest down), so results do not depend on the tile size.
template <int N, int S, int LPU>
__device__ __forceinline__ void halve(float (&v)[N]) {
  constexpr int M = (LPU / 2) >> S, Hf = (N >> S) / 2;
#pragma unroll
  for (int i = 0; i < Hf; i++) v[i] += __shfl_xor_sync(0xffffffffu, v[Hf + i], M);
}

template <int NA, int T, int UW>
__device__ __forceinline__ void wreduce(float (&v)[NA * T], float (&r)[NA]) {
  constexpr int LT = Log2<T>::v, LG = Roles<UW>::LG, LPU = Roles<UW>::LPU;
  static_assert((1 << LT) == T && LT <= LG, "T must be a power of two <= lanes per unit");
  if constexpr (LT >= 1) halve<NA * T, 0, LPU>(v);
  if constexpr (LT >= 2) halve<NA * T, 1, LPU>(v);
  if constexpr (LT >= 3) halve<NA * T, 2, LPU>(v);
  if constexpr (LT >= 4) halve<NA * T, 3, LPU>(v);
  if constexpr (LT >= 5) halve<NA * T, 4, LPU>(v);
#pragma unroll
  for (int s = LT; s < LG; s++) {
#pragma unroll
    for (int a = 0; a < NA; a++) v[a] += __shfl_xor_sync(0xffffffffu, v[a], (LPU / 2) >> s);
  }
#pragma unroll
  for (int a = 0; a < NA; a++) r[a] = v[a];
}

__device__ __forceinline__ void named_bar_sync(int id, int threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

// Contraction of a tile of T nodes (rows of X: NVX per node, H floats each)
// against this thread's register weights. Returns true on the lanes that hold
// the final sums of (node node_of_lane<T, UW>(lane), unit ro.unit()) in r[a]
// (the lead lanes of the part-0 warps). HTS: X already carries h~ (the sum of
// the NCH children) as row NV of every node; otherwise it is summed from the
// child rows in registers. Products are packed FFMA2 over (even, odd) k pairs
// -- half the FP32 issue slots of scalar FFMA, leaving room for the loads and
// shuffles; the two halves are added before the reduction. UW > 1: the parts
// meet through `xs` (>= 16 (UW - 1) NA T floats) and one named barrier per unit
// group (ids 1 .. 16 / UW), parts added in order 0, 1, ...
template <class PH, int H, int T, int UW, bool HTS = false>
__device__ __forceinline__ bool contract_w(const float *X, const WRegs<H> &w, float (&r)[PH::NA],
                                           const Roles<UW> &ro, float *xs) {
  constexpr int KC = WShape<H>::KC;
  constexpr int NV = PH::NV;
  constexpr int NVX = HTS ? NV + 1 : NV;
  constexpr int QB = KC >= 4 ? 4 : 2;  // k block held in registers at a time
  constexpr int QP = QB / 2;           // ... in f2 pairs
  const int lane = threadIdx.x & 31;
  const int g = node_of_lane<T, UW>(lane);
  f2 acc[PH::NA * T];
#pragma unroll
  for (int i = 0; i < PH::NA * T; i++) acc[i] = 0ull;  // (+0.0f, +0.0f)
#pragma unroll
  for (int t = 0; t < T; t++) {
    const float *Xt = X + (size_t)((t ^ g) * NVX) * H;  // slot t holds node t ^ g
#pragma unroll
    for (int q = 0; q < KC; q += QB) {
      f2 x[NV + 1][QP];
      const int off = koff<H, UW>(ro.part, ro.c, q / 4);
#pragma unroll
      for (int j = 0; j < NVX; j++) {
        const float *p = Xt + (size_t)j * H + off;
        if constexpr (QB == 4) {
          const float4 v = *reinterpret_cast<const float4 *>(p);
          x[j][0] = f2pack(v.x, v.y);
          x[j][1] = f2pack(v.z, v.w);
        } else {
          const float2 v = *reinterpret_cast<const float2 *>(p);
          x[j][0] = f2pack(v.x, v.y);
        }
      }
      if constexpr (PH::NCH > 0 && !HTS) {
#pragma unroll
        for (int e = 0; e < QP; e++) {
          f2 s = x[0][e];
#pragma unroll
          for (int j = 1; j < PH::NCH; j++) s = f2add(s, x[j][e]);
          x[NV][e] = s;
        }
      }
#pragma unroll
      for (int p = 0; p < PH::NP; p++)
#pragma unroll
        for (int e = 0; e < QP; e++)
          acc[t * PH::NA + PH::a(p)] = f2fma(w[PH::g(p)][q / 2 + e], x[PH::v(p)][e], acc[t * PH::NA + PH::a(p)]);
    }
  }
  float v[PH::NA * T];
#pragma unroll
  for (int i = 0; i < PH::NA * T; i++) v[i] = f2sum(acc[i]);
  wreduce<PH::NA, T, UW>(v, r);
  const bool lead = lead_lane<T, UW>(lane);
  if constexpr (UW > 1) {
    // partial sums of parts 1 .. UW-1 -> xs, then part 0 adds them in order
    float *xg = xs + (size_t)ro.grp * (UW - 1) * UW * T * PH::NA;
    const int slot = (ro.ul * T + g) * PH::NA;
    if (ro.part > 0 && lead) {
#pragma unroll
      for (int a = 0; a < PH::NA; a++) xg[(size_t)(ro.part - 1) * UW * T * PH::NA + slot + a] = r[a];
    }
    named_bar_sync(1 + ro.grp, 32 * UW);
    if (ro.part == 0 && lead) {
#pragma unroll
      for (int pp = 1; pp < UW; pp++)
#pragma unroll
        for (int a = 0; a < PH::NA; a++) r[a] += xg[(size_t)(pp - 1) * UW * T * PH::NA + slot + a];
    }
    return ro.part == 0 && lead;
  }
  return lead;
}

}  // namespace wq
}  // namespace cx
