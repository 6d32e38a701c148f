// smem_engine.cuh -- contraction engine with the CTA's weight rows resident in
// SHARED memory (forward.cu's general kernel and forward_big.cu's pipelined
// large-batch kernel): lane = hidden unit (32 per CTA), the 8 warps split the
// contraction dimension, partial sums are reduced through shared memory.
#pragma once
#include <cuda_runtime.h>

#include "fwd_common.cuh"

namespace cx {
namespace sme {
using namespace fwd;

constexpr int kWarps = kFwdThreads / 32;

// ---------------------------------------------------------------------------
// Product tables: product p adds W[gate g(p)] . vec[v(p)] into acc a(p).
// Vector index NV denotes the child sum h~ (computed on the fly).
// ---------------------------------------------------------------------------
struct PhLstmLeaf {  // [i; o; u] = W_iou x
  static constexpr int G0 = 0, NG = 3, NV = 1, NA = 3, NP = 3;
  static constexpr bool HT = false;
  __device__ static constexpr int g(int p) { return p; }
  __device__ static constexpr int v(int p) { return 0; }
  __device__ static constexpr int a(int p) { return p; }
};
template <int MAXC>
struct PhLstmLevel {  // [i; o; u] = U_iou h~ ; f_k = U_f h_k
  static constexpr int G0 = 0, NG = 4, NV = MAXC, NA = 3 + MAXC, NP = 3 + MAXC;
  static constexpr bool HT = true;
  __device__ static constexpr int g(int p) { return p < 3 ? p : 3; }
  __device__ static constexpr int v(int p) { return p < 3 ? MAXC : p - 3; }
  __device__ static constexpr int a(int p) { return p; }
};
struct PhGruLeaf {  // z = W_z x ; g = W_h x
  static constexpr int G0 = 0, NG = 2, NV = 1, NA = 2, NP = 2;
  static constexpr bool HT = false;
  __device__ static constexpr int g(int p) { return p; }
  __device__ static constexpr int v(int p) { return 0; }
  __device__ static constexpr int a(int p) { return p; }
};
template <int MAXC>
struct PhGruA {  // z = U_z h~ ; r_k = U_r h_k   (gates 0, 1 of the resident set)
  static constexpr int G0 = 0, NG = 2, NV = MAXC, NA = 1 + MAXC, NP = 1 + MAXC;
  static constexpr bool HT = true;
  __device__ static constexpr int g(int p) { return p < 1 ? 0 : 1; }
  __device__ static constexpr int v(int p) { return p < 1 ? MAXC : p - 1; }
  __device__ static constexpr int a(int p) { return p; }
};
struct PhGruB {  // U_h s   (gate 2 of the resident set; vector 0 = s)
  static constexpr int G0 = 2, NG = 1, NV = 1, NA = 1, NP = 1;
  static constexpr bool HT = false;
  __device__ static constexpr int g(int p) { return 0; }
  __device__ static constexpr int v(int p) { return 0; }
  __device__ static constexpr int a(int p) { return 0; }
};
struct PhFcLevel {  // W [h_l; h_r] = W_l h_l + W_r h_r
  static constexpr int G0 = 0, NG = 2, NV = 2, NA = 1, NP = 2;
  static constexpr bool HT = false;
  __device__ static constexpr int g(int p) { return p; }
  __device__ static constexpr int v(int p) { return p; }
  __device__ static constexpr int a(int p) { return 0; }
};
struct PhDagProj {  // W_x x
  static constexpr int G0 = 0, NG = 1, NV = 1, NA = 1, NP = 1;
  static constexpr bool HT = false;
  __device__ static constexpr int g(int p) { return 0; }
  __device__ static constexpr int v(int p) { return 0; }
  __device__ static constexpr int a(int p) { return 0; }
};
template <int MAXC>
struct PhDagLevel {  // U h~
  static constexpr int G0 = 0, NG = 1, NV = MAXC, NA = 1, NP = 1;
  static constexpr bool HT = true;
  __device__ static constexpr int g(int p) { return 0; }
  __device__ static constexpr int v(int p) { return MAXC; }
  __device__ static constexpr int a(int p) { return 0; }
};

// Lane = unit (u < 32), warp w covers k in [w H/8, (w+1) H/8).
// Ws: [gate][unit][H + 4] (row padding keeps float4 reads conflict-free);
// X : [T][NV][H] (broadcast reads).
template <class PH, int T>
__device__ __forceinline__ void fma_engine(const float *__restrict__ Ws, const float *__restrict__ X,
                                           int H, float (&acc)[PH::NA][T]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int HP = H + 4;
#pragma unroll
  for (int a = 0; a < PH::NA; a++)
#pragma unroll
    for (int t = 0; t < T; t++) acc[a][t] = 0.f;
  const int kc = H / kWarps;
  const int kb = warp * kc;
  constexpr int NG_USED = PH::NG;
  for (int k = kb; k < kb + kc; k += 4) {
    float4 w[NG_USED];
#pragma unroll
    for (int g = 0; g < NG_USED; g++)
      w[g] = *reinterpret_cast<const float4 *>(Ws + (size_t)((PH::G0 + g) * kUG + lane) * HP + k);
#pragma unroll
    for (int t = 0; t < T; t++) {
      float4 v[PH::NV + 1];
#pragma unroll
      for (int j = 0; j < PH::NV; j++)
        v[j] = *reinterpret_cast<const float4 *>(X + (size_t)(t * PH::NV + j) * H + k);
      if constexpr (PH::HT) {
        v[PH::NV] = v[0];
#pragma unroll
        for (int j = 1; j < PH::NV; j++) v[PH::NV] = add4(v[PH::NV], v[j]);
      }
#pragma unroll
      for (int p = 0; p < PH::NP; p++) fma4(acc[PH::a(p)][t], w[PH::g(p)], v[PH::v(p)]);
    }
  }
}

// Cross-warp reduction of the K-split partial sums through `red` (aliases X).
// Thread (t = tid / 32, u = lane) receives the full sums of node t, unit u.
template <int NA, int T>
__device__ __forceinline__ void reduce_acc(float *red, const float (&acc)[NA][T], float (&out)[NA]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();  // everyone is done reading X
#pragma unroll
  for (int a = 0; a < NA; a++)
#pragma unroll
    for (int t = 0; t < T; t++) red[((warp * NA + a) * T + t) * 32 + lane] = acc[a][t];
  __syncthreads();
  const int t = threadIdx.x >> 5;
#pragma unroll
  for (int a = 0; a < NA; a++) {
    float s = 0.f;
    if (t < T) {
#pragma unroll
      for (int w = 0; w < kWarps; w++) s += red[((w * NA + a) * T + t) * 32 + lane];
    }
    out[a] = s;
  }
}


}  // namespace sme
}  // namespace cx
