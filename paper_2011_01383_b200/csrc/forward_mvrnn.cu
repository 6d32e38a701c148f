// forward_mvrnn.cu -- MV-RNN persistent forward (Table 2; reading Q9).
//
// MV-RNN [Socher et al. 2012] carries a vector a and a matrix A per node:
//   leaf      (a, A) = (Emb[w], Mw[w])
//   internal  a_n = tanh(W [B a; A b] + beta),  A_n = W_M [A; B]
// (left child (a, A), right child (b, B)). The matrix product W_M [A; B] is
// 2 H^3 flops per node and dominates, so the cell is NODE-parallel (SURVEY
// §8(a) a7 "node-parallel at H=64"): every CTA keeps W and W_M resident in
// shared memory and evaluates whole nodes; each level's nodes are split
// across all CTAs, one grid barrier per level as in the other cells.
// Leaf matrices are never copied: a child that is a leaf (new id >=
// first_leaf -- the paper's one-comparison leaf check) is read
// straight from the Mw table.
#include <cuda_runtime.h>

#include "common.cuh"
#include "fwd_kernels.cuh"

namespace cx {
namespace {

constexpr int kT = kFwdThreads;

__device__ __forceinline__ void chunk_of_m(int M, int Gn, int g, int &lo, int &hi) {
  int q = M / Gn, r = M % Gn;
  lo = g * q + min(g, r);
  hi = lo + q + (g < r ? 1 : 0);
}
__device__ __forceinline__ int owner_of_m(int pos, int M, int Gn) {
  int q = M / Gn, r = M % Gn, big = r * (q + 1);
  return pos < big ? pos / (q + 1) : r + (pos - big) / q;
}

template <int H>
struct MvLayout {
  static constexpr int WP = 2 * H + 4;  // W row stride ([H][2H] padded)
  static constexpr int AP = H + 4;      // [A; B] row stride
  static constexpr size_t w = (size_t)H * WP;
  static constexpr size_t wmt = (size_t)2 * H * H;  // W_M^T [2H][H]
  static constexpr size_t ab = (size_t)2 * H * AP;
  static constexpr size_t vec = 4 * (size_t)H;      // a, b, p (2H)
  static constexpr size_t bytes = sizeof(float) * (w + wmt + ab + vec);
};

// CTAs per node at a level of M nodes (G CTAs): 4 or 2 when the level is that
// small and the per-thread row count RT divides
template <int RT>
__device__ __forceinline__ int split_factor(int M, int G) {
  return (RT >= 4 && 4 * M <= G) ? 4 : (RT >= 2 && 2 * M <= G) ? 2 : 1;
}

// rows [r0 + ti*RR, +RR) x cols [tj*4H/64 ..) of W_M [A; B] (thread (ti, tj) of 16 x 16)
template <int RR, int H, int AP>
__device__ __forceinline__ void mv_rows(const float *WMt, const float *AB, float *dst, int r0, int ti,
                                        int tj) {
  constexpr int RC = H / 16;  // columns per thread
  float acc[RR][RC];
#pragma unroll
  for (int r = 0; r < RR; r++)
#pragma unroll
    for (int c = 0; c < RC; c++) acc[r][c] = 0.f;
  for (int k = 0; k < 2 * H; k++) {
    float w[RR], x[RC];
#pragma unroll
    for (int r = 0; r < RR; r++) w[r] = WMt[(size_t)k * H + r0 + ti * RR + r];
#pragma unroll
    for (int c = 0; c < RC; c++) x[c] = AB[(size_t)k * AP + tj * RC + c];
#pragma unroll
    for (int r = 0; r < RR; r++)
#pragma unroll
      for (int c = 0; c < RC; c++) acc[r][c] = fmaf(w[r], x[c], acc[r][c]);
  }
#pragma unroll
  for (int r = 0; r < RR; r++)
#pragma unroll
    for (int c = 0; c < RC; c++) dst[(size_t)(r0 + ti * RR + r) * H + tj * RC + c] = acc[r][c];
}

template <int H>
__global__ void __launch_bounds__(kT, 1) mvrnn_kernel(FwdArgs a) {
  using Lay = MvLayout<H>;
  extern __shared__ __align__(16) float smem[];
  float *Ws = smem;              // W [H][WP]
  float *WMt = Ws + Lay::w;      // W_M^T [2H][H]
  float *AB = WMt + Lay::wmt;    // [A; B] [2H][AP]
  float *av = AB + Lay::ab;      // a [H]
  float *bv = av + H;            // b [H]
  float *pv = bv + H;            // p = [B a; A b] [2H]
  __shared__ int s_own, s_cin[2], s_leafw[2], s_isleaf[2];

  griddep_wait();
  if (*reinterpret_cast<volatile int *>(&a.hdr->status) != CX_OK) return;
  const int L = a.hdr->num_levels, first_leaf = a.hdr->first_leaf, n = a.n;
  const int tid = threadIdx.x, G = gridDim.x, g = blockIdx.x;
  const float *Mw = a.w[0], *W = a.w[1], *beta = a.w[2], *WM = a.w[3];
  const size_t HH = (size_t)H * H;
  unsigned epoch = 0;

  // resident weights (model persistence)
  for (int idx = tid; idx < H * 2 * H; idx += kT) {
    int i = idx / (2 * H), k = idx - i * 2 * H;
    Ws[i * Lay::WP + k] = __ldg(W + idx);
    WMt[(size_t)k * H + i] = __ldg(WM + idx);
  }

  // ---- leaf phase: (a, A) = (Emb[w], Mw[w]) -------------------------------
  {
    int lo, hi;
    chunk_of_m(n - first_leaf, G, g, lo, hi);
    for (int i = first_leaf + lo; i < first_leaf + hi; i++) {
      int own = __ldg(a.perm + i);
      int w = __ldg(a.words + own);
      if (w < 0 || w >= a.V) {
        if (tid == 0) latch_error(a.hdr, CX_E_WORD_RANGE, own);
        w = 0;
      }
      for (int u = tid; u < H; u += kT) a.h_out[(size_t)own * H + u] = __ldg(a.emb + (size_t)w * H + u);
      if (a.aux_out) {
        const float4 *src = reinterpret_cast<const float4 *>(Mw + w * HH);
        float4 *dst = reinterpret_cast<float4 *>(a.aux_out + own * HH);
        for (int q = tid; q < (int)(HH / 4); q += kT) dst[q] = __ldg(src + q);
      }
    }
  }

  // ---- internal levels ------------------------------------------------------
  constexpr int RT = H / 16;    // rows per thread in the A_n product

  constexpr int TPO = kT / H;   // threads per output of W p (k interleaved)
  const int ti = tid >> 4, tj = tid & 15;
  // node bookkeeping (depends on the linearization only): children, their
  // input ids, leaf flags and words; the first node of each level is loaded
  // (and its leaf children's Mw matrices prefetched into L2) while the CTA
  // waits at the level barrier
  auto load_node = [&](int i) {
    int own = __ldg(a.perm + i);
    s_own = own;
    int nc = 0;
    int c[2] = {-1, -1};
    for (int k = 0; k < a.maxc; k++) {
      int ck = __ldg(a.chn + (size_t)k * n + i);
      if (ck < 0) break;
      if (k < 2) c[k] = ck;
      nc++;
    }
    if (nc != 2) {
      latch_error(a.hdr, CX_E_ARITY, own);
      if (c[1] < 0) c[1] = c[0];
    }
    for (int k = 0; k < 2; k++) {
      s_cin[k] = __ldg(a.perm + c[k]);
      s_isleaf[k] = c[k] >= first_leaf;
      int w = 0;
      if (s_isleaf[k]) {
        w = __ldg(a.words + s_cin[k]);
        if (w < 0 || w >= a.V) w = 0;  // latched by the leaf phase
      }
      s_leafw[k] = w;
    }
  };
  for (int l = 1; l < L; l++) {
    grid_arrive(a.bar, epoch);
    const int base = __ldg(a.lbeg + l), M = __ldg(a.lsize + l);
    // a level with at most G/F nodes: F (4 or 2) CTAs per node, each computing
    // 1/F of the W_M [A; B] rows (the matrix product dominates the node)
    const int F = split_factor<RT>(M, G);
    const int half = g % F;  // this CTA's part of the node
    int lo, hi;
    if (F > 1) {
      lo = min(g / F, M);
      hi = min(lo + 1, M);
    } else {
      chunk_of_m(M, G, g, lo, hi);
    }
    if (tid == 0 && lo < hi) {
      load_node(base + lo);
      for (int k = 0; k < 2; k++)
        if (s_isleaf[k]) {
          const char *src = reinterpret_cast<const char *>(Mw + s_leafw[k] * HH);
          for (size_t off = 0; off < HH * sizeof(float); off += 128)
            asm volatile("prefetch.global.L2 [%0];" ::"l"(src + off));
        }
    }
    grid_wait(a.bar, G, epoch);
    for (int i = base + lo; i < base + hi; i++) {
      if (tid == 0 && i != base + lo) load_node(i);
      __syncthreads();
      // gather a, b and [A; B]
      for (int u = tid; u < 2 * H; u += kT) {
        int k = u / H, e = u - k * H;
        (k ? bv : av)[e] = __ldcg(a.h_out + (size_t)s_cin[k] * H + e);
      }
      for (int q = tid; q < (int)(2 * HH / 4); q += kT) {
        int k = q / (int)(HH / 4), e = 4 * (q - k * (int)(HH / 4));
        const float *src = s_isleaf[k] ? Mw + s_leafw[k] * HH : a.Abuf + (size_t)s_cin[k] * HH;
        float4 v = s_isleaf[k] ? __ldg(reinterpret_cast<const float4 *>(src + e)) : ldcg4(src + e);
        int r = e / H, col = e - r * H;
        *reinterpret_cast<float4 *>(AB + (size_t)(k * H + r) * Lay::AP + col) = v;
      }
      __syncthreads();
      // p = [B a; A b]: 2H outputs, 2 threads each (k interleaved)
      {
        int o = tid >> 1, half = tid & 1;
        float s = 0.f;
        if (o < 2 * H) {
          // o < H: (B a)[o] with B = AB rows H..2H-1 ; else (A b)[o-H] with A = rows 0..H-1
          const float *row = o < H ? AB + (size_t)(H + o) * Lay::AP : AB + (size_t)(o - H) * Lay::AP;
          const float *x = o < H ? av : bv;
          for (int k = half; k < H; k += 2) s = fmaf(row[k], x[k], s);
        }
        s += __shfl_xor_sync(0xffffffffu, s, 1);
        if (o < 2 * H && half == 0) pv[o] = s;
      }
      __syncthreads();
      // a_n = tanh(W p + beta): TPO threads per output, k interleaved
      {
        int o = tid / TPO, q = tid % TPO;
        float s = 0.f;
        for (int k = q; k < 2 * H; k += TPO) s = fmaf(Ws[o * Lay::WP + k], pv[k], s);
#pragma unroll
        for (int d = TPO / 2; d >= 1; d >>= 1) s += __shfl_xor_sync(0xffffffffu, s, d);
        if (q == 0 && half == 0) a.h_out[(size_t)s_own * H + o] = tanhf_(s + __ldg(beta + o));
      }
      // A_n = W_M [A; B]: thread (ti, tj) computes rows ti*RT.., cols tj*RT..
      // (split: this CTA's half of the rows, RT/2 per thread)
      float *An = a.Abuf + (size_t)s_own * HH;
      if constexpr (RT >= 4) {
        if (F == 4) mv_rows<RT / 4, H, Lay::AP>(WMt, AB, An, half * (H / 4), ti, tj);
      }
      if constexpr (RT >= 2) {
        if (F == 2) mv_rows<RT / 2, H, Lay::AP>(WMt, AB, An, half * (H / 2), ti, tj);
      }
      if (F == 1) mv_rows<RT, H, Lay::AP>(WMt, AB, An, 0, ti, tj);
      __syncthreads();
    }
  }

  // ---- packed roots (rows this CTA wrote) ------------------------------------
  if (a.root_out) {
    const int R = a.hdr->num_roots;
    for (int r = 0; r < R; r++) {
      int i = __ldg(a.roots + r);
      int lvl = __ldg(a.hnew + i);
      int own;
      if (lvl == 0) {
        own = owner_of_m(i - first_leaf, n - first_leaf, G);
      } else {
        const int Ml = __ldg(a.lsize + lvl), pos = i - __ldg(a.lbeg + lvl);
        const int F = split_factor<H / 16>(Ml, G);
        own = F > 1 ? F * pos : owner_of_m(pos, Ml, G);  // split levels: part 0 wrote h
      }
      if (own != g) continue;
      int src = __ldg(a.perm + i);
      for (int u = tid; u < H; u += kT)
        a.root_out[(size_t)r * H + u] = __ldcg(a.h_out + (size_t)src * H + u);
    }
  }

  __syncthreads();
  if (tid == 0) {
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

template <int H>
bool plan_h(int num_sms, FwdPlan *p, int *Gn, int *Gu) {
  auto k = mvrnn_kernel<H>;
  size_t smem = MvLayout<H>::bytes;
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
  *Gn = num_sms;
  *Gu = 1;
  p->ctas = num_sms;
  p->threads = kT;
  p->smem = smem;
  p->kernel = (const void *)k;
  p->family = 5;
  return true;
}

}  // namespace

bool mvrnn_plan(int H, int num_sms, FwdPlan *plan, int *Gn, int *Gu) {
  switch (H) {
    case 16: return plan_h<16>(num_sms, plan, Gn, Gu);
    case 32: return plan_h<32>(num_sms, plan, Gn, Gu);
    case 64: return plan_h<64>(num_sms, plan, Gn, Gu);
    default: return false;
  }
}

}  // namespace cx
