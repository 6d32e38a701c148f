// forward_single.cu -- the one-launch path for tiny forests and element-wise
// cells: cx_linearize_forward as ONE kernel in which every
// CTA linearizes the batch in its own shared memory (lin_single.cuh, CTA 0
// also writes the cx_linearization outputs) and then evaluates the structures
// it owns (structure g -> CTA g mod #CTAs; structures are independent, P.3
// P:759-761) with __syncthreads as the level barrier: no grid barrier and no
// second launch.
//
// Recursion unrolling (§3.1, evaluated P:1617-1621). For
// TreeRNN (Listing 1, h = tanh(h_l + h_r)) every hidden unit is an independent
// recursion, so a thread that owns (node, unit) can compute its children's
// unit inline, keeping them in registers ("reuse of the children's hidden
// state via fast on-chip caches") -- the paper's "computation for one node in
// one GPU thread block, thus avoiding additional global barriers when
// unrolled". UNROLL = U evaluates U levels per barrier: a node at the top of a
// U-level band recomputes nothing (trees: every node has one parent) and a
// node whose parent lies outside the band is finished on its own. With U = 1
// it is the level-synchronous schedule of Listing 2. TreeFC mixes units
// (h = tanh(W [h_l; h_r] + b)), so a band would need its children's full
// vectors: it runs level-synchronously (U = 1) only.
//
// State: the rows of every node live in shared memory (new numbering) when
// n H floats fit, and are also written to h_out (input numbering) for the
// caller; otherwise h_out itself is the state (a CTA only reads rows it wrote,
// ordered by __syncthreads).
#include <cuda_runtime.h>

#include <cstdlib>

#include "fwd_common.cuh"
#include "lin_single.cuh"
#include "lin_warp.cuh"

namespace cx {
namespace {
using namespace fwd;

constexpr int kScThreads = 256;
constexpr int kScCnt = 2048;  // linearizer count table (ints)

__host__ __device__ inline size_t sc_smem_ints(int n, int maxc) {
  return lin_sm_ints(n, maxc, kScCnt) + (size_t)maxc * n + 2 * (size_t)n + 64;
}
constexpr size_t kScSmem = 200 * 1024;  // dynamic shared memory of the kernel

template <int CELL, int UNROLL>
__global__ void __launch_bounds__(kScThreads) sc_kernel(FwdArgs a) {
  extern __shared__ __align__(16) int sm[];
  const int n = a.n, maxc = a.maxc, H = a.H, tid = threadIdx.x;
  unsigned long long *ferr = reinterpret_cast<unsigned long long *>(&a.bar->pad[0]);
  trace_mark(a, 0);
  LinPrefetch pf{a.words, a.emb, H, a.V};
  int *chn = sm + lin_sm_ints(n, maxc, kScCnt);
  const bool tiny = lin_warp_applies(n, maxc);
  if (tiny && tid >= 32) {
    // warp 0 linearizes; the others fetch the word ids and pull the nodes'
    // embedding rows into L2 meanwhile (fire-and-forget prefetches)
    for (int v = tid - 32; v < n; v += blockDim.x - 32) {
      const int wd = __ldg(a.words + v);
      if (wd >= 0 && wd < a.V)
        for (int q = 0; q < H; q += 32) asm volatile("prefetch.global.L2 [%0];" ::"l"(a.emb + (size_t)wd * H + q));
    }
  }
  const LinOut lo = tiny ? lin_warp_body(a.lin, sm, blockIdx.x == 0, chn)
                         : lin_single_body(a.lin, sm, kScCnt, blockIdx.x == 0, chn, pf);
  trace_mark(a, 20);
  if (!lo.ok) {
    fused_exit(a, ferr);
    return;
  }
  const LinSm ls = lin_carve(sm, n, maxc);
  const int L = lo.L, G = gridDim.x;
  int *lev = chn + (size_t)maxc * n;  // level of every new id
  for (int l = 0; l < L; l++)
    for (int i = ls.lb[l] + tid; i < ls.lb[l] + ls.ls[l]; i += blockDim.x) lev[i] = l;
  // a DAG whose structures share nodes: CTA 0 evaluates everything
  bool one = false;
  if (a.kind == CX_DAG) {
    bool bad = false;
    for (int i = tid; i < n; i += blockDim.x)
      for (int k = 0; k < maxc; k++) {
        const int c = chn[(size_t)k * n + i];
        if (c >= 0 && ls.sid[c] != ls.sid[i]) bad = true;
      }
    one = __syncthreads_or(bad);
  } else {
    __syncthreads();
  }
  auto mine = [&](int i) { return (one ? 0 : ls.sid[i] % G) == (int)blockIdx.x; };
  trace_mark(a, 21);
  // state rows: shared memory when they fit (after the ints), else h_out
  float *hs = reinterpret_cast<float *>(lev + n + 4);
  const bool on_chip = (size_t)(reinterpret_cast<char *>(hs + (size_t)n * H) -
                                reinterpret_cast<char *>(sm)) <= dynamic_smem_bytes();
  auto hrow = [&](int i) { return on_chip ? hs + (size_t)i * H : a.h_out + (size_t)ls.perm[i] * H; };
  auto hput = [&](int i, int u, float v) {  // state + caller output
    if (on_chip) {
      hs[(size_t)i * H + u] = v;
      a.h_out[(size_t)ls.perm[i] * H + u] = v;
    } else {
      a.h_out[(size_t)ls.perm[i] * H + u] = v;
    }
  };
  auto latch_word = [&](int own) {
    atomicMax(ferr, ~(((unsigned long long)CX_E_WORD_RANGE << 32) | (unsigned)own));
  };
  // binary cells: both children present (else CX_E_ARITY, clamped)
  auto kids = [&](int i, int &c0, int &c1) {
    c0 = chn[i];
    c1 = maxc > 1 ? chn[n + i] : -1;
    if (c0 < 0 || c1 < 0) {
      atomicMax(ferr, ~(((unsigned long long)CX_E_ARITY << 32) | (unsigned)ls.perm[i]));
      if (c0 < 0) c0 = i;  // memory safety only: outputs are unspecified
      if (c1 < 0) c1 = c0;
    }
  };
  // ---- leaves: h = Emb[word] (TreeRNN / TreeFC leaves are a pure gather) ----
  {
    const int b = ls.lb[0], e = b + ls.ls[0];
    for (int idx = tid; idx < (e - b) * H; idx += blockDim.x) {
      const int i = b + idx / H, u = idx % H;
      if (!mine(i)) continue;
      const int own = ls.perm[i];
      int wd = __ldg(a.words + own);
      if (wd < 0 || wd >= a.V) {
        if (u == 0) latch_word(own);
        wd = 0;
      }
      hput(i, u, __ldg(a.emb + (size_t)wd * H + u));
    }
  }
  __syncthreads();
  trace_mark(a, 22);
  // ---- internal levels, UNROLL levels per barrier ---------------------------
  for (int l0 = 1; l0 < L; l0 += UNROLL) {
    const int ltop = min(L - 1, l0 + UNROLL - 1);
    if constexpr (CELL == CX_TREERNN) {
      // thread (node, unit) for every node of the band that is the band's
      // top for its subtree: its parent is above the band (or it is a root)
      const int b = ls.lb[ltop], e = ls.lb[l0] + ls.ls[l0];  // ids of levels ltop .. l0
      for (int idx = tid; idx < (e - b) * H; idx += blockDim.x) {
        const int i = b + idx / H, u = idx % H;
        if (!mine(i)) continue;
        const int par = ls.par[ls.perm[i]];  // input id of the parent (trees), -1 root
        if (par >= 0 && lev[ls.inv[par]] <= ltop) continue;  // finished by its parent
        // evaluate the subtree below i inside the band: an explicit stack of
        // pending nodes (<= UNROLL levels deep), unit u only
        if constexpr (UNROLL == 1) {
          int c0, c1;
          kids(i, c0, c1);
          hput(i, u, tanhf_(hrow(c0)[u] + hrow(c1)[u]));
        } else {
          // UNROLL == 2: children in the band (level l0) are computed inline
          int c0, c1;
          kids(i, c0, c1);
          float v[2];
          const int cs[2] = {c0, c1};
#pragma unroll
          for (int k = 0; k < 2; k++) {
            const int c = cs[k];
            if (lev[c] >= l0 && lev[i] > lev[c]) {  // the child lies in the band: inline
              int g0, g1;
              kids(c, g0, g1);
              v[k] = tanhf_(hrow(g0)[u] + hrow(g1)[u]);
              hput(c, u, v[k]);  // the caller's output for the child
            } else {
              v[k] = hrow(c)[u];
            }
          }
          hput(i, u, tanhf_(v[0] + v[1]));
        }
      }
    } else {  // CX_TREEFC, level-synchronous: h = tanh(W [h_l; h_r] + b)
      const int b = ls.lb[l0], e = b + ls.ls[l0];
      for (int idx = tid; idx < (e - b) * H; idx += blockDim.x) {
        const int i = b + idx / H, u = idx % H;
        if (!mine(i)) continue;
        int c0, c1;
        kids(i, c0, c1);
        const float *wr = a.w[0] + (size_t)u * 2 * H;
        const float *h0 = hrow(c0), *h1 = hrow(c1);
        float s0 = 0.f, s1 = 0.f;
        for (int k = 0; k < H; k++) {
          s0 = fmaf(__ldg(wr + k), h0[k], s0);
          s1 = fmaf(__ldg(wr + H + k), h1[k], s1);
        }
        hput(i, u, tanhf_(s0 + s1 + __ldg(a.w[1] + u)));
      }
    }
    __syncthreads();
    trace_mark(a, 2 + l0);
  }
  // ---- packed roots ----------------------------------------------------------
  if (a.root_out)
    for (int idx = tid; idx < n * H; idx += blockDim.x) {
      const int i = idx / H, u = idx % H;
      if (!mine(i) || ls.indeg[ls.perm[i]] != 0) continue;
      a.root_out[(size_t)ls.sid[i] * H + u] = hrow(i)[u];
    }
  trace_mark(a, a.trace_slots - 1);
  fused_exit(a, ferr);
}

constexpr int kScMaxWork = 1 << 22;  // TreeFC: n H^2 multiply-adds per launch

template <int CELL, int U>
bool sc_plan_one(int n, int maxc, int H, FwdPlan *p, int *Gn, int *Gu) {
  const size_t smem = sizeof(int) * sc_smem_ints(n, maxc);
  // + the state rows when they fit (the kernel checks %dynamic_smem_size); the
  // launch asks for no more shared memory than it uses
  const size_t with_rows = smem + sizeof(float) * ((size_t)n * H + 16);
  auto k = sc_kernel<CELL, U>;
  constexpr int kMaxDev = 64;
  static int set[kMaxDev];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDev) return false;
  if (smem > kScSmem) return false;
  if (!set[dev]) {
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kScSmem) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    set[dev] = 1;
  }
  // one CTA per ~16 nodes (a structure of the tiny configs), at most one per SM
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int G = n < 16 ? 1 : (n / 16 < sms ? n / 16 : sms);
  *Gn = G;
  *Gu = 1;
  p->ctas = G;
  p->threads = kScThreads;
  p->smem = with_rows <= kScSmem ? with_rows : smem;
  p->kernel = (const void *)k;
  p->cluster = 1;
  p->fused = true;
  p->family = 7;
  return true;
}

}  // namespace

// One-launch single-CTA-per-structure path (cx_linearize_forward): TreeRNN
// (unrolled by CX_UNROLL, default 2) for any batch whose linearizer fits one
// CTA's shared memory; TreeFC for tiny batches (n H^2 <= kScMaxWork).
bool single_plan(int cell, int H, int maxc, int n, FwdPlan *p, int *Gn, int *Gu) {
  if (maxc > 2 || n < 1) return false;
  if (cell == CX_TREERNN) {
    const char *e = std::getenv("CX_UNROLL");
    const int U = e ? std::atoi(e) : 2;
    if (U == 1) return sc_plan_one<CX_TREERNN, 1>(n, maxc, H, p, Gn, Gu);
    return sc_plan_one<CX_TREERNN, 2>(n, maxc, H, p, Gn, Gu);
  }
  if (cell == CX_TREEFC && (size_t)n * H * H <= (size_t)kScMaxWork)
    return sc_plan_one<CX_TREEFC, 1>(n, maxc, H, p, Gn, Gu);
  return false;
}

}  // namespace cx
