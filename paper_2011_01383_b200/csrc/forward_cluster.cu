// forward_cluster.cu -- latency path: one thread-block cluster per group of
// structures, hardware cluster barriers between levels, child state exchanged
// through distributed shared memory (DSMEM).
//
// Structures of a batch are independent (property P.3),
// so a level barrier only has to cover the CTAs that evaluate the same
// structures. A cluster of CS = H / 16 CTAs (16 at H = 256) owns whole
// structures (structure g -> cluster g mod #clusters) and each of its CTAs
// owns 16 hidden units with register-resident weights (rw_engine.cuh):
//   * every CTA keeps, in its own shared memory, its 16-unit slice of h (and of
//     the TreeLSTM memory cell / DAG-RNN input projection) for every node;
//   * a tile of T nodes pulls its children's full rows from the CS slices
//     (DSMEM loads, the paper's rnn_cache of App. A.3), contracts
//     them against the register weights and writes its own slice locally;
//   * one barrier.cluster (release/acquire) per level -- ~0.3 us measured --
//     replaces the ~1.1 us grid barrier, and nothing goes through L2 on the
//     level-to-level path (h_out is written for the caller only).
// The structure of every node comes from cx_linearize (structure[]); for a
// DAG whose structures share nodes, every node falls back to cluster 0
// (still correct, just serial over one cluster).
#include <cooperative_groups.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <climits>
#include <type_traits>

#include "lin_single.cuh"
#include "rw_engine.cuh"
#include "warp_engine.cuh"

namespace cg = cooperative_groups;

namespace cx {
namespace {
using namespace fwd;
using namespace rw;
using namespace wq;

constexpr int kCUnits = kRUG;  // units per CTA (16)

// dtype = CX_BF16 on this (FMA) path: the contraction operands -- weights,
// input rows x, gathered child states -- are rounded to bf16 where they are
// produced (weight registers, gathered / imported / pushed rows); products
// and sums stay fp32, as on the tensor cores (reading Q18). Outputs stay fp32.
__device__ __forceinline__ float rbf(float x) { return __bfloat162float(__float2bfloat16_rn(x)); }
__device__ __forceinline__ float4 rbf4(float4 v) {
  return make_float4(rbf(v.x), rbf(v.y), rbf(v.z), rbf(v.w));
}
// round rows [0, cnt) of H floats at X in place (block-wide; caller syncs)
template <int H>
__device__ __forceinline__ void round_rows(float *X, int cnt) {
  for (int idx = threadIdx.x; idx < cnt * H / 4; idx += blockDim.x) {
    float4 *p = reinterpret_cast<float4 *>(X) + idx;
    *p = rbf4(*p);
  }
}
template <int H>
__device__ __forceinline__ void round_wregs(WRegs<H> &w) {
#pragma unroll
  for (int g = 0; g < 4; g++)
#pragma unroll
    for (int j = 0; j < WShape<H>::KC / 2; j++) {
      float lo, hi;
      asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(w[g][j]));
      w[g][j] = f2pack(rbf(lo), rbf(hi));
    }
}

// DAG-RNN level: U h~ + W_x x in one accumulator. Rows per node in X: the
// MAXC children, x (vector MAXC), then h~ (vector MAXC + 1, the HTS row).
template <int MAXC>
struct CDagLevel : PhBase<2, MAXC + 1, MAXC, 1, 2> {
  __device__ static constexpr int g(int p) { return p == 0 ? 1 : 0; }
  __device__ static constexpr int v(int p) { return p == 0 ? MAXC + 1 : MAXC; }
  __device__ static constexpr int a(int p) { return 0; }
};

template <int CELL, int MAXC>
struct CCfg;
// RPN: X rows per node at a level; AUX: a per-node aux slice in shared memory
// (TreeLSTM's memory cell; DAG-RNN recomputes W_x x at the node's level instead
// of keeping its projection, which halves the per-node footprint)
template <int MAXC>
struct CCfg<CX_TREELSTM, MAXC> {
  // LEAFB: leaves per bookkeeping + gather block; sequences (MAXC = 1) have
  // one leaf per chain, and the smaller X buffer lets 1000-node chain batches
  // keep their per-node slices on chip
  // TMAX: nodes per level tile (3 + MAXC packed accumulators per node must
  // stay in registers); TLEAF: leaves per leaf tile (3 accumulators)
  static constexpr int TMAX = 4, TLEAF = 8, NVMAX = MAXC, NAMAX = 3 + MAXC,
                       LEAFB = MAXC == 1 ? 16 : 24, RPN = MAXC + 1;
  static constexpr bool AUX = true;
};
template <int MAXC>
struct CCfg<CX_DAGRNN, MAXC> {
  static constexpr int TMAX = 16, TLEAF = 16, NVMAX = MAXC, NAMAX = 1, LEAFB = 32, RPN = MAXC + 2;
  static constexpr bool AUX = false;
};

template <int CELL, int H, int MAXC>
struct CLayout {
  using C = CCfg<CELL, MAXC>;
  static constexpr size_t xl = (size_t)C::TMAX * C::RPN * H, xb = (size_t)C::LEAFB * H;
  static constexpr size_t x_floats = xl > xb ? xl : xb;
  // fixed floats: tile buffer and the per-node aux slice (TreeLSTM memory
  // cell) -- then the ints, then region R: the per-node h slices (barrier +
  // pull mode) or the push-mode arrays. (The warp engine needs no reduction
  // buffers.)
  __host__ __device__ static size_t fixed_floats(int n) {
    return x_floats + (C::AUX ? (size_t)kCUnits * n : 0);
  }
  static size_t r_min_bytes(int n) { return sizeof(float) * (size_t)kCUnits * n + 16; }
  static size_t ints(int n, int maxc, int L) { return (size_t)(3 + maxc) * n + 4 * (size_t)L + 64; }
  static size_t bytes(int n, int maxc, int L) {
    return sizeof(float) * fixed_floats(n) + sizeof(int) * ints(n, maxc, L) + r_min_bytes(n);
  }
};

// Max nodes the cluster path takes (per-node slices live in shared memory).
constexpr int kClusterMaxN = 1536;  // and the shared-memory check of the plan
// Fused linearize + forward: count-table entries of the
// in-kernel single-CTA linearizer, and its extra shared memory (ints): the
// linearizer's arrays stand in for the prologue's perm/label/level arrays,
// plus the remapped children, the cluster's level lists and their offsets.
constexpr int kFusedCnt = 2048;
__host__ __device__ inline size_t fused_extra_ints(int n, int maxc) {
  return lin_sm_ints(n, maxc, kFusedCnt) + (size_t)maxc * n + 3 * (size_t)n + 64;
}

// run tile<T>() for the smallest power of two T >= cnt (T <= TM; warp-uniform)
template <int TM, class F>
__device__ __forceinline__ void dispatch_tile(int cnt, F &&f) {
  if constexpr (TM >= 16) {
    if (cnt > 8) { f(std::integral_constant<int, 16>{}); return; }
  }
  if constexpr (TM >= 8) {
    if (cnt > 4) { f(std::integral_constant<int, 8>{}); return; }
  }
  if (cnt > 2) f(std::integral_constant<int, 4>{});
  else if (cnt == 2) f(std::integral_constant<int, 2>{});
  else f(std::integral_constant<int, 1>{});
}

struct CS {  // shared-memory carve of one CTA
  float *X, *hsl, *aux;
  int *perm, *lab, *chn, *list, *lbeg, *lsize, *coff, *ccur;  // coff/ccur: this cluster's level lists
};

// Pull the full H-rows of `rows` (new ids, -1 = zeros) from the CS slices into
// X (RPN rows per node: the NV children, ..., their sum h~ in the last row).
template <int H, int NV, int RPN = NV + 1, class ROW>
__device__ __forceinline__ void pull_rows(cg::cluster_group &cl, const CS &s, int cnt, ROW row,
                                          bool bf16ops) {
  constexpr int CSZ = H / kCUnits;
  constexpr int Q = kCUnits / 4;  // float4 per slice
  const int total = cnt * CSZ * Q;
  for (int idx = threadIdx.x; idx < total; idx += blockDim.x) {
    const int q = idx % Q, r = idx / Q;
    const int peer = r % CSZ, t = r / CSZ;
    const float *remote = cl.map_shared_rank(s.hsl, peer);
    float4 v[NV];
#pragma unroll
    for (int j = 0; j < NV; j++) {
      const int c = row(t, j);
      v[j] = c >= 0 ? *reinterpret_cast<const float4 *>(remote + (size_t)c * kCUnits + 4 * q)
                    : make_float4(0.f, 0.f, 0.f, 0.f);
      if (bf16ops) v[j] = rbf4(v[j]);
    }
    float4 sum = v[0];
#pragma unroll
    for (int j = 0; j < NV; j++) {
      *reinterpret_cast<float4 *>(s.X + (size_t)(t * RPN + j) * H + peer * kCUnits + 4 * q) = v[j];
      if (j) { sum.x += v[j].x; sum.y += v[j].y; sum.z += v[j].z; sum.w += v[j].w; }
    }
    *reinterpret_cast<float4 *>(s.X + (size_t)(t * RPN + RPN - 1) * H + peer * kCUnits + 4 * q) = sum;
  }
}

// ---------------------------------------------------------------------------
// The kernel. Thread (warp w, lane c) holds the k-chunk c of every gate row of
// hidden unit unit0 + w (warp_engine.cuh): tiles are contracted and their
// gates evaluated without any block-wide reduction; one __syncthreads per
// tile stages the finished h slices for the push (or ends a pull-mode tile).
//
// FUSED: the kernel linearizes the batch itself (every CTA redundantly runs
// the single-CTA linearizer of lin_single.cuh on its own shared memory, so no
// grid-wide synchronisation is needed; CTA 0 also writes the cx_linearization
// outputs). Forward data errors are latched into a workspace word and merged
// into the header by the last CTA out, after CTA 0 has written it.
// EARLY (fused TreeLSTM): the leaves are evaluated before the linearizer (see
// the phase below).
template <int CELL, int H, int MAXC, bool FUSED>
__global__ void __launch_bounds__(kRThreads, 1) ck_kernel(FwdArgs a) {
  using Cfg = CCfg<CELL, MAXC>;
  using Lay = CLayout<CELL, H, MAXC>;
  constexpr int KC = WShape<H>::KC;
  constexpr int TMAX = Cfg::TMAX;
  extern __shared__ __align__(16) float smem[];
  constexpr int LEAFB = Cfg::LEAFB;
  __shared__ int s_nodes[LEAFB];
  __shared__ int s_word[LEAFB];
  __shared__ float s_bias[4 * kCUnits];
  // push mode: the new h slices of up to SG nodes (several tiles of a level)
  // are staged, then pushed after ONE __syncthreads (double-buffered)
  constexpr int SG = 32;
  static_assert(SG % TMAX == 0 && SG % Cfg::TLEAF == 0 && SG >= LEAFB, "stage groups align with tiles");
  __shared__ __align__(16) float s_stage[2][SG * kCUnits];

  cg::cluster_group cl = cg::this_cluster();
  const int maxc = a.maxc;
  const int crank = (int)cl.block_rank();
  const int cid = blockIdx.x / (int)cl.num_blocks(), ncl = gridDim.x / (int)cl.num_blocks();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int hu = lane & 15;  // half-warp lane: row-piece and push mapping
  const int unit0 = crank * kCUnits;
  const Roles<1> ro(warp, lane);  // one unit per warp (UW = 1, warp_engine.cuh)
  const int myu = unit0 + warp;  // this warp's hidden unit
  const bool latch = crank == 0;
  trace_mark(a, 0);

  // ---- weights -> registers (first the leaf / projection gates): inputs only,
  // so this overlaps cx_linearize under programmatic dependent launch --------
  WRegs<H> w;
  Gate gs[4];
  int ng;
  if constexpr (CELL == CX_TREELSTM) {
    gs[0] = {a.w[0], 0, H, 0}; gs[1] = {a.w[0], H, H, 0}; gs[2] = {a.w[0], 2 * H, H, 0};
    ng = 3;
  } else {
    gs[0] = {a.w[0], 0, H, 0}; gs[1] = {a.w[1], 0, H, 0};
    ng = 2;
  }
  auto load_leaf_weights = [&]() {
    load_wregs_w<4, H, 1>(w, gs, ng, myu, ro);
    if (a.bf16ops) round_wregs<H>(w);
    if constexpr (CELL == CX_TREELSTM) {
      if (tid < 4 * kCUnits) {
        int g = tid / kCUnits, uu = tid % kCUnits;
        const float *b = g < 3 ? a.w[2] + g * H : a.w[4];
        s_bias[tid] = __ldg(b + unit0 + uu);
      }
    } else {
      if (tid < kCUnits) s_bias[tid] = __ldg(a.w[2] + unit0 + tid);
    }
  };
  auto load_rec_weights = [&]() {  // TreeLSTM recurrent gates U_iou, U_f
    gs[0] = {a.w[1], 0, H, 0}; gs[1] = {a.w[1], H, H, 0}; gs[2] = {a.w[1], 2 * H, H, 0};
    gs[3] = {a.w[3], 0, H, 0};
    load_wregs_w<4, H, 1>(w, gs, 4, myu, ro);
    if (a.bf16ops) round_wregs<H>(w);
  };
  constexpr bool EARLY = FUSED && CELL == CX_TREELSTM;
  if constexpr (FUSED && !EARLY) {
    // fire-and-forget L2 prefetch of this thread's weight rows; the register
    // loads follow the in-kernel linearization (loads in flight would queue
    // ahead of the linearizer's own children loads)
    for (int g = 0; g < ng; g++) {
      const float *src = gs[g].base + (size_t)(gs[g].r0 + myu) * gs[g].ld + gs[g].c0 + 4 * lane;
      asm volatile("prefetch.global.L2 [%0];" ::"l"(src));
    }
  } else if constexpr (!FUSED) {
    load_leaf_weights();
  }
  if constexpr (CELL == CX_TREELSTM) {
    for (int g = 0; g < 4; g++) {
      const float *src = (g < 3 ? a.w[1] + (size_t)(g * H + myu) * H
                                : a.w[3] + (size_t)myu * H) + 4 * lane;
      asm volatile("prefetch.global.L2 [%0];" ::"l"(src));
    }
  }
  unsigned long long *ferr = reinterpret_cast<unsigned long long *>(&a.bar->pad[0]);
  auto latch_word = [&](int own) {
    if constexpr (FUSED) atomicMax(ferr, ~(((unsigned long long)CX_E_WORD_RANGE << 32) | (unsigned)own));
    else latch_error(a.hdr, CX_E_WORD_RANGE, own);
  };
  int L, first_leaf, R;
  const int n = a.n;
  LinSm ls;
  int *fint = nullptr;
  const size_t fixed = Lay::fixed_floats(n);
  float *const X = smem;

  // ---- EARLY leaf phase (fused TreeLSTM): a leaf's cell needs no linearization
  // -- only its word -- so the leaves are evaluated at kernel entry, spread over
  // ALL clusters by input id (cluster c takes ids [c n / ncl, (c+1) n / ncl)),
  // h into h_out and c into cbuf (aux_out or workspace), both in input
  // numbering; one release increment of a grid-wide counter per CTA publishes
  // them. The linearizer then runs while those stores drain, and each cluster
  // imports its internal nodes' leaf children from L2 after one acquire of the
  // counter (complete long before). A leaf is a node whose first child slot is
  // absent; malformed inputs are caught by the linearizer (its codes rank
  // below CX_E_WORD_RANGE) and outputs are then unspecified.
  if constexpr (EARLY) {
    load_leaf_weights();
    // the chunk's leaves and their word ids (one round trip for both), then
    // every leaf row gathered at once into E (all of the shared memory is free
    // before the linearizer runs; blocks of EB rows if the chunk is larger)
    int lo, hi;
    chunk_of(n, ncl, cid, lo, hi);
    const int span = hi - lo;
    // (+ TLEAF slack rows: a partial tile reads, and discards, rows past its end)
    const int EB = min(span, (int)(((size_t)dynamic_smem_bytes() - 8 * (size_t)span - 64) /
                                   (sizeof(float) * H)) - Cfg::TLEAF);
    float *E = smem;
    int *elist = reinterpret_cast<int *>(smem + (size_t)(EB + Cfg::TLEAF) * H), *ewd = elist + span;
    __shared__ int s_wc[kRNW];
    int ecnt = 0;
    for (int base = lo; base < hi; base += blockDim.x) {  // compact the chunk's leaves
      const int v = base + tid;
      bool f = false;
      int wd = 0;
      if (v < hi) {
        const int c0 = __ldg(a.lin.ch + v);
        wd = __ldg(a.words + v);
        f = c0 == -1;
      }
      const unsigned bal = __ballot_sync(0xffffffffu, f);
      if (lane == 0) s_wc[warp] = __popc(bal);
      __syncthreads();
      int before = ecnt, tot = 0;
      for (int ww = 0; ww < kRNW; ww++) {
        if (ww < warp) before += s_wc[ww];
        tot += s_wc[ww];
      }
      if (f) {
        if (wd < 0 || wd >= a.V) {
          if (latch) latch_word(v);
          wd = 0;
        }
        const int pos = before + __popc(bal & ((1u << lane) - 1u));
        elist[pos] = v;
        ewd[pos] = wd;
      }
      ecnt += tot;
      __syncthreads();
    }
    trace_mark(a, 13);
    for (int b0 = 0; b0 < ecnt; b0 += EB) {
      const int cntb = min(EB, ecnt - b0);
      if (b0) __syncthreads();  // E is overwritten
      gather_rows_c<1, H>(E, cntb, [&](int t, int) { return a.emb + (size_t)ewd[b0 + t] * H; });
      __syncthreads();
      if (a.bf16ops) {
        round_rows<H>(E, cntb);
        __syncthreads();
      }
      trace_mark(a, 14);
      for (int t0 = 0; t0 < cntb; t0 += Cfg::TLEAF) {
        const int cntt = min(Cfg::TLEAF, cntb - t0);
        auto tile = [&](auto tt) {
          constexpr int T = decltype(tt)::value;
          float r[3];
          const bool act = contract_w<RLstmLeaf, H, T, 1>(E + (size_t)t0 * H, w, r, ro, nullptr);
          const int tn = node_of_lane<T, 1>(lane);
          if (act && tn < cntt) {
            const size_t o = (size_t)elist[b0 + t0 + tn] * H + myu;
            const float cc = sigmoidf_(r[0] + s_bias[warp]) * tanhf_(r[2] + s_bias[32 + warp]);
            a.h_out[o] = sigmoidf_(r[1] + s_bias[16 + warp]) * tanhf_(cc);
            a.cbuf[o] = cc;
          }
        };
        dispatch_tile<Cfg::TLEAF>(cntt, tile);
      }
    }
    trace_mark(a, 15);
    __syncthreads();  // the linearizer reuses the shared memory
    if (tid == 0) {
      __threadfence();
      red_release_add_u32(&a.bar->count, 1u);
    }
    load_rec_weights();  // the recurrent gates -> registers, overlapping the linearizer
    trace_mark(a, 21);
  }
  if constexpr (FUSED) {
    fint = reinterpret_cast<int *>(smem + fixed);
    LinPrefetch pf{a.words, a.emb, H, a.V};
    if (EARLY) pf.words = nullptr;  // no leaf rows left to fetch
    const LinOut lo = lin_single_body(a.lin, fint, kFusedCnt, blockIdx.x == 0,
                                      fint + lin_sm_ints(n, maxc, kFusedCnt), pf);
    trace_mark(a, 20);
    if (!lo.ok) {
      fused_exit(a, ferr);
      return;
    }
    if (!EARLY) load_leaf_weights();
    ls = lin_carve(fint, n, maxc);
    L = lo.L;
    first_leaf = lo.first_leaf;
    R = lo.num_roots;
  } else {
    griddep_wait();
    if (*reinterpret_cast<volatile int *>(&a.hdr->status) != CX_OK) return;
    L = a.hdr->num_levels;
    first_leaf = a.hdr->first_leaf;
    R = a.hdr->num_roots;
  }
  (void)first_leaf;

  CS s;
  s.X = X;
  s.aux = smem + Lay::x_floats;  // TreeLSTM only
  int *int_end;
  if constexpr (FUSED) {  // the linearizer's shared-memory results
    s.perm = ls.perm;
    s.lab = ls.sid;
    s.lbeg = ls.lb;
    s.lsize = ls.ls;
    s.chn = fint + lin_sm_ints(n, maxc, kFusedCnt);
    s.list = s.chn + (size_t)maxc * n;
    s.coff = s.list + n;
    s.ccur = s.coff + n + 1;
    int_end = fint + fused_extra_ints(n, maxc);
  } else {
    s.perm = reinterpret_cast<int *>(smem + fixed);
    s.lab = s.perm + n;
    s.list = s.lab + n;
    s.chn = s.list + n;
    s.lbeg = s.chn + (size_t)maxc * n;
    s.lsize = s.lbeg + L;
    s.coff = s.lsize + L;      // [L + 1] start of level l in this cluster's list
    s.ccur = s.coff + L + 1;   // [L] fill cursors
    int_end = s.ccur + L;
  }
  // region R: everything after the ints, up to the end of the dynamic smem
  char *Rb = reinterpret_cast<char *>((reinterpret_cast<uintptr_t>(int_end) + 15) & ~uintptr_t(15));
  const size_t r_bytes = (size_t)dynamic_smem_bytes() - (size_t)(Rb - reinterpret_cast<char *>(smem));
  s.hsl = reinterpret_cast<float *>(Rb);  // barrier + pull mode

  // ---- prologue: structure labels (root index, propagated top-down) --------
  if constexpr (!FUSED) {
    for (int l = tid; l < L; l += blockDim.x) {
      s.lbeg[l] = __ldg(a.lbeg + l);
      s.lsize[l] = __ldg(a.lsize + l);
    }
    for (int v = tid; v < n; v += blockDim.x) {
      s.perm[v] = __ldg(a.perm + v);
      s.lab[v] = __ldg(a.sid + v);  // structure index (cx_linearize)
    }
    for (int e = tid; e < maxc * n; e += blockDim.x) s.chn[e] = __ldg(a.chn + e);
    __syncthreads();
  }
  bool one_cluster = false;
  if (a.kind == CX_DAG) {  // structures sharing a node: one cluster does everything
    bool bad = false;
    for (int i = tid; i < n; i += blockDim.x)
      for (int k = 0; k < maxc; k++) {
        int c = s.chn[k * n + i];
        if (c < 0) break;
        if (s.lab[c] != s.lab[i]) bad = true;
      }
    one_cluster = __syncthreads_or(bad);
  }

  // ---- this cluster's nodes, bucketed by level once ---------------------------
  for (int l = tid; l < L; l += blockDim.x) s.ccur[l] = 0;
  __syncthreads();
  // this cluster evaluates node i (new id)
  auto mine = [&](int i) { return (one_cluster ? 0 : s.lab[i] % ncl) == cid; };
  // level of new id i: ids are level-contiguous, root-most level first
  auto level_of = [&](int i) {
    int lo = 0, hi = L - 1;  // find l with lbeg[l] <= i < lbeg[l] + lsize[l]
    while (lo < hi) {
      int mid = (lo + hi) >> 1;
      if (i >= s.lbeg[mid]) hi = mid; else lo = mid + 1;
    }
    return lo;
  };
  for (int i = tid; i < n; i += blockDim.x)
    if (mine(i)) atomicAdd(&s.ccur[level_of(i)], 1);
  __syncthreads();
  if (warp == 0) {  // exclusive scan of the per-level counts (level 0 first)
    int acc = 0;
    for (int b0 = 0; b0 < L; b0 += 32) {
      int l = b0 + lane;
      int x = l < L ? s.ccur[l] : 0, incl = x;
      for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      if (l < L) s.coff[l] = acc + incl - x;
      acc += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) s.coff[L] = acc;
  }
  __syncthreads();
  // fill in ascending new id inside each level, so every CTA of the cluster
  // builds the SAME list (push mode addresses a node's rows by its position):
  // g = #mine before i by a block-wide scan; levels are contiguous id ranges,
  // root-most first, so #mine before level l's first id = coff[L] - coff[l + 1]
  {
    __shared__ int s_wsum[kRNW];
    int G = 0;
    for (int c0 = 0; c0 < n; c0 += blockDim.x) {
      const int i = c0 + tid;
      const bool f = i < n && mine(i);
      const unsigned bal = __ballot_sync(0xffffffffu, f);
      if (lane == 0) s_wsum[warp] = __popc(bal);
      __syncthreads();
      int before = G;
      for (int ww = 0; ww < warp; ww++) before += s_wsum[ww];
      int tot = 0;
      for (int ww = 0; ww < kRNW; ww++) tot += s_wsum[ww];
      if (f) {
        const int l = level_of(i);
        const int g = before + __popc(bal & ((1u << lane) - 1u));
        s.list[s.coff[l] + g - (s.coff[L] - s.coff[l + 1])] = i;
      }
      G += tot;
      __syncthreads();
    }
  }
  trace_mark(a, 1);

  // ---- push mode (trees: one parent per node) --------------------------------
  // Every internal node of this cluster owns MAXC rows of H floats in region R
  // (level-major, in list order: row (p - coff[1]) * MAXC + k for the k-th
  // child of the node at list position p). The epilogue that finishes a node
  // writes its 16-unit slice of h straight into its parent's row in all CS
  // CTAs of the cluster (st.async, DSMEM), each store signalling the
  // receiving CTA's mbarrier of the parent's level. A level starts when its
  // mbarrier has received all its rows: no cluster barrier, no pull and no
  // release fence on the level-to-level path. Falls back to the barrier + pull
  // mode (per cluster, uniformly) when the rows do not fit in region R.
  bool push = false;
  unsigned long long *mb = nullptr;
  int *prow = nullptr, *plev = nullptr;
  float *XA = nullptr;
  if constexpr (CELL == CX_TREELSTM) {
    if (a.kind != CX_DAG && L > 1 && !a.push_off) {
      char *q = Rb;
      mb = reinterpret_cast<unsigned long long *>(q);
      q += ((size_t)8 * L + 15) & ~size_t(15);
      prow = reinterpret_cast<int *>(q);
      plev = prow + n;
      q += ((size_t)8 * n + 15) & ~size_t(15);
      XA = reinterpret_cast<float *>(q);
      // + slack: a partial last tile reads (discarded) rows past the level end
      const size_t rows = (size_t)(s.coff[L] - s.coff[1] + TMAX) * MAXC;
      push = (size_t)(q - Rb) + rows * H * sizeof(float) <= r_bytes;
    }
  }
  if (push) {
    for (int v = tid; v < n; v += blockDim.x) prow[v] = -1;
    for (int l = tid; l < L; l += blockDim.x) s.ccur[l] = 0;
    __syncthreads();
    for (int p = s.coff[1] + tid; p < s.coff[L]; p += blockDim.x) {
      const int i = s.list[p], lv = level_of(i);
      int nc = 0;
#pragma unroll
      for (int k = 0; k < MAXC; k++) {
        const int c = k < maxc ? s.chn[k * n + i] : -1;
        const int row = (p - s.coff[1]) * MAXC + k;
        if (c >= 0) {
          prow[c] = row;
          plev[c] = lv;
          if (!EARLY || c < first_leaf) nc++;  // EARLY: leaf rows are imported, not pushed
        } else {  // absent child: a zero row nobody pushes into
          float4 *z = reinterpret_cast<float4 *>(XA + (size_t)row * H);
          for (int q4 = 0; q4 < H / 4; q4++) z[q4] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
      atomicAdd(&s.ccur[lv], nc);
    }
    for (int l = 1 + tid; l < L; l += blockDim.x) mbar_init(&mb[l], 1);
    fence_mbar_init_cluster();
    __syncthreads();
    for (int l = 1 + tid; l < L; l += blockDim.x)
      if (s.coff[l + 1] > s.coff[l] && s.ccur[l] > 0)
        mbar_expect_tx(&mb[l], (unsigned)s.ccur[l] * H * 4u);
  }
  // EARLY: import this cluster's leaves (list positions [0, coff[1])) from L2
  // once every CTA has published its share: push mode -- the full h row into
  // the parent's slot row; both modes -- this CTA's 16-unit slice of c (the
  // parents' forget-gate term), and of h in pull mode
  if constexpr (EARLY) {
    trace_mark(a, 17);
    if (tid == 0) {
      unsigned long long spins = 0;
      while (ld_relaxed_u32(&a.bar->count) < gridDim.x)
        if (++spins > (1ull << 26)) __trap();
      (void)ld_acquire_u32(&a.bar->count);
    }
    __syncthreads();
    trace_mark(a, 18);
    const int nl0 = s.coff[1];
    constexpr int Q4 = H / 4;
    // cp.async (L2 -> shared, all pieces in flight at once, one wait)
    if (push)
      for (int idx = tid; idx < nl0 * Q4; idx += blockDim.x) {
        const int v = s.list[idx / Q4], q = idx % Q4, pr = prow[v];
        if (pr >= 0) cp_async16(XA + (size_t)pr * H + 4 * q, a.h_out + (size_t)s.perm[v] * H + 4 * q);
      }
    constexpr int Q16 = kCUnits / 4;  // 16-byte pieces of a 16-unit slice
    for (int idx = tid; idx < nl0 * Q16; idx += blockDim.x) {
      const int v = s.list[idx / Q16], qq = idx % Q16;
      const size_t o = (size_t)s.perm[v] * H + unit0 + 4 * qq;
      cp_async16(s.aux + (size_t)v * kCUnits + 4 * qq, a.cbuf + o);
      if (!push) cp_async16(s.hsl + (size_t)v * kCUnits + 4 * qq, a.h_out + o);
      else if (a.root_out && prow[v] < 0)  // a single-node tree: its leaf is its root
        *reinterpret_cast<float4 *>(a.root_out + (size_t)s.lab[v] * H + unit0 + 4 * qq) =
            ldcg4(a.h_out + o);
    }
    cp_async_wait_all();
    if (push && a.bf16ops)  // each thread rounds the pieces it copied itself
      for (int idx = tid; idx < nl0 * Q4; idx += blockDim.x) {
        const int v = s.list[idx / Q4], q = idx % Q4, pr = prow[v];
        if (pr >= 0) {
          float4 *d = reinterpret_cast<float4 *>(XA + (size_t)pr * H + 4 * q);
          *d = rbf4(*d);
        }
      }
    trace_mark(a, 22);
  }
  if (push) {
    // every CTA of the cluster has initialised its mbarriers before any push
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
  }

  // The level barrier of pull mode is split: arrive (release: this CTA's state
  // slices are published to the cluster), then the caller's outputs of the
  // level just finished go to global memory, then wait (acquire). Issued before
  // the arrive, those global stores would stall the release fence (ncu: the
  // barrier's MEMBAR was the top stall).
  auto cl_arrive = [] { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); };
  auto cl_wait = [] { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); };
  // h_out (and TreeLSTM c into aux_out) of this cluster's nodes at list
  // positions [pb, pe), this CTA's 16 units: 64-byte row pieces
  auto put_outputs = [&](int pb, int pe) {
    const bool wa = CELL == CX_TREELSTM && a.aux_out;
    for (int idx = tid; idx < (pe - pb) * kCUnits; idx += blockDim.x) {
      const int v = s.list[pb + idx / kCUnits], uu = idx % kCUnits;
      const size_t o = (size_t)s.perm[v] * H + unit0 + uu;
      a.h_out[o] = s.hsl[(size_t)v * kCUnits + uu];
      if (wa) a.aux_out[o] = s.aux[(size_t)v * kCUnits + uu];
    }
  };
  // push mode, node v (tile slot t) finished with h = hh, c = cc at this warp's
  // unit: caller outputs straight from the epilogue, the h value into the stage
  int sb = 0;  // stage buffer of the current group (double-buffered)
  auto emit = [&](int v, int t, float hh, float cc) {  // t: position in the stage group
    const size_t o = (size_t)s.perm[v] * H + myu;
    a.h_out[o] = hh;
    if (CELL == CX_TREELSTM && a.aux_out) a.aux_out[o] = cc;
    if (a.root_out && prow[v] < 0) a.root_out[(size_t)s.lab[v] * H + myu] = hh;
    s_stage[sb][t * kCUnits + warp] = a.bf16ops ? rbf(hh) : hh;  // the parent's operand
  };
  // ... then (after __syncthreads) lane hu of node t's half-warp sends the
  // 64-byte slice to CTA hu's row of the parent
  auto push_slice = [&](int v, int t) {
    constexpr int CSZ = H / kCUnits;  // CTAs of the cluster: lane hu < CSZ serves CTA hu
    const int pr = prow[v];
    if (pr < 0 || hu >= CSZ) return;
    const unsigned dst = mapa_rank(smem_addr(XA + (size_t)pr * H + unit0), (unsigned)hu);
    const unsigned bar = mapa_rank(smem_addr(&mb[plev[v]]), (unsigned)hu);
    const float4 *src = reinterpret_cast<const float4 *>(&s_stage[sb][t * kCUnits]);
#pragma unroll
    for (int q4 = 0; q4 < kCUnits / 4; q4++) st_async_v4(dst + 16u * q4, src[q4], bar);
  };
  // after the last tile of a stage group (nodes gl[0 .. cntg)): stage
  // complete, push, flip the stage buffer
  auto flush = [&](const int *gl, int cntg) {
    __syncthreads();
    if (tid < cntg * kCUnits) push_slice(gl[tid >> 4], tid >> 4);
    sb ^= 1;
  };

  // ---- leaf / projection phase (done at entry when EARLY) --------------------
  if (!EARLY) {
    // this cluster's leaves (level 0). TreeLSTM: [i; o; u] = W_iou x + b;
    // DAG-RNN: h = tanh(W_x x + b) (internal nodes add W_x x at their level)
    const int cnt = s.coff[1];
    for (int b0 = 0; b0 < cnt; b0 += LEAFB) {
      const int cntb = min(LEAFB, cnt - b0);
      if (tid < cntb) {
        int v = s.list[b0 + tid];
        int own = s.perm[v];
        int wd = __ldg(a.words + own);
        if (wd < 0 || wd >= a.V) {
          if (latch) latch_word(own);
          wd = 0;
        }
        s_nodes[tid] = v;
        s_word[tid] = wd;
      }
      __syncthreads();
      gather_rows_c<1, H>(X, cntb, [&](int t, int) { return a.emb + (size_t)s_word[t] * H; });
      __syncthreads();
      if (a.bf16ops) {
        round_rows<H>(X, cntb);
        __syncthreads();
      }
      for (int t0 = 0; t0 < cntb; t0 += Cfg::TLEAF) {
        const int cntt = min(Cfg::TLEAF, cntb - t0);
        auto tile = [&](auto tt) {
          constexpr int T = decltype(tt)::value;
          const int tn = node_of_lane<T, 1>(lane);
          bool lead;
          if constexpr (CELL == CX_TREELSTM) {
            float r[3];
            lead = contract_w<RLstmLeaf, H, T, 1>(X + (size_t)t0 * H, w, r, ro, nullptr) && tn < cntt;
            if (lead) {
              const int v = s_nodes[t0 + tn];
              const float cc = sigmoidf_(r[0] + s_bias[warp]) * tanhf_(r[2] + s_bias[32 + warp]);
              const float hh = sigmoidf_(r[1] + s_bias[16 + warp]) * tanhf_(cc);
              s.aux[(size_t)v * kCUnits + warp] = cc;
              if (push) emit(v, t0 + tn, hh, cc);
              else s.hsl[(size_t)v * kCUnits + warp] = hh;
            }
            if (push && t0 + Cfg::TLEAF >= cntb) flush(s_nodes, cntb);
          } else {
            float r[1];
            lead = contract_w<RDagLeaf, H, T, 1>(X + (size_t)t0 * H, w, r, ro, nullptr) && tn < cntt;
            if (lead) s.hsl[(size_t)s_nodes[t0 + tn] * kCUnits + warp] = tanhf_(r[0] + s_bias[warp]);
          }
        };
        dispatch_tile<Cfg::TLEAF>(cntt, tile);
      }
      __syncthreads();  // X and s_nodes are overwritten by the next block
    }
    if constexpr (CELL == CX_TREELSTM) load_rec_weights();
  }
  trace_mark(a, 2);
  if (!push) {
    cl_arrive();
    if (!EARLY) put_outputs(s.coff[0], s.coff[1]);  // the leaves (level 0)
    cl_wait();
  }

  // ---- internal levels: one cluster barrier per level (pull mode) or one
  // mbarrier wait per level (push mode) ---------------------------------------
  for (int l = 1; l < L; l++) {
    const int tb = 24 + 5 * l;  // debug trace slots of this level's first tile
    const int lbase = s.coff[l], cnt = s.coff[l + 1] - lbase;
    if (l < 20) trace_mark(a, tb);
    if (push && cnt > 0 && s.ccur[l] > 0) {  // this level's pushed child rows have arrived
      // watchdog: a lost row would otherwise spin forever; trap (sticky launch
      // error, reported as CX_E_CUDA) instead of hanging the device
      unsigned long long spins = 0;
      while (!mbar_try_wait_cluster(&mb[l], 0))
        if (++spins > (1ull << 24)) __trap();
    }
    for (int t0 = 0; t0 < cnt; t0 += TMAX) {
      const int cntt = min(TMAX, cnt - t0);
      // tile node t and its children come straight from the shared-memory
      // level list and child table (no per-tile staging barrier)
      const int *tl = s.list + lbase + t0;
      auto child = [&](int t, int k) { return k < maxc ? s.chn[k * n + tl[t]] : -1; };
      if (t0 == 0 && l < 20) trace_mark(a, tb + 1);
      if (!push) {
        if constexpr (CELL == CX_DAGRNN) {  // x rows (L2; prefetched in the fused kernel)
          constexpr int q4 = H / 4, RPN = Cfg::RPN;
          for (int idx = tid; idx < cntt * q4; idx += blockDim.x) {
            const int t = idx / q4, c = idx - t * q4;
            const int own = s.perm[tl[t]];
            int wd = __ldg(a.words + own);
            if (wd < 0 || wd >= a.V) {
              if (latch && c == 0) latch_word(own);
              wd = 0;
            }
            *reinterpret_cast<float4 *>(s.X + (size_t)(t * RPN + MAXC) * H + 4 * c) =
                a.bf16ops ? rbf4(ldcg4(a.emb + (size_t)wd * H + 4 * c)) : ldcg4(a.emb + (size_t)wd * H + 4 * c);
          }
        }
        pull_rows<H, Cfg::NVMAX, Cfg::RPN>(cl, s, cntt, child, a.bf16ops);
        __syncthreads();
      }
      auto tile = [&](auto tt) {
        constexpr int T = decltype(tt)::value;
        const int tn = node_of_lane<T, 1>(lane);
        bool lead;
        if constexpr (CELL == CX_TREELSTM) {
          float r[3 + MAXC];
          if (push)  // the MAXC child rows of each node, h~ summed in registers
            lead = contract_w<RLstmLevel<MAXC>, H, T, 1, false>(
                XA + (size_t)(lbase + t0 - s.coff[1]) * MAXC * H, w, r, ro, nullptr);
          else
            lead = contract_w<RLstmLevel<MAXC>, H, T, 1, true>(s.X, w, r, ro, nullptr);
          lead = lead && tn < cntt;
          if (t0 == 0 && l < 20) trace_mark(a, tb + 3);
          if (lead) {
            const int v = tl[tn];
            float cc = sigmoidf_(r[0] + s_bias[warp]) * tanhf_(r[2] + s_bias[32 + warp]);
            const float bf = s_bias[48 + warp];
#pragma unroll
            for (int k = 0; k < MAXC; k++) {
              const int c = child(tn, k);
              if (c >= 0) cc += sigmoidf_(r[3 + k] + bf) * s.aux[(size_t)c * kCUnits + warp];
            }
            const float hh = sigmoidf_(r[1] + s_bias[16 + warp]) * tanhf_(cc);
            s.aux[(size_t)v * kCUnits + warp] = cc;
            if (push) emit(v, (t0 % SG) + tn, hh, cc);
            else s.hsl[(size_t)v * kCUnits + warp] = hh;
          }
          if (t0 == 0 && l < 20) trace_mark(a, tb + 2);
          if (push && ((t0 + TMAX) % SG == 0 || t0 + TMAX >= cnt)) {
            const int g0 = t0 - t0 % SG;
            flush(s.list + lbase + g0, t0 + cntt - g0);
          }
        } else {
          float r[1];
          lead = contract_w<CDagLevel<MAXC>, H, T, 1, true>(s.X, w, r, ro, nullptr) && tn < cntt;
          if (lead) s.hsl[(size_t)tl[tn] * kCUnits + warp] = tanhf_(r[0] + s_bias[warp]);
        }
        if (!push) __syncthreads();
      };
      dispatch_tile<TMAX>(cntt, tile);
      if (t0 == 0 && l < 20) trace_mark(a, tb + 4);
    }
    if (!push) {
      cl_arrive();
      put_outputs(lbase, lbase + cnt);
      cl_wait();
    }
    trace_mark(a, 3 + l);
  }

  // ---- packed root states (this CTA's units of this cluster's roots) --------
  // (push mode: written by the epilogue)
  if (a.root_out && !push) {
    if constexpr (FUSED) {  // roots: in-degree 0; their structure index is their slot
      for (int p = warp; p < s.coff[L]; p += kRNW) {  // this cluster's nodes
        const int v = s.list[p];
        if (ls.indeg[s.perm[v]] != 0) continue;
        if (lane < kCUnits)
          a.root_out[(size_t)s.lab[v] * H + unit0 + lane] = s.hsl[(size_t)v * kCUnits + lane];
      }
    } else {
      for (int r = warp; r < R; r += kRNW) {
        const int v = __ldg(a.roots + r);
        if (!mine(v)) continue;
        if (lane < kCUnits) a.root_out[(size_t)r * H + unit0 + lane] = s.hsl[(size_t)v * kCUnits + lane];
      }
    }
  }
  trace_mark(a, a.trace_slots - 1);
  if constexpr (FUSED) fused_exit(a, ferr);
  else publish_and_exit(a);
}

template <int CELL, int H, int MAXC, bool FUSED>
bool cplan_one(int n, int maxc, int L_bound, int num_roots_hint, FwdPlan *p, int *Gn, int *Gu) {
  constexpr int CSZ = H / kCUnits;
  using Lay = CLayout<CELL, H, MAXC>;
  auto k = ck_kernel<CELL, H, MAXC, FUSED>;
  size_t need = Lay::bytes(n, maxc, L_bound);
  if (FUSED)  // the linearizer's arrays replace the prologue's int arrays
    need = need - sizeof(int) * Lay::ints(n, maxc, L_bound) + sizeof(int) * fused_extra_ints(n, maxc);
  // per-device cache (caller holds the api mutex): the largest dynamic shared
  // memory a CTA can have, the attribute setup and the co-resident clusters.
  // The kernel always gets all of it: region R beyond `need` holds the push
  // mode's rows (forward_cluster.cu header).
  constexpr int kMaxDev = 64;
  static int max_dyn[kMaxDev], cached_max[kMaxDev];
  static bool done[kMaxDev];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDev) return false;
  if (!done[dev]) {
    int optin = 0;
    cudaFuncAttributes fa;
    if (cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess ||
        cudaFuncGetAttributes(&fa, (const void *)k) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    const int dyn = (optin - (int)fa.sharedSizeBytes) & ~127;
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (CSZ > 8) cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaGetLastError();
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(CSZ * 8);
    cfg.blockDim = dim3(kRThreads);
    cfg.dynamicSmemBytes = dyn;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CSZ;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int m = 0;
    if (cudaOccupancyMaxActiveClusters(&m, (const void *)k, &cfg) != cudaSuccess) m = 0;
    cudaGetLastError();
    max_dyn[dev] = dyn;
    cached_max[dev] = m;
    done[dev] = true;
  }
  if (need > (size_t)max_dyn[dev] || cached_max[dev] < 1) return false;
  int ncl = cached_max[dev];
  if (num_roots_hint > 0 && num_roots_hint < ncl) ncl = num_roots_hint;
  *Gn = ncl;
  *Gu = CSZ;
  p->ctas = ncl * CSZ;
  p->threads = kRThreads;
  p->smem = (size_t)max_dyn[dev];
  p->kernel = (const void *)k;
  p->cluster = CSZ;
  p->fused = FUSED;
  p->family = 3;
  return true;
}

template <int CELL, int H, bool FUSED>
bool cplan_cell(int n, int maxc, int L_bound, int roots, FwdPlan *p, int *Gn, int *Gu) {
  if (maxc <= 1) return cplan_one<CELL, H, 1, FUSED>(n, maxc, L_bound, roots, p, Gn, Gu);
  if (maxc <= 2) return cplan_one<CELL, H, 2, FUSED>(n, maxc, L_bound, roots, p, Gn, Gu);
  if (maxc <= 4) return cplan_one<CELL, H, 4, FUSED>(n, maxc, L_bound, roots, p, Gn, Gu);
  return false;
}

template <bool FUSED>
bool cplan(int cell, int H, int maxc, int n, int roots, FwdPlan *p, int *Gn, int *Gu) {
  if (n > kClusterMaxN || n < 1) return false;
  const int L_bound = n;  // level arrays sized for the worst case
  switch (cell) {
    case CX_TREELSTM:
      if (H == 256) return cplan_cell<CX_TREELSTM, 256, FUSED>(n, maxc, L_bound, roots, p, Gn, Gu);
      if (H == 128) return cplan_cell<CX_TREELSTM, 128, FUSED>(n, maxc, L_bound, roots, p, Gn, Gu);
      if (H == 64) return cplan_cell<CX_TREELSTM, 64, FUSED>(n, maxc, L_bound, roots, p, Gn, Gu);
      return false;
    case CX_DAGRNN:
      if (H == 256) return cplan_cell<CX_DAGRNN, 256, FUSED>(n, maxc, L_bound, roots, p, Gn, Gu);
      if (H == 128) return cplan_cell<CX_DAGRNN, 128, FUSED>(n, maxc, L_bound, roots, p, Gn, Gu);
      if (H == 64) return cplan_cell<CX_DAGRNN, 64, FUSED>(n, maxc, L_bound, roots, p, Gn, Gu);
      return false;
  }
  return false;
}

}  // namespace

// Cluster path for small batches: TreeLSTM and DAG-RNN, H in {64, 128, 256},
// n <= kClusterMaxN. `roots` (<= 0: unknown) caps the number of clusters.
bool cluster_plan(int cell, int H, int maxc, int n, int roots, FwdPlan *p, int *Gn, int *Gu) {
  return cplan<false>(cell, H, maxc, n, roots, p, Gn, Gu);
}

// The same kernel with the single-CTA linearizer fused into its prologue
// (cx_linearize_forward); false when the shared memory does not fit.
bool fused_plan(int cell, int H, int maxc, int n, FwdPlan *p, int *Gn, int *Gu) {
  return cplan<true>(cell, H, maxc, n, 0, p, Gn, Gu);
}

}  // namespace cx
