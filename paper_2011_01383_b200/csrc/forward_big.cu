// forward_big.cu -- throughput path for LARGE batches (TreeLSTM, DAG-RNN):
// the persistent grid kernel of forward.cu (32 units per CTA, weight rows
// resident in shared memory, one grid barrier per level) with every CTA
// running a 3-stage software pipeline over its tiles of a level:
//   stage A  bookkeeping of tile j+2 loaded into registers (independent loads:
//            the recurrent state lives in the linearized numbering, so child
//            rows are addressed by the children's new ids directly);
//   stage B  child rows (and the children's memory-cell slices) of tile j+1
//            copied global -> shared with cp.async (zero-fill for absent
//            children) into the second buffer;
//   stage C  contraction of tile j against the resident weights, fused gates.
// Loads of later tiles therefore overlap the FMA work of the current one
// instead of serialising three dependent round trips per tile.
// State: hs [n][H] (h, new numbering), cs [n][H] (TreeLSTM c) or ps [n][H]
// (DAG-RNN input projections), all in the workspace; h_out / aux_out (input
// numbering) are written for the caller; root states are copied after a final
// grid barrier.
#include <cuda_runtime.h>

#include <type_traits>

#include "smem_engine.cuh"

namespace cx {
namespace {
using namespace fwd;
using namespace sme;

constexpr int kBTMax = 8;  // largest tile (nodes)

__device__ __forceinline__ void cp_async16_zfill(void *smem, const void *gmem, bool valid) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  int n = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "r"(n) : "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait_group() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

template <int CELL, int MAXC>
struct BCfg;
// T: tile (nodes, <= 8: the epilogue maps node t = tid / 32 over 256 threads);
// S: pipeline stages (buffers in flight). DAG-RNN tiles carry little math, so
// its pipeline is deeper to keep DRAM-latency gathers in flight; TreeLSTM is
// bounded by shared memory (128 KiB of resident weights).
template <int MAXC>
struct BCfg<CX_TREELSTM, MAXC> {
  static constexpr int NG = 4, NV = MAXC, NA = 3 + MAXC, NAUX = MAXC;  // aux: children's c slices
  static constexpr int T = 8, S = 2;
};
template <int MAXC>
struct BCfg<CX_DAGRNN, MAXC> {
  static constexpr int NG = 1, NV = MAXC, NA = 1, NAUX = 1;  // aux: own projection slice
  static constexpr int T = 8, S = 4;
};

struct BMeta {
  int cnt;
  int node[kBTMax];         // new id
  int own[kBTMax];          // input id (output row)
  int ch[kBTMax][kMaxC];    // children new ids, -1 absent
  int word[kBTMax];         // leaf / projection phases
};

template <int CELL, int H, int MAXC>
struct BLayout {
  using C = BCfg<CELL, MAXC>;
  static constexpr size_t w = (size_t)C::NG * kUG * (H + 4);
  static constexpr size_t wl = (size_t)(CELL == CX_TREELSTM ? 3 : 1) * kUG * (H + 4);
  static constexpr size_t wmax = w > wl ? w : wl;
  static constexpr size_t x = (size_t)C::T * (C::NV > 1 ? C::NV : 1) * H;  // one stage
  static constexpr size_t red = (size_t)kWarps * C::NA * C::T * 32;
  static constexpr size_t aux = (size_t)C::T * C::NAUX * 32;              // one stage
  static constexpr size_t bytes = sizeof(float) * (wmax + C::S * x + red + C::S * aux);
};

template <int CELL, int H, int MAXC>
__global__ void __launch_bounds__(kFwdThreads, 1) big_kernel(FwdArgs a) {
  using Cf = BCfg<CELL, MAXC>;
  using Lay = BLayout<CELL, H, MAXC>;
  constexpr int NV = Cf::NV, NAUX = Cf::NAUX, kBT = Cf::T, S = Cf::S;
  static_assert(kBT <= kFwdThreads / 32, "epilogue covers tid / 32 < T");
  extern __shared__ __align__(16) float smem[];
  __shared__ BMeta meta[S];
  __shared__ float s_bias[4 * kUG];

  griddep_wait();
  if (*reinterpret_cast<volatile int *>(&a.hdr->status) != CX_OK) return;
  const int L = a.hdr->num_levels, first_leaf = a.hdr->first_leaf, n = a.n;
  const int gn = blockIdx.x / a.Gu, gu = blockIdx.x % a.Gu;
  const int tid = threadIdx.x, lane = tid & 31;
  const int unit0 = gu * kUG;
  const bool latch = gu == 0;
  float *Ws = smem;
  float *const Xbase = Ws + Lay::wmax;
  float *red = Xbase + S * Lay::x;
  float *const Abase = red + Lay::red;
  auto Xb = [&](int b) { return Xbase + (size_t)b * Lay::x; };
  auto Ab = [&](int b) { return Abase + (size_t)b * Lay::aux; };
  // TreeLSTM computation hoisting: with fewer
  // vocabulary words than nodes the leaf cell is evaluated once per word (state
  // rows [0, V)), internal node i lives at row V + i, parents read leaf
  // children from their word's row, and the leaves' outputs are copied at the end
  const bool lstm_hoist = CELL == CX_TREELSTM && a.V < n;
  const int sbase = lstm_hoist ? a.V : 0;
  const size_t R = (size_t)n + sbase;       // state rows
  float *hs = a.pbuf;                       // [R][H] h (workspace)
  float *st = a.pbuf + R * H;               // [R][H] c (LSTM) or projections (DAG)
  int *wn = reinterpret_cast<int *>(a.pbuf + 2 * R * H);  // [n] word of new id
  unsigned epoch = 0;

  // biases of the owned units
  if constexpr (CELL == CX_TREELSTM) {
    if (tid < 4 * kUG) {
      int g = tid / kUG;
      const float *b = g < 3 ? a.w[2] + g * H : a.w[4];
      s_bias[tid] = __ldg(b + unit0 + (tid % kUG));
    }
  } else {
    if (tid < kUG) s_bias[tid] = __ldg(a.w[2] + unit0 + tid);
  }

  // ---- leaf-phase gates -> shared memory ------------------------------------
  {
    const float *base = a.w[0];
    const int ng = CELL == CX_TREELSTM ? 3 : 1;
    const int HP = H + 4, q = H / 4;
    for (int row = tid >> 5; row < ng * kUG; row += kWarps) {
      const float *src = base + (size_t)((row >> 5) * H + unit0 + (row & 31)) * H;
      for (int c = lane; c < q; c += 32) cp_async16(Ws + (size_t)row * HP + 4 * c, src + 4 * c);
    }
    cp_async_commit();
  }

  // DAG-RNN computation hoisting: the input projection
  // W_x x + b depends only on the word, so with fewer vocabulary words than
  // nodes it is computed once per word (st rows [0, V)) and every level --
  // leaves included, as a level without children -- reads its node's word row
  const bool dag_hoist = CELL == CX_DAGRNN && a.V < n;
  const bool hoist_rows = dag_hoist || lstm_hoist;  // leaf/projection pass over word rows
  // ---- words of this CTA's leaf-phase nodes, in the new numbering -----------
  const int lo0 = CELL == CX_DAGRNN ? 0 : first_leaf;
  int plo, phi;
  chunk_of(n - lo0, a.Gn, gn, plo, phi);
  plo += lo0;
  phi += lo0;
  {
    for (int i = plo + tid; i < phi; i += blockDim.x) {
      const int own = __ldg(a.perm + i);
      int w = __ldg(a.words + own);
      if (w < 0 || w >= a.V) {
        if (latch) latch_error(a.hdr, CX_E_WORD_RANGE, own);
        w = 0;
      }
      wn[i] = w;  // every unit group writes the same value (benign)
    }
  }
  __syncthreads();
  // hoisted TreeLSTM: level bookkeeping (prefetched before a level barrier
  // completes) maps leaf children through other CTAs' wn entries
  if (lstm_hoist) grid_sync(a.bar, gridDim.x, epoch);

  // ---------------------------------------------------------------------------
  // One pipelined pass over [lo, hi). `leaf` selects the leaf/projection phase.
  // ---------------------------------------------------------------------------
  auto load_meta_regs = [&](int i0, int cnt, int &r_own, int (&r_ch)[kMaxC], int &r_word,
                            bool leaf) {
    if (tid < cnt) {
      const int i = i0 + tid;
      if (leaf && hoist_rows) {  // leaf / projection pass over word rows
        r_own = -1;
        r_word = i;
        return;
      }
      r_own = __ldg(a.perm + i);
      if (leaf) {
        r_word = __ldcg(wn + i);
      } else {
        if (dag_hoist) r_word = __ldcg(wn + i);
#pragma unroll
        for (int k = 0; k < kMaxC; k++) r_ch[k] = k < a.maxc ? __ldg(a.chn + (size_t)k * n + i) : -1;
        if (lstm_hoist) {  // state rows: a leaf child's word row, else V + child
#pragma unroll
          for (int k = 0; k < kMaxC; k++)
            if (r_ch[k] >= 0) r_ch[k] = r_ch[k] >= first_leaf ? __ldcg(wn + r_ch[k]) : sbase + r_ch[k];
        }
      }
    }
  };
  auto store_meta = [&](BMeta &M, int i0, int cnt, int r_own, const int (&r_ch)[kMaxC], int r_word,
                        bool leaf) {
    if (tid == 0) M.cnt = cnt;
    if (tid < cnt) {
      M.node[tid] = i0 + tid;
      M.own[tid] = r_own;
      if (leaf) {
        M.word[tid] = r_word;
      } else {
        if (dag_hoist) M.word[tid] = r_word;
        bool absent = false;
#pragma unroll
        for (int k = 0; k < kMaxC; k++) {
          absent = absent || r_ch[k] < 0;
          M.ch[tid][k] = absent ? -1 : r_ch[k];
        }
      }
    }
  };
  auto gather = [&](const BMeta &M, int buf, bool leaf) {
    const int cnt = M.cnt;
    float *X = Xb(buf);
    constexpr int q = H / 4;
    const int nvl = leaf ? 1 : NV;
    for (int idx = tid; idx < cnt * nvl * q; idx += blockDim.x) {
      const int row = idx / q, c = idx - row * q;
      const int t = row / nvl, j = row - t * nvl;
      const float *src;
      bool valid = true;
      if (leaf) {
        src = a.emb + (size_t)M.word[t] * H;
      } else {
        const int ch = M.ch[t][j];
        valid = ch >= 0;
        src = hs + (size_t)(valid ? ch : 0) * H;
      }
      cp_async16_zfill(X + (size_t)row * H + 4 * c, src + 4 * c, valid);
    }
    if (!leaf) {
      float *A = Ab(buf);
      constexpr int q8 = kUG / 4;  // float4 per 32-unit slice
      for (int idx = tid; idx < cnt * NAUX * q8; idx += blockDim.x) {
        const int r = idx / q8, c = idx - r * q8;
        const int t = r / NAUX, k = r - t * NAUX;
        int src_row;
        bool valid;
        if constexpr (CELL == CX_TREELSTM) {
          src_row = M.ch[t][k];
          valid = src_row >= 0;
        } else {
          src_row = dag_hoist ? M.word[t] : M.node[t];  // the node's projection row
          valid = true;
        }
        cp_async16_zfill(A + (size_t)r * 32 + 4 * c, st + (size_t)(valid ? src_row : 0) * H + unit0 + 4 * c,
                         valid);
      }
    }
    cp_async_commit();
  };

  auto pass = [&](int lo, int hi, bool leaf, bool prefetched) {
    const int ntiles = (hi - lo + kBT - 1) / kBT;
    if (ntiles <= 0) return;
    int r_own = 0, r_word = 0, r_ch[kMaxC];
#pragma unroll
    for (int k = 0; k < kMaxC; k++) r_ch[k] = -1;
    // bookkeeping of tiles 0 .. S-1 (levels: the first two were loaded while
    // the CTA waited at the grid barrier)
    for (int j = prefetched ? 2 : 0; j < S && j < ntiles; j++) {
      load_meta_regs(lo + j * kBT, min(kBT, hi - lo - j * kBT), r_own, r_ch, r_word, leaf);
      store_meta(meta[j], lo + j * kBT, min(kBT, hi - lo - j * kBT), r_own, r_ch, r_word, leaf);
    }
    __syncthreads();
    for (int j = 0; j < S - 1; j++) {
      if (j < ntiles) gather(meta[j], j, leaf);
      else cp_async_commit();  // empty group keeps the group count uniform
    }
    for (int j = 0; j < ntiles; j++) {
      const int b = j % S;
      if (j + S - 1 < ntiles) gather(meta[(j + S - 1) % S], (j + S - 1) % S, leaf);
      else cp_async_commit();
      // stage A: bookkeeping of tile j + S into registers (consumed after compute)
      const int i2 = lo + (j + S) * kBT;
      const int cnt2 = j + S < ntiles ? min(kBT, hi - i2) : 0;
      load_meta_regs(i2, cnt2, r_own, r_ch, r_word, leaf);
      cp_async_wait_group<S - 1>();  // tile j's group has landed
      __syncthreads();
      // stage C: contraction + fused gates of tile j
      const BMeta &M = meta[b];
      const float *X = Xb(b);
      const float *A = Ab(b);
      const int t = tid >> 5, u = lane, unit = unit0 + u;
      const int cnt = M.cnt;
      if constexpr (CELL == CX_TREELSTM) {
        if (leaf) {
          float acc[3][kBT], s3[3];
          fma_engine<PhLstmLeaf, kBT>(Ws, X, H, acc);
          reduce_acc<3, kBT>(red, acc, s3);
          if (t < cnt) {
            const int i = M.node[t];
            float cc = sigmoidf_(s3[0] + s_bias[u]) * tanhf_(s3[2] + s_bias[64 + u]);
            float hh = sigmoidf_(s3[1] + s_bias[32 + u]) * tanhf_(cc);
            hs[(size_t)i * H + unit] = hh;  // hoisted: i is the word row
            st[(size_t)i * H + unit] = cc;
            if (!lstm_hoist) {
              const size_t o = (size_t)M.own[t] * H + unit;
              a.h_out[o] = hh;
              if (a.aux_out) a.aux_out[o] = cc;
            }
          }
        } else {
          float acc[3 + MAXC][kBT], s5[3 + MAXC];
          fma_engine<PhLstmLevel<MAXC>, kBT>(Ws, X, H, acc);
          reduce_acc<3 + MAXC, kBT>(red, acc, s5);
          if (t < cnt) {
            const int i = M.node[t];
            float cc = sigmoidf_(s5[0] + s_bias[u]) * tanhf_(s5[2] + s_bias[64 + u]);
            const float bf = s_bias[96 + u];
#pragma unroll
            for (int k = 0; k < MAXC; k++)
              if (M.ch[t][k] >= 0) cc += sigmoidf_(s5[3 + k] + bf) * A[(t * NAUX + k) * 32 + u];
            float hh = sigmoidf_(s5[1] + s_bias[32 + u]) * tanhf_(cc);
            hs[(size_t)(sbase + i) * H + unit] = hh;
            st[(size_t)(sbase + i) * H + unit] = cc;
            const size_t o = (size_t)M.own[t] * H + unit;
            a.h_out[o] = hh;
            if (a.aux_out) a.aux_out[o] = cc;
          }
        }
      } else {  // DAG-RNN
        if (leaf) {  // projection of every node; leaves finish
          float acc[1][kBT], s1[1];
          fma_engine<PhDagProj, kBT>(Ws, X, H, acc);
          reduce_acc<1, kBT>(red, acc, s1);
          if (t < cnt) {
            const int i = M.node[t];
            const float p = s1[0] + s_bias[u];
            st[(size_t)i * H + unit] = p;
            if (!dag_hoist && i >= first_leaf) {
              const float hh = tanhf_(p);
              hs[(size_t)i * H + unit] = hh;
              a.h_out[(size_t)M.own[t] * H + unit] = hh;
            }
          }
        } else {
          float acc[1][kBT], s1[1];
          fma_engine<PhDagLevel<MAXC>, kBT>(Ws, X, H, acc);
          reduce_acc<1, kBT>(red, acc, s1);
          if (t < cnt) {
            const int i = M.node[t];
            const float hh = tanhf_(s1[0] + A[t * NAUX * 32 + u]);
            hs[(size_t)i * H + unit] = hh;
            a.h_out[(size_t)M.own[t] * H + unit] = hh;
          }
        }
      }
      __syncthreads();  // buffers of tile j are free
      if (cnt2 > 0) store_meta(meta[b], i2, cnt2, r_own, r_ch, r_word, leaf);
      __syncthreads();
    }
  };

  // ---- leaf phase (TreeLSTM leaves / DAG-RNN projections of all nodes) -------
  cp_async_wait_all();
  __syncthreads();
  if (hoist_rows) {
    int wlo, whi;
    chunk_of(a.V, a.Gn, gn, wlo, whi);
    pass(wlo, whi, true, false);
  } else {
    pass(plo, phi, true, false);
  }
  __syncthreads();
  // recurrent gates (TreeLSTM: U_iou, U_f; DAG-RNN: U): land during the barrier
  {
    const int HP = H + 4, q = H / 4;
    for (int row = tid >> 5; row < Cf::NG * kUG; row += kWarps) {
      const int g = row >> 5, u = row & 31;
      const float *src;
      if constexpr (CELL == CX_TREELSTM) src = g < 3 ? a.w[1] + (size_t)(g * H + unit0 + u) * H
                                                     : a.w[3] + (size_t)(unit0 + u) * H;
      else src = a.w[1] + (size_t)(unit0 + u) * H;
      for (int c = lane; c < q; c += 32) cp_async16(Ws + (size_t)row * HP + 4 * c, src + 4 * c);
    }
    cp_async_commit();
  }

  // ---- levels -----------------------------------------------------------------
  const int lstart = dag_hoist ? 0 : 1;  // hoisted DAG-RNN: leaves are a level
  for (int l = lstart; l < L; l++) {
    const int base = __ldg(a.lbeg + l), M = __ldg(a.lsize + l);
    int lo, hi;
    chunk_of(M, a.Gn, gn, lo, hi);
    lo += base;
    hi += base;
    grid_arrive(a.bar, epoch);
    // bookkeeping of the first two tiles while the barrier completes
    static_assert(S >= 2, "at least double buffering");
    {
      int r_own = 0, r_word = 0, r_ch[kMaxC];
#pragma unroll
      for (int k = 0; k < kMaxC; k++) r_ch[k] = -1;
      const int c0 = max(0, min(kBT, hi - lo)), c1 = max(0, min(kBT, hi - lo - kBT));
      load_meta_regs(lo, c0, r_own, r_ch, r_word, false);
      store_meta(meta[0], lo, c0, r_own, r_ch, r_word, false);
      load_meta_regs(lo + kBT, c1, r_own, r_ch, r_word, false);
      store_meta(meta[1], lo + kBT, c1, r_own, r_ch, r_word, false);
    }
    grid_wait(a.bar, gridDim.x, epoch);
    if (l == lstart) {
      cp_async_wait_all();
      __syncthreads();
    }
    pass(lo, hi, false, true);
  }
  cp_async_wait_all();

  // state row of new id i
  auto srow = [&](int i) -> size_t {
    return lstm_hoist ? (size_t)(i >= first_leaf ? __ldcg(wn + i) : sbase + i) : (size_t)i;
  };
  // ---- hoisted TreeLSTM leaves: caller outputs from their word's row --------
  if (lstm_hoist) {
    if (L == 1) grid_sync(a.bar, gridDim.x, epoch);  // else a level barrier ordered it
    const int q = H / 4;
    const int gw = (blockIdx.x * blockDim.x + tid) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    for (int j = first_leaf + gw; j < n; j += nw) {  // a warp per leaf row
      const int own = __ldg(a.perm + j);
      const size_t w = (size_t)__ldcg(wn + j) * H;
      for (int c = lane; c < q; c += 32) {
        __stcs(reinterpret_cast<float4 *>(a.h_out + (size_t)own * H) + c, ldcg4(hs + w + 4 * c));
        if (a.aux_out)
          __stcs(reinterpret_cast<float4 *>(a.aux_out + (size_t)own * H) + c, ldcg4(st + w + 4 * c));
      }
    }
  }
  // ---- packed root states (after a final barrier every row of hs is final) ---
  if (a.root_out) {
    grid_sync(a.bar, gridDim.x, epoch);
    const int R = a.hdr->num_roots;
    const int q = H / 4;
    for (int idx = blockIdx.x * blockDim.x + tid; idx < R * q; idx += gridDim.x * blockDim.x) {
      const int r = idx / q, c = idx - r * q;
      const size_t i = srow(__ldg(a.roots + r));
      *reinterpret_cast<float4 *>(a.root_out + (size_t)r * H + 4 * c) = ldcg4(hs + i * H + 4 * c);
    }
  }
  publish_and_exit(a);
}

template <int CELL, int H, int MAXC>
bool bplan_one(int num_sms, FwdPlan *p, int *Gn, int *Gu) {
  constexpr size_t smem = BLayout<CELL, H, MAXC>::bytes;
  if (smem > 227 * 1024) return false;
  auto k = big_kernel<CELL, H, MAXC>;
  static bool set_dev[kMaxDevices];  // per device (attributes are per context)
  const int dev = device_slot();
  if (dev < 0) return false;
  if (!set_dev[dev]) {
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    cudaGetLastError();
    set_dev[dev] = true;
  }
  *Gu = H / kUG;
  *Gn = num_sms / *Gu;
  p->ctas = *Gn * *Gu;
  p->threads = kFwdThreads;
  p->smem = smem;
  p->kernel = (const void *)k;
  p->family = 4;
  p->cluster = 1;
  p->big = true;
  return true;
}

template <int CELL, int H>
bool bplan_cell(int maxc, int num_sms, FwdPlan *p, int *Gn, int *Gu) {
  if (maxc <= 1) return bplan_one<CELL, H, 1>(num_sms, p, Gn, Gu);
  if (maxc <= 2) return bplan_one<CELL, H, 2>(num_sms, p, Gn, Gu);
  if (maxc <= 4) return bplan_one<CELL, H, 4>(num_sms, p, Gn, Gu);
  return false;
}

}  // namespace

// Large-batch path: TreeLSTM / DAG-RNN, H in {128, 256}.
bool big_plan(int cell, int H, int maxc, int num_sms, FwdPlan *p, int *Gn, int *Gu) {
  switch (cell) {
    case CX_TREELSTM:
      if (H == 256) return bplan_cell<CX_TREELSTM, 256>(maxc, num_sms, p, Gn, Gu);
      if (H == 128) return bplan_cell<CX_TREELSTM, 128>(maxc, num_sms, p, Gn, Gu);
      return false;
    case CX_DAGRNN:
      if (H == 256) return bplan_cell<CX_DAGRNN, 256>(maxc, num_sms, p, Gn, Gu);
      if (H == 128) return bplan_cell<CX_DAGRNN, 128>(maxc, num_sms, p, Gn, Gu);
      return false;
  }
  return false;
}

// workspace floats of the large-batch path: hs, st ([n][H] each) + words [n]
size_t big_workspace_bytes(int cell, int H, int n, int V) {
  const size_t R = (size_t)n + (cell == CX_TREELSTM && V < n ? (size_t)V : 0);  // hoisted word rows
  return sizeof(float) * (2 * R * H) + sizeof(int) * (size_t)n + 256;
}

}  // namespace cx
