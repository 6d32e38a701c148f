// lin_single.cuh -- the single-CTA linearizer as a device
// function, shared by the standalone cx_linearize kernel (linearize.cu) and
// the fused linearize + forward kernel (forward_cluster.cu, SURVEY §8(f) f1:
// "the single-CTA linearizer runs [inside the forward launch]").
//
// Every working array lives in shared memory; the only global traffic is one
// coalesced read of `children` and, when `write_global`, fire-and-forget
// stores of the cx_linearization outputs (no dependent global round trip on
// the latency path). Algorithm and numbering: see linearize.cu's header
// (§4.2, App. B, reading Q4).
#pragma once
#include <cuda_runtime.h>

#include <climits>

#include "common.cuh"
#include "lin_kernels.cuh"

namespace cx {

// smem (ints): ch[maxc*n] | hgt | indeg | perm | inv | lb | ls | sid | par [n each] | cnt[cap]
struct LinSm {
  int *ch, *hgt, *indeg, *perm, *inv, *lb, *ls, *sid, *par, *cnt;
};
__host__ __device__ inline size_t lin_sm_ints(int n, int maxc, int cnt_cap) {
  return (size_t)(maxc + 8) * n + cnt_cap;
}
__device__ __forceinline__ LinSm lin_carve(int *sm, int n, int maxc) {
  LinSm s;
  s.ch = sm;
  s.hgt = s.ch + (size_t)maxc * n;
  s.indeg = s.hgt + n;
  s.perm = s.indeg + n;
  s.inv = s.perm + n;
  s.lb = s.inv + n;
  s.ls = s.lb + n;
  s.sid = s.ls + n;
  s.par = s.sid + n;
  s.cnt = s.par + n;
  return s;
}

struct LinOut {
  int ok;          // no data error latched
  int L;           // levels
  int num_roots;
  int first_leaf;  // = lb[0]
};

__device__ __noinline__ inline void lin_latch(unsigned long long *err, int code, int v) {
  atomicMin(err, ((unsigned long long)(unsigned)code << 32) | (unsigned)v);
}

// Optional L2 prefetch of each node's input row Emb[words[v]] (fused forward):
// node v is handled by CTA v mod gridDim, its word id load overlaps the
// children load and the prefetch is fire-and-forget.
struct LinPrefetch {
  const int32_t *words = nullptr;
  const float *emb = nullptr;
  int H = 0, V = 0;
};

// Run a1..a6 with the calling CTA. `cnt_cap` = entries of the count table.
// `write_global`: write the cx_linearization arrays and header of `a`.
// `chn_s` (optional): remapped children [maxc][n] also kept in shared memory.
// `pf`: optional prefetch of the nodes' input rows. Every thread returns the
// same LinOut.
__device__ __forceinline__ LinOut lin_single_body(const LinArgs &a, int *sm, int cnt_cap,
                                                  bool write_global, int *chn_s,
                                                  const LinPrefetch &pf) {
  __shared__ unsigned long long s_err;
  __shared__ int s_count, s_round, s_max;
  const int n = a.n, maxc = a.maxc, tid = threadIdx.x, nthr = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5;
  const LinSm s = lin_carve(sm, n, maxc);
  int *ch = s.ch, *hgt = s.hgt, *indeg = s.indeg, *perm = s.perm, *inv = s.inv, *lb = s.lb,
      *ls_s = s.ls, *sid = s.sid, *par = s.par;

  if (write_global) lin_mark(a, 0);
  int pf_w = -1;
  if (pf.words) {
    const long long pv = blockIdx.x + (long long)gridDim.x * tid;
    if (pv < n) pf_w = __ldg(pf.words + pv);
  }
  // the children, as 4-byte cp.async copies: every piece in flight at once
  // (one HBM round trip, not one per loop iteration); waited before the
  // barrier below
#pragma unroll 1
  for (int i = tid; i < maxc * n; i += nthr) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(ch + i);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(a.ch + i) : "memory");
  }
  if (pf_w >= 0 && pf_w < pf.V) {
    const float *row = pf.emb + (size_t)pf_w * pf.H;
#pragma unroll 1
    for (int q = 0; q < pf.H; q += 32) asm volatile("prefetch.global.L2 [%0];" ::"l"(row + q));
  }
#pragma unroll 1
  for (int v = tid; v < n; v += nthr) {
    indeg[v] = 0;
    hgt[v] = -1;
    par[v] = -1;  // parent pointer (trees/sequences)
    sid[v] = INT_MAX;
  }
  if (tid == 0) {
    s_err = kNoError;
    s_count = 0;
    s_round = 0;
    s_max = 0;
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();

  // a1: validation + in-degree; errors latched in shared memory (lowest key).
  // For trees and sequences the same pass records parent pointers (par[]) and
  // the number of children (inv[], free until a4) for the walk-up below.
  const bool tree_like = a.kind != CX_DAG;
  int *parent = par, *pending = inv;
#pragma unroll 1
  for (int v = tid; v < n; v += nthr) {
    bool absent = false;
    int nc = 0;
#pragma unroll 1
    for (int k = 0; k < maxc; k++) {
      int c = ch[k * n + v];
      if (c == -1) {
        absent = true;
        continue;
      }
      nc++;
      if (absent) lin_latch(&s_err, CX_E_CHILD_LAYOUT, v);
      if (c < 0 || c >= n) {
        lin_latch(&s_err, CX_E_CHILD_RANGE, v);
        continue;
      }
      atomicAdd(&indeg[c], 1);
      if (tree_like) parent[c] = v;
#pragma unroll 1
      for (int k2 = 0; k2 < k; k2++)
        if (ch[k2 * n + v] == c) lin_latch(&s_err, CX_E_KIND, v);
    }
    if (nc == 0) hgt[v] = 0;
    pending[v] = nc;
  }
  __syncthreads();
  if (tree_like)
#pragma unroll 1
    for (int v = tid; v < n; v += nthr)
      if (indeg[v] > 1) lin_latch(&s_err, CX_E_KIND, v);
  __syncthreads();
  if (write_global) lin_mark(a, 1);
  bool failed = s_err != kNoError;

  // a2: heights, h = 0 for a leaf, else 1 + max over the children.
  // Trees/sequences: every leaf walks up its parent chain; at each parent it
  // raises the height (atomicMax) and decrements the pending count -- only
  // the last arriving child continues, so every node is finalised exactly
  // once and no block barrier is needed per level. DAGs (and hmode 1, for
  // measurement): Jacobi rounds, one __syncthreads_or each (round r finalises
  // exactly the nodes of height r; no progress => CX_E_CYCLE on every node on
  // or above a cycle, the lowest id wins). Measured on B200 (b10, 390 nodes):
  // walk-up 3.5k cycles, rounds 7.7k, an asynchronous polling pass 10k (the
  // 16 polling warps starve the one on the critical path).
  int L = 0;
  if (!failed && n > 0) {
    int hmax = 0;
    if (tree_like && a.hjacobi != 1) {
#pragma unroll 1
      for (int v = tid; v < n; v += nthr) {
        // start at leaves only: an immutable test (a node's pending count can
        // reach 0 while this loop runs, when the walk of its last child passes
        // through it; re-walking it would decrement its parent twice)
        if (ch[v] != -1) continue;
        int cur = v, hc = 0;
        while (true) {
          int p = parent[cur];
          if (p < 0) break;
          atomicMax(&hgt[p], hc + 1);
          __threadfence_block();
          if (atomicSub(&pending[p], 1) != 1) break;
          __threadfence_block();
          cur = p;
          hc = atomicAdd(&hgt[p], 0);  // every child's atomicMax precedes its decrement
        }
        hmax = max(hmax, hc);
      }
      __syncthreads();
      bool unfinished = false;
#pragma unroll 1
      for (int v = tid; v < n; v += nthr)
        if (pending[v] > 0) {  // on or above a cycle
          lin_latch(&s_err, CX_E_CYCLE, v);
          unfinished = true;
        }
      if (__syncthreads_or(unfinished)) failed = true;
      for (int o = 16; o; o >>= 1) hmax = max(hmax, __shfl_xor_sync(0xffffffffu, hmax, o));
      if (lane == 0) atomicMax(&s_round, hmax);
      __syncthreads();
      L = s_round + 1;
    } else {
      // each thread walks only its unfinished nodes (ids tid + j * nthr, a
      // bitmask): a round costs one pass over the open frontier, not over n
      const int J = (n + nthr - 1) / nthr;
      unsigned todo = 0;
      if (J <= 32) {
#pragma unroll 1
        for (int j = 0; j < J; j++) {
          const int v = tid + j * nthr;
          if (v < n && hgt[v] < 0) todo |= 1u << j;
        }
      }
      int r = 0;
      bool progress = true;
      while (progress) {
        r++;
        bool any = false;
        if (maxc <= 2) {
          // branch-free round (the common binary / unary DAGs): every load of
          // a node is issued before any test (tools/micro/jacobi_round.cu:
          // 690 vs 1,260 cycles per round for 10 grids of 10 x 10)
#pragma unroll 1
          for (int v = tid; v < n; v += nthr) {
            const int h = hgt[v];
            const int c0 = ch[v], c1 = maxc == 2 ? ch[n + v] : -1;
            const int h0 = c0 >= 0 ? hgt[c0] : 0, h1 = c1 >= 0 ? hgt[c1] : 0;
            if (h < 0 && h0 >= 0 && h0 < r && h1 >= 0 && h1 < r) {
              hgt[v] = r;
              any = true;
            }
          }
        } else if (J <= 32) {
          unsigned t = todo;
          while (t) {
            const int j = __ffs(t) - 1;
            t &= t - 1;
            const int v = tid + j * nthr;
            bool ok = true;
#pragma unroll 1
            for (int k = 0; k < maxc; k++) {
              const int c = ch[k * n + v];
              if (c == -1) break;
              const int hc = hgt[c];
              if (hc < 0 || hc >= r) {
                ok = false;
                break;
              }
            }
            if (ok) {
              hgt[v] = r;
              todo &= ~(1u << j);
              any = true;
            }
          }
        } else {
#pragma unroll 1
          for (int v = tid; v < n; v += nthr) {
            if (hgt[v] >= 0) continue;
            bool ok = true;
#pragma unroll 1
            for (int k = 0; k < maxc; k++) {
              int c = ch[k * n + v];
              if (c == -1) break;
              int hc = hgt[c];
              if (hc < 0 || hc >= r) {
                ok = false;
                break;
              }
            }
            if (ok) {
              hgt[v] = r;
              any = true;
            }
          }
        }
        progress = __syncthreads_or(any);
      }
      bool unfinished = false;
#pragma unroll 1
      for (int v = tid; v < n; v += nthr)
        if (hgt[v] < 0) {
          lin_latch(&s_err, CX_E_CYCLE, v);
          unfinished = true;
        }
      if (__syncthreads_or(unfinished)) failed = true;
      L = r;
    }
  }
  if (write_global) lin_mark(a, 2);

  if (!failed && n > 0) {
    // a3: per-(level, id segment) counts + roots row, always in shared memory:
    // S segments of `seg` ids (one warp each), S shrinks when L is large.
    const int nw = nthr >> 5;
    int S = min(nw, max(1, cnt_cap / (L + 1)));
    S = min(S, (n + 31) / 32);
    const int seg = 32 * ((((n + 31) / 32) + S - 1) / S);
    S = (n + seg - 1) / seg;
    int *cnt = s.cnt;
#pragma unroll 1
    for (int e = tid; e < (L + 1) * S; e += nthr) cnt[e] = 0;
    __syncthreads();
    const unsigned lt = (1u << lane) - 1u;
    if (warp < S) {
      const int sg = warp, end = min(n, (sg + 1) * seg);
#pragma unroll 1
      for (int base = sg * seg; base < end; base += 32) {
        int v = base + lane;
        bool valid = v < end;
        int hv = valid ? hgt[v] : -1;
        unsigned m = __match_any_sync(0xffffffffu, hv);
        if (valid && (m & lt) == 0) cnt[hv * S + sg] += __popc(m);
        unsigned rb = __ballot_sync(0xffffffffu, valid && indeg[v] == 0);
        if (lane == 0 && rb) cnt[L * S + sg] += __popc(rb);
        __syncwarp();
      }
    }
    __syncthreads();
    if (write_global) lin_mark(a, 3);
    // exclusive scan in the order (level L-1 .. 0) x (segment 0 .. S-1): warp w
    // takes levels w, w + nw, ...; level totals, then a warp-0 scan over them
#pragma unroll 1
    for (int l = warp; l < L; l += nw) {
      int x = lane < S ? cnt[l * S + lane] : 0;  // S <= 32 when L < cnt_cap/32
      int incl = x;
      for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      if (S <= 32) {
        if (lane < S) cnt[l * S + lane] = incl - x;  // within-level offset
        if (lane == 31) ls_s[l] = incl;               // level size
      } else {
        // wide tables (tiny L): serial per level
        if (lane == 0) {
          int acc = 0;
#pragma unroll 1
          for (int s2 = 0; s2 < S; s2++) {
            int c = cnt[l * S + s2];
            cnt[l * S + s2] = acc;
            acc += c;
          }
          ls_s[l] = acc;
        }
      }
    }
    if (warp == nw - 1) {  // roots row
      int acc = 0;
#pragma unroll 1
      for (int b = 0; b < S; b += 32) {
        int x = b + lane < S ? cnt[L * S + b + lane] : 0;
        int incl = x;
        for (int o = 1; o < 32; o <<= 1) {
          int y = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += y;
        }
        if (b + lane < S) cnt[L * S + b + lane] = acc + incl - x;
        acc += __shfl_sync(0xffffffffu, incl, 31);
      }
      if (lane == 0) s_count = acc;
    }
    __syncthreads();
    // level begins: exclusive scan of level sizes from level L-1 down (warp 0)
    if (warp == 0) {
      int acc = 0, mx = 0;
#pragma unroll 1
      for (int b = 0; b < L; b += 32) {
        int l = L - 1 - (b + lane);
        int x = l >= 0 ? ls_s[l] : 0;
        int incl = x;
        for (int o = 1; o < 32; o <<= 1) {
          int y = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += y;
        }
        if (l >= 0) {
          lb[l] = acc + incl - x;
          if (write_global) {
            a.lbeg[l] = acc + incl - x;
            a.lsize[l] = x;
          }
          mx = max(mx, x);
        }
        acc += __shfl_sync(0xffffffffu, incl, 31);
      }
      for (int o = 16; o; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      if (lane == 0) s_max = mx;
    }
    __syncthreads();
    if (write_global) lin_mark(a, 4);
    // a4: stable scatter (each warp walks its segment in id order)
    if (warp < S) {
      const int sg = warp, end = min(n, (sg + 1) * seg);
      int rbase = cnt[L * S + sg];
#pragma unroll 1
      for (int base = sg * seg; base < end; base += 32) {
        int v = base + lane;
        bool valid = v < end;
        int hv = valid ? hgt[v] : -1;
        unsigned m = __match_any_sync(0xffffffffu, hv);
        int leader = __ffs(m) - 1;
        int b = (valid && lane == leader) ? lb[hv] + cnt[hv * S + sg] : 0;
        b = __shfl_sync(0xffffffffu, b, leader);
        int nid = b + __popc(m & lt);
        bool isroot = valid && indeg[v] == 0;
        unsigned rb = __ballot_sync(0xffffffffu, isroot);
        __syncwarp();
        if (valid && lane == leader) cnt[hv * S + sg] += __popc(m);
        if (valid) {
          perm[nid] = v;
          inv[v] = nid;
          if (write_global) {
            a.perm[nid] = v;
            a.inv[v] = nid;
            a.hnew[nid] = hv;
          }
          if (isroot) {
            if (write_global) a.roots[rbase + __popc(rb & lt)] = nid;
            sid[nid] = rbase + __popc(rb & lt);
          }
        }
        rbase += __popc(rb);
        __syncwarp();
      }
    }
    __syncthreads();
    if (write_global) lin_mark(a, 5);
    // a5: remap children to new ids
#pragma unroll 1
    for (int i = tid; i < n; i += nthr) {
      int v = perm[i];
#pragma unroll 1
      for (int k = 0; k < maxc; k++) {
        int c = ch[k * n + v];
        const int r = c == -1 ? -1 : inv[c];
        if (write_global) a.chn[(long long)k * n + i] = r;
        if (chn_s) chn_s[k * n + i] = r;
      }
    }
    // a6: structure of every node. Trees/sequences: walk up to the root (roots
    // already hold their index); DAGs: the smallest root index reaching the
    // node, propagated top-down one level per round.
    if (tree_like) {
      __syncthreads();
#pragma unroll 1
      for (int i = tid; i < n; i += nthr) {
        int v = perm[i], p = parent[v];
        if (p < 0) continue;
        while (p >= 0) {
          v = p;
          p = parent[v];
        }
        sid[i] = sid[inv[v]];
      }
      __syncthreads();
    } else {
#pragma unroll 1
      for (int l = L - 1; l >= 1; l--) {
        const int b = lb[l], e = b + ls_s[l];
#pragma unroll 1
        for (int i = b + tid; i < e; i += nthr) {
          const int si = sid[i], v = perm[i];
          if (maxc <= 2) {  // all loads of the node issued before the atomics
            const int c0 = ch[v], c1 = maxc == 2 ? ch[n + v] : -1;
            const int n0 = c0 >= 0 ? inv[c0] : -1, n1 = c1 >= 0 ? inv[c1] : -1;
            if (n0 >= 0) atomicMin(&sid[n0], si);
            if (n1 >= 0) atomicMin(&sid[n1], si);
          } else {
#pragma unroll 1
            for (int k = 0; k < maxc; k++) {
              int c = ch[k * n + v];
              if (c == -1) break;
              atomicMin(&sid[inv[c]], si);
            }
          }
        }
        __syncthreads();
      }
    }
    if (write_global)
#pragma unroll 1
      for (int i = tid; i < n; i += nthr) a.sid[i] = sid[i];
  }

  // header (one thread; plain stores)
  __syncthreads();
  if (write_global) lin_mark(a, 6);
  const unsigned long long key = s_err;
  LinOut out;
  out.ok = key == kNoError;
  out.L = n > 0 && out.ok ? L : 0;
  out.num_roots = n > 0 && out.ok ? s_count : 0;
  out.first_leaf = n > 0 && out.ok ? lb[0] : 0;
  if (write_global && tid == 0) {
    cx_lin_header *h = a.hdr;
    h->err_key = key;
    h->num_nodes = n;
    if (key != kNoError) {
      h->status = (int)(key >> 32);
      h->bad_node = (int)(key & 0xffffffffu);
      h->num_levels = 0;
    } else {
      h->status = CX_OK;
      h->bad_node = -1;
      h->num_levels = out.L;
      h->num_roots = out.num_roots;
      h->num_leaves = n - out.first_leaf;
      h->first_leaf = out.first_leaf;
      h->max_level_size = n > 0 ? s_max : 0;
    }
  }
  return out;
}

}  // namespace cx
